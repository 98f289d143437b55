// selector.h — host-side tile selector (see selector.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/mbci.h"

namespace mbci {

// Largest reduction dims the ABI accepts (K: live k loop in 64-column chunks on kernel 0;
// L: h chunks of <= 128 columns on the grid, PAPER.md:230-233 / Table II G3-G6).
constexpr int64_t kMaxK = 65536;
constexpr int64_t kMaxL = 65536;

void model_terms(int64_t batch, int64_t M, int64_t N, int64_t K, int64_t L, int64_t TM,
                 int64_t TN, int64_t TK, int64_t TH, int32_t s, const mbci_hw_t& hw,
                 double out[5]);
bool rule3_reject(int64_t size, int64_t tile);
int64_t tc_smem_bytes(int32_t k_steps, int32_t BN, int32_t TL, int32_t stages, int32_t b_layout,
                      int32_t* a_bytes, int32_t* b_stage, int32_t* d_stage);
int32_t tmem_alloc_cols(int32_t BN, int32_t TL);
bool tc_eligible(const mbci_chain_desc_t& d);

// SMEM carve-up of the persistent ping-pong attention kernel (chain_tc4.cuh): Q pair buffers,
// a K/V ring, barriers (l and the TMEM slot live in static shared memory).
struct Tc4Layout {
  int32_t q_bytes, b_stage, d_stage, q_bufs, smem_total;
};
bool tc4_layout(int32_t k_steps, int32_t TL, int32_t stages, int32_t b_layout, Tc4Layout* out,
                int32_t smem_max = 232448);
// Kernel 5 (chain_tc5.cuh, L <= 64): the same SMEM carve-up with 20 + 2·stages barriers.
bool tc5_layout(int32_t k_steps, int32_t TL, int32_t stages, int32_t b_layout, Tc4Layout* out,
                int32_t smem_max = 232448);
// rule3 = false skips Rule 3 entirely: an explicitly forced plan only has to be
// legal (SMEM / TMEM / TMA), not preferred.
int enumerate_plans(const mbci_chain_desc_t& d, const mbci_hw_t& hw,
                    std::vector<mbci_plan_t>& out, bool rule3 = true);
void hw_default(mbci_hw_t* hw);
// PAPER.md Fig. 7 funnel over the paper's own search space (prune.cpp).
mbci_status_t prune_funnel(int64_t M, int64_t N, int64_t K, int64_t H, int32_t elem_bytes, int64_t shm_max,
                           mbci_funnel_t* f);

}  // namespace mbci
