// chain_tc.cuh — the fused MBCI chain E = op(A·B)·D on sm_100a tensor cores.
//
// One CTA owns one work unit (batch index β, a 128-row m-tile, an h-chunk of TL output
// columns): the paper's spatial loops m and h bound to blockIdx (Rule 1).
// K <= 128 makes the k loop dead, so the A tile is loaded ONCE per CTA and
// E is stored once per CTA after the n loop (S_E hoisted).  The
// intermediate C never leaves the SM: S = A·B_j lands in tensor memory, the inter-GEMM op
// turns it into P (16-bit) in place, and GEMM2 reads P straight from tensor memory.
//
// Warp roles (224 threads):
//   warps 0-3  "row warps": thread t owns output row t (TMEM lane t); softmax / scale /
//              convert of S_j into P_j, lazy O rescale, epilogue (E = O / l).
//   warp 4     TMA producer: A once, then B_j into a `stages`-deep SMEM ring.
//   warp 5     tcgen05 issuer (one elected lane) + TMEM allocator.
//   warp 6     TMA producer: D_j into its own `stages`-deep ring (B and D slots are
//              released separately: B_j after G1(j), D_j after G2(j)).
// Issue order of the MMA warp: G1(0) G1(1) G2(0) G1(2) G2(1) ... G2(nt-1), so the row
// warps convert S_j while the tensor core runs G2(j-1) and G1(j+1) (S double-buffered).
//
// TMEM columns: S_0 [0,BN), S_1 [BN,2BN), O [2BN, 2BN+TLP).  P_j (16-bit, packed two per
// 32-bit column) overwrites the first BN/2 columns of S_{j&1}.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "ptx.cuh"

namespace mbci {

struct TcParams {
  int32_t M, N, K, L;
  int32_t batch, l_m, l_h;
  int32_t TL;        // output columns per CTA (multiple of 16, the h tile)
  int32_t k_steps;   // ceil(K / 16); 0 => C = 0
  int32_t stages;
  int32_t op;        // 0 none, 1 scale, 2 softmax
  int32_t causal;    // softmax: key n visible to row m only if n <= m (R18)
  float scale;       // SCALE multiplier, or softmax scale * log2(e)
  const int32_t* valid_len;
  void* E;
  int64_t ld_e, bs_e;
  uint32_t a_bytes;        // A tile bytes in SMEM (= TMA transaction bytes)
  uint32_t b_stage_bytes;  // one B stage
  uint32_t d_stage_bytes;  // one D stage
  uint32_t kp_rows;        // B (layout 0) box rows = 16 * k_steps (64 when A is streamed)
  int32_t kc;              // 0: A resident (K <= 128); else K > 128 streamed in kc chunks of 64 columns:
                           // ring entry (j, c) = [A[:, 64c:64c+64] | B_j[64c:64c+64]] (live k loop,
                           // PAPER.md:230-233 with L_A in k scope)
  uint32_t tmem_cols;
  uint32_t idesc1, idesc2;
  uint64_t* trace;   // optional per-CTA event timestamps (debug; see mbci_chain_set_trace)
  // Third contraction (mbci_chain3): E = op2(scale2 · O') · F with O' = op(A·B)·D
  // (softmax-normalised).  The CTA keeps the whole L (TL = L padded, one h chunk for D) and the grid's
  // h index walks H in chunks of TH columns; O' -> P2 (16-bit, TMEM) -> G3 (TS MMA, F from SMEM).
  int32_t c3;        // 0: two-GEMM chain
  int32_t H, TH;
  int32_t op2;       // 0 none, 1 scale, 3 relu, 4 gelu
  float scale2;
  uint32_t f_bytes;  // F tile (L rows x TH columns) in SMEM
  uint32_t idesc3;
  // Split-N partial runs (as Tc4Params): keys [key_off, key_off + N) of the full sequence; SOFTMAX
  // writes the natural-log row log-sum-exp of that key range to lse[β·M + m] (nullptr: not written).
  int32_t key_off;
  float* lse;
};

// Trace slots (kTraceSlots x u64 per CTA, globaltimer ns unless noted).
constexpr int kTraceSlots = 128;
enum : int {
  kTrStart = 0, kTrSetup = 1, kTrSmid = 2, kTrAFull = 3, kTrEpi = 4, kTrEnd = 5,
  kTrTile0 = 8, kTrPerTile = 7, kTrTiles = 16,
  // per tile j at kTrTile0 + kTrPerTile * j + {0: S ready, 1: S loaded, 2: max done, 3: exp done,
  //                                           4: P arrived, 5: G1 issued, 6: G2 issued}
};
#define MBCI_TR(j, k) (kTrTile0 + kTrPerTile * (j) + (k))

constexpr int kRowThreads = 128;
constexpr int kThreads = 224;
constexpr float kRescaleTau = 8.0f;   // lazy rescale threshold, log2 units (P <= 2^8)

template <bool BF16, int BN, int KCH, int BL, int DCH>
__global__ void __launch_bounds__(kThreads, BN == 64 ? 2 : 1)
    k_chain_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmF,
               const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int S = p.stages;
  uint8_t* sA = smem;
  uint8_t* sB = sA + p.a_bytes;
  uint8_t* sD = sB + S * p.b_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + S * p.d_stage_bytes);
  uint64_t* a_full = bars;
  uint64_t* b_full = bars + 1;
  uint64_t* d_full = b_full + S;
  uint64_t* b_empty = d_full + S;   // B_j's slot is free once G1(j) has read it
  uint64_t* d_empty = b_empty + S;  // D_j's slot is free once G2(j) has read it
  uint64_t* s_full = d_empty + S;   // [2]
  uint64_t* p_full = s_full + 2;    // [2]
  uint64_t* o_done = p_full + 2;    // [1] one completion per G2(i)
  uint64_t* o_final = o_done + 1;   // [1] one completion after the last G2
  uint64_t* p2_full = o_final + 1;  // [1] chain3: row warps wrote P2 (128 arrivals)
  uint64_t* f_full = p2_full + 1;   // [1] chain3: F tile landed
  uint64_t* e3_full = f_full + 1;   // [1] chain3: G3 completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(e3_full + 1);
  uint8_t* sF = reinterpret_cast<uint8_t*>(bars) + 1024;   // chain3: F tile after the barrier block

  const int warp = threadIdx.x >> 5;
  const int unit = blockIdx.x;
  uint64_t* tr = p.trace ? p.trace + static_cast<int64_t>(blockIdx.x) * kTraceSlots : nullptr;
  if (tr && threadIdx.x == 0) {
    tr[kTrStart] = ptx::globaltimer();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[kTrSmid] = smid;
  }
  const int ht = unit % p.l_h;
  const int mt = (unit / p.l_h) % p.l_m;
  const int beta = unit / (p.l_h * p.l_m);
  const int m0 = mt * 128;
  const int h0 = p.c3 ? 0 : ht * p.TL;    // D / O columns of this CTA (chain3: the whole L)
  const int h3 = ht * p.TH;                // chain3: F / E columns of this CTA

  int n_lim = p.N;
  if (p.op == 2 && p.valid_len != nullptr) n_lim = min(max(p.valid_len[beta] - p.key_off, 0), p.N);
  // causal (R18): row m sees keys n <= m; the CTA's tiles end at its last row's limit
  const int row_lim = (p.op == 2 && p.causal) ? min(n_lim, m0 + static_cast<int>(threadIdx.x) + 1) : n_lim;
  if (p.op == 2 && p.causal) n_lim = min(n_lim, m0 + 128);
  const int nt = (n_lim + BN - 1) / BN;

  if (threadIdx.x == kRowThreads) {
    ptx::mbar_init(a_full, 1);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&b_full[s], 1);
      ptx::mbar_init(&d_full[s], 1);
      ptx::mbar_init(&b_empty[s], 1);
      ptx::mbar_init(&d_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&p_full[b], kRowThreads);
    }
    ptx::mbar_init(o_done, 1);
    ptx::mbar_init(o_final, 1);
    ptx::mbar_init(p2_full, kRowThreads);
    ptx::mbar_init(f_full, 1);
    ptx::mbar_init(e3_full, 1);
    ptx::fence_mbar_init();
    if (p.c3 && nt > 0) ptx::tma_prefetch(&tmF);
    if (nt > 0) {  // maps are only encoded when the operands exist
      if (p.k_steps > 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
      }
      ptx::tma_prefetch(&tmD);
    }
  }
  if (warp == 5) ptx::tmem_alloc(tmem_slot, p.tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tr && threadIdx.x == 0) tr[kTrSetup] = ptx::globaltimer();

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer: A, B_j
    const bool elected = ptx::elect_one();   // one elect.sync per warp (all 32 lanes take part)
    if (elected && nt > 0 && p.k_steps > 0 && p.kc > 0) {
      // live k loop: (A chunk, B chunk) pairs, A re-read from L2 for every key tile
      for (int j = 0, e = 0; j < nt; ++j) {
        for (int c = 0; c < p.kc; ++c, ++e) {
          const int s = e % S;
          if (e >= S) ptx::mbar_wait(&b_empty[s], ((e / S) - 1) & 1);
          uint8_t* dst = sB + s * p.b_stage_bytes;
          ptx::mbar_arrive_expect_tx(&b_full[s], p.b_stage_bytes);
          ptx::tma_load_3d(dst, &tmA, &b_full[s], c * 64, m0, beta);
          if constexpr (BL == 1) {
            ptx::tma_load_3d(dst + 16384, &tmB, &b_full[s], c * 64, j * BN, beta);
          } else {
#pragma unroll
            for (int nb = 0; nb < BN / 64; ++nb)
              ptx::tma_load_3d(dst + 16384 + nb * (64 * 128), &tmB, &b_full[s], j * BN + nb * 64, c * 64, beta);
          }
        }
      }
    } else if (elected && nt > 0 && p.k_steps > 0) {
      ptx::mbar_arrive_expect_tx(a_full, p.a_bytes);
#pragma unroll
      for (int c = 0; c < KCH; ++c) ptx::tma_load_3d(sA + c * 16384, &tmA, a_full, c * 64, m0, beta);
      for (int j = 0; j < nt; ++j) {
        const int s = j % S;
        if (j >= S) ptx::mbar_wait(&b_empty[s], ((j / S) - 1) & 1);
        uint8_t* dst = sB + s * p.b_stage_bytes;
        ptx::mbar_arrive_expect_tx(&b_full[s], p.b_stage_bytes);
        if constexpr (BL == 1) {
#pragma unroll
          for (int c = 0; c < KCH; ++c)
            ptx::tma_load_3d(dst + c * (BN * 128), &tmB, &b_full[s], c * 64, j * BN, beta);
        } else {
#pragma unroll
          for (int c = 0; c < BN / 64; ++c)
            ptx::tma_load_3d(dst + c * (p.kp_rows * 128), &tmB, &b_full[s], j * BN + c * 64, 0, beta);
        }
      }
    }
  } else if (warp == 6) {
    // ------------------------------------------------------------ TMA producer: D_j (and F)
    const bool elected6 = ptx::elect_one();
    if (elected6 && nt > 0 && p.c3) {   // chain3: the F tile once, up front
      ptx::mbar_arrive_expect_tx(f_full, p.f_bytes);
      for (int c = 0; c < p.TH / 64; ++c)
        ptx::tma_load_3d(sF + c * (p.TL * 128), &tmF, f_full, h3 + c * 64, 0, beta);
    }
    if (elected6 && nt > 0) {
      for (int j = 0; j < nt; ++j) {
        const int s = j % S;
        if (j >= S) ptx::mbar_wait(&d_empty[s], ((j / S) - 1) & 1);
        uint8_t* ddst = sD + s * p.d_stage_bytes;
        ptx::mbar_arrive_expect_tx(&d_full[s], p.d_stage_bytes);
#pragma unroll
        for (int c = 0; c < DCH; ++c)
          ptx::tma_load_3d(ddst + c * (BN * 128), &tmD, &d_full[s], h0 + c * 64, j * BN, beta);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ tcgen05 issuer
    if (ptx::elect_one() && nt > 0) {
      const uint32_t tO = tmem + 2 * BN;
      if (p.k_steps > 0 && p.kc == 0) ptx::mbar_wait(a_full, 0);
      if (tr) tr[kTrAFull] = ptx::globaltimer();
      const uint32_t a_base = ptx::smem_u32(sA);
      for (int j = 0; j <= nt; ++j) {
        if (j < nt && p.kc > 0) {   // live k loop: S_j = sum over chunks c of A_c · B_j,c
          const int buf = j & 1;
          for (int c = 0; c < p.kc; ++c) {
            const int e = j * p.kc + c, s = e % S;
            ptx::mbar_wait(&b_full[s], (e / S) & 1);
            ptx::tc_fence_after();
            const uint32_t e_base = ptx::smem_u32(sB + s * p.b_stage_bytes);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const uint64_t ad = ptx::sdesc_sw128(e_base + ks * 32, 16, 1024);
              uint64_t bd;
              if constexpr (BL == 1)
                bd = ptx::sdesc_sw128(e_base + 16384 + ks * 32, 16, 1024);
              else
                bd = ptx::sdesc_sw128(e_base + 16384 + ks * 2048, 64 * 128, 1024);
              ptx::mma_ss(tmem + buf * BN, ad, bd, p.idesc1, (c > 0 || ks > 0) ? 1u : 0u);
            }
            ptx::mma_commit(&b_empty[s]);
          }
          if (tr && j < kTrTiles) tr[MBCI_TR(j, 5)] = ptx::globaltimer();
          ptx::mma_commit(&s_full[buf]);
        } else if (j < nt) {
          const int s = j % S, buf = j & 1;
          if (p.k_steps > 0) {
            ptx::mbar_wait(&b_full[s], (j / S) & 1);
            ptx::tc_fence_after();
            const uint32_t b_base = ptx::smem_u32(sB + s * p.b_stage_bytes);
            for (int ks = 0; ks < p.k_steps; ++ks) {
              const uint64_t ad =
                  ptx::sdesc_sw128(a_base + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
              uint64_t bd;
              if constexpr (BL == 1)
                bd = ptx::sdesc_sw128(b_base + (ks >> 2) * (BN * 128) + (ks & 3) * 32, 16, 1024);
              else
                bd = ptx::sdesc_sw128(b_base + ks * 2048, p.kp_rows * 128, 1024);
              ptx::mma_ss(tmem + buf * BN, ad, bd, p.idesc1, ks > 0 ? 1u : 0u);
            }
            if (tr && j < kTrTiles) tr[MBCI_TR(j, 5)] = ptx::globaltimer();
            ptx::mma_commit(&b_empty[s]);
          }
          ptx::mma_commit(&s_full[buf]);
        }
        if (j >= 1) {
          const int i = j - 1, s = i % S, buf = i & 1;
          ptx::mbar_wait(&p_full[buf], (i >> 1) & 1);
          ptx::mbar_wait(&d_full[s], (i / S) & 1);
          ptx::tc_fence_after();
          const uint32_t d_base = ptx::smem_u32(sD + s * p.d_stage_bytes);
#pragma unroll
          for (int ks = 0; ks < BN / 16; ++ks) {
            const uint64_t dd = ptx::sdesc_sw128(d_base + ks * 2048, BN * 128, 1024);
            ptx::mma_ts(tO, tmem + buf * BN + ks * 8, dd, p.idesc2, (i > 0 || ks > 0) ? 1u : 0u);
          }
          if (tr && i < kTrTiles) tr[MBCI_TR(i, 6)] = ptx::globaltimer();
          ptx::mma_commit(&d_empty[s]);
          ptx::mma_commit(o_done);
          if (i == nt - 1) ptx::mma_commit(o_final);
        }
      }
      if (p.c3) {   // G3: E3 = P2 · F_h (P2 from TMEM columns [0, TL/2) of S_0, F MN-major in SMEM)
        ptx::mbar_wait(p2_full, 0);
        ptx::mbar_wait(f_full, 0);
        ptx::tc_fence_after();
        const uint32_t tE3 = tmem + 2 * BN + p.TL;
        const uint32_t f_base = ptx::smem_u32(sF);
        for (int ks = 0; ks < p.TL / 16; ++ks) {
          const uint64_t fd = ptx::sdesc_sw128(f_base + ks * 2048, p.TL * 128, 1024);
          ptx::mma_ts(tE3, tmem + ks * 8, fd, p.idesc3, ks > 0 ? 1u : 0u);
        }
        ptx::mma_commit(e3_full);
      }
    }
  } else {
    // ------------------------------------------------------------ row warps (0-3)
    const int row = threadIdx.x;  // TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t tS = tmem + lane_off;
    const uint32_t tO = tmem + lane_off + 2 * BN;
    const int TLP = p.TL;
    float m_run = 0.f, l_run = 0.f;
    const float sc = p.scale;

    for (int j = 0; j < nt; ++j) {
      const int buf = j & 1;
      ptx::mbar_wait(&s_full[buf], (j >> 1) & 1);
      const bool trj = tr && threadIdx.x == 0 && j < kTrTiles;
      if (trj) tr[MBCI_TR(j, 0)] = ptx::globaltimer();
      ptx::tc_fence_after();
      uint32_t sr[BN];
      if (p.k_steps > 0) {
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) ptx::tmem_ld32(tS + buf * BN + c * 32, &sr[c * 32]);
        ptx::tmem_wait_ld();
      } else {
#pragma unroll
        for (int c = 0; c < BN; ++c) sr[c] = 0u;
      }
      float s[BN];
#pragma unroll
      for (int c = 0; c < BN; ++c) s[c] = __uint_as_float(sr[c]);
      if (trj) tr[MBCI_TR(j, 1)] = ptx::globaltimer_after(sr[BN - 1]);
      uint32_t pk[BN / 2];
      if (p.op == 2) {
        const int valid = row_lim - j * BN;  // >= BN for a full tile (this thread's row)
        const bool full = valid >= BN;
        // tile max of z = sc * S over valid keys (sc >= 0: max S; sc < 0: min S)
        float mx;
        if (full) {
          if (sc >= 0.f) {
            float m0v = s[0], m1v = s[1];
#pragma unroll
            for (int c = 2; c + 3 < BN; c += 4) {
              m0v = ptx::max3(m0v, s[c], s[c + 1]);
              m1v = ptx::max3(m1v, s[c + 2], s[c + 3]);
            }
            mx = ptx::max3(m0v, m1v, ptx::max3(s[BN - 2], s[BN - 1], s[0]));
          } else {
            float m0v = s[0], m1v = s[1];
#pragma unroll
            for (int c = 2; c + 3 < BN; c += 4) {
              m0v = ptx::min3(m0v, s[c], s[c + 1]);
              m1v = ptx::min3(m1v, s[c + 2], s[c + 3]);
            }
            mx = ptx::min3(m0v, m1v, ptx::min3(s[BN - 2], s[BN - 1], s[0]));
          }
        } else if (sc >= 0.f) {
          mx = -INFINITY;
#pragma unroll
          for (int c = 0; c < BN; ++c) mx = (c < valid) ? fmaxf(mx, s[c]) : mx;
        } else {
          mx = INFINITY;
#pragma unroll
          for (int c = 0; c < BN; ++c) mx = (c < valid) ? fminf(mx, s[c]) : mx;
        }
        const float m_tile = mx * sc;
        if (trj) tr[MBCI_TR(j, 2)] = ptx::globaltimer_after(__float_as_uint(mx));
        if (j == 0) {
          m_run = m_tile;
        } else {
          // warp-uniform decision (tcgen05.ld/st are warp-collective)
          const bool need = __any_sync(0xffffffffu, m_tile > m_run + kRescaleTau);
          if (need) {
            const float m_new = fmaxf(m_run, m_tile);
            const float alpha = ptx::ex2(m_run - m_new);
            l_run *= alpha;
            m_run = m_new;
            // G2(j-1) has landed in O.  Parity waits are only unambiguous one phase ahead:
            // s_full(j) completing implies G2(j-2) completed (tcgen05 ops retire in issue
            // order), so o_done has completed j-1 or j times here.
            ptx::mbar_wait(o_done, (j - 1) & 1);
            ptx::tc_fence_after();
            for (int c0 = 0; c0 < TLP; c0 += 16) {
              uint32_t r[16];
              ptx::tmem_ld16(tO + c0, r);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int q = 0; q < 16; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) * alpha);
              ptx::tmem_st16(tO + c0, r);
            }
          }
        }
        const float neg_m = -m_run;
        float ls = 0.f;
#pragma unroll
        for (int c = 0; c < BN / 2; ++c) {
          float p0 = ptx::ex2(fmaf(s[2 * c], sc, neg_m));
          float p1 = ptx::ex2(fmaf(s[2 * c + 1], sc, neg_m));
          if (!full) {
            p0 = (2 * c < valid) ? p0 : 0.f;
            p1 = (2 * c + 1 < valid) ? p1 : 0.f;
          }
          ls += p0 + p1;
          pk[c] = ptx::pack2<BF16>(p0, p1);
        }
        l_run += ls;
        if (trj) tr[MBCI_TR(j, 3)] = ptx::globaltimer_after(__float_as_uint(ls));
      } else if (p.op == 1) {
#pragma unroll
        for (int c = 0; c < BN / 2; ++c) pk[c] = ptx::pack2<BF16>(s[2 * c] * sc, s[2 * c + 1] * sc);
      } else if (p.op >= 3) {   // RELU / GELU of scale * S
#pragma unroll
        for (int c = 0; c < BN / 2; ++c)
          pk[c] = ptx::pack2<BF16>(ptx::act(p.op, s[2 * c] * sc), ptx::act(p.op, s[2 * c + 1] * sc));
      } else {
#pragma unroll
        for (int c = 0; c < BN / 2; ++c) pk[c] = ptx::pack2<BF16>(s[2 * c], s[2 * c + 1]);
      }
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) ptx::tmem_st32(tS + buf * BN + c * 32, &pk[c * 32]);
      ptx::tmem_wait_st();
      // consume o_done's phase for G2(j - 1) every tile (it completes once per G2; the rescale
      // above may already have waited on it): no phase goes unobserved, so parity waits stay
      // unambiguous and compute-sanitizer --tool synccheck finds no missing wait
      if (j >= 1) ptx::mbar_wait(o_done, (j - 1) & 1);
      ptx::tc_fence_before();
      ptx::mbar_arrive(&p_full[buf]);
      if (trj) tr[MBCI_TR(j, 4)] = ptx::globaltimer();
    }

    // ------------------------------------------------------------ epilogue
    if (nt > 0) {
      // o_done may still be two phases behind here, so the last G2 has its own barrier.
      ptx::mbar_wait(o_final, 0);
      ptx::tc_fence_after();
    }
    if (tr && threadIdx.x == 0) tr[kTrEpi] = ptx::globaltimer();
    float inv = (p.op == 2) ? (l_run > 0.f ? 1.0f / l_run : 0.f) : 1.0f;
    const int gm = m0 + row;
    if (p.lse != nullptr && p.op == 2 && ht == 0 && !p.c3 && gm < p.M)   // one h chunk writes it
      p.lse[static_cast<int64_t>(beta) * p.M + gm] = l_run > 0.f ? (m_run + log2f(l_run)) * 0.69314718055994531f : -INFINITY;
    uint32_t tOut = tO;
    int outc = TLP, ncols = min(TLP, p.L - h0), ecol0 = h0;
    if (p.c3) {
      // P2 = cvt(op2(scale2 · O / l)) into TMEM columns [0, TL/2) of S_0 (every G2 has completed)
      if (nt > 0) {
        for (int c0 = 0; c0 < TLP; c0 += 32) {
          uint32_t r[32], pk2[16];
          ptx::tmem_ld32(tO + c0, r);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            float v0 = __uint_as_float(r[2 * q]) * inv, v1 = __uint_as_float(r[2 * q + 1]) * inv;
            if (p.op2 != 0) {
              v0 = ptx::act(p.op2, p.scale2 * v0);
              v1 = ptx::act(p.op2, p.scale2 * v1);
            }
            pk2[q] = ptx::pack2<BF16>(v0, v1);
          }
          ptx::tmem_st16(tS + c0 / 2, pk2);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(p2_full);
        ptx::mbar_wait(e3_full, 0);
        ptx::tc_fence_after();
      }
      tOut = tmem + lane_off + 2 * BN + p.TL;
      outc = p.TH;
      ncols = min(p.TH, p.H - h3);
      ecol0 = h3;
      inv = 1.0f;
    }
    using T16 = uint16_t;
    T16* erow = reinterpret_cast<T16*>(p.E) + static_cast<int64_t>(beta) * p.bs_e +
                static_cast<int64_t>(gm) * p.ld_e + ecol0;
    for (int c0 = 0; c0 < outc; c0 += 16) {
      uint32_t r[16];
      if (nt > 0) {
        ptx::tmem_ld16(tOut + c0, r);
        ptx::tmem_wait_ld();
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) r[q] = 0u;
      }
      uint32_t w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        w[q] = ptx::pack2<BF16>(__uint_as_float(r[2 * q]) * inv, __uint_as_float(r[2 * q + 1]) * inv);
      if (gm < p.M) {
        if (c0 + 16 <= ncols) {
          uint4* dst = reinterpret_cast<uint4*>(erow + c0);
          dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
          dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        } else {
          for (int q = 0; q < 16 && c0 + q < ncols; ++q)
            erow[c0 + q] = static_cast<T16>((w[q >> 1] >> ((q & 1) * 16)) & 0xFFFFu);
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[kTrEnd] = ptx::globaltimer();
  if (warp == 5) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, p.tmem_cols);
  }
}

}  // namespace mbci
