// selector.cpp — host-side tile selector for the fused chain (no GPU needed).
//
// The paper's pipeline (§III-§IV) adapted to the one kernel structure this build
// ships (the flat expression mh(n(k(L_A,L_B,C_C),L_D,C_E),S_E) with k dead):
//   * candidates: tile sizes T_M = 128 (tcgen05 M), T_N = BN in {64,128}, T_K = K padded
//     to 16 (dead k loop), T_H = TL in multiples of 16 up to L padded
//     ("multiples of 16"), and a B200 pipeline depth (stages 2..4);
//   * Rule 3 (padding) on N and L; if it rejects every candidate the rule is
//     skipped (it is a pruning heuristic, not a legality rule — DESIGN.md R17);
//   * Rule 4 becomes the exact SMEM budget (<= smem_max) and the TMEM budget
//     (2*BN + TL <= 512 columns): sm_100 sizes are known, no 1.2 slack is needed;
//   * Eqs. (2)-(5) for every survivor (t_mem, t_comp, alpha, t_estm);
//   * a B200 score t_b200 = max(t_HBM, t_tensor, t_SFU, t_issue) x wave quantisation
//     + per-wave fixed latency, which the selector minimises (the paper's smooth alpha only
//     says "more blocks is better"; DESIGN.md §5 explains the extension).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/mbci.h"
#include "selector.h"

namespace mbci {

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

void model_terms(int64_t batch, int64_t M, int64_t N, int64_t K, int64_t L, int64_t TM,
                 int64_t TN, int64_t TK, int64_t TH, int32_t s, const mbci_hw_t& hw,
                 double out[5]) {
  const double b = static_cast<double>(batch);
  const double lm = static_cast<double>(cdiv(M, TM)), lh = static_cast<double>(cdiv(L, TH));
  const double ln = static_cast<double>(cdiv(N, TN)), lk = static_cast<double>(cdiv(K, TK));
  // Eq. (3): sum over Load/Store of TS x prod(Lp_set) / W
  const double la_trip = (lk == 1.0) ? b * lm : b * lm * lh * ln * lk;  // dead k: L_A -> m scope
  double mem = 0.0;
  mem += static_cast<double>(TM * TK * s) * la_trip;           // L_A
  mem += static_cast<double>(TK * TN * s) * b * lm * lh * ln * lk;  // L_B
  mem += static_cast<double>(TN * TH * s) * b * lm * lh * ln;  // L_D
  mem += static_cast<double>(TM * TH * s) * b * lm * lh;       // S_E (hoisted out of n)
  // Eq. (4): sum over Compute of Fp x prod(Lp_set) / P
  double comp = 0.0;
  comp += 2.0 * TM * TN * TK * (b * lm * lh * ln * lk);  // C_C
  comp += 2.0 * TM * TN * TH * (b * lm * lh * ln);       // C_E
  const double t_mem = mem / hw.W;
  const double t_comp = comp / hw.P;
  const double n_block = b * lm * lh;
  const double alpha = (n_block + hw.n_sm) / n_block;  // Eq. (5)
  out[0] = t_mem;
  out[1] = t_comp;
  out[2] = alpha;
  out[3] = (t_mem + t_comp) * alpha;  // Eq. (2)
  out[4] = n_block;
}

// PAPER.md:288 Rule 3.
bool rule3_reject(int64_t size, int64_t tile) {
  if (tile <= 0) return true;
  if (size % tile == 0) return false;
  if ((size & (size - 1)) == 0) return true;
  const double pad = static_cast<double>(cdiv(size, tile) * tile - size);
  return pad / static_cast<double>(size) >= 0.05;
}

int64_t tc_smem_bytes(int32_t k_steps, int32_t BN, int32_t TL, int32_t stages, int32_t b_layout,
                      int32_t* a_bytes, int32_t* b_stage, int32_t* d_stage) {
  const int32_t kp = 16 * k_steps;
  const int32_t kch = std::max<int32_t>(1, static_cast<int32_t>(cdiv(kp, 64)));
  const int32_t dch = static_cast<int32_t>(cdiv(TL, 64));
  const bool stream = k_steps > 8;   // K > 128: live k loop, ring entry = A chunk + B chunk (64 columns)
  const int32_t a = (k_steps > 0 && !stream) ? kch * 16384 : 0;
  const int32_t b = k_steps == 0 ? 0
                    : stream     ? 16384 + BN * 128
                                 : (b_layout == 1 ? kch * BN * 128 : (BN / 64) * kp * 128);
  const int32_t d = dch * BN * 128;
  if (a_bytes) *a_bytes = a;
  if (b_stage) *b_stage = b;
  if (d_stage) *d_stage = d;
  const int32_t n_bars = 1 + 4 * stages + 4 + 2;
  return static_cast<int64_t>(a) + static_cast<int64_t>(stages) * (b + d) + 8 * n_bars + 16 +
         1024;  // + alignment slack for the 1024-B swizzle atoms
}

bool tc4_layout(int32_t k_steps, int32_t TL, int32_t stages, int32_t b_layout, Tc4Layout* out,
                int32_t smem_max) {
  if (TL > 128 || k_steps < 1) return false;   // TMEM: NSB S buffers + O_0, O_1
  if (TL <= 64 && stages < 3) return false;      // NSB = 3 releases K/V slot g at tile g + 2
  int32_t a, b, d;
  tc_smem_bytes(k_steps, 128, TL, stages, b_layout, &a, &b, &d);
  for (int32_t q_bufs = 2; q_bufs >= 1; --q_bufs) {
    const int32_t bars = 8 * (18 + 2 * stages);
    const int32_t total = q_bufs * 2 * a + stages * (b + d) + bars + 1024;
    if (total + 5120 <= smem_max) {   // 4 KB of (l, m) + slack stay for static shared memory
      if (out) *out = Tc4Layout{a, b, d, q_bufs, total};
      return true;
    }
  }
  return false;
}

bool tc5_layout(int32_t k_steps, int32_t TL, int32_t stages, int32_t b_layout, Tc4Layout* out,
                int32_t smem_max) {
  // TMEM: S_0, S_1 (128 columns) + P_0, P_1 (64) + O_0, O_1 (64) = 512 columns, so L <= 64
  if (TL > 64 || k_steps < 1 || stages < 2) return false;
  int32_t a, b, d;
  tc_smem_bytes(k_steps, 128, TL, stages, b_layout, &a, &b, &d);
  for (int32_t q_bufs = 2; q_bufs >= 1; --q_bufs) {
    const int32_t bars = 8 * (20 + 2 * stages);
    const int32_t e_stage = 16384;   // E staging for the TMA-store epilogue (128 rows x 128 B)
    const int32_t total = q_bufs * 2 * a + stages * (b + d) + e_stage + bars + 1024;
    if (total + 5120 <= smem_max) {   // 4 KB of (l, m) + slack stay for static shared memory
      if (out) *out = Tc4Layout{a, b, d, q_bufs, total};
      return true;
    }
  }
  return false;
}

int32_t tmem_alloc_cols(int32_t BN, int32_t TL) {
  const int32_t need = 2 * BN + TL;
  int32_t c = 32;
  while (c < need) c <<= 1;
  return c;
}

bool tc_eligible(const mbci_chain_desc_t& d) {
  if (d.dtype != MBCI_F16 && d.dtype != MBCI_BF16) return false;
  if (d.K > kMaxK || d.L > kMaxL) return false;
  // TMA: every row / batch stride a multiple of 16 bytes (8 elements)
  const int64_t strides[8] = {d.ld_a, d.ld_b, d.ld_d, d.ld_e, d.bs_a, d.bs_b, d.bs_d, d.bs_e};
  for (int64_t v : strides)
    if (v % 8 != 0) return false;
  if (d.M > (int64_t(1) << 31) - 256 || d.N > (int64_t(1) << 31) - 256) return false;
  return true;
}

// Round-1 measurement: kernel 0 runs ~2.2-2.6x slower than the roofline-style score below
// (C2 24.3 vs 9.3 us); the persistent kernels 4 and 5 are scored from their measured per-tile
// cost.  The common factor keeps the two kinds of score comparable.
constexpr double kModelToB200 = 2.4;

static void score_b200(const mbci_chain_desc_t& d, const mbci_hw_t& hw, mbci_plan_t& p) {
  const int32_t s = (d.dtype == MBCI_F32) ? 4 : 2;
  const double b = static_cast<double>(d.batch);
  const double bytes = b * static_cast<double>(d.M * d.K + d.K * d.N + d.N * d.L + d.M * d.L) * s;
  const double t_hbm = bytes / hw.W;
  const int64_t lm = cdiv(d.M, p.BM), lh = cdiv(d.L, p.TL), nt = cdiv(d.N, p.BN);
  const double rows = static_cast<double>(lm * p.BM), keys = static_cast<double>(nt * p.BN);
  double t_tc, t_sfu = 0.0, t_issue;
  const double elems = b * static_cast<double>(lh) * rows * keys;  // C elements computed
  if (p.kernel != 1) {   // every tcgen05 family
    t_tc = b * lh * 2.0 * rows * keys * (p.TK + p.TL) / hw.P;
    if (d.op == MBCI_OP_SOFTMAX) t_sfu = elems / (hw.n_sm * hw.sfu_per_clk_sm * hw.clock_hz);
    const double instr = (d.op == MBCI_OP_SOFTMAX) ? 5.0 : 1.5;  // thread-instructions/element
    t_issue = elems * instr / (hw.n_sm * 128.0 * hw.clock_hz);
  } else {
    // CUDA cores: 2 FMAs per (m,n,k) and (m,n,l), 128 FMA lanes per SM
    t_tc = b * 2.0 * d.M * d.N * (d.K + d.L) / (hw.n_sm * 256.0 * hw.clock_hz);
    t_issue = t_tc;
  }
  if (p.kernel == 4 || p.kernel == 5 || p.kernel == 6) {
    // persistent pair units dealt round-robin (ceil(units / n_sm) rounds per SM).
    const int64_t units = b == 0 ? 0 : static_cast<int64_t>(b) * cdiv(d.M, 256);
    const int64_t ntm = std::max<int64_t>(1, nt);
    const int64_t rounds = units / hw.n_sm, rem = units % hw.n_sm;
    // a last round of <= n_sm / 2 units runs as half items (keys split over the two slots)
    const bool halves = rem > 0 && 2 * rem <= hw.n_sm && ntm % 2 == 0 && d.mask == MBCI_MASK_NONE &&
                        p.stages >= (p.TL <= 64 ? 4 : 3);
    const int64_t tail_tiles = rem > 0 ? (halves ? ntm / 2 : ntm) : 0;
    // Calibrated on B200 (tools/trace_chain4.py): one 256 x 128 score tile of a pair unit costs
    // (kernel 4) ~0.75 us + 6 ns per unit of (K + L) (d = 64: 1.5 us, d = 128: 2.3 us) on an SM,
    // (kernel 5, separate P) ~0.35 us + 5 ns per unit of (K + L) (d = 64: 1.0 us), plus ~3 us of
    // prologue / epilogue per launch (~2 us with programmatic dependent launch, kernel 5).
    // NONE / SCALE (no exponentials): the issuer and tensor pipe bound the tile.
    const double kd = static_cast<double>(p.TK + p.TL);
    double t_pair;
    if (p.kernel == 4)
      t_pair = d.op == MBCI_OP_SOFTMAX ? 0.75e-6 + 6.0e-9 * kd : 0.15e-6 + 4.0e-9 * kd;
    else
      t_pair = d.op == MBCI_OP_SOFTMAX ? 0.35e-6 + 5.0e-9 * kd : 0.12e-6 + 3.0e-9 * kd;
    t_pair *= 1.965e9 / hw.clock_hz;
    // kernel 6 measures within noise of kernel 5 on softmax and slower on NONE / SCALE
    // (round 2, profiles/r2_k5_k6_prefetch_ab.txt): it ranks just behind kernel 5
    if (p.kernel == 6) t_pair *= 1.001;
    const double fixed = p.kernel >= 5 ? 2.0e-6 : 3.0e-6;
    // Ties go to the deeper ring: softmax up to the 4 stages that keep two Q buffers at d = 64;
    // the linear ops (long items, no exponentials) to the deepest ring that still keeps two Q
    // buffers (kernel 5 on C4 K = L = 16: 4 -> 7 stages 44.8 -> 43.0 us, profiles/r2_k5_ring_sweep.txt).
    int32_t pref = std::min<int32_t>(p.stages, 4);
    if (p.kernel >= 5 && d.op != MBCI_OP_SOFTMAX) {
      Tc4Layout lay;
      pref = (tc5_layout(p.TK / 16, p.TL, p.stages, d.b_layout, &lay, hw.smem_max) && lay.q_bufs == 2) ? p.stages : 0;
    }
    p.t_b200 = std::max(t_hbm, static_cast<double>(rounds * ntm + tail_tiles) * t_pair) + fixed -
               1e-12 * pref + (p.kernel == 6 ? 1e-9 : 0.0);
    return;
  }
  int32_t occ = 1;
  if (p.kernel == 0) {
    occ = std::max<int32_t>(1, std::min<int32_t>(hw.smem_max / std::max<int32_t>(1, p.smem_bytes),
                                                 hw.tmem_cols / std::max<int32_t>(1, p.tmem_cols)));
    occ = std::min<int32_t>(occ, 2);
  } else {
    occ = 8;
  }
  const double slots = static_cast<double>(hw.n_sm) * occ;
  const double waves = std::ceil(static_cast<double>(p.n_block) / slots);
  const double q = p.n_block > 0 ? waves * slots / static_cast<double>(p.n_block) : 1.0;
  const double t_fixed = waves * 1.0e-6 / occ;  // prologue + epilogue latency per wave
  p.t_b200 = (std::max(std::max(t_hbm, t_tc), std::max(t_sfu, t_issue)) * q + t_fixed) * kModelToB200;
}

static void fill_model(const mbci_chain_desc_t& d, const mbci_hw_t& hw, int32_t s, mbci_plan_t& p) {
  double t[5];
  model_terms(d.batch, d.M, d.N, d.K, d.L, p.BM, p.BN, p.TK, p.TL, s, hw, t);
  p.t_mem = t[0];
  p.t_comp = t[1];
  p.alpha = t[2];
  p.t_estm = t[3];
  p.n_block = static_cast<int64_t>(t[4]);
  score_b200(d, hw, p);
}

int enumerate_plans(const mbci_chain_desc_t& d, const mbci_hw_t& hw,
                    std::vector<mbci_plan_t>& out, bool rule3) {
  out.clear();
  const int32_t s = (d.dtype == MBCI_F32) ? 4 : 2;
  if (tc_eligible(d)) {
    const int32_t k_steps = static_cast<int32_t>(cdiv(d.K, 16));
    const int32_t lpad = static_cast<int32_t>(std::max<int64_t>(16, cdiv(d.L, 16) * 16));
    // Persistent families (kernels 5 and 4): one 128-key tile per step with the ragged last
    // tile masked and only the L real columns stored, so Rule 3's padding waste
    // does not apply to them; they need K >= 1 (a live G1) and N >= 1.
    if (k_steps >= 1 && k_steps <= 8 && d.N >= 1) {   // K <= 128: Q tiles resident (dead k loop)
      for (int kern : {6, 5, 4}) {
        if (kern == 6 && (d.mask & MBCI_MASK_CAUSAL)) continue;   // kernel 6 has no causal rows
        for (int32_t st = 2; st <= 8; ++st) {
          Tc4Layout lay;
          const bool ok = kern >= 5 ? tc5_layout(k_steps, lpad, st, d.b_layout, &lay, hw.smem_max)
                                    : tc4_layout(k_steps, lpad, st, d.b_layout, &lay, hw.smem_max);
          if (!ok) continue;
          mbci_plan_t p{};
          p.kernel = kern;
          p.BM = 256;
          p.BN = 128;
          p.TK = 16 * k_steps;
          p.TL = lpad;
          p.stages = st;
          p.smem_bytes = lay.smem_total;
          p.tmem_cols = 512;
          fill_model(d, hw, s, p);
          out.push_back(p);
        }
      }
    }
    // Kernel 0 (one CTA per 128-row m tile and h chunk; also the K = 0 chain): the paper's
    // space of BN and TL with Rule 3 (skipped if it rejects every tile, R17).
    const size_t n0 = out.size();
    for (int pass = 0; pass < 2 && out.size() == n0; ++pass) {
      const bool apply_rule3 = rule3 && (pass == 0);
      for (int32_t BN : {64, 128}) {
        if (apply_rule3 && d.N > 0 && rule3_reject(d.N, BN)) continue;
        for (int32_t TL = 16; TL <= std::min<int32_t>(lpad, 128); TL += 16) {   // L > 128: h chunks on the grid
          if (apply_rule3 && d.L > 0 && rule3_reject(d.L, TL)) continue;
          if (2 * BN + TL > hw.tmem_cols) continue;  // TMEM budget
          for (int32_t st = 2; st <= 4; ++st) {
            const int64_t smem = tc_smem_bytes(k_steps, BN, TL, st, d.b_layout, nullptr, nullptr, nullptr);
            if (smem > hw.smem_max) continue;  // exact SMEM budget (Rule 4 on sm_100)
            mbci_plan_t p{};
            p.kernel = 0;
            p.BM = 128;
            p.BN = BN;
            p.TK = std::max<int32_t>(16, 16 * k_steps);
            p.TL = TL;
            p.stages = st;
            p.smem_bytes = static_cast<int32_t>(smem);
            p.tmem_cols = tmem_alloc_cols(BN, TL);
            fill_model(d, hw, s, p);
            out.push_back(p);
          }
        }
      }
    }
  } else {
    // fp32 on tcgen05 (kernel 7, 3xTF32, chain_tf32.cuh): one CTA per (β, 128-row tile), 64-key
    // tiles for K, L <= 64 and 32-key tiles up to K, L <= 128, any strides.  Scored from its synchronous per-tile structure (load +
    // split, GEMM1, op, GEMM2 ~1.2 us per tile on a CTA) and ranked ahead of the CUDA-core path.
    const bool tf32_ok = d.dtype == MBCI_F32 && d.K >= 1 && d.K <= 128 && d.L <= 128 && d.N >= 1 &&
                         d.batch * cdiv(d.M, 128) <= (int64_t(1) << 31) - 1;
    const bool tf32_wide = d.K > 64 || d.L > 64;   // 32-key tiles, 128 O columns
    if (tf32_ok) {
      mbci_plan_t p{};
      p.kernel = 7;
      p.BM = 128;
      p.BN = tf32_wide ? 32 : 64;
      p.TK = static_cast<int32_t>(cdiv(d.K, 8) * 8);
      p.TL = static_cast<int32_t>(std::max<int64_t>(16, cdiv(d.L, 16) * 16));
      p.stages = 1;
      p.smem_bytes = tf32_wide ? 2 * (4 * 128 * 128 + 4 * 32 * 128 + 1 * 128 * 128) + 1024
                               : 2 * (2 * 128 * 128 + 2 * 64 * 128 + 2 * 64 * 128) + 1024;
      p.tmem_cols = 256;
      double t[5];
      model_terms(d.batch, d.M, d.N, d.K, d.L, 128, p.BN, p.TK, p.TL, s, hw, t);
      p.t_mem = t[0];
      p.t_comp = t[1];
      p.alpha = t[2];
      p.t_estm = t[3];
      p.n_block = d.batch * cdiv(d.M, 128);
      const double waves = std::ceil(static_cast<double>(p.n_block) / hw.n_sm);
      p.t_b200 = waves * static_cast<double>(cdiv(d.N, p.BN)) * 1.2e-6 * (1.965e9 / hw.clock_hz) + 3.0e-6;
      out.push_back(p);
    }
    const int64_t smem = d.N * 4 + 64;
    if (smem <= hw.smem_max) {
      mbci_plan_t p{};
      p.kernel = 1;
      p.BM = 1;
      p.BN = static_cast<int32_t>(std::max<int64_t>(1, d.N));
      p.TK = static_cast<int32_t>(std::max<int64_t>(1, d.K));
      p.TL = static_cast<int32_t>(std::max<int64_t>(1, d.L));
      p.stages = 1;
      p.smem_bytes = static_cast<int32_t>(smem);
      p.tmem_cols = 0;
      double t[5];
      model_terms(d.batch, d.M, d.N, d.K, d.L, 1, std::max<int64_t>(1, d.N),
                  std::max<int64_t>(1, d.K), std::max<int64_t>(1, d.L), s, hw, t);
      p.t_mem = t[0];
      p.t_comp = t[1];
      p.alpha = t[2];
      p.t_estm = t[3];
      p.n_block = static_cast<int64_t>(t[4]);
      score_b200(d, hw, p);
      if (tf32_ok) p.t_b200 += 1.0;   // the CUDA-core path is the fallback once kernel 7 is legal
      out.push_back(p);
    }
  }
  std::stable_sort(out.begin(), out.end(), [](const mbci_plan_t& a, const mbci_plan_t& b) {
    if (a.t_b200 != b.t_b200) return a.t_b200 < b.t_b200;
    return a.t_estm < b.t_estm;
  });
  return static_cast<int>(out.size());
}

void hw_default(mbci_hw_t* hw) {
  hw->W = 6534.8e9;     // measured copy bandwidth on this pool's B200 (MEASURED_PEAKS.json)
  hw->P = 1637.0e12;    // measured cuBLAS bf16 burst (MEASURED_PEAKS.json)
  hw->n_sm = 148;
  hw->smem_max = 232448;
  hw->tmem_cols = 512;
  hw->sfu_per_clk_sm = 16.0;
  hw->clock_hz = 1.965e9;
}

}  // namespace mbci
