// chain_tc5.cuh — persistent ping-pong fused chain E = op(A·B)·D on sm_100a, head dims <= 64,
// with a separate P buffer per slot (the default kernel for L <= 64).
//
// Same arithmetic and work layout as chain_tc4.cuh (mbci.h; PAPER.md:196 chain, :498 softmax
// between the GEMMs, :489 batched layout; units = (β, pair of 128-row m tiles) bound to a
// persistent grid, PAPER.md:285 Rule 1; k loop dead for K <= 128; S_E hoisted,
// PAPER.md:232-233; half items for the last partial round).  What differs is the TMEM layout
// and, from it, the dependency graph of a step:
//
//   kernel 4 (d <= 64):  three 128-column S buffers rotated over both slots, P aliasing S.  The
//     next S tile of slot x can only be written once the OTHER slot's G2 has read the P that
//     occupies the buffer, so a slot's next score tile waits for p_full(1-x) -> G2 -> G1 ->
//     s_full: ~0.5 us of every 1.5 us step on C2 (round-2 trace, profiles/r2_SUMMARY.md).
//   kernel 5:  S_0, S_1 (128 columns each), P_0, P_1 (64 columns of packed 16-bit P each),
//     O_0, O_1 (64 columns each) = 512 columns.  S_x is released (s_free) as soon as softmax x
//     has the row in registers, so G1(x, j+1) runs while softmax x computes the exponentials of
//     tile j; P_x is released (p_free) by the commit after G2(x, j).  Each slot's chain only
//     involves its own buffers, so the two slots no longer serialise each other.
//
// One tcgen05 issuer thread per slot (warps 12 and 14), each in its own order, per step g:
//     wait s_free(x, g) -> G1(x, g + 1) -> commit s_full(x)
//     wait p_full(x, g) -> G2(x, g)     -> commit p_free(x) [+ kv_empty, o_full]
// (flags bit 8, the default: event-driven — both hand-offs polled, G1 and G2 issued in whichever
// order their inputs complete, so a late K tile no longer holds back the G2 the softmax waits on)
// so neither slot's next score tile waits behind the other slot's hand-offs (a single issuer
// serialising both slots cost ~0.45 us per step on C2: it blocked on the full MMA issue queue
// after each G2 before it could issue the other slot's G1).  Deadlock-free: every wait is for
// work whose own inputs were issued earlier in the same slot's order; a K/V entry is released
// after both readers' commits (kv_empty counts 2), Q after both slots' last G1 (q_empty 2).
//
// Softmax: 8 warps, warp w serves slot x = w >> 2 and TMEM lane quadrant q = w & 3 (rows 32q ..
// 32q + 31): a whole 128-column S row per thread in registers (setmaxnreg 184).  Exp-phase turns
// (flags bit 0): warp w of slot 0 and warp w + 4 of slot 1 share SMSP q; their exponential
// phases alternate (named barriers 1-4: slot 0's turn, 5-8: slot 1's), so the MUFU serves one
// warp at a time while the other loads S and takes its row max.  In isolation one warp reaches
// 14.5 ex2/clk/SM with 2/8 of the pairs on the FMA-pipe polynomial (tools/exp_sched_bench.cu).
// The single-thread roles (issuers, TMA) wait with mbarrier.try_wait, which suspends the thread,
// instead of spinning on test_wait: a spinning thread takes issue slots from the softmax warp of
// its SMSP (flags bit 2 restores spinning, for A/B measurements).
//
// Epilogue (warps 8-11): E = O / l packed to 16 bits into a 128-B-swizzled shared tile and
// written by one TMA bulk tensor store per 128-row tile (per-thread 16-B global stores from
// the epilogue warps stretched the softmax warps' MUFU phases ~2x on the shared MIO queue).
//
// P_x hand-off: with the event-driven issuers (flags bit 8) G2 of the previous step has long
// released P_x when a step's exponentials start, so (flags bit 12, the default) the softmax waits
// for p_free first and stores each 16-column chunk of P as soon as it is computed (16 packed
// registers live instead of 64).  Without bit 12 the exponentials go to registers and the wait
// comes only before P is written (the order that paid with the in-order issuers).  A lazy rescale
// of O_x waits first either way.
//
// Programmatic dependent launch: every CTA lets the next grid of the stream be scheduled at
// once (griddepcontrol.launch_dependents) and waits for its prerequisite grids before its
// first global-memory access (griddepcontrol.wait), so barrier initialisation, TMEM
// allocation and descriptor prefetch of step i + 1 overlap the tail of step i.
//
// Warps: 0-7 softmax | 8-11 epilogue | 12 tcgen05 issuer of slot 0 + TMEM allocator | 13 TMA
//        producer | 14 tcgen05 issuer of slot 1 | 15 idle.  setmaxnreg: 184 / 80 / 64.
#pragma once
#include "chain_tc4.cuh"

namespace mbci {

constexpr uint32_t kT5PCol = 256;   // P_0 at 256, P_1 at 320
constexpr uint32_t kT5OCol = 384;   // O_0 at 384, O_1 at 448

constexpr uint32_t kT5EStage = 16384;   // E staging: 128 rows x 128 B (64 16-bit columns), 128-B swizzle
constexpr int kT5Threads = 512;

// t4_exp_row (chain_tc4.cuh) with the exp-phase hand-over folded in: after chunk `arrive_after`
// (of 4 chunks of 16 column pairs) the other slot's warp of this SMSP may start its turn
// (bar != 0), so the two warps overlap on the MUFU for the remaining chunks.  The packed 16-bit
// P row stays in registers (`pk`, 64 words: the S registers die as the pairs are consumed) and is
// written to TMEM by the caller once G2 of the previous step has released P_x — so the
// exponentials of step g overlap G2(g - 1) instead of waiting for it.
template <bool BF16, int EMU, bool MASKED>
__device__ __forceinline__ void t5_exp_row(uint32_t (&pk)[64], const uint32_t (&sr)[kT4BN], float sc, float m,
                                           int valid, float2& l2a, float2& l2b, int arrive_after, uint32_t bar) {
  const float2 sc2 = make_float2(sc, sc);
  const float2 nm2 = make_float2(-m, -m);
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int cp = ch * 16 + c;
      const float2 z = __ffma2_rn(make_float2(__uint_as_float(sr[2 * cp]), __uint_as_float(sr[2 * cp + 1])), sc2, nm2);
      float2 e;
      if (EMU > 0 && ((cp * EMU) & 7) < EMU) {
        e = t4_exp2_poly(z);
      } else {
        e.x = ptx::ex2(z.x);
        e.y = ptx::ex2(z.y);
      }
      if (MASKED) {
        e.x = (2 * cp < valid) ? e.x : 0.f;
        e.y = (2 * cp + 1 < valid) ? e.y : 0.f;
      }
      if (c & 1) l2b = __fadd2_rn(l2b, e); else l2a = __fadd2_rn(l2a, e);
      pk[cp] = ptx::pack2<BF16>(e.x, e.y);
    }
    if (bar != 0 && ch == arrive_after) ptx::named_bar_arrive(bar, 64);
  }
}

// NONE / SCALE / RELU / GELU: the packed 16-bit row of op(s·S) into registers (the caller stores it
// once G2 of the previous step has released P_x)
template <bool BF16, bool ACT, bool SCALED = true>
__device__ __forceinline__ void t5_cvt_row_impl(uint32_t (&pk)[64], const uint32_t (&sr)[kT4BN], float sc, int op) {
  const float2 sc2 = make_float2(sc, sc);
#pragma unroll
  for (int cp = 0; cp < 64; ++cp) {
    float2 z;
    if constexpr (SCALED)
      z = __fmul2_rn(make_float2(__uint_as_float(sr[2 * cp]), __uint_as_float(sr[2 * cp + 1])), sc2);
    else   // NONE (scale 1): P = cvt(S), no multiply
      z = make_float2(__uint_as_float(sr[2 * cp]), __uint_as_float(sr[2 * cp + 1]));
    if constexpr (ACT) {
      z.x = ptx::act(op, z.x);
      z.y = ptx::act(op, z.y);
    }
    pk[cp] = ptx::pack2<BF16>(z.x, z.y);
  }
}
template <bool BF16, bool NOMUL_NONE>
__device__ __forceinline__ void t5_cvt_row(uint32_t (&pk)[64], const uint32_t (&sr)[kT4BN], float sc, int op) {
  if (op >= 3) t5_cvt_row_impl<BF16, true>(pk, sr, sc, op);   // one uniform branch per tile
  else if (NOMUL_NONE && op == 0) t5_cvt_row_impl<BF16, false, false>(pk, sr, sc, op);
  else t5_cvt_row_impl<BF16, false>(pk, sr, sc, op);
}

// As t5_exp_row, but each chunk's 16 packed P words go to TMEM (P_x, already released by G2 of the
// previous step) as soon as they are computed: 16 packed registers live instead of 64 (flags bit 12)
template <bool BF16, int EMU, bool MASKED>
__device__ __forceinline__ void t5_exp_row_st(uint32_t tP, const uint32_t (&sr)[kT4BN], float sc, float m, int valid,
                                              float2& l2a, float2& l2b, int arrive_after, uint32_t bar) {
  const float2 sc2 = make_float2(sc, sc);
  const float2 nm2 = make_float2(-m, -m);
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    uint32_t pk[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int cp = ch * 16 + c;
      const float2 z = __ffma2_rn(make_float2(__uint_as_float(sr[2 * cp]), __uint_as_float(sr[2 * cp + 1])), sc2, nm2);
      float2 e;
      if (EMU > 0 && ((cp * EMU) & 7) < EMU) {
        e = t4_exp2_poly(z);
      } else {
        e.x = ptx::ex2(z.x);
        e.y = ptx::ex2(z.y);
      }
      if (MASKED) {
        e.x = (2 * cp < valid) ? e.x : 0.f;
        e.y = (2 * cp + 1 < valid) ? e.y : 0.f;
      }
      if (c & 1) l2b = __fadd2_rn(l2b, e); else l2a = __fadd2_rn(l2a, e);
      pk[c] = ptx::pack2<BF16>(e.x, e.y);
    }
    ptx::tmem_st16(tP + ch * 16, pk);
    if (bar != 0 && ch == arrive_after) ptx::named_bar_arrive(bar, 64);
  }
}

// P_x <- the packed row (64 columns of 16-bit pairs), 16 columns per tcgen05.st
__device__ __forceinline__ void t5_store_p(uint32_t tP, const uint32_t (&pk)[64]) {
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) ptx::tmem_st16(tP + ch * 16, &pk[ch * 16]);
}

// L2 prefetch of this CTA's first items (Q tiles and every K/V tile they read), up to
// p.pf_bytes, issued by the TMA thread BEFORE griddepcontrol.wait: with programmatic dependent
// launch the CTA is resident while the previous grid drains, so the HBM latency of its first
// loads overlaps that tail (L2 is coherent: the loads after the wait still see the previous
// grid's writes).  Key padding is ignored here (valid_len may be written by the previous grid).
template <int KCH, int BL>
__device__ __forceinline__ void t5_prefetch_l2(const Tc4Params& p, const CUtensorMap* tmA, const CUtensorMap* tmB,
                                               const CUtensorMap* tmD) {
  int64_t bytes = 0;
  const int ntv = (p.N + kT4BN - 1) / kT4BN;
  for (int i = blockIdx.x; i < p.items && bytes < p.pf_bytes; i += gridDim.x) {
    T4Item it;
    it.decode(p, i);
    const int beta = it.u / p.l_mp;
    const int m0 = (it.u - beta * p.l_mp) * 256 + (it.half > 0 ? 128 : 0);
    const int nq = (it.half < 0 && m0 + 128 < p.M) ? 2 : 1;
    for (int x = 0; x < nq; ++x)
#pragma unroll
      for (int c = 0; c < KCH; ++c) ptx::tma_prefetch_l2_3d(tmA, c * 64, m0 + x * 128, beta);
    bytes += nq * p.q_bytes;
    for (int t = 0; t < ntv && bytes < p.pf_bytes; ++t) {
      if constexpr (BL == 1) {
#pragma unroll
        for (int c = 0; c < KCH; ++c) ptx::tma_prefetch_l2_3d(tmB, c * 64, t * kT4BN, beta);
      } else {
#pragma unroll
        for (int c = 0; c < kT4BN / 64; ++c) ptx::tma_prefetch_l2_3d(tmB, t * kT4BN + c * 64, 0, beta);
      }
      ptx::tma_prefetch_l2_3d(tmD, 0, t * kT4BN, beta);
      bytes += p.b_stage_bytes + p.d_stage_bytes;
    }
  }
}

template <bool BF16, int KCH, int BL, int EMU>
__global__ void __launch_bounds__(kT5Threads, 1)
    k_chain_tc5(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmE,
                const Tc4Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ uint32_t tmem_base_slot;
  __shared__ float l_sm[2][2][128];   // [slot][active-item parity][row]: row sum of p
  __shared__ float m_sm[2][2][128];   // [slot][parity][row]: running max (log2) the p were taken against

  const int S = p.stages;
  const uint32_t kv_stage = p.b_stage_bytes + p.d_stage_bytes;
  uint8_t* sQ = smem;                                      // [q_bufs][2][q_bytes]
  uint8_t* sKV = sQ + p.q_bufs * 2 * p.q_bytes;            // [S][K | V]
  uint8_t* sE = sKV + S * kv_stage;                        // E staging (TMA-store epilogue)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sE + kT5EStage);
  uint64_t* q_full = bars;          // [2]
  uint64_t* q_empty = bars + 2;     // [2]
  uint64_t* o_full = bars + 4;      // [2] last G2_x of an item completed
  uint64_t* o_free = bars + 6;      // [2] epilogue read O_x (128 arrivals)
  uint64_t* l_full = bars + 8;      // [2] softmax x published l (one arrival per warp: 4)
  uint64_t* l_free = bars + 10;     // [2] epilogue read l_sm[x][ai & 1] (128 arrivals)
  uint64_t* s_full = bars + 12;     // [2] G1_x landed in S_x (commit)
  uint64_t* s_free = bars + 14;     // [2] softmax x holds S_x in registers (one arrival per warp: 4)
  uint64_t* p_full = bars + 16;     // [2] softmax x wrote P_x (one arrival per warp: 4)
  uint64_t* p_free = bars + 18;     // [2] G2_x read P_x and updated O_x (commit)
  uint64_t* kv_full = bars + 20;    // [S] K_g and V_g landed
  uint64_t* kv_empty = kv_full + S; // [S] the G2s reading the entry completed (two commits)

  const int warp = threadIdx.x >> 5;
  // The linear ops NONE / SCALE / RELU / GELU run their own instantiation (EMU < 0), which carries
  // only the linear path (no scale-1 multiply for NONE).  The softmax instantiations (EMU >= 0) keep
  // the code they were tuned with: code placement alone moved C2 from 17.4 to 18.1-18.6 us when the
  // linear path changed or was compiled out of them (profiles/r2_k5_layout_ab.txt)
  constexpr bool kLinear = EMU < 0;
  const int lin_op = p.op == 2 ? 0 : p.op;
#define MBCI_T5_OP (kLinear ? lin_op : p.op)
  // Work-skipping diagnostics (MBCI_T4_DEBUG, trace build only; results are wrong by design):
  // 1 softmax and 16 epilogue keep only their barrier protocol, 2 / 4 the issuers skip the G2 / G1
  // MMAs (commits stay), 64 "TMA only": the issuers release each ring entry as soon as it lands
  // and every other role idles, 128 the softmax ignores s_full / p_free (free-running, timing only).
#if MBCI_TRACE
  const int dbg = p.dbg;
#else
  constexpr int dbg = 0;
#endif
#if MBCI_TRACE
  uint64_t* tr = p.trace ? p.trace + static_cast<int64_t>(blockIdx.x) * kT4TraceSlots : nullptr;
#else
  constexpr uint64_t* tr = nullptr;
#endif
  if (tr && threadIdx.x == 0) {
    tr[0] = ptx::globaltimer();
    tr[4] = t4_clk();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[2] = smid;
  }
  if (threadIdx.x == 0) ptx::grid_dep_launch();
  auto load_entry = [&](int s, int tile, int beta) {
    uint8_t* kdst = sKV + s * kv_stage;
    uint8_t* vdst = kdst + p.b_stage_bytes;
    ptx::mbar_arrive_expect_tx(&kv_full[s], p.b_stage_bytes + p.d_stage_bytes);
    if constexpr (BL == 1) {
#pragma unroll
      for (int c = 0; c < KCH; ++c)
        ptx::tma_load_3d(kdst + c * (kT4BN * 128), &tmB, &kv_full[s], c * 64, tile * kT4BN, beta);
    } else {
#pragma unroll
      for (int c = 0; c < kT4BN / 64; ++c)
        ptx::tma_load_3d(kdst + c * (p.kp_rows * 128), &tmB, &kv_full[s], tile * kT4BN + c * 64, 0, beta);
    }
    ptx::tma_load_3d(vdst, &tmD, &kv_full[s], 0, tile * kT4BN, beta);   // L <= 64: one 64-column box
  };
  auto load_q = [&](int qb, int m0, int beta, bool two) {
    ptx::mbar_arrive_expect_tx(&q_full[qb], (two ? 2u : 1u) * p.q_bytes);
    for (int x = 0; x < (two ? 2 : 1); ++x) {
      uint8_t* dst = sQ + (qb * 2 + x) * p.q_bytes;
#pragma unroll
      for (int c = 0; c < KCH; ++c)
        ptx::tma_load_3d(dst + c * 16384, &tmA, &q_full[qb], c * 64, m0 + x * 128, beta);
    }
  };
  // The TMA warp initialises the barriers; the first item's Q and ring entries go out before
  // the CTA-wide barrier (after the prerequisite grid completed), overlapping TMEM allocation.
  int pre_entries = 0;
  if (warp == 13 && ptx::elect_one()) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 2);   // each slot's issuer commits after its last G1
      ptx::mbar_init(&o_full[i], 1);
      ptx::mbar_init(&o_free[i], 128);
      ptx::mbar_init(&l_full[i], 4);
      ptx::mbar_init(&l_free[i], 128);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 4);
      ptx::mbar_init(&p_full[i], 4);
      ptx::mbar_init(&p_free[i], 1);
    }
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 2);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    ptx::tma_prefetch(&tmD);
    if (p.pf_bytes > 0) t5_prefetch_l2<KCH, BL>(p, &tmA, &tmB, &tmD);
    ptx::grid_dep_wait();
    for (int i = blockIdx.x; i < p.items; i += gridDim.x) {
      T4Item it;
      it.decode(p, i);
      const int beta = it.u / p.l_mp;
      const int m0 = (it.u - beta * p.l_mp) * 256 + (it.half > 0 ? 128 : 0);
      const int nt = it.tiles(t4_unit_nlim(p, it.u));
      if (nt == 0) continue;
      load_q(0, m0, beta, it.half < 0 && m0 + 128 < p.M);
      const int per = it.half >= 0 ? 2 : 1;
      // only the first step's ring entries go out with Q (p.burst = 0: the whole ring): all 148
      // CTAs filling their rings at once queue ~24 MB in L2 / HBM ahead of the first step's data
      pre_entries = min(S, p.burst > 0 ? per : nt * per);
      for (int e = 0; e < pre_entries; ++e) load_entry(e, e / per + (e % per) * nt, beta);
      break;
    }
  }
  if (warp == 12) ptx::tmem_alloc(&tmem_base_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  ptx::grid_dep_wait();   // every role reads valid_len / writes E only after the prerequisite grid
  const uint32_t tmem = tmem_base_slot;
  if (tr && threadIdx.x == 0) tr[1] = ptx::globaltimer();
  const int G = gridDim.x;

  if (warp >= 12) {
    ptx::setmaxnreg_dec<64>();
    // single-thread roles: try_wait (suspending) unless flags bit 2 asks for spinning
    const bool spin = (p.flags & 4) != 0;
    auto wait1 = [&](uint64_t* bar, uint32_t parity) {
      if (spin) ptx::mbar_spin(bar, parity); else ptx::mbar_wait(bar, parity);
    };
    // flags bit 7: the TMA producer sleeps in its waits (suspend-time hint) to free issue slots
    auto wait_tma = [&](uint64_t* bar, uint32_t parity) {
      if (p.flags & 128) ptx::mbar_wait_lazy(bar, parity); else wait1(bar, parity);
    };
    if (warp == 13) {
      // ============================================================ TMA producer
      if (ptx::elect_one()) {
        int g = 0, ai = 0;   // g: ring entries used so far
        for (int i = blockIdx.x; i < p.items; i += G) {
          T4Item it;
          it.decode(p, i);
          const int beta = it.u / p.l_mp;
          const int m0 = (it.u - beta * p.l_mp) * 256 + (it.half > 0 ? 128 : 0);
          const int nt = it.tiles(t4_unit_nlim(p, it.u));
          if (nt == 0) continue;
          const int qb = ai % p.q_bufs;
          if (ai >= p.q_bufs) wait_tma(&q_empty[qb], ((ai / p.q_bufs) - 1) & 1);
          if (ai > 0 || pre_entries == 0) load_q(qb, m0, beta, it.half < 0 && m0 + 128 < p.M);
          ++ai;
          for (int j = 0; j < nt; ++j) {
            for (int x = 0; x < (it.half >= 0 ? 2 : 1); ++x, ++g) {
              if (g < pre_entries) continue;
              const int tile = j + x * nt;   // half item: slot 1 takes tiles [nt, 2 nt)
              const int s = g % S;
              if (g >= S) wait_tma(&kv_empty[s], ((g / S) - 1) & 1);
              else if (g == pre_entries && pre_entries > 0) wait1(&kv_full[pre_entries - 1], 0);   // first step landed
              if (tr && g < kT4TrTiles) tr[460 + g] = t4_clk();
              load_entry(s, tile, beta);
            }
          }
        }
      }
    } else if (warp == 12 || warp == 14) {
      // ============================================================ tcgen05 issuers (one per slot)
      if (ptx::elect_one()) {
        const int x = warp == 12 ? 0 : 1;
        const uint64_t dA = ptx::sdesc_sw128(0, 16, 1024);
        const uint64_t dB = (BL == 1) ? ptx::sdesc_sw128(0, 16, 1024) : ptx::sdesc_sw128(0, p.kp_rows * 128, 1024);
        const uint64_t dD = ptx::sdesc_sw128(0, kT4BN * 128, 1024);
        const uint32_t sQ0 = ptx::smem_u32(sQ), sKV0 = ptx::smem_u32(sKV);
        const uint32_t idesc1 = p.idesc1, idesc2 = p.idesc2;
        const int k_steps = p.k_steps;
        const uint32_t dS = tmem + x * 128;
        const uint32_t tO = tmem + kT5OCol + x * 64;
        const uint32_t tP = tmem + kT5PCol + x * 64;
        T4Cursor c1, c2;   // c1: step of the next G1 (one ahead of c2), c2: step of the next G2
        c1.init(p, G);
        c2 = c1;
        // G1(x) of step c1: S_x = Q_x · K_(tile of slot x)  (ready: its inputs were tested already)
        auto issue_g1 = [&](bool ready = false) {
          int kst;
          uint32_t kph;
          c1.entry(x, S, kst, kph);
          if (!ready) {
            if (c1.j == 0) wait1(&q_full[c1.qb], c1.qph);
            wait1(&kv_full[kst], kph);
          }
          ptx::tc_fence_after();
          const uint32_t q_lo = (sQ0 + (c1.qb * 2 + (c1.hf ? 0 : x)) * p.q_bytes) >> 4;   // half: one Q tile
          const uint32_t k_lo = (sKV0 + kst * kv_stage) >> 4;
#pragma unroll
          for (int ks = 0; ks < 4 * KCH; ++ks) {
            if (ks < k_steps) {
              const uint64_t ad = dA + q_lo + (ks >> 2) * 1024 + (ks & 3) * 2;
              const uint64_t bd = (BL == 1) ? dB + k_lo + (ks >> 2) * (kT4BN * 8) + (ks & 3) * 2
                                            : dB + k_lo + ks * 128;
              if (!(dbg & 4)) ptx::mma_ss(dS, ad, bd, idesc1, ks > 0 ? 1u : 0u);
            }
          }
          ptx::mma_commit(&s_full[x]);
          if (tr && c1.g < kT4TrTiles) tr[T4TR(c1.g, 14 + x)] = t4_clk();
          if (c1.j == c1.nt - 1) ptx::mma_commit(&q_empty[c1.qb]);   // this slot's last read of Q
          c1.advance(p, G);
        };
        if (dbg & 64) {   // TMA only: release every entry of this slot as soon as it lands
          for (; c1.valid; c1.advance(p, G)) {
            if (c1.j == 0) wait1(&q_full[c1.qb], c1.qph);
            int kst;
            uint32_t kph;
            c1.entry(x, S, kst, kph);
            wait1(&kv_full[kst], kph);
            ptx::mbar_arrive(&kv_empty[kst]);
            if (c1.hf) ptx::mbar_arrive(&kv_empty[kst]);
            if (c1.j == c1.nt - 1) ptx::mbar_arrive(&q_empty[c1.qb]);
          }
          c2.valid = false;
        }
        if (c1.valid) issue_g1();
        // G2(x) of step c2: O_x += P_x · V_(tile of slot x)  (its inputs are complete)
        auto issue_g2 = [&]() {
          if (tr && c2.g < kT4TrTiles) tr[T4TR(c2.g, 10 + x)] = t4_clk();
          ptx::tc_fence_after();
          int vst;
          uint32_t vph;
          c2.entry(x, S, vst, vph);
          const uint32_t v_lo = (sKV0 + vst * kv_stage + p.b_stage_bytes) >> 4;
          const uint32_t acc0 = c2.j > 0 ? 1u : 0u;
#pragma unroll
          for (int ks = 0; ks < kT4BN / 16; ++ks)
            if (!(dbg & 2)) ptx::mma_ts(tO, tP + ks * 8, dD + v_lo + ks * 128, idesc2, ks > 0 ? 1u : acc0);
          ptx::mma_commit(&p_free[x]);
          if (tr && c2.g < kT4TrTiles) tr[T4TR(c2.g, 12 + x)] = t4_clk();
          ptx::mma_commit(&kv_empty[vst]);
          if (c2.hf) ptx::mma_commit(&kv_empty[vst]);
          if (c2.j == c2.nt - 1) ptx::mma_commit(&o_full[x]);
          c2.advance(p, G);
        };
        if (p.flags & 256) {
          // Event-driven order (flags bit 8): poll both hand-offs and issue G2(c2) as soon as P_x is
          // written and G1(c1) as soon as S_x is free and its K tile has landed, whichever comes
          // first, so a late K tile no longer holds back the G2 the softmax waits on (p_free).
          // Phases stay unambiguous: G1(c1) needs s_free of step c1 - 1, which the softmax only
          // arrives after S(c1 - 1) exists; G2(c2) needs p_full of step c2 < c1.
          const uint64_t t0 = ptx::globaltimer();
          uint32_t idle = 0;
          while (c2.valid) {
            bool did = false;
            if (c1.valid && ptx::mbar_test(&s_free[x], (c1.g - 1) & 1) &&
                (c1.j != 0 || ptx::mbar_test(&q_full[c1.qb], c1.qph))) {
              int kst;
              uint32_t kph;
              c1.entry(x, S, kst, kph);
              if (ptx::mbar_test(&kv_full[kst], kph)) {
                issue_g1(true);
                did = true;
              }
            }
            if (c2.g < c1.g && ptx::mbar_test(&p_full[x], c2.g & 1) &&
                (c2.j != 0 || c2.ai == 0 || ptx::mbar_test(&o_free[x], (c2.ai - 1) & 1))) {
              issue_g2();
              did = true;
            }
            if (!did) {
              // sleep (suspend-time hint) on the first unmet input in the softmax's own order — S_x
              // free comes before P_x written — then re-test both
              uint64_t* bar;
              uint32_t par;
              if (c1.valid && !ptx::mbar_test(&s_free[x], (c1.g - 1) & 1)) {
                bar = &s_free[x];
                par = (c1.g - 1) & 1;
              } else if (c1.valid && c1.j == 0 && !ptx::mbar_test(&q_full[c1.qb], c1.qph)) {
                bar = &q_full[c1.qb];
                par = c1.qph;
              } else if (c2.g < c1.g) {
                bar = &p_full[x];
                par = c2.g & 1;
              } else {
                int kst;
                c1.entry(x, S, kst, par);
                bar = &kv_full[kst];
              }
              if (!(p.flags & 4)) ptx::mbar_try_wait_hint(ptx::smem_u32(bar), par, 100);   // bit 2: pure polling
              if (((++idle) & 1023u) == 0 && ptx::globaltimer() - t0 > 4000000000ull) __trap();
            }
          }
        }
        uint32_t ph = 0;   // parity of step c2.g (s_free / p_full phases count this slot's steps)
        while (c2.valid) {
          if (c1.valid) {
            wait1(&s_free[x], ph);   // softmax x has S(x, step c2) in registers
            issue_g1();
          }
          wait1(&p_full[x], ph);
          if (tr && c2.g < kT4TrTiles) tr[T4TR(c2.g, 10 + x)] = t4_clk();
          if (c2.j == 0 && c2.ai > 0) wait1(&o_free[x], (c2.ai - 1) & 1);
          ptx::tc_fence_after();
          int vst;
          uint32_t vph;
          c2.entry(x, S, vst, vph);
          const uint32_t v_lo = (sKV0 + vst * kv_stage + p.b_stage_bytes) >> 4;
          const uint32_t acc0 = c2.j > 0 ? 1u : 0u;
#pragma unroll
          for (int ks = 0; ks < kT4BN / 16; ++ks)
            if (!(dbg & 2)) ptx::mma_ts(tO, tP + ks * 8, dD + v_lo + ks * 128, idesc2, ks > 0 ? 1u : acc0);
          ptx::mma_commit(&p_free[x]);
          if (tr && c2.g < kT4TrTiles) tr[T4TR(c2.g, 12 + x)] = t4_clk();
          // kv_empty counts two arrivals: one per slot on a shared entry, or both from the one
          // slot that reads a half item's entry
          ptx::mma_commit(&kv_empty[vst]);
          if (c2.hf) ptx::mma_commit(&kv_empty[vst]);
          if (c2.j == c2.nt - 1) ptx::mma_commit(&o_full[x]);
          c2.advance(p, G);
          ph ^= 1;
        }
      }
    }
  } else if (warp >= 8) {
    // ============================================================ epilogue (warps 8-11)
    ptx::setmaxnreg_dec<80>();
    // flags bit 7: the epilogue sleeps in its waits (suspend-time hint) to free issue slots
    auto wait_epi = [&](uint64_t* bar, uint32_t parity) {
      if (p.flags & 1024) ptx::mbar_wait_backoff(bar, parity);   // bit 10: sleep between polls
      else if (p.flags & 128) ptx::mbar_wait_lazy(bar, parity);
      else ptx::mbar_wait(bar, parity);
    };
    const int row = threadIdx.x - 256;   // TMEM lane (warp 8+w reads lanes 32w..32w+31)
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const bool leader = threadIdx.x == 256;
    const uint32_t sE0 = ptx::smem_u32(sE) + row * 128;
    int ai = 0;
    // E tile (beta, rows gm0 .. gm0 + 127) = w0·O_0 + w1·O_1 (one slot: w1 = 0), packed to 16
    // bits into the 128-B-swizzled staging tile, then one TMA bulk tensor store (clipped to L
    // columns and M rows by the tensor map).  O is released (o_free) once read.
    auto emit = [&](int beta, int gm0, int x0, float w0, int x1, float w1, int nt) {
      if (dbg & 16) {
        if (nt > 0) {
          ptx::mbar_arrive(&o_free[x0]);
          if (x1 >= 0) ptx::mbar_arrive(&o_free[x1]);
        }
        return;
      }
      if (leader) ptx::tma_store_wait_read();   // the previous store has read the staging
      ptx::named_bar_sync(9, 128);
      const uint32_t tA = tmem + lane_off + kT5OCol + x0 * 64, tB = tmem + lane_off + kT5OCol + x1 * 64;
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t w[8];
        if (c0 < p.TL && nt > 0) {
          uint32_t r0[16];
          ptx::tmem_ld16(tA + c0, r0);
          if (x1 >= 0) {
            uint32_t r1[16];
            ptx::tmem_ld16(tB + c0, r1);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 8; ++q)
              w[q] = ptx::pack2<BF16>(w0 * __uint_as_float(r0[2 * q]) + w1 * __uint_as_float(r1[2 * q]),
                                      w0 * __uint_as_float(r0[2 * q + 1]) + w1 * __uint_as_float(r1[2 * q + 1]));
          } else {
            ptx::tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 8; ++q)
              w[q] = ptx::pack2<BF16>(w0 * __uint_as_float(r0[2 * q]), w0 * __uint_as_float(r0[2 * q + 1]));
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) w[q] = 0u;
        }
        const int ck = c0 >> 3;   // 16-B chunk index of this 16-column group (two chunks)
        ptx::st_shared_v4(sE0 + ((ck ^ (row & 7)) << 4), w[0], w[1], w[2], w[3]);
        ptx::st_shared_v4(sE0 + (((ck + 1) ^ (row & 7)) << 4), w[4], w[5], w[6], w[7]);
      }
      if (nt > 0) {
        ptx::tc_fence_before();
        ptx::mbar_arrive(&o_free[x0]);
        if (x1 >= 0) ptx::mbar_arrive(&o_free[x1]);
      }
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(9, 128);
      if (leader) {
        ptx::tma_store_3d(&tmE, sE, 0, gm0, beta);
        ptx::tma_store_commit();
      }
    };
    for (int i = (dbg & 64) ? p.items : blockIdx.x; i < p.items; i += G) {
      T4Item it;
      it.decode(p, i);
      const int beta = it.u / p.l_mp;
      const int m0 = (it.u - beta * p.l_mp) * 256;
      const int nt = it.tiles(t4_unit_nlim(p, it.u));
      if (it.half >= 0) {
        // half item: both slots hold partial (O, m, l) of the same 128 rows; merge by
        // log-sum-exp (exact in real arithmetic, R4)
        float l[2], m[2];
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          wait_epi(&o_full[x], ai & 1);
          wait_epi(&l_full[x], ai & 1);
          l[x] = l_sm[x][ai & 1][row];
          m[x] = m_sm[x][ai & 1][row];
          ptx::mbar_arrive(&l_free[x]);
        }
        ptx::tc_fence_after();
        float w0 = 1.f, w1 = 1.f, inv = 1.f;   // NONE / SCALE: E = O_0 + O_1
        if (MBCI_T5_OP == 2) {
          const float mstar = fmaxf(l[0] > 0.f ? m[0] : -INFINITY, l[1] > 0.f ? m[1] : -INFINITY);
          w0 = l[0] > 0.f ? ptx::ex2(m[0] - mstar) : 0.f;
          w1 = l[1] > 0.f ? ptx::ex2(m[1] - mstar) : 0.f;
          const float Lsum = l[0] * w0 + l[1] * w1;
          inv = Lsum > 0.f ? 1.0f / Lsum : 0.f;
          t4_store_lse(p, beta, m0 + it.half * 128 + row, mstar, Lsum);
        }
        emit(beta, m0 + it.half * 128, 0, w0 * inv, 1, w1 * inv, nt);
        ++ai;
        continue;
      }
#pragma unroll 1
      for (int x = 0; x < 2; ++x) {
        float l = 0.f, mr = 0.f;
        if (nt > 0) {
          wait_epi(&o_full[x], ai & 1);
          ptx::tc_fence_after();
          if (tr && x == 0 && row == 0 && ai < 4) tr[490 + 4 * ai] = t4_clk();
          wait_epi(&l_full[x], ai & 1);
          l = l_sm[x][ai & 1][row];
          mr = m_sm[x][ai & 1][row];
          ptx::mbar_arrive(&l_free[x]);
        }
        t4_store_lse(p, beta, m0 + x * 128 + row, mr, l);
        if (m0 + x * 128 >= p.M) {   // a pair whose second tile is past M: nothing to store
          if (nt > 0) {
            ptx::tc_fence_before();
            ptx::mbar_arrive(&o_free[x]);
          }
          continue;
        }
        emit(beta, m0 + x * 128, x, l > 0.f ? 1.0f / l : 0.f, -1, 0.f, nt);
        if (tr && row == 0 && ai < 4) tr[490 + 4 * ai + 1 + x] = t4_clk();
      }
      if (nt > 0) ++ai;
    }
    if (leader) ptx::tma_store_wait_read();   // the staging must outlive the bulk stores' reads
  } else {
    // ============================================================ softmax (warps 0-7)
    ptx::setmaxnreg_inc<184>();   // a whole 128-column S row lives in registers
    const int x = warp >> 2;               // slot
    const int row = threadIdx.x & 127;     // TMEM lane
    const bool lane0 = (threadIdx.x & 31) == 0;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_off + x * 128;
    const uint32_t tP = tmem + lane_off + kT5PCol + x * 64;
    const uint32_t tO = tmem + lane_off + kT5OCol + x * 64;
    const float sc = p.scale;
    // Exp-phase turns (flags bit 0, softmax only): named barriers 1-4 = slot 0's turn on SMSP q,
    // 5-8 = slot 1's; slot 0 goes first.
    const bool turns = (p.flags & 1) != 0 && MBCI_T5_OP == 2;
    // flags bit 11: on SOFTMAX the softmax warps poll s_full / p_free with test_wait instead of
    // try_wait (C2 -1.3 %; on the linear ops polling costs 7 %, so they keep try_wait)
    const bool sm_spin = (p.flags & 2048) != 0 && MBCI_T5_OP == 2;
    auto wait_sm = [&](uint64_t* bar, uint32_t parity) {
      if (sm_spin) ptx::mbar_spin(bar, parity); else ptx::mbar_wait(bar, parity);
    };
    const uint32_t bar_mine = 1 + (warp & 3) + 4 * x, bar_other = 1 + (warp & 3) + 4 * (1 - x);
    const int turn_chunk = 3 - ((p.flags >> 4) & 3);   // flags bits 4-5: hand over 0-3 chunks early
    int g = 0, ai = 0;
    for (int i = (dbg & 64) ? p.items : blockIdx.x; i < p.items; i += G) {
      T4Item it;
      it.decode(p, i);
      const int beta = it.u / p.l_mp;
      const int nt = it.tiles(t4_unit_nlim(p, it.u));
      if (nt == 0) continue;
      const int n_lim = t4_nlim(p, beta) - (it.half >= 0 ? x * nt * kT4BN : 0);
      const int m_row = (it.u - beta * p.l_mp) * 256 + x * 128 + row;   // causal: no half items
      float m_run = 0.f;
      float2 l2 = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
      for (int j = 0; j < nt; ++j, ++g) {
        const uint32_t ph = g & 1;
        if (!(dbg & 128)) wait_sm(&s_full[x], ph);   // 128: free-running softmax (timing only)
        ptx::tc_fence_after();
        if (tr && row == 0 && g < kT4TrTiles) tr[T4TR(g, x)] = t4_clk();
        if (dbg & 1) {   // barrier protocol only
          __syncwarp();
          if (lane0) ptx::mbar_arrive(&s_free[x]);
          if (g > 0) wait_sm(&p_free[x], ph ^ 1u);
          __syncwarp();
          if (lane0) ptx::mbar_arrive(&p_full[x]);
          continue;
        }
        const int valid = (p.causal ? min(n_lim, m_row + 1) : n_lim) - j * kT4BN;   // this thread's row
        const bool full = __all_sync(0xffffffffu, valid >= kT4BN);                   // warp-uniform
        uint32_t sr[kT4BN];
#pragma unroll
        for (int c = 0; c < kT4BN / 32; ++c) ptx::tmem_ld32(tS + c * 32, &sr[c * 32]);
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane0) ptx::mbar_arrive(&s_free[x]);   // S_x may be overwritten by G1(x, g + 1)
        if (MBCI_T5_OP != 2) {
          // NONE / SCALE: padded keys have S = 0 and zero V rows (TMA fill), no masking needed
          if (p.flags & 512) {   // convert first, then wait for G2_x(g - 1) to release P_x
            uint32_t pk[64];
            t5_cvt_row<BF16, kLinear>(pk, sr, sc, MBCI_T5_OP);
            if (g > 0) wait_sm(&p_free[x], ph ^ 1u);
            ptx::tc_fence_after();
            t5_store_p(tP, pk);
          } else {
            if (g > 0) wait_sm(&p_free[x], ph ^ 1u);   // G2_x(g - 1) has read P_x
            ptx::tc_fence_after();
            t4_cvt_row<BF16, kLinear>(tP, sr, sc, MBCI_T5_OP);
          }
        } else {
          float mx;
          if (full)
            mx = sc >= 0.f ? t4_row_extreme<false, false>(sr, valid) : t4_row_extreme<true, false>(sr, valid);
          else
            mx = sc >= 0.f ? t4_row_extreme<false, true>(sr, valid) : t4_row_extreme<true, true>(sr, valid);
          const float m_tile = mx * sc;
          if (tr && row == 0 && g < kT4TrTiles) tr[T4TR(g, 2 + x)] = t4_clk_after(__float_as_uint(mx));
          // P_x (and, for a rescale, O_x) is free once G2_x(g - 1) completed.  Without a rescale
          // the wait is deferred until the exponentials are in registers (flags bit 3 restores
          // the early wait, for A/B measurements).
          bool p_ready = g == 0;
          if (!p_ready && (p.flags & 8)) {
            if (!(dbg & 128)) wait_sm(&p_free[x], ph ^ 1u);
            ptx::tc_fence_after();
            p_ready = true;
          }
          if (j == 0) {
            m_run = m_tile;
          } else if (__any_sync(0xffffffffu, m_tile > m_run + kT4Tau)) {
            // warp-uniform (tcgen05.ld/st are warp-collective); O_x must hold G2_x(g - 1)
            if (!p_ready) {
              if (!(dbg & 128)) wait_sm(&p_free[x], ph ^ 1u);
              ptx::tc_fence_after();
              p_ready = true;
            }
            const float m_new = fmaxf(m_run, m_tile);
            const float alpha = ptx::ex2(m_run - m_new);
            l2.x *= alpha;
            l2.y *= alpha;
            l2b.x *= alpha;
            l2b.y *= alpha;
            m_run = m_new;
            for (int c0 = 0; c0 < p.TL; c0 += 16) {
              uint32_t r[16];
              ptx::tmem_ld16(tO + c0, r);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int k = 0; k < 16; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) * alpha);
              ptx::tmem_st16(tO + c0, r);
            }
          }
          if (turns && (x == 1 || g > 0)) ptx::named_bar_sync(bar_mine, 64);
          if (tr && row == 0 && g < kT4TrTiles) tr[T4TR(g, 4 + x)] = t4_clk();   // exps start
          // the other slot's warp may start its turn after chunk turn_chunk of this one's
          if (p.flags & 4096) {   // bit 12: P_x released first, each chunk stored as computed
            if (!p_ready) {
              if (!(dbg & 128)) wait_sm(&p_free[x], ph ^ 1u);
              ptx::tc_fence_after();
              p_ready = true;
            }
            if (full)
              t5_exp_row_st<BF16, EMU, false>(tP, sr, sc, m_run, valid, l2, l2b, turn_chunk, turns ? bar_other : 0u);
            else
              t5_exp_row_st<BF16, 0, true>(tP, sr, sc, m_run, valid, l2, l2b, turn_chunk, turns ? bar_other : 0u);
            if (tr && row == 0 && g < kT4TrTiles) tr[T4TR(g, 6 + x)] = t4_clk();   // exps done
          } else {
          uint32_t pk[64];
          if (full)
            t5_exp_row<BF16, EMU, false>(pk, sr, sc, m_run, valid, l2, l2b, turn_chunk, turns ? bar_other : 0u);
          else
            t5_exp_row<BF16, 0, true>(pk, sr, sc, m_run, valid, l2, l2b, turn_chunk, turns ? bar_other : 0u);
          if (tr && row == 0 && g < kT4TrTiles) tr[T4TR(g, 6 + x)] = t4_clk();   // exps done
          if (!p_ready) {
            if (!(dbg & 128)) wait_sm(&p_free[x], ph ^ 1u);
            ptx::tc_fence_after();
          }
          t5_store_p(tP, pk);
          }
        }
        ptx::tmem_wait_st();
        if (tr && row == 0 && g < kT4TrTiles) tr[T4TR(g, 8 + x)] = t4_clk();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane0) ptx::mbar_arrive(&p_full[x]);
      }
      // l_full's parity protocol allows one phase in flight: publishing l of item ai waits
      // until the epilogue has read item ai - 1's.
      if (ai >= 1) ptx::mbar_wait(&l_free[x], (ai - 1) & 1);
      l_sm[x][ai & 1][row] = MBCI_T5_OP == 2 ? (l2.x + l2.y) + (l2b.x + l2b.y) : 1.0f;   // E = O / l
      m_sm[x][ai & 1][row] = m_run;
      __syncwarp();
      if (lane0) ptx::mbar_arrive(&l_full[x]);
      ++ai;
    }
    if (turns && !(dbg & 1) && x == 0 && g > 0) ptx::named_bar_sync(bar_mine, 64);   // slot 1's last hand-back
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[3] = ptx::globaltimer();
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}
#undef MBCI_T5_OP

}  // namespace mbci
