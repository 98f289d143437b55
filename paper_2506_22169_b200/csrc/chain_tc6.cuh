// chain_tc6.cuh — kernel 6: kernel 5 (chain_tc5.cuh) with every score row split across TWO softmax
// warps, so each SMSP runs four softmax warps instead of two.
//
// Same arithmetic, work items, TMEM layout (S_0, S_1, P_0, P_1, O_0, O_1 = 512 columns), barrier
// protocol and issuer / TMA / epilogue roles as kernel 5 (PAPER.md:196 chain, :498 softmax
// between the GEMMs, :489 batched layout; Rule 1 spatial loops on the persistent grid, :285; dead
// k loop, :253; S_E hoisted, :232-233).  What differs is the softmax:
//
//   kernel 5: one warp per (slot, TMEM lane quadrant) owns a whole 128-column S row: 128 S
//     registers, a 480-instruction unrolled exponential block, and per tile a ~460-cycle TMEM
//     load during which that warp issues nothing.  Measured (round 2, profiles/r2_*): the exp
//     phase of one warp ran at half its isolated rate, `no_instruction` (i-cache, L0 ~6 KB) was
//     the top stall of the exp loop, and two warps per SMSP could not hide the TMEM latency.
//   kernel 6: warps w and w + 8 (same SMSP, same lanes) share the rows of slot x = (w >> 2) & 1:
//     half h = w >> 3 owns key columns [64h, 64h + 64) of each S tile.  Per tile each warp loads
//     64 columns, takes its partial row max, swaps it with its partner through shared memory
//     (one 64-thread named barrier per (slot, quadrant)), computes 64 exponentials (a 240-
//     instruction block shared by all 16 warps) and writes its 32 packed P columns.  The two
//     halves keep separate row sums, added by the epilogue; the lazy-rescale decision is
//     identical in both (same combined row max), each rescales its half of O_x's 16-column
//     chunks.
//
// Warps: 0-15 softmax (w & 3 = lane quadrant, (w >> 2) & 1 = slot, w >> 3 = column half) |
//        16-19 epilogue | 20 tcgen05 issuer of slot 0 + TMEM allocator | 21 TMA producer |
//        22 tcgen05 issuer of slot 1 | 23 idle.  768 threads; setmaxnreg 96 / 56 / 40.
#pragma once
#include "chain_tc4.cuh"
#include "chain_tc5.cuh"

namespace mbci {

// 24 warps = 6 per SMSP, so ptxas gives every thread 80 registers at launch (the per-SMSP file
// holds 512 per lane); setmaxnreg then moves them: 16 x 96 + 4 x 56 + 4 x 40 = 24 x 80.
constexpr int kT6Threads = 768;

// p = 2^(sc·S − m) for the 64 scores of a half row (registers) into 32 packed 16-bit words `pk`,
// two packed partial sums.  MASKED: columns >= valid give 0.  After chunk `arrive_after` (of 2
// chunks of 16 pairs) the other slot's warps of this SMSP may start their exponentials (bar != 0).
template <bool BF16, int EMU, bool MASKED>
__device__ __forceinline__ void t6_exp_half(uint32_t (&pk)[32], const uint32_t (&sr)[64], float sc, float m,
                                            int valid, float2& l2a, float2& l2b, int arrive_after, uint32_t bar) {
  const float2 sc2 = make_float2(sc, sc);
  const float2 nm2 = make_float2(-m, -m);
#pragma unroll
  for (int ch = 0; ch < 2; ++ch) {
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
    if (bar != 0 && ch == arrive_after) ptx::named_bar_arrive(bar, 128);
  }
}

// NONE / SCALE: P = cvt(scale · S) for a 64-column half row
template <bool BF16, bool ACT>
__device__ __forceinline__ void t6_cvt_half_impl(uint32_t tP, const uint32_t (&sr)[64], float sc, int op) {
  const float2 sc2 = make_float2(sc, sc);
#pragma unroll
  for (int ch = 0; ch < 2; ++ch) {
    uint32_t pk[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int cp = ch * 16 + c;
      float2 z = __fmul2_rn(make_float2(__uint_as_float(sr[2 * cp]), __uint_as_float(sr[2 * cp + 1])), sc2);
      if constexpr (ACT) {
        z.x = ptx::act(op, z.x);
        z.y = ptx::act(op, z.y);
      }
      pk[c] = ptx::pack2<BF16>(z.x, z.y);
    }
    ptx::tmem_st16(tP + ch * 16, pk);
  }
}
template <bool BF16>
__device__ __forceinline__ void t6_cvt_half(uint32_t tP, const uint32_t (&sr)[64], float sc, int op) {
  if (op >= 3) t6_cvt_half_impl<BF16, true>(tP, sr, sc, op);
  else t6_cvt_half_impl<BF16, false>(tP, sr, sc, op);
}

// Extreme (max, or min for a negative scale) of a 64-column half row; MASKED: first `valid` only.
template <bool MIN, bool MASKED>
__device__ __forceinline__ float t6_half_extreme(const uint32_t (&sr)[64], int valid) {
  if constexpr (MASKED) {
    float mx = MIN ? INFINITY : -INFINITY;
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      const float v = __uint_as_float(sr[c]);
      if (c < valid) mx = MIN ? fminf(mx, v) : fmaxf(mx, v);
    }
    return mx;
  } else {
    float a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      a[q] = MIN ? fminf(__uint_as_float(sr[2 * q]), __uint_as_float(sr[2 * q + 1]))
                 : fmaxf(__uint_as_float(sr[2 * q]), __uint_as_float(sr[2 * q + 1]));
#pragma unroll
    for (int c = 16; c < 64; c += 16)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = t4_red<MIN>(a[q], __uint_as_float(sr[c + 2 * q]), __uint_as_float(sr[c + 2 * q + 1]));
    return t4_red<MIN>(t4_red<MIN>(a[0], a[1], a[2]), t4_red<MIN>(a[3], a[4], a[5]), MIN ? fminf(a[6], a[7]) : fmaxf(a[6], a[7]));
  }
}

template <bool BF16, int KCH, int BL, int EMU>
__global__ void __launch_bounds__(kT6Threads, 1)
    k_chain_tc6(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmE,
                const Tc4Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ uint32_t tmem_base_slot;
  __shared__ float l_sm[2][2][2][128];   // [slot][column half][active-item parity][row]: partial row sums
  __shared__ float m_sm[2][2][128];      // [slot][parity][row]: running max (log2) the p were taken against
  __shared__ float xmax[2][2][2][128];   // [tile parity][slot][column half][row]: partial row extremes

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
  uint64_t* l_full = bars + 8;      // [2] softmax x published l (one arrival per warp: 8)
  uint64_t* l_free = bars + 10;     // [2] epilogue read l_sm[x][ai & 1] (128 arrivals)
  uint64_t* s_full = bars + 12;     // [2] G1_x landed in S_x (commit)
  uint64_t* s_free = bars + 14;     // [2] softmax x holds S_x in registers (one arrival per warp: 8)
  uint64_t* p_full = bars + 16;     // [2] softmax x wrote P_x (one arrival per warp: 8)
  uint64_t* p_free = bars + 18;     // [2] G2_x read P_x and updated O_x (commit)
  uint64_t* kv_full = bars + 20;    // [S] K_g and V_g landed
  uint64_t* kv_empty = kv_full + S; // [S] the G2s reading the entry completed (two commits)

  const int warp = threadIdx.x >> 5;
  // Diagnostics (trace build only): 256 = exp-throughput probe — every softmax warp runs its
  // exponential block kProbeReps times on one S tile (with the exp-phase turns when enabled),
  // 512 adds the per-tile TMEM load and row max; no other role works.  Results are garbage.
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
  if (warp == 21 && !(dbg & 256) && ptx::elect_one()) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 2);   // each slot's issuer commits after its last G1
      ptx::mbar_init(&o_full[i], 1);
      ptx::mbar_init(&o_free[i], 128);
      ptx::mbar_init(&l_full[i], 8);
      ptx::mbar_init(&l_free[i], 128);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 8);
      ptx::mbar_init(&p_full[i], 8);
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
  if (warp == 20) ptx::tmem_alloc(&tmem_base_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  ptx::grid_dep_wait();   // every role reads valid_len / writes E only after the prerequisite grid
  const uint32_t tmem = tmem_base_slot;
  if (tr && threadIdx.x == 0) tr[1] = ptx::globaltimer();
  const int G = gridDim.x;

  if (warp >= 20) {
    ptx::setmaxnreg_dec<40>();
    // single-thread roles: try_wait (suspending) unless flags bit 2 asks for spinning
    const bool spin = (p.flags & 4) != 0;
    auto wait1 = [&](uint64_t* bar, uint32_t parity) {
      if (spin) ptx::mbar_spin(bar, parity); else ptx::mbar_wait(bar, parity);
    };
    if (warp == 21) {
      // ============================================================ TMA producer
      if (!(dbg & 256) && ptx::elect_one()) {
        int g = 0, ai = 0;   // g: ring entries used so far
        for (int i = blockIdx.x; i < p.items; i += G) {
          T4Item it;
          it.decode(p, i);
          const int beta = it.u / p.l_mp;
          const int m0 = (it.u - beta * p.l_mp) * 256 + (it.half > 0 ? 128 : 0);
          const int nt = it.tiles(t4_unit_nlim(p, it.u));
          if (nt == 0) continue;
          const int qb = ai % p.q_bufs;
          if (ai >= p.q_bufs) wait1(&q_empty[qb], ((ai / p.q_bufs) - 1) & 1);
          if (ai > 0 || pre_entries == 0) load_q(qb, m0, beta, it.half < 0 && m0 + 128 < p.M);
          ++ai;
          for (int j = 0; j < nt; ++j) {
            for (int x = 0; x < (it.half >= 0 ? 2 : 1); ++x, ++g) {
              if (g < pre_entries) continue;
              const int tile = j + x * nt;   // half item: slot 1 takes tiles [nt, 2 nt)
              const int s = g % S;
              if (g >= S) wait1(&kv_empty[s], ((g / S) - 1) & 1);
              else if (g == pre_entries && pre_entries > 0) wait1(&kv_full[pre_entries - 1], 0);   // first step landed
              if (tr && g < kT4TrTiles) tr[460 + g] = t4_clk();
              load_entry(s, tile, beta);
            }
          }
        }
      }
    } else if (warp == 20 || warp == 22) {
      // ============================================================ tcgen05 issuers (one per slot)
      if (!(dbg & 256) && ptx::elect_one()) {
        const int x = warp == 20 ? 0 : 1;
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
        // G1(x) of step c1: S_x = Q_x · K_(tile of slot x)
        auto issue_g1 = [&]() {
          if (c1.j == 0) wait1(&q_full[c1.qb], c1.qph);
          int kst;
          uint32_t kph;
          c1.entry(x, S, kst, kph);
          wait1(&kv_full[kst], kph);
          ptx::tc_fence_after();
          const uint32_t q_lo = (sQ0 + (c1.qb * 2 + (c1.hf ? 0 : x)) * p.q_bytes) >> 4;   // half: one Q tile
          const uint32_t k_lo = (sKV0 + kst * kv_stage) >> 4;
#pragma unroll
          for (int ks = 0; ks < 4 * KCH; ++ks) {
            if (ks < k_steps) {
              const uint64_t ad = dA + q_lo + (ks >> 2) * 1024 + (ks & 3) * 2;
              const uint64_t bd = (BL == 1) ? dB + k_lo + (ks >> 2) * (kT4BN * 8) + (ks & 3) * 2
                                            : dB + k_lo + ks * 128;
              ptx::mma_ss(dS, ad, bd, idesc1, ks > 0 ? 1u : 0u);
            }
          }
          ptx::mma_commit(&s_full[x]);
          if (tr && c1.g < kT4TrTiles) tr[T4TR(c1.g, 14 + x)] = t4_clk();
          if (c1.j == c1.nt - 1) ptx::mma_commit(&q_empty[c1.qb]);   // this slot's last read of Q
          c1.advance(p, G);
        };
        if (c1.valid) issue_g1();
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
            ptx::mma_ts(tO, tP + ks * 8, dD + v_lo + ks * 128, idesc2, ks > 0 ? 1u : acc0);
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
  } else if (warp >= 16) {
    // ============================================================ epilogue (warps 16-19)
    ptx::setmaxnreg_dec<56>();
    const int row = threadIdx.x - 512;   // TMEM lane (warp 16+w reads lanes 32w..32w+31)
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const bool leader = threadIdx.x == 512;
    const uint32_t sE0 = ptx::smem_u32(sE) + row * 128;
    int ai = 0;
    // E tile (beta, rows gm0 .. gm0 + 127) = w0·O_0 + w1·O_1 (one slot: w1 = 0), packed to 16
    // bits into the 128-B-swizzled staging tile, then one TMA bulk tensor store (clipped to L
    // columns and M rows by the tensor map).  O is released (o_free) once read.
    auto emit = [&](int beta, int gm0, int x0, float w0, int x1, float w1, int nt) {
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
    for (int i = (dbg & 256) ? p.items : blockIdx.x; i < p.items; i += G) {
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
          ptx::mbar_wait(&o_full[x], ai & 1);
          ptx::mbar_wait(&l_full[x], ai & 1);
          l[x] = l_sm[x][0][ai & 1][row] + l_sm[x][1][ai & 1][row];
          m[x] = m_sm[x][ai & 1][row];
          ptx::mbar_arrive(&l_free[x]);
        }
        ptx::tc_fence_after();
        float w0 = 1.f, w1 = 1.f, inv = 1.f;   // NONE / SCALE: E = O_0 + O_1
        if (p.op == 2) {
          const float mstar = fmaxf(l[0] > 0.f ? m[0] : -INFINITY, l[1] > 0.f ? m[1] : -INFINITY);
          w0 = l[0] > 0.f ? ptx::ex2(m[0] - mstar) : 0.f;
          w1 = l[1] > 0.f ? ptx::ex2(m[1] - mstar) : 0.f;
          const float Lsum = l[0] * w0 + l[1] * w1;
          inv = Lsum > 0.f ? 1.0f / Lsum : 0.f;
        }
        emit(beta, m0 + it.half * 128, 0, w0 * inv, 1, w1 * inv, nt);
        ++ai;
        continue;
      }
#pragma unroll 1
      for (int x = 0; x < 2; ++x) {
        float l = 0.f;
        if (nt > 0) {
          ptx::mbar_wait(&o_full[x], ai & 1);
          ptx::tc_fence_after();
          if (tr && x == 0 && row == 0 && ai < 4) tr[490 + 4 * ai] = t4_clk();
          ptx::mbar_wait(&l_full[x], ai & 1);
          l = l_sm[x][0][ai & 1][row] + l_sm[x][1][ai & 1][row];
          ptx::mbar_arrive(&l_free[x]);
        }
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
    // ============================================================ softmax (warps 0-15)
    ptx::setmaxnreg_inc<96>();
    const int x = (warp >> 2) & 1;         // slot
    const int h = warp >> 3;               // column half of the S tile
    const int row = threadIdx.x & 127;     // TMEM lane
    const bool lane0 = (threadIdx.x & 31) == 0;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_off + x * 128 + h * 64;
    const uint32_t tP = tmem + lane_off + kT5PCol + x * 64 + h * 32;
    const uint32_t tO = tmem + lane_off + kT5OCol + x * 64;
    const uint32_t pair_bar = 1 + x * 4 + (warp & 3);   // warps w and w ^ 8 (no turns)
    // Exp-phase turns (flags bit 0, softmax only): on SMSP q the two warps of slot 0 and the two of
    // slot 1 take turns on the MUFU; named barrier 1 + q + 4x (128 threads: slot x's two warps
    // wait, the other slot's two arrive) opens slot x's turn and also carries the partner's
    // partial row max.  Slot 1 pre-arrives once so slot 0 starts; slot 0 consumes slot 1's last
    // hand-over after its loop.
    const bool turns = (p.flags & 1) != 0 && p.op == 2;
    const uint32_t bar_mine = 1 + (warp & 3) + 4 * x, bar_other = 1 + (warp & 3) + 4 * (1 - x);
    const int turn_chunk = 1 - ((p.flags >> 4) & 1);   // flags bit 4: hand over one chunk early
    if (turns && x == 1) ptx::named_bar_arrive(bar_other, 128);
    const float sc = p.scale;
    int g = 0, ai = 0;
    if (dbg & 256) {
      constexpr int kProbeReps = 64;
      float2 la = make_float2(0.f, 0.f), lb = la;
      const uint64_t c0 = t4_clk();
      for (int r = 0; r < kProbeReps; ++r) {
        uint32_t sr[64];
        ptx::tmem_ld32(tS, &sr[0]);
        ptx::tmem_ld32(tS + 32, &sr[32]);
        ptx::tmem_wait_ld();
        if (dbg & 512) {
          float mx = t6_half_extreme<false, false>(sr, 64);
          la.x += mx;
        }
        if (turns) ptx::named_bar_sync(bar_mine, 128);
        uint32_t pk[32];
        t6_exp_half<BF16, EMU, false>(pk, sr, sc, 0.5f, 64, la, lb, turn_chunk, turns ? bar_other : 0u);
        ptx::tmem_st16(tP, &pk[0]);
        ptx::tmem_st16(tP + 16, &pk[16]);
        ptx::tmem_wait_st();
      }
      const uint64_t c1 = t4_clk();
      if (tr && (threadIdx.x & 31) == 0) tr[8 + warp] = c1 - c0;
      if (la.x + la.y + lb.x + lb.y == 1.2345f) l_sm[0][0][0][0] = 1.f;
    } else
    for (int i = blockIdx.x; i < p.items; i += G) {
      T4Item it;
      it.decode(p, i);
      const int beta = it.u / p.l_mp;
      const int nt = it.tiles(t4_unit_nlim(p, it.u));
      if (nt == 0) continue;
      const int n_lim = t4_nlim(p, beta) - (it.half >= 0 ? x * nt * kT4BN : 0) - h * 64;
      float m_run = 0.f;
      float2 l2 = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
      for (int j = 0; j < nt; ++j, ++g) {
        const uint32_t ph = g & 1;
        ptx::mbar_wait(&s_full[x], ph);
        ptx::tc_fence_after();
        if (tr && row == 0 && h == 0 && g < kT4TrTiles) tr[T4TR(g, x)] = t4_clk();
        const int valid = n_lim - j * kT4BN;   // valid columns of this half (may be <= 0 or >= 64)
        const bool full = valid >= 64;
        uint32_t sr[64];
        ptx::tmem_ld32(tS, &sr[0]);
        ptx::tmem_ld32(tS + 32, &sr[32]);
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane0) ptx::mbar_arrive(&s_free[x]);   // S_x may be overwritten by G1(x, g + 1)
        if (p.op != 2) {
          // NONE / SCALE: padded keys have S = 0 and zero V rows (TMA fill), no masking needed
          if (g > 0) ptx::mbar_wait(&p_free[x], ph ^ 1u);   // G2_x(g - 1) has read P_x
          ptx::tc_fence_after();
          t6_cvt_half<BF16>(tP, sr, sc, p.op);
        } else {
          float mx;
          if (full)
            mx = sc >= 0.f ? t6_half_extreme<false, false>(sr, valid) : t6_half_extreme<true, false>(sr, valid);
          else
            mx = sc >= 0.f ? t6_half_extreme<false, true>(sr, valid) : t6_half_extreme<true, true>(sr, valid);
          // combine with the partner half (same rows, other 64 columns)
          xmax[ph][x][h][row] = mx;
          if (turns) ptx::named_bar_sync(bar_mine, 128); else ptx::named_bar_sync(pair_bar, 64);
          const float mo = xmax[ph][x][h ^ 1][row];
          mx = sc >= 0.f ? fmaxf(mx, mo) : fminf(mx, mo);
          const float m_tile = mx * sc;
          if (tr && row == 0 && h == 0 && g < kT4TrTiles) tr[T4TR(g, 2 + x)] = t4_clk_after(__float_as_uint(mx));
          // P_x (and, for a rescale, O_x) is free once G2_x(g - 1) completed; without a rescale the
          // wait is deferred until the exponentials are in registers
          bool p_ready = g == 0;
          if (j == 0) {
            m_run = m_tile;
          } else if (__any_sync(0xffffffffu, m_tile > m_run + kT4Tau)) {
            // warp-uniform and identical in both halves (same rows, same combined max); each
            // half rescales its 16-column chunks of O_x
            if (!p_ready) {
              ptx::mbar_wait(&p_free[x], ph ^ 1u);
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
            for (int c0 = h * 16; c0 < p.TL; c0 += 32) {
              uint32_t r[16];
              ptx::tmem_ld16(tO + c0, r);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int k = 0; k < 16; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) * alpha);
              ptx::tmem_st16(tO + c0, r);
            }
          }
          if (tr && row == 0 && h == 0 && g < kT4TrTiles) tr[T4TR(g, 4 + x)] = t4_clk();   // exps start
          uint32_t pk[32];
          const uint32_t hand = turns ? bar_other : 0u;
          if (full)
            t6_exp_half<BF16, EMU, false>(pk, sr, sc, m_run, valid, l2, l2b, turn_chunk, hand);
          else
            t6_exp_half<BF16, 0, true>(pk, sr, sc, m_run, valid, l2, l2b, turn_chunk, hand);
          if (tr && row == 0 && h == 0 && g < kT4TrTiles) tr[T4TR(g, 6 + x)] = t4_clk();   // exps done
          if (!p_ready) {
            ptx::mbar_wait(&p_free[x], ph ^ 1u);
            ptx::tc_fence_after();
          }
          ptx::tmem_st16(tP, &pk[0]);
          ptx::tmem_st16(tP + 16, &pk[16]);
        }
        ptx::tmem_wait_st();
        if (tr && row == 0 && h == 0 && g < kT4TrTiles) tr[T4TR(g, 8 + x)] = t4_clk();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane0) ptx::mbar_arrive(&p_full[x]);
      }
      // l_full's parity protocol allows one phase in flight: publishing l of item ai waits
      // until the epilogue has read item ai - 1's.
      if (ai >= 1) ptx::mbar_wait(&l_free[x], (ai - 1) & 1);
      l_sm[x][h][ai & 1][row] = p.op == 2 ? (l2.x + l2.y) + (l2b.x + l2b.y) : (h == 0 ? 1.0f : 0.0f);   // E = O / l
      if (h == 0) m_sm[x][ai & 1][row] = m_run;
      __syncwarp();
      if (lane0) ptx::mbar_arrive(&l_full[x]);
      ++ai;
    }
    if (turns && x == 0) ptx::named_bar_sync(bar_mine, 128);   // slot 1's last hand-over
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[3] = ptx::globaltimer();
  if (warp == 20) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace mbci
