// chain_tc2.cuh — persistent, two-slot, stream-K version of the fused chain on sm_100a.
//
// What it computes is exactly chain_tc.cuh's E = op(A·B)·D (mbci.h); how the work is laid out:
//
// * Persistent cooperative grid, one CTA per SM.  A CTA runs TWO independent pipelines
//   ("slots"), each with its own softmax warpgroup, tcgen05 issuer warp and TMA warp, its own
//   half of tensor memory (256 columns) and its own SMEM ring.  Two softmax warps per SMSP
//   keep the MUFU (ex2) pipe fed while the other slot is in a max / load / store / epilogue
//   phase (one warp per SMSP reaches only ~70% of the ex2 rate — tools/microbench.cu).
// * Work = the paper's spatial loops m, h bound to units (β, m-tile, h-chunk), PAPER.md:285,
//   times the n loop cut into BN-key tiles.  The flat list of (unit, n-tile) "tile-works" is
//   split evenly over all slots (stream-K).  A unit cut between slots is finished by the slot
//   holding its first tile; every other piece stores its partial (O, m, l) to a workspace and
//   raises a flag, and the finisher merges (log-sum-exp for softmax, a sum otherwise).  The
//   merge is exact in real arithmetic (online-softmax identity) — DESIGN.md §5.
// *//   Per slot, TMEM columns: S_0 [0,BN), S_1 [BN,2BN) fp32 (double-buffered), O [2BN, +TLP).
//   P_j (16-bit, two per column) overwrites the first BN/2 columns of S_{j&1} after the
//   softmax warps have read S_j.  The MMA warp issues G1(j+1) before G2(j), so S_{j+1} is
//   ready while softmax(j) runs; tcgen05 ops retire in issue order, which orders G1(j+2)'s
//   write of S_{j&1} after G2(j)'s read of P_j without an explicit barrier.
// * The TMA warp polls its B and D rings independently (B_j is needed at G1(j), D_j only at
//   G2(j), one softmax later), so neither ring waits behind the other.
//
// Warps: 0-3 softmax slot 0 | 4-7 softmax slot 1 | 8 MMA slot 0 | 9 MMA slot 1 |
//        10 TMA slot 0 | 11 TMA slot 1.   384 threads; setmaxnreg gives the softmax
//        warpgroups 208 registers and warps 8-11 88 (<= 168 x 384 allocated at launch).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "ptx.cuh"

namespace mbci {

struct Tc2Params {
  int32_t M, N, K, L;
  int32_t batch, l_m, l_h;
  int32_t TL;             // output columns per unit (multiple of 16)
  int32_t k_steps;        // ceil(K/16); 0 => C = 0
  int32_t stages;         // B/D ring depth per slot
  int32_t a_bufs;         // A buffers per slot (1 or 2)
  int32_t op;             // 0 none, 1 scale, 2 softmax
  float scale;            // SCALE multiplier or softmax scale*log2(e)
  const int32_t* valid_len;
  void* E;
  int64_t ld_e, bs_e;
  uint32_t a_bytes, b_stage_bytes, d_stage_bytes, kp_rows;
  uint32_t slot_bytes;    // SMEM bytes per slot (1024-aligned)
  uint32_t idesc1, idesc2;
  int32_t W;              // total tile-works = units * tpu   (host guarantees W * n_slots < 2^62)
  int32_t tpu;            // n-tiles per unit = max(1, ceil(N / BN))
  int32_t n_slots;        // slots_per_cta * gridDim.x
  int32_t slots_per_cta;  // 2 (default) or 1 (slot 1 idles; diagnostics)
  float* ws;              // partial O: [n_slots][128][TLP] fp32, then m,l: [n_slots][2][128]
  int32_t* flags;         // [n_slots], 0 between launches
  uint64_t* trace;
};

constexpr int kT2Threads = 384;
#ifndef MBCI_TRACE
#define MBCI_TRACE 0
#endif
#ifndef MBCI_ISSUER_SPIN
#define MBCI_ISSUER_SPIN 1
#endif
#if MBCI_ISSUER_SPIN
#define MBCI_ISSUER_WAIT(bar, par) ptx::mbar_spin(bar, par)
#else
#define MBCI_ISSUER_WAIT(bar, par) ptx::mbar_wait(bar, par)
#endif
constexpr float kT2Tau = 8.0f;

__device__ __forceinline__ int32_t slot_lo(int32_t s, const Tc2Params& p) {
  return static_cast<int32_t>((static_cast<int64_t>(s) * p.W) / p.n_slots);
}
__device__ __forceinline__ int32_t slot_of_tile(int32_t t, const Tc2Params& p) {
  return static_cast<int32_t>(((static_cast<int64_t>(t) + 1) * p.n_slots - 1) / p.W);
}

// One piece of a slot's tile stream: unit u's nominal n-tiles [t0, t1); tiles >= nv are masked.
struct Piece {
  int32_t unit, t0, t1, nv, n_lim, beta, m0, h0;
  __device__ __forceinline__ int tiles() const { return max(0, min(t1, nv) - t0); }
};

template <int BN>
__device__ __forceinline__ Piece make_piece(const Tc2Params& p, int32_t t, int32_t hi) {
  Piece pc;
  pc.unit = t / p.tpu;
  pc.t0 = t - pc.unit * p.tpu;
  pc.t1 = min(p.tpu, pc.t0 + (hi - t));
  const int32_t uh = pc.unit / p.l_h;
  pc.h0 = (pc.unit - uh * p.l_h) * p.TL;
  pc.beta = uh / p.l_m;
  pc.m0 = (uh - pc.beta * p.l_m) * 128;
  int n_lim = p.N;
  if (p.op == 2 && p.valid_len != nullptr) n_lim = min(max(__ldg(p.valid_len + pc.beta), 0), p.N);
  pc.n_lim = n_lim;
  pc.nv = (n_lim + BN - 1) / BN;
  return pc;
}

// Walks the valid tiles of a slot's stream in order (the TMA warp keeps one per ring).
template <int BN>
struct TileIter {
  int32_t t, hi;   // next nominal tile, end
  Piece pc;
  int32_t jj, nt;  // index inside the current piece, its valid tiles
  int32_t g;       // stream index of the current valid tile
  int32_t piece;   // index of the current non-empty piece (-1 before the first)
  __device__ __forceinline__ void init(int32_t lo, int32_t hi_) {
    t = lo; hi = hi_; jj = 0; nt = 0; g = 0; piece = -1;
  }
  // move to the next valid tile (or stay on the current one if jj < nt); false when the
  // stream is exhausted.  new_piece is set when the tile is the first of a non-empty piece.
  __device__ __forceinline__ bool next(const Tc2Params& p, bool& new_piece) {
    new_piece = false;
    while (jj >= nt) {
      if (t >= hi) return false;
      pc = make_piece<BN>(p, t, hi);
      t += pc.t1 - pc.t0;
      nt = pc.tiles();
      jj = 0;
      if (nt > 0) { new_piece = true; ++piece; }
    }
    return true;
  }
};

template <bool BF16, int BN, int KCH, int BL, int DCH>
__global__ void __launch_bounds__(kT2Threads, 1)
    k_chain_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, const Tc2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem_base = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ uint32_t tmem_slot_addr;

  const int warp = threadIdx.x >> 5;
  const int slot = (warp < 8) ? (warp >> 2) : (warp & 1);   // 0-3,8,10 -> 0 ; 4-7,9,11 -> 1
  const int S = p.stages;
  uint8_t* sA = smem_base + slot * p.slot_bytes;
  uint8_t* sB = sA + p.a_bufs * p.a_bytes;
  uint8_t* sD = sB + S * p.b_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + S * p.d_stage_bytes);
  uint64_t* a_full = bars;             // [2]
  uint64_t* a_empty = bars + 2;        // [2]
  uint64_t* b_full = bars + 4;         // [S]
  uint64_t* b_empty = b_full + S;
  uint64_t* d_full = b_empty + S;
  uint64_t* d_empty = d_full + S;
  uint64_t* s_full = d_empty + S;   // [2] G1(j) landed in S_{j&1}
  uint64_t* p_full = s_full + 2;    // [2] softmax wrote P_j into S_{j&1}
  uint64_t* o_done = p_full + 2;    // one completion per G2 (lazy O rescale)
  uint64_t* o_final = o_done + 1;   // one completion per non-empty piece (epilogue)

  const int32_t gslot = static_cast<int32_t>(blockIdx.x) * p.slots_per_cta + slot;
  const bool slot_on = slot < p.slots_per_cta;
  const int32_t lo = slot_on ? slot_lo(gslot, p) : 0, hi = slot_on ? slot_lo(gslot + 1, p) : 0;
#if MBCI_TRACE
  uint64_t* tr = (p.trace && slot_on) ? p.trace + static_cast<int64_t>(gslot) * 256 : nullptr;
#else
  constexpr uint64_t* tr = nullptr;   // tracing compiled out (build with -DMBCI_TRACE=1)
#endif

  if (threadIdx.x == 0 || threadIdx.x == 128) {
    if (tr) {
      tr[0] = ptx::globaltimer();
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[2] = smid;
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&a_full[i], 1);
      ptx::mbar_init(&a_empty[i], 1);
    }
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&b_full[s], 1);
      ptx::mbar_init(&b_empty[s], 1);
      ptx::mbar_init(&d_full[s], 1);
      ptx::mbar_init(&d_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&p_full[b], 128);
    }
    ptx::mbar_init(o_done, 1);
    ptx::mbar_init(o_final, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 10 && lo < hi) {
    if (p.k_steps > 0) {
      ptx::tma_prefetch(&tmA);
      ptx::tma_prefetch(&tmB);
    }
    ptx::tma_prefetch(&tmD);
  }
  if (warp == 8) ptx::tmem_alloc(&tmem_slot_addr, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_slot_addr + slot * 256;
  const uint32_t tO = tbase + 2 * BN;
  if (tr && (threadIdx.x == 0 || threadIdx.x == 128)) tr[1] = ptx::globaltimer();

  if (warp >= 8) {
    if constexpr (BN > 64) ptx::setmaxnreg_dec<88>();
    if (warp >= 10) {
      // ============================================================ TMA producer (slot)
      if (ptx::elect_one()) {
        TileIter<BN> ib, id;   // B ring (+ A per piece) and D ring advance independently
        ib.init(lo, hi);
        id.init(lo, hi);
        bool nb = false, nd = false;
        bool more_b = ib.next(p, nb);
        bool more_d = id.next(p, nd);
        bool a_pending = more_b && nb;   // the B iterator entered a piece whose A is not loaded
        while (more_b || more_d) {
          bool progressed = false;
          if (more_b) {
            bool ok = true;
            if (a_pending) {
              if (p.k_steps > 0) {
                const int ab = ib.piece % p.a_bufs;
                if (ib.piece >= p.a_bufs && !ptx::mbar_test(&a_empty[ab], ((ib.piece / p.a_bufs) - 1) & 1)) {
                  ok = false;
                } else {
                  ptx::mbar_arrive_expect_tx(&a_full[ab], p.a_bytes);
#pragma unroll
                  for (int c = 0; c < KCH; ++c)
                    ptx::tma_load_3d(sA + ab * p.a_bytes + c * 16384, &tmA, &a_full[ab], c * 64, ib.pc.m0,
                                     ib.pc.beta);
                }
              }
              if (ok) a_pending = false;
            }
            if (ok) {
              bool issued = true;
              if (p.k_steps > 0) {
                const int s = ib.g % S;
                if (ib.g < S || ptx::mbar_test(&b_empty[s], ((ib.g / S) - 1) & 1)) {
                  const int j = ib.pc.t0 + ib.jj;
                  uint8_t* dst = sB + s * p.b_stage_bytes;
                  if (tr && ib.g < 8) tr[8 + 16 * ib.g + 14] = ptx::globaltimer();
                  ptx::mbar_arrive_expect_tx(&b_full[s], p.b_stage_bytes);
                  if constexpr (BL == 1) {
#pragma unroll
                    for (int c = 0; c < KCH; ++c)
                      ptx::tma_load_3d(dst + c * (BN * 128), &tmB, &b_full[s], c * 64, j * BN, ib.pc.beta);
                  } else {
#pragma unroll
                    for (int c = 0; c < BN / 64; ++c)
                      ptx::tma_load_3d(dst + c * (p.kp_rows * 128), &tmB, &b_full[s], j * BN + c * 64, 0,
                                       ib.pc.beta);
                  }
                } else {
                  issued = false;
                }
              }
              if (issued) {
                ++ib.jj;
                ++ib.g;
                more_b = ib.next(p, nb);
                a_pending = more_b && nb;
                progressed = true;
              }
            }
          }
          if (more_d) {
            const int s = id.g % S;
            if (id.g < S || ptx::mbar_test(&d_empty[s], ((id.g / S) - 1) & 1)) {
              const int j = id.pc.t0 + id.jj;
              uint8_t* ddst = sD + s * p.d_stage_bytes;
              if (tr && id.g < 8) tr[8 + 16 * id.g + 15] = ptx::globaltimer();
              ptx::mbar_arrive_expect_tx(&d_full[s], p.d_stage_bytes);
#pragma unroll
              for (int c = 0; c < DCH; ++c)
                ptx::tma_load_3d(ddst + c * (BN * 128), &tmD, &d_full[s], id.pc.h0 + c * 64, j * BN, id.pc.beta);
              ++id.jj;
              ++id.g;
              more_d = id.next(p, nd);
              progressed = true;
            }
          }
          if (!progressed) __nanosleep(32);
        }
      }
    } else {
      // ============================================================ tcgen05 issuer (slot)
      if (ptx::elect_one()) {
        const uint32_t idesc1 = p.idesc1, idesc2 = p.idesc2;
        const int k_steps = p.k_steps, a_bufs = p.a_bufs;
        const uint32_t a_bytes = p.a_bytes, b_stage = p.b_stage_bytes, d_stage = p.d_stage_bytes;
        // descriptor templates; per MMA only the 14-bit start-address field changes
        const uint64_t dA = ptx::sdesc_sw128(0, 16, 1024);
        const uint64_t dB = (BL == 1) ? ptx::sdesc_sw128(0, 16, 1024) : ptx::sdesc_sw128(0, p.kp_rows * 128, 1024);
        const uint64_t dD = ptx::sdesc_sw128(0, BN * 128, 1024);
        const uint32_t sA0 = ptx::smem_u32(sA), sB0 = ptx::smem_u32(sB), sD0 = ptx::smem_u32(sD);
        int32_t t = lo;
        int32_t g = 0, piece = 0;
        int32_t prev_s = -1;           // D slot of the pending G2 (-1: none)
        bool prev_first = false, prev_last = false;
        while (true) {
          Piece pc;
          int nt = 0;
          bool have = false;
          while (t < hi) {
            pc = make_piece<BN>(p, t, hi);
            t += pc.t1 - pc.t0;
            nt = pc.tiles();
            if (nt > 0) { have = true; break; }
          }
          // retire the previous piece's last G2 before touching a new A (or at the end)
          if (prev_s >= 0) {
            const int gi = g - 1, sp = prev_s;
            MBCI_ISSUER_WAIT(&p_full[gi & 1], (gi >> 1) & 1);
            if (tr && gi < 8) tr[8 + 16 * gi + 12] = ptx::globaltimer();
            MBCI_ISSUER_WAIT(&d_full[sp], (gi / S) & 1);
            ptx::tc_fence_after();
            const uint32_t d_lo = (sD0 + sp * d_stage) >> 4;
            const uint32_t tPb = tbase + (gi & 1) * BN;
#pragma unroll
            for (int ks = 0; ks < BN / 16; ++ks)
              ptx::mma_ts(tO, tPb + ks * 8, dD + d_lo + ks * 128, idesc2, (!prev_first || ks > 0) ? 1u : 0u);
            if (tr && gi < 8) tr[8 + 16 * gi + 13] = ptx::globaltimer();
            ptx::mma_commit(&d_empty[sp]);
            ptx::mma_commit(o_done);
            if (prev_last) ptx::mma_commit(o_final);
            prev_s = -1;
          }
          if (!have) break;
          const int ab = piece % a_bufs;
          if (k_steps > 0) MBCI_ISSUER_WAIT(&a_full[ab], (piece / a_bufs) & 1);
          const uint32_t a_lo = (sA0 + ab * a_bytes) >> 4;
          for (int jj = 0; jj < nt; ++jj, ++g) {
            const int s = g % S;
            // ---- G1(g): S_{g&1} = A · B_j  (its previous P was read by G2(g-2), issued earlier)
            if (tr && g < 8) tr[8 + 16 * g + 10] = ptx::globaltimer();
            if (k_steps > 0) {
              MBCI_ISSUER_WAIT(&b_full[s], (g / S) & 1);
              if (tr && g < 8) tr[128 + 8 * g + 0] = ptx::globaltimer();
              ptx::tc_fence_after();
              const uint32_t b_lo = (sB0 + s * b_stage) >> 4;
              for (int ks = 0; ks < k_steps; ++ks) {
                const uint32_t ao = (ks >> 2) * 1024 + (ks & 3) * 2;             // (16384 B, 32 B) >> 4
                const uint32_t bo = (BL == 1) ? (ks >> 2) * (BN * 8) + (ks & 3) * 2 : ks * 128;
                ptx::mma_ss(tbase + (g & 1) * BN, dA + a_lo + ao, dB + b_lo + bo, idesc1, ks > 0 ? 1u : 0u);
                if (tr && g < 8 && ks < 4) tr[128 + 8 * g + 1 + ks] = ptx::globaltimer();
              }
              ptx::mma_commit(&b_empty[s]);
              if (tr && g < 8) tr[128 + 8 * g + 5] = ptx::globaltimer();
              if (jj == nt - 1) ptx::mma_commit(&a_empty[ab]);
            } else {
              ptx::tc_fence_after();
            }
            ptx::mma_commit(&s_full[g & 1]);
            if (tr && g < 8) tr[8 + 16 * g + 11] = ptx::globaltimer();
            // ---- G2(g-1): O += P · D_{j-1}, one tile behind G1 so both overlap softmax
            if (prev_s >= 0) {
              const int gi = g - 1, sp = prev_s;
              MBCI_ISSUER_WAIT(&p_full[gi & 1], (gi >> 1) & 1);
              if (tr && gi < 8) tr[8 + 16 * gi + 12] = ptx::globaltimer();
              MBCI_ISSUER_WAIT(&d_full[sp], (gi / S) & 1);
              ptx::tc_fence_after();
              const uint32_t d_lo = (sD0 + sp * d_stage) >> 4;
              const uint32_t tPb = tbase + (gi & 1) * BN;
#pragma unroll
              for (int ks = 0; ks < BN / 16; ++ks)
                ptx::mma_ts(tO, tPb + ks * 8, dD + d_lo + ks * 128, idesc2, (!prev_first || ks > 0) ? 1u : 0u);
              if (tr && gi < 8) tr[8 + 16 * gi + 13] = ptx::globaltimer();
              ptx::mma_commit(&d_empty[sp]);
              ptx::mma_commit(o_done);
              if (prev_last) ptx::mma_commit(o_final);
            }
            prev_s = s;
            prev_first = (jj == 0);
            prev_last = (jj == nt - 1);
          }
          ++piece;
        }
      }
    }
  } else {
    // ============================================================== softmax warps (slot)
    if constexpr (BN > 64) ptx::setmaxnreg_inc<208>();
    const int wq = warp & 3;                 // TMEM lane quadrant
    const int row = wq * 32 + (threadIdx.x & 31);
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const float sc = p.scale;
    const int TLP = p.TL;
    constexpr int TLMAX = DCH * 64;
    int32_t t = lo;
    int32_t g = 0;
    int32_t pieces_done = 0;
    while (t < hi) {
      const Piece pc = make_piece<BN>(p, t, hi);
      t += pc.t1 - pc.t0;
      const int nt = pc.tiles();
      float m_run = -INFINITY, l_run = 0.f;
      for (int jj = 0; jj < nt; ++jj, ++g) {
        const int j = pc.t0 + jj;
        ptx::mbar_wait(&s_full[g & 1], (g >> 1) & 1);
        const bool trj = tr && (row & 31) == 0 && g < 8;   // lane 0 of each warp
        if (trj && row == 0) tr[8 + 16 * g + 0] = ptx::globaltimer();
        ptx::tc_fence_after();
        uint32_t sr[BN];
        if (p.k_steps > 0) {
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) ptx::tmem_ld32(tbase + (g & 1) * BN + lane_off + c * 32, &sr[c * 32]);
          ptx::tmem_wait_ld();
        } else {
#pragma unroll
          for (int c = 0; c < BN; ++c) sr[c] = 0u;
        }
        if (trj) tr[8 + 16 * g + 1 + wq] = ptx::globaltimer();
        float s[BN];
#pragma unroll
        for (int c = 0; c < BN; ++c) s[c] = __uint_as_float(sr[c]);
        bool rescale = false;
        float alpha = 1.f;
        const int valid = pc.n_lim - j * BN;
        const bool full = valid >= BN;
        if (p.op == 2) {
          float mx;
          if (full) {
            float a0 = s[0], a1 = s[1];
            if (sc >= 0.f) {
#pragma unroll
              for (int c = 2; c + 3 < BN; c += 4) {
                a0 = ptx::max3(a0, s[c], s[c + 1]);
                a1 = ptx::max3(a1, s[c + 2], s[c + 3]);
              }
              mx = ptx::max3(a0, a1, ptx::max3(s[BN - 2], s[BN - 1], s[0]));
            } else {
#pragma unroll
              for (int c = 2; c + 3 < BN; c += 4) {
                a0 = ptx::min3(a0, s[c], s[c + 1]);
                a1 = ptx::min3(a1, s[c + 2], s[c + 3]);
              }
              mx = ptx::min3(a0, a1, ptx::min3(s[BN - 2], s[BN - 1], s[0]));
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
          if (jj == 0) {
            m_run = m_tile;
          } else if (__any_sync(0xffffffffu, m_tile > m_run + kT2Tau)) {
            const float m_new = fmaxf(m_run, m_tile);
            alpha = ptx::ex2(m_run - m_new);
            l_run *= alpha;
            m_run = m_new;
            rescale = true;
          }
        }
        if (trj && row == 0) tr[8 + 16 * g + 5] = ptx::globaltimer();
        if (rescale) {
          // O must hold G2(g-1).  s_full(g) completing implies G2(g-2) retired (in-order), so
          // o_done has completed g-1 or g times: the parity wait below is unambiguous.
          ptx::mbar_wait(o_done, (g - 1) & 1);
          ptx::tc_fence_after();
          for (int c0 = 0; c0 < TLP; c0 += 16) {
            uint32_t r[16];
            ptx::tmem_ld16(tO + lane_off + c0, r);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) * alpha);
            ptx::tmem_st16(tO + lane_off + c0, r);
          }
        }
        if (p.op == 2) {
          const float neg_m = -m_run;
          float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
          for (int c32 = 0; c32 < BN / 64; ++c32) {
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int e = c32 * 64 + 2 * c;
              float p0 = ptx::ex2(fmaf(s[e], sc, neg_m));
              float p1 = ptx::ex2(fmaf(s[e + 1], sc, neg_m));
              if (!full) {
                p0 = (e < valid) ? p0 : 0.f;
                p1 = (e + 1 < valid) ? p1 : 0.f;
              }
              ls0 += p0;
              ls1 += p1;
              pk[c] = ptx::pack2<BF16>(p0, p1);
            }
            ptx::tmem_st32(tbase + (g & 1) * BN + lane_off + c32 * 32, pk);
          }
          l_run += ls0 + ls1;
        } else {
#pragma unroll
          for (int c32 = 0; c32 < BN / 64; ++c32) {
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int e = c32 * 64 + 2 * c;
              pk[c] = p.op == 1 ? ptx::pack2<BF16>(s[e] * sc, s[e + 1] * sc) : ptx::pack2<BF16>(s[e], s[e + 1]);
            }
            ptx::tmem_st32(tbase + (g & 1) * BN + lane_off + c32 * 32, pk);
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_full[g & 1]);
        if (trj) tr[8 + 16 * g + 6 + wq] = ptx::globaltimer();
      }

      // ---------------------------------------------------------- piece epilogue
      float o[TLMAX];
      if (nt > 0) {
        ptx::mbar_wait(o_final, pieces_done & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < TLMAX; c0 += 16) {
          if (c0 < TLP) {
            uint32_t r[16];
            ptx::tmem_ld16(tO + lane_off + c0, r);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q) o[c0 + q] = __uint_as_float(r[q]);
          }
        }
        ++pieces_done;
      } else {
#pragma unroll
        for (int c = 0; c < TLMAX; ++c) o[c] = 0.f;
      }
      if (p.op != 2) {
        m_run = 0.f;
      } else if (nt == 0) {
        m_run = -INFINITY;
        l_run = 0.f;
      }
      float* ws_o = p.ws;                                                 // [P][128][TLP]
      float* ws_ml = p.ws + static_cast<int64_t>(p.n_slots) * 128 * TLP;  // [P][2][128]
      if (pc.t0 != 0) {
        // not the unit's first tile: publish the partial (O, m, l) for the finisher
        float* wo = ws_o + (static_cast<int64_t>(gslot) * 128 + row) * TLP;
#pragma unroll
        for (int c0 = 0; c0 < TLMAX; c0 += 4)
          if (c0 < TLP) __stcg(reinterpret_cast<float4*>(wo + c0), make_float4(o[c0], o[c0 + 1], o[c0 + 2], o[c0 + 3]));
        __stcg(ws_ml + gslot * 256 + row, m_run);
        __stcg(ws_ml + gslot * 256 + 128 + row, l_run);
        ptx::named_bar_sync(1 + slot, 128);
        if (row == 0) {
          __threadfence();
          ptx::st_release_gpu(p.flags + gslot, 1);
        }
      } else {
        // finisher: merge the partials of the unit's later pieces (held by later slots)
        const int32_t s_end = slot_of_tile(pc.unit * p.tpu + p.tpu - 1, p);
        for (int32_t q = gslot + 1; q <= s_end; ++q) {
          if (row == 0) {
            ptx::spin_acquire_gpu(p.flags + q, 1);
            __threadfence();
            p.flags[q] = 0;   // reset for the next launch (only this thread waits on it)
          }
          ptx::named_bar_sync(1 + slot, 128);
          const float* qo = ws_o + (static_cast<int64_t>(q) * 128 + row) * TLP;
          const float m2 = __ldcg(ws_ml + q * 256 + row);
          const float l2 = __ldcg(ws_ml + q * 256 + 128 + row);
          float a = 1.f, b = 1.f;
          if (p.op == 2) {
            const float mm = fmaxf(m_run, m2);
            a = (mm == -INFINITY) ? 0.f : ptx::ex2(m_run - mm);
            b = (mm == -INFINITY) ? 0.f : ptx::ex2(m2 - mm);
            l_run = l_run * a + l2 * b;
            m_run = mm;
          }
#pragma unroll
          for (int c0 = 0; c0 < TLMAX; c0 += 4) {
            if (c0 < TLP) {
              const float4 v = __ldcg(reinterpret_cast<const float4*>(qo + c0));
              o[c0] = o[c0] * a + v.x * b;
              o[c0 + 1] = o[c0 + 1] * a + v.y * b;
              o[c0 + 2] = o[c0 + 2] * a + v.z * b;
              o[c0 + 3] = o[c0 + 3] * a + v.w * b;
            }
          }
        }
        const float inv = (p.op == 2) ? (l_run > 0.f ? 1.0f / l_run : 0.f) : 1.0f;
        const int gm = pc.m0 + row;
        const int ncols = min(TLP, p.L - pc.h0);
        uint16_t* erow = reinterpret_cast<uint16_t*>(p.E) + static_cast<int64_t>(pc.beta) * p.bs_e +
                         static_cast<int64_t>(gm) * p.ld_e + pc.h0;
        if (gm < p.M) {
#pragma unroll
          for (int c0 = 0; c0 < TLMAX; c0 += 16) {
            if (c0 < ncols) {
              uint32_t w[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) w[q] = ptx::pack2<BF16>(o[c0 + 2 * q] * inv, o[c0 + 2 * q + 1] * inv);
              if (c0 + 16 <= ncols) {
                uint4* dst = reinterpret_cast<uint4*>(erow + c0);
                dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
              } else {
#pragma unroll
                for (int q = 0; q < 16; ++q)
                  if (c0 + q < ncols) erow[c0 + q] = static_cast<uint16_t>((w[q >> 1] >> ((q & 1) * 16)) & 0xFFFFu);
              }
            }
          }
        }
      }
    }
    if (tr && row == 0) tr[5] = ptx::globaltimer();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_slot_addr, 512);
  }
}

}  // namespace mbci
