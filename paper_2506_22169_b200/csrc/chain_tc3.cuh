// chain_tc3.cuh — persistent stream-K fused chain, two Q tiles per CTA sharing every B/D tile.
//
// Same arithmetic as chain_tc.cuh (E = op(A·B)·D, mbci.h); the layout of the work:
//
// * Persistent cooperative grid, one CTA per SM.  A work unit is (β, a PAIR of 128-row m-tiles,
//   an h-chunk) — the paper's spatial loops m, h bound to CTAs (Rule 1) — and its
//   n loop is cut into BN = 128-key tiles.  The flat list of (unit, n-tile) tile-works is split
//   evenly over the CTAs (stream-K); a unit cut between CTAs is finished by the CTA holding its
//   first tile, the other pieces publish partial (O, m, l) and a flag, and the finisher merges
//   them (online-softmax identity, exact in real arithmetic).
// * Each B_j / D_j tile is loaded once and feeds both Q tiles, so the single tcgen05 issuer
//   amortises every barrier wait and B/D handshake over 2 x 128 x 128 scores (tools/
//   commit_bench.cu, handoff_bench.cu: a wait costs ~200 cycles, an MMA issue ~50).
// * TMEM (512 columns): S_0 [0,128) S_1 [128,256) fp32, O_0 [256, 256+TL) O_1 [256+TL, 256+2TL).
//   P_x (16-bit, two per column) overwrites the first 64 columns of S_x after softmax x read S_x.
//   Issue order per tile j: G2_0(j-1) G1_0(j) G2_1(j-1) G1_1(j): G1_x(j) rewrites S_x only after
//   G2_x(j-1) read P_x (tcgen05 ops retire in issue order), and s_full_x(j) therefore also
//   certifies that O_x holds G2_x(j-1) — the softmax warps may rescale O_x without another wait.
//
// Warps: 0-3 softmax of Q tile 0 | 4-7 softmax of Q tile 1 | 8 tcgen05 issuer | 9 TMA producer.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "ptx.cuh"

#ifndef MBCI_TRACE
#define MBCI_TRACE 0
#endif

namespace mbci {

struct Tc3Params {
  int32_t M, N, K, L;
  int32_t batch, l_mp, l_h;  // m-tile PAIRS per batch, h-chunks
  int32_t TL;                // output columns per unit (multiple of 16, <= 128)
  int32_t k_steps;           // ceil(K/16); 0 => C = 0
  int32_t stages;            // B/D ring depth
  int32_t q_bufs;            // Q-pair buffers (1 or 2)
  int32_t op;                // 0 none, 1 scale, 2 softmax
  float scale;               // SCALE multiplier or softmax scale*log2(e)
  const int32_t* valid_len;
  void* E;
  int64_t ld_e, bs_e;
  uint32_t q_bytes;          // one Q tile (128 rows x K), both tiles of a pair = 2 * q_bytes
  uint32_t b_stage_bytes, d_stage_bytes, kp_rows;
  uint32_t idesc1, idesc2;
  int32_t W;                 // tile-works = units * tpu
  int32_t tpu;               // n-tiles per unit = max(1, ceil(N / 128))
  int32_t n_ctas;            // gridDim.x
  float* ws;                 // partials: O [n_ctas][256][TL] fp32, then (m, l) [n_ctas][2][256]
  int32_t* flags;            // [n_ctas], 0 between launches
  uint64_t* trace;
};

constexpr int kT3Threads = 320;
constexpr int kT3BN = 128;
constexpr float kT3Tau = 8.0f;

struct Piece3 {
  int32_t unit, t0, t1, nv, n_lim, beta, m0, h0;
  __device__ __forceinline__ int tiles() const { return max(0, min(t1, nv) - t0); }
};

__device__ __forceinline__ int32_t cta_lo(int32_t c, const Tc3Params& p) {
  return static_cast<int32_t>((static_cast<int64_t>(c) * p.W) / p.n_ctas);
}
__device__ __forceinline__ int32_t cta_of_tile(int32_t t, const Tc3Params& p) {
  return static_cast<int32_t>(((static_cast<int64_t>(t) + 1) * p.n_ctas - 1) / p.W);
}

__device__ __forceinline__ Piece3 make_piece3(const Tc3Params& p, int32_t t, int32_t hi) {
  Piece3 pc;
  pc.unit = t / p.tpu;
  pc.t0 = t - pc.unit * p.tpu;
  pc.t1 = min(p.tpu, pc.t0 + (hi - t));
  const int32_t uh = pc.unit / p.l_h;
  pc.h0 = (pc.unit - uh * p.l_h) * p.TL;
  pc.beta = uh / p.l_mp;
  pc.m0 = (uh - pc.beta * p.l_mp) * 256;
  int n_lim = p.N;
  if (p.op == 2 && p.valid_len != nullptr) n_lim = min(max(__ldg(p.valid_len + pc.beta), 0), p.N);
  pc.n_lim = n_lim;
  pc.nv = (n_lim + kT3BN - 1) / kT3BN;
  return pc;
}

struct TileIter3 {
  int32_t t, hi;
  Piece3 pc;
  int32_t jj, nt, g, piece;
  __device__ __forceinline__ void init(int32_t lo, int32_t hi_) {
    t = lo; hi = hi_; jj = 0; nt = 0; g = 0; piece = -1;
  }
  __device__ __forceinline__ bool next(const Tc3Params& p, bool& new_piece) {
    new_piece = false;
    while (jj >= nt) {
      if (t >= hi) return false;
      pc = make_piece3(p, t, hi);
      t += pc.t1 - pc.t0;
      nt = pc.tiles();
      jj = 0;
      if (nt > 0) { new_piece = true; ++piece; }
    }
    return true;
  }
};

template <bool BF16, int KCH, int BL, int DCH>
__global__ void __launch_bounds__(kT3Threads, 1)
    k_chain_tc3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, const Tc3Params p) {
  constexpr int BN = kT3BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ uint32_t tmem_base_addr;

  const int warp = threadIdx.x >> 5;
  const int S = p.stages;
  uint8_t* sQ = smem;                                   // [q_bufs][2][q_bytes]
  uint8_t* sB = sQ + p.q_bufs * 2 * p.q_bytes;          // [S][b_stage]
  uint8_t* sD = sB + S * p.b_stage_bytes;               // [S][d_stage]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + S * p.d_stage_bytes);
  uint64_t* q_full = bars;            // [2]
  uint64_t* q_empty = bars + 2;       // [2]
  uint64_t* b_full = bars + 4;        // [S]
  uint64_t* d_full = b_full + S;      // [S]
  uint64_t* kv_empty = d_full + S;    // [S]
  uint64_t* s_full = kv_empty + S;    // [2] per Q tile
  uint64_t* p_full = s_full + 2;      // [2] per Q tile (128 arrivals)
  uint64_t* o_final = p_full + 2;     // one completion per non-empty piece

  const int32_t cta = static_cast<int32_t>(blockIdx.x);
  const int32_t lo = cta_lo(cta, p), hi = cta_lo(cta + 1, p);
#if MBCI_TRACE
  uint64_t* tr = p.trace ? p.trace + static_cast<int64_t>(cta) * 256 : nullptr;
#else
  constexpr uint64_t* tr = nullptr;
#endif

  if (threadIdx.x == 0) {
    if (tr) {
      tr[0] = ptx::globaltimer();
      tr[6] = clock64();
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 128);
    }
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&b_full[s], 1);
      ptx::mbar_init(&d_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    ptx::mbar_init(o_final, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 9 && lo < hi) {
    if (p.k_steps > 0) {
      ptx::tma_prefetch(&tmA);
      ptx::tma_prefetch(&tmB);
    }
    ptx::tma_prefetch(&tmD);
  }
  if (warp == 8) ptx::tmem_alloc(&tmem_base_addr, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_addr;

  if (warp == 9) {
    // ================================================================ TMA producer
    if (ptx::elect_one()) {
      const int k_steps = p.k_steps, q_bufs = p.q_bufs;
      const uint32_t q_bytes = p.q_bytes, b_stage = p.b_stage_bytes, d_stage = p.d_stage_bytes;
      TileIter3 ib, id;
      ib.init(lo, hi);
      id.init(lo, hi);
      bool nb = false, nd = false;
      bool more_b = ib.next(p, nb);
      bool more_d = id.next(p, nd);
      bool q_pending = more_b && nb;
      while (more_b || more_d) {
        bool progressed = false;
        if (more_b) {
          bool ok = true;
          if (q_pending) {
            if (k_steps > 0) {
              const int qb = ib.piece % q_bufs;
              if (ib.piece >= q_bufs && !ptx::mbar_test(&q_empty[qb], ((ib.piece / q_bufs) - 1) & 1)) {
                ok = false;
              } else {
                uint8_t* dst = sQ + qb * 2 * q_bytes;
                ptx::mbar_arrive_expect_tx(&q_full[qb], 2 * q_bytes);
#pragma unroll
                for (int x = 0; x < 2; ++x)
#pragma unroll
                  for (int c = 0; c < KCH; ++c)
                    ptx::tma_load_3d(dst + x * q_bytes + c * 16384, &tmA, &q_full[qb], c * 64, ib.pc.m0 + 128 * x,
                                     ib.pc.beta);
              }
            }
            if (ok) q_pending = false;
          }
          if (ok) {
            const int s = ib.g % S;
            if (ib.g < S || ptx::mbar_test(&kv_empty[s], ((ib.g / S) - 1) & 1)) {
              if (k_steps > 0) {
                const int j = ib.pc.t0 + ib.jj;
                uint8_t* dst = sB + s * b_stage;
                if (tr && ib.g < 8) tr[8 + 16 * ib.g + 10] = ptx::globaltimer();
                ptx::mbar_arrive_expect_tx(&b_full[s], b_stage);
                if constexpr (BL == 1) {
#pragma unroll
                  for (int c = 0; c < KCH; ++c)
                    ptx::tma_load_3d(dst + c * (BN * 128), &tmB, &b_full[s], c * 64, j * BN, ib.pc.beta);
                } else {
#pragma unroll
                  for (int c = 0; c < BN / 64; ++c)
                    ptx::tma_load_3d(dst + c * (p.kp_rows * 128), &tmB, &b_full[s], j * BN + c * 64, 0, ib.pc.beta);
                }
              }
              ++ib.jj;
              ++ib.g;
              more_b = ib.next(p, nb);
              q_pending = more_b && nb;
              progressed = true;
            }
          }
        }
        if (more_d && id.g < ib.g) {   // D_j's slot is released together with B_j's (kv_empty)
          const int s = id.g % S;
          const int j = id.pc.t0 + id.jj;
          uint8_t* ddst = sD + s * d_stage;
          if (tr && id.g < 8) tr[8 + 16 * id.g + 11] = ptx::globaltimer();
          ptx::mbar_arrive_expect_tx(&d_full[s], d_stage);
#pragma unroll
          for (int c = 0; c < DCH; ++c)
            ptx::tma_load_3d(ddst + c * (BN * 128), &tmD, &d_full[s], id.pc.h0 + c * 64, j * BN, id.pc.beta);
          ++id.jj;
          ++id.g;
          more_d = id.next(p, nd);
          progressed = true;
        }
        if (!progressed) __nanosleep(20);
      }
    }
  } else if (warp == 8) {
    // ================================================================ tcgen05 issuer
    if (ptx::elect_one()) {
      const uint32_t idesc1 = p.idesc1, idesc2 = p.idesc2;
      const int k_steps = p.k_steps, q_bufs = p.q_bufs;
      const uint32_t q_bytes = p.q_bytes, b_stage = p.b_stage_bytes, d_stage = p.d_stage_bytes;
      const uint64_t dA = ptx::sdesc_sw128(0, 16, 1024);
      const uint64_t dB = (BL == 1) ? ptx::sdesc_sw128(0, 16, 1024) : ptx::sdesc_sw128(0, p.kp_rows * 128, 1024);
      const uint64_t dD = ptx::sdesc_sw128(0, BN * 128, 1024);
      const uint32_t sQ0 = ptx::smem_u32(sQ), sB0 = ptx::smem_u32(sB), sD0 = ptx::smem_u32(sD);
      const uint32_t TL = static_cast<uint32_t>(p.TL);
      int32_t t = lo;
      int32_t g = 0, piece = 0;
      // G1_x(g): S_x = Q_x · B_j
      auto g1 = [&](int x, uint32_t q_lo, int s) {
        const uint32_t b_lo = (sB0 + s * b_stage) >> 4;
        const uint32_t qx = q_lo + x * (q_bytes >> 4);
        for (int ks = 0; ks < k_steps; ++ks) {
          const uint32_t ao = (ks >> 2) * 1024 + (ks & 3) * 2;
          const uint32_t bo = (BL == 1) ? (ks >> 2) * (BN * 8) + (ks & 3) * 2 : ks * 128;
          ptx::mma_ss(tmem + x * BN, dA + qx + ao, dB + b_lo + bo, idesc1, ks > 0 ? 1u : 0u);
        }
      };
      // G2_x(g): O_x += P_x · D_j
      auto g2 = [&](int x, int s, bool first) {
        const uint32_t d_lo = (sD0 + s * d_stage) >> 4;
        const uint32_t tO = tmem + 256 + x * TL;
#pragma unroll
        for (int ks = 0; ks < BN / 16; ++ks)
          ptx::mma_ts(tO, tmem + x * BN + ks * 8, dD + d_lo + ks * 128, idesc2, (!first || ks > 0) ? 1u : 0u);
      };
      while (t < hi) {
        const Piece3 pc = make_piece3(p, t, hi);
        t += pc.t1 - pc.t0;
        const int nt = pc.tiles();
        if (nt <= 0) continue;
        const int qb = piece % q_bufs;
        if (k_steps > 0) ptx::mbar_wait(&q_full[qb], (piece / q_bufs) & 1);
        const uint32_t q_lo = (sQ0 + qb * 2 * q_bytes) >> 4;
        // prologue: G1 of the piece's first tile for both Q tiles
        {
          const int s = g % S;
          if (k_steps > 0) {
            ptx::mbar_wait(&b_full[s], (g / S) & 1);
            ptx::tc_fence_after();
            g1(0, q_lo, s);
            ptx::mma_commit(&s_full[0]);
            g1(1, q_lo, s);
            ptx::mma_commit(&s_full[1]);
            if (nt == 1) ptx::mma_commit(&q_empty[qb]);
          } else {
            ptx::tc_fence_after();
            ptx::mma_commit(&s_full[0]);
            ptx::mma_commit(&s_full[1]);
          }
        }
        for (int jj = 0; jj < nt; ++jj, ++g) {
          const int s = g % S;
          const bool more = jj + 1 < nt;
          const int s1 = (g + 1) % S;
          ptx::mbar_wait(&d_full[s], (g / S) & 1);
          if (tr && g < 8) tr[8 + 16 * g + 4] = ptx::globaltimer();
          // Q tile 0: G2_0(g) then G1_0(g+1)
          ptx::mbar_wait(&p_full[0], g & 1);
          if (tr && g < 8) tr[8 + 16 * g + 5] = ptx::globaltimer();
          ptx::tc_fence_after();
          g2(0, s, jj == 0);
          if (more) {
            if (k_steps > 0) {
              ptx::mbar_wait(&b_full[s1], ((g + 1) / S) & 1);
              ptx::tc_fence_after();
              g1(0, q_lo, s1);
            }
            ptx::mma_commit(&s_full[0]);
          }
          if (tr && g < 8) tr[8 + 16 * g + 6] = ptx::globaltimer();
          // Q tile 1: G2_1(g) then G1_1(g+1)
          ptx::mbar_wait(&p_full[1], g & 1);
          if (tr && g < 8) tr[8 + 16 * g + 7] = ptx::globaltimer();
          ptx::tc_fence_after();
          g2(1, s, jj == 0);
          ptx::mma_commit(&kv_empty[s]);     // B_g and D_g fully consumed
          if (more) {
            if (k_steps > 0) g1(1, q_lo, s1);
            ptx::mma_commit(&s_full[1]);
            if (jj + 2 == nt && k_steps > 0) ptx::mma_commit(&q_empty[qb]);
          } else {
            ptx::mma_commit(o_final);
          }
          if (tr && g < 8) tr[8 + 16 * g + 8] = ptx::globaltimer();
        }
        ++piece;
      }
    }
  } else {
    // ================================================================ softmax warps
    const int x = warp >> 2;                 // Q tile of this warpgroup
    const int wq = warp & 3;                 // TMEM lane quadrant
    const int row = wq * 32 + (threadIdx.x & 31);
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tSx = tmem + x * BN + lane_off;
    const uint32_t tOx = tmem + 256 + x * p.TL + lane_off;
    const float sc = p.scale;
    const int TLP = p.TL;
    constexpr int TLMAX = DCH * 64;
    int32_t t = lo;
    int32_t g = 0;
    int32_t pieces_done = 0;
    while (t < hi) {
      const Piece3 pc = make_piece3(p, t, hi);
      t += pc.t1 - pc.t0;
      const int nt = pc.tiles();
      float m_run = -INFINITY, l_run = 0.f;
      for (int jj = 0; jj < nt; ++jj, ++g) {
        const int j = pc.t0 + jj;
        ptx::mbar_wait(&s_full[x], g & 1);
        const bool trj = tr && row == 0 && g < 8;
        if (trj) tr[8 + 16 * g + 0 + 2 * x] = ptx::globaltimer();
        ptx::tc_fence_after();
        // Two passes over S in TMEM (32 columns at a time keeps ~70 live registers): pass 1 the
        // row max, pass 2 exp2 / convert, writing P_x in place (chunk c of S -> columns 16c.. of
        // P, all already consumed).
        const bool has_s = p.k_steps > 0;
        const int valid = pc.n_lim - j * BN;
        const bool full = valid >= BN;
        auto load_chunk = [&](int c, float (&v)[32]) {
          if (has_s) {
            ptx::tmem_ld32(tSx + c * 32, reinterpret_cast<uint32_t*>(v));
            ptx::tmem_wait_ld();
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = 0.f;
          }
        };
        if (p.op == 2) {
          float mx = (sc >= 0.f) ? -INFINITY : INFINITY;
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) {
            float v[32];
            load_chunk(c, v);
            if (full) {
              if (sc >= 0.f) {
#pragma unroll
                for (int q = 0; q < 32; q += 2) mx = ptx::max3(mx, v[q], v[q + 1]);
              } else {
#pragma unroll
                for (int q = 0; q < 32; q += 2) mx = ptx::min3(mx, v[q], v[q + 1]);
              }
            } else {
#pragma unroll
              for (int q = 0; q < 32; ++q)
                if (c * 32 + q < valid) mx = (sc >= 0.f) ? fmaxf(mx, v[q]) : fminf(mx, v[q]);
            }
          }
          const float m_tile = mx * sc;
          if (jj == 0) {
            m_run = m_tile;
          } else if (__any_sync(0xffffffffu, m_tile > m_run + kT3Tau)) {
            // O_x already holds G2_x(g-1): s_full_x(g) retired after it (issue order)
            const float m_new = fmaxf(m_run, m_tile);
            const float alpha = ptx::ex2(m_run - m_new);
            l_run *= alpha;
            m_run = m_new;
            for (int c0 = 0; c0 < TLP; c0 += 16) {
              uint32_t r[16];
              ptx::tmem_ld16(tOx + c0, r);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int q = 0; q < 16; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) * alpha);
              ptx::tmem_st16(tOx + c0, r);
            }
          }
          const float neg_m = -m_run;
          float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) {
            float v[32];
            load_chunk(c, v);
            uint32_t pk[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const int e = c * 32 + 2 * q;
              float p0 = ptx::ex2(fmaf(v[2 * q], sc, neg_m));
              float p1 = ptx::ex2(fmaf(v[2 * q + 1], sc, neg_m));
              if (!full) {
                p0 = (e < valid) ? p0 : 0.f;
                p1 = (e + 1 < valid) ? p1 : 0.f;
              }
              ls0 += p0;
              ls1 += p1;
              pk[q] = ptx::pack2<BF16>(p0, p1);
            }
            ptx::tmem_st16(tSx + c * 16, pk);
          }
          l_run += ls0 + ls1;
        } else {
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) {
            float v[32];
            load_chunk(c, v);
            uint32_t pk[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              pk[q] = p.op == 1 ? ptx::pack2<BF16>(v[2 * q] * sc, v[2 * q + 1] * sc) : ptx::pack2<BF16>(v[2 * q], v[2 * q + 1]);
            ptx::tmem_st16(tSx + c * 16, pk);
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_full[x]);
        if (trj) tr[8 + 16 * g + 1 + 2 * x] = ptx::globaltimer();
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
            ptx::tmem_ld16(tOx + c0, r);
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
      const int prow = x * 128 + row;                                    // row inside the pair
      float* ws_o = p.ws;                                                // [C][256][TLP]
      float* ws_ml = p.ws + static_cast<int64_t>(p.n_ctas) * 256 * TLP;  // [C][2][256]
      if (pc.t0 != 0) {
        float* wo = ws_o + (static_cast<int64_t>(cta) * 256 + prow) * TLP;
#pragma unroll
        for (int c0 = 0; c0 < TLMAX; c0 += 4)
          if (c0 < TLP) __stcg(reinterpret_cast<float4*>(wo + c0), make_float4(o[c0], o[c0 + 1], o[c0 + 2], o[c0 + 3]));
        __stcg(ws_ml + cta * 512 + prow, m_run);
        __stcg(ws_ml + cta * 512 + 256 + prow, l_run);
        ptx::named_bar_sync(1, 256);
        if (threadIdx.x == 0) {
          __threadfence();
          ptx::st_release_gpu(p.flags + cta, 1);
        }
      } else {
        const int32_t c_end = cta_of_tile(pc.unit * p.tpu + p.tpu - 1, p);
        for (int32_t q = cta + 1; q <= c_end; ++q) {
          if (threadIdx.x == 0) {
            ptx::spin_acquire_gpu(p.flags + q, 1);
            __threadfence();
            p.flags[q] = 0;   // reset for the next launch (only this thread waits on it)
          }
          ptx::named_bar_sync(1, 256);
          const float* qo = ws_o + (static_cast<int64_t>(q) * 256 + prow) * TLP;
          const float m2 = __ldcg(ws_ml + q * 512 + prow);
          const float l2 = __ldcg(ws_ml + q * 512 + 256 + prow);
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
        const int gm = pc.m0 + prow;
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
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) {
    tr[5] = ptx::globaltimer();
    tr[7] = clock64();
  }
  if (warp == 8) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace mbci
