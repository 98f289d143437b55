// chain_tc4.cuh — persistent ping-pong fused chain E = op(A·B)·D on sm_100a.
//
// Same arithmetic as chain_tc.cuh (mbci.h; PAPER.md:196 chain, :498 softmax between the GEMMs,
// :489 batched layout); a different layout of the work, built for the MUFU (ex2) + tensor-core
// balance of d <= 128 attention on B200 (op = SOFTMAX) and reused for the plain chains (NONE /
// SCALE: the warpgroups only convert S to 16-bit P):
//
// * Persistent grid (one CTA per SM).  A unit is (β, a PAIR of 128-row m-tiles) — the paper's
//   spatial loop m bound to CTAs (Rule 1) with the whole L in the CTA (the h loop
//   is dead for L <= 128) — and units are dealt round-robin to CTAs.  K = A's width <= 128 makes
//   the k loop dead, so both Q tiles of a unit are loaded once and E is stored
//   once per unit after the n loop (S_E hoisted).
// * Each K_j / V_j tile (B_j, D_j) is loaded once and feeds both Q tiles ("slots").  The two
//   softmax warpgroups work on the two slots; the single tcgen05 issuer interleaves the slots,
//   so while one slot's warpgroup computes exponentials the tensor core serves the other.
//   The look-ahead G1s cross unit boundaries: the next unit's first S tiles are computed while
//   the current unit's last P is still being produced (Q is double-buffered when SMEM allows).
// * A separate epilogue warpgroup drains O (E = O / l, cvt, store), so the softmax warpgroups
//   start the next unit at once; O_x is released to the next unit's first G2 by `o_free`.
// * TMEM (512 columns): NSB fp32 S buffers of 128 columns rotated over the slot-tile sequence,
//   then O_0, O_1 (see NSB below).  P (16-bit, two per column) overwrites the first 64 columns
//   of the S buffer it came from.  tcgen05 ops of one thread complete in issue order, so a G1
//   rewrites a buffer only after the G2 that read its P.
// * Exponentials: z = s·log2(e)·S − m with packed f32x2 FMA; p = 2^z on the MUFU (ex2.approx)
//   or, for EMU of every 8 column pairs (default 2, MBCI_T4_EMU), on the FMA pipe (Cody–Waite
//   split + degree-3 minimax polynomial, max rel. error 8.8e-5 < the 16-bit P rounding), so
//   both pipes share the work.
//   Lazy rescale: the running max only moves when a tile's max exceeds it by > τ = 8 (log2),
//   exact in real arithmetic (R4).
//
// * Wave quantisation: a last, partial round of <= n_SM / 2 units runs as "half" items (one
//   128-row Q tile, the two slots split its key tiles, the epilogue merges them by log-sum-exp),
//   so that round costs half the tiles (Tc4Params).
//
// Warps: 0-3 softmax slot 0 | 4-7 softmax slot 1 | 8-11 epilogue | 12 tcgen05 issuer + TMEM
//        allocator | 13 TMA producer | 14-15 idle.  setmaxnreg moves registers to the softmax
//        warpgroups (184 each: a whole 128-column S row in registers) from the others (80 / 64).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "ptx.cuh"

#ifndef MBCI_TRACE
#define MBCI_TRACE 0
#endif

namespace mbci {

struct Tc4Params {
  int32_t M, N, K, L;
  int32_t batch, l_mp;     // 256-row pair units per β
  int32_t units;           // batch * l_mp
  int32_t TL;              // L padded to 16 (<= 128): O columns per slot
  int32_t k_steps;         // ceil(K / 16) >= 1
  int32_t stages;          // K/V ring depth
  int32_t q_bufs;          // Q-pair buffers (1 or 2)
  int32_t op;              // 2 softmax; 1 scale, 0 none (P = cvt(scale * S), E = O)
  int32_t causal;          // softmax: key n visible to row m only if n <= m (R18)
  float scale;             // softmax: scale * log2(e); SCALE: the multiplier; NONE: 1
  const int32_t* valid_len;
  void* E;
  int64_t ld_e, bs_e;
  uint32_t q_bytes;        // one 128-row Q tile
  uint32_t b_stage_bytes, d_stage_bytes, kp_rows;
  uint32_t idesc1, idesc2;
  // Work items (one per CTA round): items [0, half_from) are whole pair units (item = unit).
  // When the last, partial round would leave SMs idle, its r units become 2r "half" items
  // [half_from, items): one 128-row Q tile each, whose two slots split the key tiles (slot x
  // takes tiles [x·h, x·h + h), h = nt_max / 2) and whose epilogue merges the two partial
  // (O, m, l) rows inside the CTA (log-sum-exp).  Only without key padding and with nt_max even.
  int32_t items, half_from, nt_max;
  uint64_t* trace;         // [gridDim.x][kT4TraceSlots] (MBCI_TRACE builds only)
  int32_t flags;           // kernel 5: bit 0 = exp-phase turns between the two slots' warps of an
                           // SMSP, bit 2 = issuer / TMA threads spin on test_wait (A/B only)
  int32_t burst;           // kernels 5 / 6: 1 = the prologue issues only the first step's K/V entries
  int32_t pf_bytes;        // kernels 5 / 6: L2 prefetch budget per CTA before the grid-dependency wait
  int32_t dbg;             // diagnostics only (MBCI_T4_DEBUG): 1 = softmax skips its TMEM/math work,
                           // 2 = issuer skips the G2 MMAs, 4 = issuer skips the G1 MMAs
  // Split-N partial runs (mbci_chain_run_partial): this launch sees keys
  // [key_off, key_off + N) of the full sequence (valid_len counts full-sequence keys), and, for
  // SOFTMAX, writes the row log-sum-exp of its key range to lse[β·M + m] (nullptr: not written).
  int32_t key_off;
  float* lse;
};

constexpr int kT4Threads = 512;
constexpr int kT4BN = 128;
constexpr float kT4Tau = 8.0f;
constexpr int kT4TraceSlots = 512;
// trace layout per CTA (MBCI_TRACE builds): [0] start (globaltimer ns) [1] setup [2] smid [3] end,
// [4] clock64 at start; per flat tile g < 40 and slot x, SM clock64 at 8 + 12*g + {0+x: S ready,
// 2+x: tile max done, 4+x: P stored, 6+x: P seen by the issuer, 8+x: G2 issued, 10+x: G1(g+1)
// issued, 12: issuer starts waiting for K_g, 13: K_g landed, 14+x: issuer starts waiting for P};
// [460 + g] TMA issues the K/V load of tile g; per unit u < 4 at 490 + 4*u + {0: o_full seen, 1: slot 0 stored, 2: slot 1 stored}.
#define T4TR(g, k) (8 + 16 * (g) + (k))
constexpr int kT4TrTiles = 28;
__device__ __forceinline__ uint64_t t4_clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
__device__ __forceinline__ uint64_t t4_clk_after(uint32_t dep) {
  uint64_t c;
  asm volatile("{\n\t.reg .u32 d;\n\tmov.u32 d, %1;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(c) : "r"(dep));
  return c;
}

__device__ __forceinline__ int t4_nlim(const Tc4Params& p, int beta) {
  int n = p.N;
  if (p.valid_len != nullptr) n = min(max(__ldg(p.valid_len + beta) - p.key_off, 0), p.N);
  return n;
}

// Split-N partial run: the natural-log row log-sum-exp of this launch's keys, ln 2 · (m + log2 l)
// with m the running max in log2 units and l the row sum of 2^(z - m); -inf when no key is valid.
__device__ __forceinline__ void t4_store_lse(const Tc4Params& p, int beta, int gm, float m, float l) {
  if (p.lse != nullptr && p.op == 2 && gm < p.M)
    p.lse[static_cast<int64_t>(beta) * p.M + gm] = l > 0.f ? (m + log2f(l)) * 0.69314718055994531f : -INFINITY;
}

// Key limit of pair unit u for its tile count: key padding and, with the causal mask (DESIGN.md
// R18), the pair's last row m0 + 255 sees keys < m0 + 256 (slot 0's rows see one tile less; that
// tile is fully masked for them).
__device__ __forceinline__ int t4_unit_nlim(const Tc4Params& p, int u) {
  const int beta = u / p.l_mp;
  int n = t4_nlim(p, beta);
  if (p.causal) n = min(n, (u - beta * p.l_mp) * 256 + 256);
  return n;
}

// Work item i -> pair unit u and, for a half item, which 128-row Q tile of it (see Tc4Params).
struct T4Item {
  int u, half;   // pair unit; -1: the whole unit, 0 / 1: which 128-row tile of it (half item)
  __device__ __forceinline__ void decode(const Tc4Params& p, int i) {
    if (i < p.half_from) {
      u = i;
      half = -1;
    } else {
      const int q = i - p.half_from;
      u = p.half_from + (q >> 1);
      half = q & 1;
    }
  }
  // steps (K/V tiles per slot) of this item given the unit's key limit; a half item's two
  // slots take half of the (unmasked, even) tile count each
  __device__ __forceinline__ int tiles(int n_lim) const {
    const int ntv = (n_lim + kT4BN - 1) / kT4BN;
    return half < 0 ? ntv : ntv / 2;
  }
};

__device__ __forceinline__ void t4_next_entry(int& st, uint32_t& ph, int S) {
  if (++st == S) { st = 0; ph ^= 1; }
}

// 2^x for a pair, on the FMA/ALU pipes.  x <= 2^22; results below 2^-127 flush towards 0.
//   x = n + f, n = floor(x) (round-down add of 1.5·2^23), f in [0, 1);
//   2^f ~= ((c3 f + c2) f + c1) f + c0 (minimax, relative error 8.8e-5); 2^n by exponent add.
__device__ __forceinline__ float2 t4_exp2_poly(float2 x) {
  constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23
  x.x = fmaxf(x.x, -127.0f);
  x.y = fmaxf(x.y, -127.0f);
  const float2 t = __fadd2_rd(x, make_float2(kMagic, kMagic));
  const float2 fl = __fadd2_rn(t, make_float2(-kMagic, -kMagic));
  const float2 f = __ffma2_rn(fl, make_float2(-1.0f, -1.0f), x);
  float2 q = __ffma2_rn(f, make_float2(0.0771190897f, 0.0771190897f),
                        make_float2(0.2275643945f, 0.2275643945f));
  q = __ffma2_rn(q, f, make_float2(0.6951461434f, 0.6951461434f));
  q = __ffma2_rn(q, f, make_float2(1.0f, 1.0f));
  float2 r;
  r.x = __uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23));
  r.y = __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23));
  return r;
}

// Row extreme of a 128-column S row held in registers (max, or min when the scale is negative):
// eight independent FMNMX3 chains.  MASKED: only the first `valid` (< 128) columns count (keys
// n >= n_lim are −inf before the softmax).
template <bool MIN>
__device__ __forceinline__ float t4_red(float a, float b, float c) {
  return MIN ? ptx::min3(a, b, c) : ptx::max3(a, b, c);
}
template <bool MIN, bool MASKED>
__device__ __forceinline__ float t4_row_extreme(const uint32_t (&sr)[kT4BN], int valid) {
  if constexpr (MASKED) {
    float mx = MIN ? INFINITY : -INFINITY;
#pragma unroll
    for (int c = 0; c < kT4BN; ++c) {
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
    for (int c = 16; c < kT4BN; c += 16)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = t4_red<MIN>(a[q], __uint_as_float(sr[c + 2 * q]), __uint_as_float(sr[c + 2 * q + 1]));
    return t4_red<MIN>(t4_red<MIN>(a[0], a[1], a[2]), t4_red<MIN>(a[3], a[4], a[5]), MIN ? fminf(a[6], a[7]) : fmaxf(a[6], a[7]));
  }
}

// p = 2^(sc·S − m) for the 128 scores of the row (registers), accumulated into two packed
// partial sums, written back as 16-bit P into TMEM columns [0, 64) of the S buffer, 16 columns
// per tcgen05.st.  MASKED: columns >= valid give p = 0.
template <bool BF16, int EMU, bool MASKED>
__device__ __forceinline__ void t4_exp_row(uint32_t tS, const uint32_t (&sr)[kT4BN], float sc, float m, int valid,
                                           float2& l2a, float2& l2b) {
  const float2 sc2 = make_float2(sc, sc);
  const float2 nm2 = make_float2(-m, -m);
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    uint32_t pk[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int cp = ch * 16 + c;   // pair index in the tile
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
    ptx::tmem_st16(tS + ch * 16, pk);
  }
}

// NONE / SCALE: P = cvt(scale * S) for the 128 scores of the row, written as 16-bit P into TMEM
// columns [0, 64) of the S buffer (no max, no exponentials, no row sum).
// RELU / GELU (op 3 / 4): P = cvt(act(scale * S)).
template <bool BF16, bool ACT, bool SCALED = true>
__device__ __forceinline__ void t4_cvt_row_impl(uint32_t tS, const uint32_t (&sr)[kT4BN], float sc, int op) {
  const float2 sc2 = make_float2(sc, sc);
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    uint32_t pk[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int cp = ch * 16 + c;
      float2 z;
      if constexpr (SCALED)
        z = __fmul2_rn(make_float2(__uint_as_float(sr[2 * cp]), __uint_as_float(sr[2 * cp + 1])), sc2);
      else   // NONE (scale 1): P = cvt(S), no multiply
        z = make_float2(__uint_as_float(sr[2 * cp]), __uint_as_float(sr[2 * cp + 1]));
      if constexpr (ACT) {
        z.x = ptx::act(op, z.x);
        z.y = ptx::act(op, z.y);
      }
      pk[c] = ptx::pack2<BF16>(z.x, z.y);
    }
    ptx::tmem_st16(tS + ch * 16, pk);
  }
}
// NOMUL_NONE: NONE converts S without its scale-1 multiply (kernel 5's linear instantiation; the
// kernels that also carry the softmax path keep the code they were tuned with, see chain_tc5.cuh)
template <bool BF16, bool NOMUL_NONE = false>
__device__ __forceinline__ void t4_cvt_row(uint32_t tS, const uint32_t (&sr)[kT4BN], float sc, int op) {
  if (op >= 3) t4_cvt_row_impl<BF16, true>(tS, sr, sc, op);   // one uniform branch per tile
  else if (NOMUL_NONE && op == 0) t4_cvt_row_impl<BF16, false, false>(tS, sr, sc, op);
  else t4_cvt_row_impl<BF16, false>(tS, sr, sc, op);
}

// Cursor over a CTA's flat sequence of key tiles (units dealt round-robin, units with no valid
// key skipped): unit u, its tile count nt, tile j inside it, the unit's Q buffer (qb, parity
// qph) and active-unit index ai, and the K/V ring stage (st, parity sph) of the tile.  Per tile
// the issuer only increments counters; divisions happen once per unit.
struct T4Cursor {
  int i, u, nt, j, ai, qb, qph, st, g;
  uint32_t sph;
  bool valid, hf;   // hf: half item (two K/V ring entries per step, one per slot)
  __device__ __forceinline__ void skip(const Tc4Params& p, int G) {
    while (i < p.items) {
      T4Item it;
      it.decode(p, i);
      nt = it.tiles(t4_unit_nlim(p, it.u));
      if (nt > 0) {
        u = it.u;
        hf = it.half >= 0;
        return;
      }
      i += G;
    }
    valid = false;
  }
  __device__ __forceinline__ void init(const Tc4Params& p, int G) {
    i = blockIdx.x; j = 0; ai = 0; qb = 0; qph = 0; st = 0; sph = 0; g = 0; valid = true; nt = 0; hf = false;
    skip(p, G);
  }
  // ring entry (stage, parity) of slot x in the current step
  __device__ __forceinline__ void entry(int x, int S, int& s, uint32_t& ph) const {
    s = st;
    ph = sph;
    if (hf && x == 1) t4_next_entry(s, ph, S);
  }
  __device__ __forceinline__ void advance(const Tc4Params& p, int G) {
    ++g;
    t4_next_entry(st, sph, p.stages);
    if (hf) t4_next_entry(st, sph, p.stages);
    if (++j >= nt) {
      j = 0;
      ++ai;
      if (++qb == p.q_bufs) { qb = 0; qph ^= 1; }
      i += G;
      skip(p, G);
    }
  }
};

// NSB: S buffers in TMEM, rotated over the flat slot-tile sequence k = 2g + x (buffer k % NSB).
//   NSB = 2 (TL > 64): S_x is reused by slot x only, G1(k+2) follows G2(k).
//   NSB = 3 (TL <= 64): three 128-column S buffers + two 64-column O; G1(k+3) follows G2(k), so
//   a slot's next S tile is computed while its softmax still runs (the softmax warpgroups never
//   wait for G2 + G1 latency), and the lazy rescale waits for G2_x(j-1) via S(k+1)'s phase.
// Commits (each ~170 cycles of issuer time, tools/sync_cost_bench.cu): per slot-tile one
// (s_full), per step one K/V release (two for a half item), plus o_full per item and slot and
// q_empty per item.
// Half items (see Tc4Params): one Q tile, slot x reads key tiles [x·nt, x·nt + nt); each step
// uses two ring entries (slot 0's, then slot 1's) and the epilogue merges the two slots' rows.
template <bool BF16, int KCH, int BL, int DCH, int EMU, int NSB>
__global__ void __launch_bounds__(kT4Threads, 1)
    k_chain_tc4(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, const Tc4Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ uint32_t tmem_base_slot;
  __shared__ float l_sm[2][2][128];   // [slot][active-item parity][row]: row sum of p
  __shared__ float m_sm[2][2][128];   // running max (log2 units) the p were taken against

  constexpr uint32_t kOCol = NSB * 128;                 // O_0 column; O_1 at kOCol + kOStride
  constexpr uint32_t kOStride = NSB == 3 ? 64 : 128;
  const int S = p.stages;
  const uint32_t kv_stage = p.b_stage_bytes + p.d_stage_bytes;
  uint8_t* sQ = smem;                                      // [q_bufs][2][q_bytes]
  uint8_t* sKV = sQ + p.q_bufs * 2 * p.q_bytes;            // [S][K | V]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + S * kv_stage);
  uint64_t* q_full = bars;          // [2]
  uint64_t* q_empty = bars + 2;     // [2]
  uint64_t* o_full = bars + 4;      // [2] last G2_x of a unit completed
  uint64_t* o_free = bars + 6;      // [2] epilogue read O_x (128 arrivals)
  uint64_t* l_full = bars + 8;      // [2] softmax x published l (128 arrivals)
  uint64_t* l_free = bars + 10;     // [2] epilogue read l_sm[x][ai & 1] (128 arrivals)
  __shared__ uint64_t dbg_bar;      // MBCI_T4_DEBUG & 8: per-group MMA latency probe
  uint64_t* s_full = bars + 12;     // [NSB] G1 landed in S buffer b
  uint64_t* p_full = s_full + 3;    // [NSB] softmax wrote P into buffer b (128 arrivals)
  uint64_t* kv_full = p_full + 3;   // [S] K_g and V_g landed (one barrier: G1 of tile g, which
                                    // precedes both G2 of the tile, is the only waiter)
  uint64_t* kv_empty = kv_full + S; // [S] the last G2 reading the entry completed (commit)

  const int warp = threadIdx.x >> 5;
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
  // The TMA warp initialises the barriers and issues the first item's Q and first K/V ring
  // entries before the CTA-wide barrier, so their HBM latency overlaps TMEM allocation and the
  // set-up of the other roles (all other threads touch the barriers only after __syncthreads).
  int pre_entries = 0;   // TMA warp: entries of the first active item already issued
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
#pragma unroll
    for (int c = 0; c < DCH; ++c)
      ptx::tma_load_3d(vdst + c * (kT4BN * 128), &tmD, &kv_full[s], c * 64, tile * kT4BN, beta);
  };
  // Q of an item into Q buffer qb (two tiles, or one for a half item / a pair past M)
  auto load_q = [&](int qb, int m0, int beta, bool two) {
    ptx::mbar_arrive_expect_tx(&q_full[qb], (two ? 2u : 1u) * p.q_bytes);
    for (int x = 0; x < (two ? 2 : 1); ++x) {
      uint8_t* dst = sQ + (qb * 2 + x) * p.q_bytes;
#pragma unroll
      for (int c = 0; c < KCH; ++c)
        ptx::tma_load_3d(dst + c * 16384, &tmA, &q_full[qb], c * 64, m0 + x * 128, beta);
    }
  };
  if (warp == 13 && ptx::elect_one()) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1);
      ptx::mbar_init(&o_full[i], 1);
      ptx::mbar_init(&o_free[i], 128);
      ptx::mbar_init(&l_full[i], 128);
      ptx::mbar_init(&l_free[i], 128);
    }
    for (int b = 0; b < NSB; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&p_full[b], 128);
    }
    ptx::mbar_init(&dbg_bar, 1);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    ptx::tma_prefetch(&tmD);
    if (!(p.dbg & 32)) {
      for (int i = blockIdx.x; i < p.items; i += gridDim.x) {
        T4Item it;
        it.decode(p, i);
        const int beta = it.u / p.l_mp;
        const int m0 = (it.u - beta * p.l_mp) * 256 + (it.half > 0 ? 128 : 0);
        const int nt = it.tiles(t4_unit_nlim(p, it.u));
        if (nt == 0) continue;
        load_q(0, m0, beta, it.half < 0 && m0 + 128 < p.M);
        const int per = it.half >= 0 ? 2 : 1;
        pre_entries = min(S, nt * per);
        for (int e = 0; e < pre_entries; ++e) load_entry(e, e / per + (e % per) * nt, beta);
        break;
      }
    }
  }
  if (warp == 12) ptx::tmem_alloc(&tmem_base_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_slot;
  if (tr && threadIdx.x == 0) tr[1] = ptx::globaltimer();
  const int G = gridDim.x;

  if (warp >= 12) {
    ptx::setmaxnreg_dec<64>();
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
          if (ai >= p.q_bufs) ptx::mbar_wait(&q_empty[qb], ((ai / p.q_bufs) - 1) & 1);
          // a fully out-of-range second tile is not loaded; a half item has one Q tile; the
          // first item's Q (and its first entries) went out before the CTA barrier
          if (ai > 0 || pre_entries == 0) load_q(qb, m0, beta, it.half < 0 && m0 + 128 < p.M);
          ++ai;
          for (int j = 0; j < nt; ++j) {
            for (int x = 0; x < (it.half >= 0 ? 2 : 1); ++x, ++g) {
              if (g < pre_entries) continue;
              const int tile = j + x * nt;   // half item: slot 1 takes tiles [nt, 2 nt)
              const int s = g % S;
              if (g >= S) ptx::mbar_wait(&kv_empty[s], ((g / S) - 1) & 1);
              if (tr && g < kT4TrTiles) tr[460 + g] = t4_clk();   // K/V load of entry g issued
              load_entry(s, tile, beta);
            }
          }
        }
      }
    } else if (warp == 12) {
      // ============================================================ tcgen05 issuer
      if (ptx::elect_one()) {
        const uint64_t dA = ptx::sdesc_sw128(0, 16, 1024);
        const uint64_t dB = (BL == 1) ? ptx::sdesc_sw128(0, 16, 1024) : ptx::sdesc_sw128(0, p.kp_rows * 128, 1024);
        const uint64_t dD = ptx::sdesc_sw128(0, kT4BN * 128, 1024);
        const uint32_t sQ0 = ptx::smem_u32(sQ), sKV0 = ptx::smem_u32(sKV);
        const uint32_t idesc1 = p.idesc1, idesc2 = p.idesc2;
        const int k_steps = p.k_steps;
        T4Cursor c1, c2;   // c1: tile of the next G1, c2: tile of the next G2
        c1.init(p, G);
        c2 = c1;
        int b1 = 0, b2 = 0;            // S buffer of the next G1 / G2
        uint32_t pph = 0;              // p_full parity of b2
        int x1 = 0;                    // slot of the next G1
        bool tail_committed = false;
        uint32_t dbg_ph = 0;
        // G1: S_b1 = Q_x1 · K_(c1 tile)
        auto issue_g1 = [&](bool kv_ready) {
          if (!c1.valid) {
            // past the CTA's last tile: one bare commit on the next buffer's s_full, so a lazy
            // rescale of the last slot-tile (which waits for "G1(k + 1)") still completes
            if (!tail_committed) ptx::mma_commit(&s_full[b1]);
            tail_committed = true;
            return;
          }
          if (x1 == 0) {
            if (tr && c1.g < kT4TrTiles) tr[T4TR(c1.g, 12)] = t4_clk();
            if (c1.j == 0) ptx::mbar_spin(&q_full[c1.qb], c1.qph);
            if (!kv_ready) ptx::mbar_spin(&kv_full[c1.st], c1.sph);
            if (c1.hf) {   // half item: slot 1's K/V is the next ring entry
              int s1;
              uint32_t ph1;
              c1.entry(1, S, s1, ph1);
              ptx::mbar_spin(&kv_full[s1], ph1);
            }
            if (tr && c1.g < kT4TrTiles) tr[T4TR(c1.g, 13)] = t4_clk();
            ptx::tc_fence_after();
          }
            const uint64_t tg1 = t4_clk();
          int kst;
          uint32_t kph;
          c1.entry(x1, S, kst, kph);
          const uint32_t q_lo = (sQ0 + (c1.qb * 2 + (c1.hf ? 0 : x1)) * p.q_bytes) >> 4;   // half: one Q tile
          const uint32_t k_lo = (sKV0 + kst * kv_stage) >> 4;
          const uint32_t dS = tmem + b1 * 128;
#pragma unroll
          for (int ks = 0; ks < 4 * KCH; ++ks) {
            if (ks < k_steps) {
              const uint64_t ad = dA + q_lo + (ks >> 2) * 1024 + (ks & 3) * 2;
              const uint64_t bd = (BL == 1) ? dB + k_lo + (ks >> 2) * (kT4BN * 8) + (ks & 3) * 2
                                            : dB + k_lo + ks * 128;
              if (!(p.dbg & 4)) ptx::mma_ss(dS, ad, bd, idesc1, ks > 0 ? 1u : 0u);
            }
          }
          ptx::mma_commit(&s_full[b1]);
          if (p.dbg & 8) {   // latency probe: issue -> completion of this G1
            ptx::mma_commit(&dbg_bar);
            ptx::mbar_spin(&dbg_bar, dbg_ph);
            dbg_ph ^= 1;
            if (tr && c1.g < kT4TrTiles) tr[T4TR(c1.g, 12 + x1)] = t4_clk() - tg1;
          }
          if (tr && c1.g < kT4TrTiles) tr[T4TR(c1.g, 10 + x1)] = t4_clk();
          if (++b1 == NSB) b1 = 0;
          if (x1 == 1) {
            if (c1.j == c1.nt - 1) ptx::mma_commit(&q_empty[c1.qb]);
            c1.advance(p, G);
          }
          x1 ^= 1;
        };
#pragma unroll 1
        for (int i = 0; i < NSB; ++i) issue_g1(false);
        int x2 = 0;
        bool p_ready = false;
        // Each mbarrier probe costs the issuer ~100-200 cycles of latency; the probes for the
        // next step are issued early (their predicates consumed later) so the latency overlaps
        // the MMAs already queued (~8 deep, tools/mma_issue_bench.cu).
        while (c2.valid) {
          if (tr && c2.g < kT4TrTiles) tr[T4TR(c2.g, 14 + x2)] = t4_clk();
          if (!p_ready) ptx::mbar_spin(&p_full[b2], pph);
          if (tr && c2.g < kT4TrTiles) tr[T4TR(c2.g, 6 + x2)] = t4_clk();
          if (c2.j == 0 && c2.ai > 0) ptx::mbar_spin(&o_free[x2], (c2.ai - 1) & 1);
          ptx::tc_fence_after();
          const bool kv_ready = c1.valid && x1 == 0 && c1.j != 0 ? ptx::mbar_test(&kv_full[c1.st], c1.sph) : false;
          // G2: O_x2 (+)= P_b2 · V_(c2 tile)
          int vst;
          uint32_t vph;
          c2.entry(x2, S, vst, vph);
          const uint32_t v_lo = (sKV0 + vst * kv_stage + p.b_stage_bytes) >> 4;
          const uint32_t tO = tmem + kOCol + x2 * kOStride;
          const uint32_t tP = tmem + b2 * 128;
          const uint32_t acc0 = c2.j > 0 ? 1u : 0u;
          const uint64_t tg2 = t4_clk();
#pragma unroll
          for (int ks = 0; ks < kT4BN / 16; ++ks)
            if (!(p.dbg & 2)) ptx::mma_ts(tO, tP + ks * 8, dD + v_lo + ks * 128, idesc2, ks > 0 ? 1u : acc0);
          if (p.dbg & 8) {   // latency probe: issue -> completion of this G2
            ptx::mma_commit(&dbg_bar);
            ptx::mbar_spin(&dbg_bar, dbg_ph);
            dbg_ph ^= 1;
            if (tr && c2.g < kT4TrTiles) tr[T4TR(c2.g, 14 + x2)] = t4_clk() - tg2;
          }
          if (tr && c2.g < kT4TrTiles) tr[T4TR(c2.g, 8 + x2)] = t4_clk();
          // K/V ring entries are released by a commit after their last reader: G2_1 of a
          // step, or each G2 of a half item's step (two entries).  (Releasing from the softmax
          // side two steps later saves this commit but deadlocks when a half item follows.)
          if (c2.hf || x2 == 1) ptx::mma_commit(&kv_empty[vst]);
          if (c2.j == c2.nt - 1) ptx::mma_commit(&o_full[x2]);
          if (++b2 == NSB) { b2 = 0; pph ^= 1; }
          if (x2 == 1) c2.advance(p, G);
          x2 ^= 1;
          issue_g1(kv_ready);   // the next G1 reuses the buffer this G2 just read
          p_ready = c2.valid ? ptx::mbar_test(&p_full[b2], pph) : false;
        }
      }
    }
  } else if (warp >= 8) {
    // ============================================================ epilogue (warps 8-11)
    ptx::setmaxnreg_dec<80>();
    const int row = threadIdx.x - 256;   // TMEM lane (warp 8+w reads lanes 32w..32w+31)
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    using T16 = uint16_t;
    int ai = 0;
    // flags bit 10 (MBCI_T4_FLAGS): the epilogue sleeps between polls of its long O waits
    auto wait_epi = [&](uint64_t* bar, uint32_t parity) {
      if (p.flags & 1024) ptx::mbar_wait_backoff(bar, parity); else ptx::mbar_wait(bar, parity);
    };
    auto store_row = [&](T16* erow, int gm, int c0, const float* v, float inv) {
      uint32_t w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = ptx::pack2<BF16>(v[2 * q] * inv, v[2 * q + 1] * inv);
      if (gm < p.M) {
        if (c0 + 16 <= p.L) {
          uint4* dst = reinterpret_cast<uint4*>(erow + c0);
          dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
          dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (c0 + q < p.L) erow[c0 + q] = static_cast<T16>((w[q >> 1] >> ((q & 1) * 16)) & 0xFFFFu);
        }
      }
    };
    for (int i = blockIdx.x; i < p.items; i += G) {
      T4Item it;
      it.decode(p, i);
      const int beta = it.u / p.l_mp;
      const int m0 = (it.u - beta * p.l_mp) * 256;
      const int nt = it.tiles(t4_unit_nlim(p, it.u));
      if (it.half >= 0) {
        // half item: both slots hold partial (O, m, l) of the same 128 rows (keys split between
        // them); merge by log-sum-exp, exact in real arithmetic (online-softmax identity)
        const int gm = m0 + it.half * 128 + row;
        T16* erow = reinterpret_cast<T16*>(p.E) + static_cast<int64_t>(beta) * p.bs_e +
                    static_cast<int64_t>(gm) * p.ld_e;
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
        if (p.op == 2) {
          const float mstar = fmaxf(l[0] > 0.f ? m[0] : -INFINITY, l[1] > 0.f ? m[1] : -INFINITY);
          w0 = l[0] > 0.f ? ptx::ex2(m[0] - mstar) : 0.f;
          w1 = l[1] > 0.f ? ptx::ex2(m[1] - mstar) : 0.f;
          const float L = l[0] * w0 + l[1] * w1;
          inv = L > 0.f ? 1.0f / L : 0.f;
          t4_store_lse(p, beta, gm, mstar, L);
        }
        const uint32_t tO0 = tmem + lane_off + kOCol, tO1 = tO0 + kOStride;
#pragma unroll 1
        for (int c0 = 0; c0 < p.TL; c0 += 16) {
          uint32_t r0[16], r1[16];
          ptx::tmem_ld16(tO0 + c0, r0);
          ptx::tmem_ld16(tO1 + c0, r1);
          ptx::tmem_wait_ld();
          float v[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = w0 * __uint_as_float(r0[q]) + w1 * __uint_as_float(r1[q]);
          store_row(erow, gm, c0, v, inv);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&o_free[0]);
        ptx::mbar_arrive(&o_free[1]);
        ++ai;
        continue;
      }
#pragma unroll 1
      for (int x = 0; x < 2; ++x) {
        const int gm = m0 + x * 128 + row;
        T16* erow = reinterpret_cast<T16*>(p.E) + static_cast<int64_t>(beta) * p.bs_e +
                    static_cast<int64_t>(gm) * p.ld_e;
        const uint32_t tO = tmem + lane_off + kOCol + x * kOStride;
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
        // whole unit: E = O / l
        const float inv = l > 0.f ? 1.0f / l : 0.f;
        t4_store_lse(p, beta, gm, mr, l);
#pragma unroll 1
        for (int c0 = 0; c0 < p.TL; c0 += 16) {
          float v[16];
          if (nt > 0) {
            uint32_t r[16];
            ptx::tmem_ld16(tO + c0, r);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = 0.f;
          }
          store_row(erow, gm, c0, v, inv);
        }
        if (nt > 0) {
          ptx::tc_fence_before();
          ptx::mbar_arrive(&o_free[x]);
        }
        if (tr && row == 0 && ai < 4) tr[490 + 4 * ai + 1 + x] = t4_clk();
      }
      if (nt > 0) ++ai;
    }
  } else {
    // ============================================================ softmax (warps 0-7)
    ptx::setmaxnreg_inc<184>();   // a whole 128-column S row lives in registers
    const int x = warp >> 2;               // slot
    const int row = threadIdx.x & 127;     // TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tO = tmem + lane_off + kOCol + x * kOStride;
    const float sc = p.scale;
    int g = 0, ai = 0;
    for (int i = blockIdx.x; i < p.items; i += G) {
      T4Item it;
      it.decode(p, i);
      const int beta = it.u / p.l_mp;
      const int nt = it.tiles(t4_unit_nlim(p, it.u));
      if (nt == 0) continue;
      // keys from this slot's first tile on (a half item's slot 1 starts at tile nt)
      const int n_lim = t4_nlim(p, beta) - (it.half >= 0 ? x * nt * kT4BN : 0);
      const int m_row = (it.u - beta * p.l_mp) * 256 + x * 128 + row;   // causal: no half items
      float m_run = 0.f;
      float2 l2 = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
      for (int j = 0; j < nt; ++j, ++g) {
        const int k = 2 * g + x, b = k % NSB;
        const uint32_t tS = tmem + lane_off + b * 128;
        ptx::mbar_wait(&s_full[b], (k / NSB) & 1);
        ptx::tc_fence_after();
        if (tr && row == 0 && g < kT4TrTiles) tr[T4TR(g, x)] = t4_clk();
        if (p.dbg & 1) {
          ptx::tc_fence_before();
          ptx::mbar_arrive(&p_full[b]);
          continue;
        }
        const int valid = (p.causal ? min(n_lim, m_row + 1) : n_lim) - j * kT4BN;   // this thread's row
        const bool full = __all_sync(0xffffffffu, valid >= kT4BN);                   // warp-uniform
        uint32_t sr[kT4BN];
#pragma unroll
        for (int c = 0; c < kT4BN / 32; ++c) ptx::tmem_ld32(tS + c * 32, &sr[c * 32]);
        ptx::tmem_wait_ld();
        if (p.op != 2) {
          // NONE / SCALE: padded keys have S = 0 and zero V rows (TMA fill), no masking needed
          t4_cvt_row<BF16>(tS, sr, sc, p.op);
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          ptx::mbar_arrive(&p_full[b]);
          continue;
        }
        float mx;
        if (full)
          mx = sc >= 0.f ? t4_row_extreme<false, false>(sr, valid) : t4_row_extreme<true, false>(sr, valid);
        else
          mx = sc >= 0.f ? t4_row_extreme<false, true>(sr, valid) : t4_row_extreme<true, true>(sr, valid);
        const float m_tile = mx * sc;
        if (tr && row == 0 && g < kT4TrTiles) tr[T4TR(g, 2 + x)] = t4_clk_after(__float_as_uint(mx));
        if (j == 0) {
          m_run = m_tile;
        } else if (__any_sync(0xffffffffu, m_tile > m_run + kT4Tau)) {
          // warp-uniform (tcgen05.ld/st are warp-collective).  O_x must hold G2_x(j-1): implied
          // by s_full for NSB = 2 (G1(k) follows G2(k-2)); for NSB = 3, G1(k + 1) is issued
          // right after G2(k + 1 - 3) = G2_x(j - 1), so its S buffer's phase certifies O_x (the
          // issuer adds a bare commit past the last tile).
          if constexpr (NSB == 3) ptx::mbar_wait(&s_full[(k + 1) % NSB], ((k + 1) / NSB) & 1);
          ptx::tc_fence_after();
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
            for (int q = 0; q < 16; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) * alpha);
            ptx::tmem_st16(tO + c0, r);
          }
        }
        if (full)
          t4_exp_row<BF16, EMU, false>(tS, sr, sc, m_run, valid, l2, l2b);
        else
          t4_exp_row<BF16, 0, true>(tS, sr, sc, m_run, valid, l2, l2b);
        ptx::tmem_wait_st();
        if (tr && row == 0 && g < kT4TrTiles) tr[T4TR(g, 4 + x)] = t4_clk();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_full[b]);
      }
      // The look-ahead G1s let a softmax run more than a unit ahead of the epilogue (units of
      // one tile), and l_full's parity protocol allows only one phase in flight: publishing l
      // of unit ai waits until the epilogue has read unit ai - 1's.
      if (ai >= 1) ptx::mbar_wait(&l_free[x], (ai - 1) & 1);
      l_sm[x][ai & 1][row] = p.op == 2 ? (l2.x + l2.y) + (l2b.x + l2b.y) : 1.0f;   // E = O / l
      m_sm[x][ai & 1][row] = m_run;
      ptx::mbar_arrive(&l_full[x]);
      ++ai;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[3] = ptx::globaltimer();
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace mbci
