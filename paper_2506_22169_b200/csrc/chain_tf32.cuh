// chain_tf32.cuh — kernel 7: the fp32 chain E = op(A·B)·D on tcgen05 tensor cores (kind::tf32)
// with 3xTF32 error compensation (SURVEY.md §8(c) reading 12; BASELINE.json north_star (3):
// "the fp32 path within 1e-5 max relative error", both contractions on tensor cores).
//
// TF32 keeps 10 mantissa bits (unit roundoff 2^-11), far above 1e-5.  Every fp32 operand x is
// split x = hi + lo with hi = RNA_tf32(x) (exactly representable in TF32) and lo = x − hi (exact in
// fp32, |lo| <= 2^-11 |x|); a product is taken as hi·hi' + hi·lo' + lo·hi' (three tcgen05.mma per
// K step, fp32 accumulation in TMEM), dropping lo·lo' (<= 2^-22 |x x'|) and the TF32 rounding of
// the lo terms (<= 2^-22).  Both contractions do this: GEMM1 S = A·B with A, B split in shared
// memory (SS MMAs), GEMM2 O += P·D with P split into two TMEM buffers (TS MMAs: P from TMEM,
// PAPER.md:196's C never leaves the SM) and D split in shared memory.
//
// Work layout (PAPER.md:285 Rule 1): one CTA per (β, 128-row m tile); the k loop is dead
// (K <= 64 here) and E is stored once after the n loop (S_E hoisted,
// PAPER.md:232-233).  Per 64-key tile the CTA's four warps load and split B_j, D_j from global
// memory straight into the 128-B-swizzled K-major layout the MMA descriptors address (D and a
// [K, N] B are transposed on the way, so every operand is K-major: no MN-major TF32 layouts),
// one elected thread issues the MMAs, and thread t owns S / P / O row t (TMEM lane t) for the
// inter-GEMM op: none, scale, or online softmax (exact rescale of O when the row max grows,
// key-padding mask), with exp2 on the MUFU (relative error ~2^-22).  O is summed over key tiles
// in fp32 registers; each tile's GEMM2 lands in TMEM afresh.
// TMEM: S [0, 64) | P_hi [64, 128) | P_lo [128, 192) | O [192, 192 + TLP), TLP = L padded to 16.
// Arbitrary (even unaligned) strides: every global access is a scalar fp32 load or store.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace mbci {

struct Tf32Params {
  int32_t M, N, K, L;
  int32_t KP;    // K padded to a multiple of 8 (the TF32 MMA K step), <= 64 (<= 128 for the wide variant)
  int32_t TLP;   // L padded to a multiple of 16 (the MMA N granularity), <= 64 (<= 128)
  int32_t op;    // 0 none, 1 scale, 2 softmax, 3 relu, 4 gelu
  int32_t causal; // softmax: key n visible to row m only if n <= m (R18)
  float scale;   // softmax: scale * log2(e); SCALE: the multiplier
  int32_t b_layout;
  const int32_t* valid_len;
  int64_t ld_a, ld_b, ld_d, ld_e;
  int64_t bs_a, bs_b, bs_d, bs_e;
  uint32_t idesc1, idesc2;   // kind::tf32, K-major A and B; N = 64 (GEMM1), N = TLP (GEMM2)
  int32_t key_off;           // split-N partial runs (as Tc4Params)
  float* lse;
};

constexpr int kTf32Threads = 128;
// Two instantiations (TfCfg<BN, OC>): BN keys per tile, OC = max O columns (= max K and L):
//   <64, 64>  K, L <= 64:  A, B, D hi/lo = 2 x (32 + 16 + 16) KB;  TMEM S | P_hi | P_lo | O = 4 x 64
//   <32, 128> K, L <= 128: A, B, D hi/lo = 2 x (64 + 16 + 16) KB;  TMEM 3 x 32 + 128
template <int BN_, int OC_>
struct TfCfg {
  static constexpr int BN = BN_, OC = OC_;
  static constexpr uint32_t A_BYTES = (OC / 32) * 128 * 128;   // K chunks of 32 fp32 x 128 rows x 128 B
  static constexpr uint32_t B_BYTES = (OC / 32) * BN * 128;    // K chunks x BN rows
  static constexpr uint32_t D_BYTES = (BN / 32) * OC * 128;    // key chunks x OC rows (l)
  static constexpr uint32_t SMEM = 2 * (A_BYTES + B_BYTES + D_BYTES) + 1024;
  static constexpr uint32_t S_COL = 0, PHI_COL = BN, PLO_COL = 2 * BN, O_COL = 3 * BN;
};
using TfSmall = TfCfg<64, 64>;
using TfWide = TfCfg<32, 128>;
constexpr uint32_t kTf32Smem = TfSmall::SMEM;      // the K, L <= 64 variant
constexpr uint32_t kTf32WideSmem = TfWide::SMEM;   // the K, L <= 128 variant

__device__ __forceinline__ void mma_ss_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_ts_tf32(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// x = hi + lo, hi = round-to-nearest (ties away) to TF32, lo exact
__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = x - hi;
}

// Byte offset of element (row, k) in a K-major, 128-B-swizzled tile of `rows` rows whose K
// extent is cut into 32-element (128-B) chunks: chunk c at c * rows * 128, row r at r * 128,
// 16-B unit u = (k % 32) / 4 stored at u ^ (r % 8).
__device__ __forceinline__ uint32_t sw128_off(int rows, int r, int k) {
  const int c = k >> 5, u = (k & 31) >> 2;
  return static_cast<uint32_t>(c * rows * 128 + r * 128 + ((u ^ (r & 7)) << 4) + (k & 3) * 4);
}

// Loads a rows x KP fp32 tile (element (r, k) = src(r, k), zero outside [0, nr) x [0, nk)) and
// stores its TF32 split into two swizzled K-major tiles; 4 consecutive k per thread and step.
// `kstride` / `rstride`: element strides of k and r in global memory.
__device__ __forceinline__ void tf32_load_split(uint8_t* dhi, uint8_t* dlo, int rows, int KP, const float* src,
                                                int nr, int nk, int64_t rstride, int64_t kstride, bool r_fast) {
  const int kq = KP >> 2;
  const int total = rows * kq;
  for (int idx = threadIdx.x; idx < total; idx += kTf32Threads) {
    int r, q;
    if (r_fast) {   // consecutive threads walk r (the contiguous global dimension)
      r = idx % rows;
      q = idx / rows;
    } else {        // consecutive threads walk k
      r = idx / kq;
      q = idx % kq;
    }
    float hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = 4 * q + e;
      const float v = (r < nr && k < nk) ? src[r * rstride + k * kstride] : 0.f;
      tf32_split(v, hi[e], lo[e]);
    }
    const uint32_t off = sw128_off(rows, r, 4 * q);
    ptx::st_shared_v4(ptx::smem_u32(dhi + off), __float_as_uint(hi[0]), __float_as_uint(hi[1]),
                      __float_as_uint(hi[2]), __float_as_uint(hi[3]));
    ptx::st_shared_v4(ptx::smem_u32(dlo + off), __float_as_uint(lo[0]), __float_as_uint(lo[1]),
                      __float_as_uint(lo[2]), __float_as_uint(lo[3]));
  }
}

// The kernel itself is compiled in k_tf32.cu only (other translation units see the parameters).
#ifdef MBCI_TF32_KERNEL
template <class CFG>
__global__ void __launch_bounds__(kTf32Threads, 1)
    k_chain_tf32(const float* __restrict__ A, const float* __restrict__ B, const float* __restrict__ D,
                 float* __restrict__ E, const Tf32Params p) {
  constexpr int kTf32BN = CFG::BN, kOC = CFG::OC;
  constexpr uint32_t kTf32ABytes = CFG::A_BYTES, kTf32BBytes = CFG::B_BYTES, kTf32DBytes = CFG::D_BYTES;
  constexpr uint32_t kTf32SCol = CFG::S_COL, kTf32PHiCol = CFG::PHI_COL, kTf32PLoCol = CFG::PLO_COL,
                     kTf32OCol = CFG::O_COL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sAhi = smem;
  uint8_t* sAlo = sAhi + kTf32ABytes;
  uint8_t* sBhi = sAlo + kTf32ABytes;
  uint8_t* sBlo = sBhi + kTf32BBytes;
  uint8_t* sDhi = sBlo + kTf32BBytes;
  uint8_t* sDlo = sDhi + kTf32DBytes;
  __shared__ uint32_t tmem_base_slot;
  __shared__ uint64_t mma_bar;

  const int l_m = (p.M + 127) / 128;
  const int beta = blockIdx.x / l_m;
  const int m0 = (blockIdx.x - beta * l_m) * 128;
  const int warp = threadIdx.x >> 5;
  const int row = threadIdx.x;   // TMEM lane / output row m0 + row
  const bool leader = threadIdx.x == 0;
  if (warp == 0) ptx::tmem_alloc(&tmem_base_slot, 256);   // 4 x 64 or 3 x 32 + 128 columns
  if (leader) {
    ptx::mbar_init(&mma_bar, 1);
    ptx::fence_mbar_init();
  }
  int n_lim = p.N;
  if (p.valid_len != nullptr) n_lim = min(max(__ldg(p.valid_len + beta) - p.key_off, 0), p.N);
  // A tile: rows m0 .. m0 + 127, K-major
  tf32_load_split(sAhi, sAlo, 128, p.KP, A + beta * p.bs_a + static_cast<int64_t>(m0) * p.ld_a, p.M - m0, p.K,
                  p.ld_a, 1, false);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_slot;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const uint32_t tS = tmem + lane_off + kTf32SCol, tPhi = tmem + lane_off + kTf32PHiCol,
                 tPlo = tmem + lane_off + kTf32PLoCol, tO = tmem + lane_off + kTf32OCol;
  const uint64_t dAhi = ptx::sdesc_sw128(ptx::smem_u32(sAhi), 16, 1024),
                 dAlo = ptx::sdesc_sw128(ptx::smem_u32(sAlo), 16, 1024),
                 dBhi = ptx::sdesc_sw128(ptx::smem_u32(sBhi), 16, 1024),
                 dBlo = ptx::sdesc_sw128(ptx::smem_u32(sBlo), 16, 1024),
                 dDhi = ptx::sdesc_sw128(ptx::smem_u32(sDhi), 16, 1024),
                 dDlo = ptx::sdesc_sw128(ptx::smem_u32(sDlo), 16, 1024);
  // causal: the CTA's last row m0 + 127 sees keys < m0 + 128; row `row` sees keys <= m0 + row
  const int cta_lim = (p.op == 2 && p.causal) ? min(n_lim, m0 + 128) : n_lim;
  const int row_lim = (p.op == 2 && p.causal) ? min(n_lim, m0 + row + 1) : n_lim;
  const int ntiles = p.op == 2 ? (cta_lim + kTf32BN - 1) / kTf32BN : (p.N + kTf32BN - 1) / kTf32BN;
  float m_run = -INFINITY, l_run = 0.f;
  // O accumulates in fp32 registers across key tiles (IEEE adds): the tensor core sums only one
  // tile's 24 products per element into TMEM (acc = 0 at each tile's first MMA), which keeps its
  // non-IEEE accumulation error at the tile scale (measured: a 1000-key chain accumulated in TMEM
  // missed 1e-5 by 2 %)
  float o[kOC];
#pragma unroll
  for (int c = 0; c < kOC; ++c) o[c] = 0.f;
  uint32_t phase = 0;
  for (int j = 0; j < ntiles; ++j) {
    const int n0 = j * kTf32BN;
    // B_j as K-major [key][k]; D_j as K-major [l][key] (transposed)
    const float* bsrc = B + beta * p.bs_b;
    if (p.b_layout == 1)   // B stored [N, K]
      tf32_load_split(sBhi, sBlo, kTf32BN, p.KP, bsrc + static_cast<int64_t>(n0) * p.ld_b, p.N - n0, p.K, p.ld_b,
                      1, false);
    else                   // B stored [K, N]: element (key, k) at k * ld_b + key
      tf32_load_split(sBhi, sBlo, kTf32BN, p.KP, bsrc + n0, p.N - n0, p.K, 1, p.ld_b, true);
    tf32_load_split(sDhi, sDlo, kOC, kTf32BN, D + beta * p.bs_d + static_cast<int64_t>(n0) * p.ld_d, p.L,
                    p.N - n0, 1, p.ld_d, true);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    // GEMM1: S = A·B_j with 3xTF32
    if (leader) {
      for (int ks = 0; ks < p.KP / 8; ++ks) {
        const uint64_t ao = static_cast<uint64_t>((ks >> 2) * (128 * 128 / 16) + (ks & 3) * 2);
        const uint64_t bo = static_cast<uint64_t>((ks >> 2) * (kTf32BN * 128 / 16) + (ks & 3) * 2);
        mma_ss_tf32(tmem + kTf32SCol, dAhi + ao, dBhi + bo, p.idesc1, ks > 0 ? 1u : 0u);
        mma_ss_tf32(tmem + kTf32SCol, dAhi + ao, dBlo + bo, p.idesc1, 1u);
        mma_ss_tf32(tmem + kTf32SCol, dAlo + ao, dBhi + bo, p.idesc1, 1u);
      }
      ptx::mma_commit(&mma_bar);
    }
    ptx::mbar_wait(&mma_bar, phase);
    phase ^= 1u;
    ptx::tc_fence_after();
    // inter-GEMM op on row `row`, 64 keys
    uint32_t s[kTf32BN];
#pragma unroll
    for (int c = 0; c < kTf32BN; c += 32) ptx::tmem_ld32(tS + c, &s[c]);
    ptx::tmem_wait_ld();
    float pv[kTf32BN];
    if (p.op == 2) {
      const int valid = row_lim - n0;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kTf32BN; ++c)
        if (c < valid) mx = fmaxf(mx, __uint_as_float(s[c]) * p.scale);
      const float m_new = fmaxf(m_run, mx);
      if (j > 0 && m_new > m_run) {   // exact online rescale (O lives in registers)
        const float alpha = ptx::ex2(m_run - m_new);
        l_run *= alpha;
#pragma unroll
        for (int c = 0; c < kOC; ++c) o[c] *= alpha;
      }
      m_run = m_new;
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < kTf32BN; ++c) {
        const float e = c < valid ? ptx::ex2(__uint_as_float(s[c]) * p.scale - m_run) : 0.f;
        pv[c] = e;
        sum += e;
      }
      l_run += sum;
    } else {
#pragma unroll
      for (int c = 0; c < kTf32BN; ++c)
        pv[c] = p.op == 0 ? __uint_as_float(s[c]) : ptx::act(p.op, p.scale * __uint_as_float(s[c]));
    }
#pragma unroll
    for (int c0 = 0; c0 < kTf32BN; c0 += 16) {
      uint32_t h[16], l[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        float hi, lo;
        tf32_split(pv[c0 + c], hi, lo);
        h[c] = __float_as_uint(hi);
        l[c] = __float_as_uint(lo);
      }
      ptx::tmem_st16(tPhi + c0, h);
      ptx::tmem_st16(tPlo + c0, l);
    }
    ptx::tmem_wait_st();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    // GEMM2: O += P·D_j with 3xTF32 (P from TMEM)
    if (leader) {
      for (int ks = 0; ks < kTf32BN / 8; ++ks) {
        const uint64_t bo = static_cast<uint64_t>((ks >> 2) * (kOC * 128 / 16) + (ks & 3) * 2);
        const uint32_t acc = ks > 0 ? 1u : 0u;
        mma_ts_tf32(tmem + kTf32OCol, tmem + kTf32PHiCol + ks * 8, dDhi + bo, p.idesc2, acc);
        mma_ts_tf32(tmem + kTf32OCol, tmem + kTf32PHiCol + ks * 8, dDlo + bo, p.idesc2, 1u);
        mma_ts_tf32(tmem + kTf32OCol, tmem + kTf32PLoCol + ks * 8, dDhi + bo, p.idesc2, 1u);
      }
      ptx::mma_commit(&mma_bar);
    }
    ptx::mbar_wait(&mma_bar, phase);   // also frees B_j / D_j and P for the next tile
    phase ^= 1u;
    ptx::tc_fence_after();
#pragma unroll
    for (int c0 = 0; c0 < kOC; c0 += 16) {
      if (c0 < p.TLP) {
        uint32_t r[16];
        ptx::tmem_ld16(tO + c0, r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c) o[c0 + c] += __uint_as_float(r[c]);
      }
    }
  }
  // epilogue: E = O (none / scale) or O / l (softmax; a row with no valid key gives 0)
  if (m0 + row < p.M) {
    float* e = E + beta * p.bs_e + static_cast<int64_t>(m0 + row) * p.ld_e;
    const float inv = p.op == 2 ? (l_run > 0.f ? 1.0f / l_run : 0.f) : 1.0f;
#pragma unroll
    for (int c = 0; c < kOC; ++c)
      if (c < p.L) e[c] = o[c] * inv;
    if (p.lse != nullptr && p.op == 2)
      p.lse[static_cast<int64_t>(beta) * p.M + m0 + row] =
          l_run > 0.f ? (m_run + log2f(l_run)) * 0.69314718055994531f : -INFINITY;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}
#endif  // MBCI_TF32_KERNEL

}  // namespace mbci
