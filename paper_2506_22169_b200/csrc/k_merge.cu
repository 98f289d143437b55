// k_merge.cu — the reduce step of split-N: R partial results of the chain, each
// over a disjoint range of the keys n, merged into E.
//
// A SOFTMAX partial r holds E_r = softmax over its keys · D (normalised by its own row sum) and
// the row log-sum-exp lse_r = ln Σ_{n in r} exp(s·C[m,n]).  Over the union of the ranges
// (PAPER.md:498 softmax over n, :196 E = C'·D):
//     E = Σ_r w_r E_r / Σ_r w_r,   w_r = exp(lse_r − max_r' lse_r')
// which is exact in real arithmetic (each E_r·exp(lse_r) is the unnormalised partial product);
// a partial whose keys are all masked has lse_r = −inf and weight 0, a row with no valid key at
// all gives E = 0.  Every other op is linear in the partial products: E = Σ_r E_r.
//
// HBM-bound: each thread owns 16 bytes of one output row (8 16-bit or 4 fp32 columns), reads the
// R lse values of its row (L1/L2 hits after the first column group) and the R 16-byte chunks of
// the partials, and writes 16 bytes; fp32 arithmetic, one rounding to the output type.  Grid-
// stride over (row, chunk); a scalar variant covers L not a multiple of the chunk or unaligned
// pointers.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>

#include "kernels.h"

namespace mbci {

namespace {

// register value -> fp32 (the 16-byte chunk is loaded once with __ldg, then unpacked here)
__device__ __forceinline__ float mg_f(float v) { return v; }
__device__ __forceinline__ float mg_f(__half v) { return __half2float(v); }
__device__ __forceinline__ float mg_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ float mg_load(const T* p) { return mg_f(__ldg(p)); }   // global memory only
template <typename T>
__device__ __forceinline__ T mg_from(float v);
template <>
__device__ __forceinline__ float mg_from<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half mg_from<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 mg_from<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// weights of row `row` (softmax): w[r] / Σ w, or all 1 (linear ops)
__device__ __forceinline__ float mg_weight(const float* lse, int64_t rows, int R, int64_t row, int r, bool softmax,
                                           float mstar, float inv) {
  if (!softmax) return 1.f;
  const float l = __ldg(lse + static_cast<int64_t>(r) * rows + row);
  return l == -INFINITY ? 0.f : __expf(l - mstar) * inv;
}

__device__ __forceinline__ void mg_row_stats(const float* lse, int64_t rows, int R, int64_t row, float& mstar,
                                             float& inv) {
  mstar = -INFINITY;
  for (int r = 0; r < R; ++r) mstar = fmaxf(mstar, __ldg(lse + static_cast<int64_t>(r) * rows + row));
  float sum = 0.f;
  if (mstar != -INFINITY)
    for (int r = 0; r < R; ++r) {
      const float l = __ldg(lse + static_cast<int64_t>(r) * rows + row);
      sum += l == -INFINITY ? 0.f : __expf(l - mstar);
    }
  inv = sum > 0.f ? 1.0f / sum : 0.f;
}

// vector variant: VE elements (16 bytes) per thread-chunk, R <= kMergeRMax parts.  Every load of a
// chunk (the R lse values of its row and the R 16-byte partial chunks) is issued before any is
// used, so a thread keeps R + R/4 independent requests in flight instead of a dependent chain.
constexpr int kMergeRMax = 8;
template <typename T>
__global__ void __launch_bounds__(256) k_merge_vec(const T* __restrict__ parts, const float* __restrict__ lse,
                                                   T* __restrict__ E, int R, int64_t rows, int64_t L, int softmax) {
  constexpr int VE = 16 / sizeof(T);
  const int64_t chunks = L / VE, total = rows * chunks, part_stride = rows * L;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / chunks, c0 = (i - row * chunks) * VE;
    uint4 v[kMergeRMax];
    float l[kMergeRMax];
#pragma unroll
    for (int r = 0; r < kMergeRMax; ++r) {
      if (r < R) {
        v[r] = __ldg(reinterpret_cast<const uint4*>(parts + r * part_stride + row * L + c0));
        l[r] = softmax ? __ldg(lse + static_cast<int64_t>(r) * rows + row) : 0.f;
      }
    }
    float w[kMergeRMax];
    float mstar = -INFINITY, sum = 0.f;
#pragma unroll
    for (int r = 0; r < kMergeRMax; ++r)
      if (r < R) mstar = fmaxf(mstar, l[r]);
#pragma unroll
    for (int r = 0; r < kMergeRMax; ++r) {
      if (r < R) {
        w[r] = !softmax ? 1.f : (l[r] == -INFINITY ? 0.f : __expf(l[r] - mstar));
        sum += w[r];
      }
    }
    const float inv = !softmax ? 1.f : (sum > 0.f ? 1.0f / sum : 0.f);
    float acc[VE];
#pragma unroll
    for (int q = 0; q < VE; ++q) acc[q] = 0.f;
#pragma unroll
    for (int r = 0; r < kMergeRMax; ++r) {
      if (r < R) {
        const T* t = reinterpret_cast<const T*>(&v[r]);
#pragma unroll
        for (int q = 0; q < VE; ++q) acc[q] = fmaf(w[r], mg_f(t[q]), acc[q]);
      }
    }
    uint4 o;
    T* ot = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int q = 0; q < VE; ++q) ot[q] = mg_from<T>(acc[q] * inv);
    *reinterpret_cast<uint4*>(E + row * L + c0) = o;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_merge_scalar(const T* __restrict__ parts, const float* __restrict__ lse,
                                                      T* __restrict__ E, int R, int64_t rows, int64_t L, int softmax) {
  const int64_t total = rows * L, part_stride = rows * L;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / L;
    float mstar = 0.f, inv = 1.f;
    if (softmax) mg_row_stats(lse, rows, R, row, mstar, inv);
    float acc = 0.f;
    for (int r = 0; r < R; ++r)
      acc = fmaf(mg_weight(lse, rows, R, row, r, softmax != 0, mstar, inv), mg_load<T>(parts + r * part_stride + i), acc);
    E[i] = mg_from<T>(acc);
  }
}

template <typename T>
cudaError_t merge_t(const void* parts, const float* lse, void* E, int R, int64_t rows, int64_t L, bool softmax,
                    bool vec, int n_sm, cudaStream_t st) {
  constexpr int VE = 16 / sizeof(T);
  vec = vec && R <= kMergeRMax;
  const int64_t work = vec ? rows * (L / VE) : rows * L;
  const int64_t blocks = (work + 255) / 256;   // one chunk per thread up to 64 blocks per SM
  const unsigned grid = static_cast<unsigned>(blocks < 64LL * n_sm ? (blocks > 0 ? blocks : 1) : 64LL * n_sm);
  if (vec)
    k_merge_vec<T><<<grid, 256, 0, st>>>(static_cast<const T*>(parts), lse, static_cast<T*>(E), R, rows, L,
                                         softmax ? 1 : 0);
  else
    k_merge_scalar<T><<<grid, 256, 0, st>>>(static_cast<const T*>(parts), lse, static_cast<T*>(E), R, rows, L,
                                            softmax ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_merge(int dtype, const void* parts, const float* lse, void* E, int R, int64_t rows, int64_t L,
                         bool softmax, bool vec, int n_sm, cudaStream_t st) {
  if (dtype == 0) return merge_t<float>(parts, lse, E, R, rows, L, softmax, vec, n_sm, st);
  if (dtype == 1) return merge_t<__half>(parts, lse, E, R, rows, L, softmax, vec, n_sm, st);
  return merge_t<__nv_bfloat16>(parts, lse, E, R, rows, L, softmax, vec, n_sm, st);
}

}  // namespace mbci
