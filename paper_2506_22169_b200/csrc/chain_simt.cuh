// chain_simt.cuh — the chain on CUDA cores, for what the tensor-core kernel does not take:
// fp32 inputs (TF32 cannot meet the 1e-5 bound; R12) and 16-bit problems whose
// strides or base addresses break TMA's 16-byte rules.  Exact fp32 FMAs, accurate expf.
//
// One CTA per output row (β, m): the C row lives in shared memory only (C never reaches
// HBM), then E[β,m,:] = op(C)·D.  Same semantics as the tensor-core path (mbci.h).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

namespace mbci {

struct SimtParams {
  int32_t M, N, K, L;
  int32_t op;
  int32_t causal;   // softmax: key n visible to row m only if n <= m (R18)
  float scale;
  int32_t b_layout;
  const int32_t* valid_len;
  int64_t ld_a, ld_b, ld_d, ld_e;
  int64_t bs_a, bs_b, bs_d, bs_e;
  int32_t key_off;   // split-N partial runs (as Tc4Params)
  float* lse;
};

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half from_f<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

constexpr int kSimtThreads = 128;

// RELU / GELU (exact erf) of x = scale * C (R19)
__device__ __forceinline__ float act_op(int op, float x) {
  if (op == 3) return fmaxf(x, 0.0f);
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}

__device__ __forceinline__ float block_reduce(float v, bool is_max, float* scratch) {
  for (int o = 16; o > 0; o >>= 1) {
    float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, w) : v + w;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  float r = scratch[0];
  for (int w = 1; w < kSimtThreads / 32; ++w) r = is_max ? fmaxf(r, scratch[w]) : r + scratch[w];
  return r;
}

template <typename T>
__global__ void __launch_bounds__(kSimtThreads)
    k_chain_simt(const T* __restrict__ A, const T* __restrict__ B, const T* __restrict__ D,
                 T* __restrict__ E, const SimtParams p) {
  extern __shared__ float c_row[];  // [N] + 8 scratch
  float* scratch = c_row + p.N;
  const int64_t beta = blockIdx.x / p.M;
  const int m = blockIdx.x % p.M;
  const T* a = A + beta * p.bs_a + static_cast<int64_t>(m) * p.ld_a;
  const T* b = B + beta * p.bs_b;
  const T* d = D + beta * p.bs_d;
  int vlen = p.N;
  if (p.op == 2 && p.valid_len != nullptr) vlen = min(max(p.valid_len[beta] - p.key_off, 0), p.N);
  if (p.op == 2 && p.causal) vlen = min(vlen, m + 1);   // key n visible to row m iff n <= m

  for (int n = threadIdx.x; n < p.N; n += blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < p.K; ++k) {
      const float bv = p.b_layout == 0 ? to_f(b[static_cast<int64_t>(k) * p.ld_b + n])
                                       : to_f(b[static_cast<int64_t>(n) * p.ld_b + k]);
      acc = fmaf(to_f(a[k]), bv, acc);
    }
    c_row[n] = (p.op == 0) ? acc : (p.op >= 3 ? act_op(p.op, p.scale * acc) : p.scale * acc);
  }
  __syncthreads();
  if (p.op == 2) {
    float mx = -INFINITY;
    for (int n = threadIdx.x; n < vlen; n += blockDim.x) mx = fmaxf(mx, c_row[n]);
    mx = block_reduce(mx, true, scratch);
    float sum = 0.f;
    for (int n = threadIdx.x; n < p.N; n += blockDim.x) {
      const float e = (n < vlen) ? expf(c_row[n] - mx) : 0.f;
      c_row[n] = e;
      sum += e;
    }
    sum = block_reduce(sum, false, scratch);
    const float inv = vlen > 0 ? 1.0f / sum : 0.f;
    if (p.lse != nullptr && threadIdx.x == 0) p.lse[beta * p.M + m] = vlen > 0 ? mx + logf(sum) : -INFINITY;
    for (int n = threadIdx.x; n < p.N; n += blockDim.x) c_row[n] *= inv;
    __syncthreads();
  }
  T* e = E + beta * p.bs_e + static_cast<int64_t>(m) * p.ld_e;
  for (int l = threadIdx.x; l < p.L; l += blockDim.x) {
    float acc = 0.f;
    for (int n = 0; n < p.N; ++n) acc = fmaf(c_row[n], to_f(d[static_cast<int64_t>(n) * p.ld_d + l]), acc);
    e[l] = from_f<T>(acc);
  }
}

}  // namespace mbci
