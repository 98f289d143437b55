// ex2_h2_bench.cu — MUFU exp2 throughput on sm_100a: ex2.approx.ftz.f32 vs ex2.approx.f16x2
// (two fp16 exponentials per instruction), raw and inside the softmax's per-pair sequence
// (z = s·S − m in fp32 FFMA2, cvt to f16x2, ex2, 16-bit accumulate, P already packed).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/ex2_h2_bench tools/ex2_h2_bench.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

#define ITERS 512
#define NP 64   // column pairs per thread (128 columns)

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2bh2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t cvt_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// MODE 0: raw f32 ex2 (independent); 1: raw f16x2 ex2; 2: f32 softmax pair sequence
// (FFMA2, 2 ex2, FADD2, cvt pack); 3: f16x2 pair sequence (FFMA2, cvt, ex2.f16x2, HADD2)
template <int MODE>
__global__ void __launch_bounds__(256, 1) k_ex(float* out, float sc, int nwarps_active) {
  const int warp = threadIdx.x >> 5;
  if (warp >= nwarps_active) return;
  float v[2 * NP];
#pragma unroll
  for (int i = 0; i < 2 * NP; ++i) v[i] = -0.01f * (i + threadIdx.x % 7);
  float2 acc = make_float2(0.f, 0.f), acc2 = make_float2(0.f, 0.f);
  uint32_t hacc[4] = {0u, 0u, 0u, 0u};
  uint32_t pk = 0;
  uint32_t h[NP];   // realistic fp16 exponents in [-10, 0]
#pragma unroll
  for (int c = 0; c < NP; ++c) h[c] = cvt_h2(-0.07f * c - 0.01f * (threadIdx.x & 7), -0.05f * c);
  const float2 nm2 = make_float2(-0.5f, -0.5f);
  for (int it = 0; it < ITERS; ++it) {
    const float2 sc2 = make_float2(sc + it * 1e-9f, sc + it * 1e-9f);   // loop-variant: no hoisting
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      if (MODE == 0) {
        acc.x += ex2f(v[2 * c]);
        acc.y += ex2f(v[2 * c + 1]);
      } else if (MODE == 1) {
        hacc[c & 3] ^= ex2h2(h[c]);
      } else if (MODE == 4) {   // conversion only: FFMA2 + F2FP
        const float2 z = __ffma2_rn(make_float2(v[2 * c], v[2 * c + 1]), sc2, nm2);
        hacc[c & 3] ^= cvt_h2(z.x, z.y);
      } else if (MODE == 5) {   // FFMA2 + F2FP + ex2.f16x2, no sum
        const float2 z = __ffma2_rn(make_float2(v[2 * c], v[2 * c + 1]), sc2, nm2);
        hacc[c & 3] ^= ex2h2(cvt_h2(z.x, z.y));
      } else if (MODE == 6) {   // raw ex2.approx.ftz.bf16x2
        hacc[c & 3] ^= ex2bh2(h[c] & 0xBFFFBFFFu);
      } else if (MODE == 2) {
        const float2 z = __ffma2_rn(make_float2(v[2 * c], v[2 * c + 1]), sc2, nm2);
        float2 e;
        e.x = ex2f(z.x);
        e.y = ex2f(z.y);
        if (c & 1) acc2 = __fadd2_rn(acc2, e); else acc = __fadd2_rn(acc, e);
        pk ^= cvt_h2(e.x, e.y);
      } else if (MODE == 3) {
        const float2 z = __ffma2_rn(make_float2(v[2 * c], v[2 * c + 1]), sc2, nm2);
        const uint32_t e = ex2h2(cvt_h2(z.x, z.y));
        hacc[c & 3] = hadd2(hacc[c & 3], e);
        pk ^= e;
      }
    }
    // keep the inputs live and loop-variant without adding work per element
    v[0] += 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc2.x + acc2.y +
      __uint_as_float(hacc[0] ^ hacc[1] ^ hacc[2] ^ hacc[3] ^ pk);
}

template <int MODE>
void run(const char* name, float* out, int warps) {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_ex<MODE><<<sms, 256>>>(out, 1.4427f, warps);
  cudaEventRecord(a);
  k_ex<MODE><<<sms, 256>>>(out, 1.4427f, warps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double exps = (double)sms * warps * 32 * ITERS * NP * 2;
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-34s warps/SMSP=%d  %.3f ms  %6.2f exps/clk/SM (at %d MHz)\n", name, warps / 4, ms,
         exps / sms / cyc, clk / 1000);
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 256 * sizeof(float));
  for (int w = 4; w <= 8; w += 4) {
    run<0>("raw ex2.approx.ftz.f32", out, w);
    run<1>("raw ex2.approx.f16x2 (2 per instr)", out, w);
    run<2>("softmax pair seq, f32 ex2", out, w);
    run<3>("softmax pair seq, f16x2 ex2", out, w);
    run<4>("FFMA2 + cvt f16x2 only", out, w);
    run<5>("FFMA2 + cvt + ex2.f16x2 (no sum)", out, w);
    run<6>("raw ex2.approx.ftz.bf16x2", out, w);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
