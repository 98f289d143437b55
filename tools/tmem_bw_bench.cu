// tmem_bw_bench.cu — TMEM read / write bandwidth per SM on sm_100a (tcgen05.ld / tcgen05.st),
// for 4, 8 and 16 warps (warp w accesses TMEM lanes 32·(w%4) .. +31).  One CTA per SM.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/tmem_bw_bench tools/tmem_bw_bench.cu
#include <cstdio>
#include <cstdint>

#define ITERS 2048

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MODE 0: read 128 columns per warp per iteration (4 x ld32, one wait)
// MODE 1: write 64 columns per warp per iteration (4 x st16, one wait)
// MODE 2: read 128 + write 64 (the softmax's per-tile traffic)
template <int MODE>
__global__ void __launch_bounds__(512, 1) k_tm(uint32_t* out, int nw) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tslot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  uint32_t acc = 0;
  if (warp < nw) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col = (uint32_t)((warp >> 2) & 3) * 128;   // 4 groups of 4 warps: 128 columns each
    const uint32_t t = tmem + lane_off + col;
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 7 + i;
    for (int it = 0; it < ITERS; ++it) {
      if (MODE == 0 || MODE == 2) {
        uint32_t a[32], b[32], c[32], d[32];
        ld32(t, a);
        ld32(t + 32, b);
        ld32(t + 64, c);
        ld32(t + 96, d);
        wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) acc ^= a[i] ^ b[i] ^ c[i] ^ d[i];
      }
      if (MODE == 1 || MODE == 2) {
        r[0] = acc + it;
        st16(t, r);
        st16(t + 16, r + 16);
        st16(t + 32, r);
        st16(t + 48, r + 16);
        wait_st();
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int MODE>
void run(const char* name, uint32_t* out, int nw) {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_tm<MODE><<<sms, 512>>>(out, nw);
  cudaEventRecord(a);
  k_tm<MODE><<<sms, 512>>>(out, nw);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double per_warp = (MODE == 0 ? 128 * 128.0 : MODE == 1 ? 64 * 128.0 : 192 * 128.0);   // bytes per iteration
  const double bytes = (double)nw * per_warp * ITERS;   // per SM
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s warps=%2d  %.3f ms  %7.1f B/clk/SM  (%.0f cycles per warp-iteration)\n", name, nw, ms, bytes / cyc,
         cyc / ITERS);
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 148 * 512 * sizeof(uint32_t));
  for (int nw : {1, 4, 8, 16}) {
    run<0>("read 128 cols / warp", out, nw);
    run<1>("write 64 cols / warp", out, nw);
    run<2>("read 128 + write 64", out, nw);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
