// How far can one thread run ahead of the tensor pipe?  Issues 16 tcgen05.mma (SS, 128x128x16)
// back to back into an idle pipe and records clock64 after each issue, then the commit wait.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "../paper_2506_22169_b200/csrc/ptx.cuh"
using namespace mbci;
__global__ void __launch_bounds__(128, 1) k(int N, uint64_t* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (warp == 1) ptx::tmem_alloc(&tslot, 512);
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1 && ptx::elect_one()) {
    const uint32_t id = ptx::idesc_f16(0, 0, 0, 128, N);
    const uint64_t dA = ptx::sdesc_sw128(ptx::smem_u32(sm), 16, 1024), dB = ptx::sdesc_sw128(ptx::smem_u32(sm + 32768), 16, 1024);
    uint64_t t[17];
    for (int rep = 0; rep < 2; ++rep) {
      const uint64_t c0 = clock64();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        ptx::mma_ss(tmem, dA + 2 * (i & 3), dB + 2 * (i & 3), id, 1);
        t[i] = clock64();
      }
      ptx::mma_commit(&bar);
      ptx::mbar_spin(&bar, rep & 1);
      t[16] = clock64();
      for (int i = 0; i < 17; ++i) out[i] = t[i] - c0;
    }
  }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 1) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}
int main() {
  uint64_t* d; cudaMalloc(&d, 17 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int N : {64, 128, 256}) {
    k<<<1, 128, 70000>>>(N, d);
    cudaError_t e = cudaDeviceSynchronize();
    uint64_t h[17]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("N=%3d issue-return clocks:", N);
    for (int i = 0; i < 16; ++i) printf(" %llu", (unsigned long long)h[i]);
    printf(" | all done %llu (%s)\n", (unsigned long long)h[16], cudaGetErrorString(e));
  }
}
