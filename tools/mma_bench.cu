// tcgen05.mma throughput by shape/kind (sm_100a): one thread issues `n` MMAs back to back and
// commits; time from first issue to the commit's mbarrier completion.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "../paper_2506_22169_b200/csrc/ptx.cuh"
using namespace mbci;
__global__ void __launch_bounds__(128, 1) k(int kind, int N, int n, uint64_t* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = 0;
  if (warp == 1) ptx::tmem_alloc(&tslot, 512);
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1 && ptx::elect_one()) {
    const uint32_t idesc_ss = ptx::idesc_f16(0, 0, 0, 128, N);      // SS, B K-major
    const uint32_t idesc_ts = ptx::idesc_f16(0, 0, 1, 128, N);      // TS, B MN-major
    const uint64_t da = ptx::sdesc_sw128(ptx::smem_u32(sm), 16, 1024);
    const uint64_t db = ptx::sdesc_sw128(ptx::smem_u32(sm + 32768), 16, 1024);
    const uint64_t dbm = ptx::sdesc_sw128(ptx::smem_u32(sm + 32768), 128 * 128, 1024);
    uint64_t best = ~0ull;
    for (int r = 0; r < 8; ++r) {
      const uint64_t c0 = clock64();
      for (int i = 0; i < n; ++i) {
        if (kind == 0) ptx::mma_ss(tmem + 256, da + 2 * (i & 3), db + 2 * (i & 3), idesc_ss, 1);
        else ptx::mma_ts(tmem + 256, tmem + 8 * (i & 7), dbm + 128 * (i & 7), idesc_ts, 1);
      }
      ptx::mma_commit(&bar);
      ptx::mbar_wait(&bar, r & 1);
      const uint64_t c1 = clock64();
      if (c1 - c0 < best) best = c1 - c0;
    }
    out[0] = best;
  }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 1) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}
int main() {
  uint64_t* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int kind : {0, 1})
    for (int N : {64, 128, 256})
      for (int n : {4, 16, 64}) {
        k<<<1, 128, 70000>>>(kind, N, n, d);
        cudaError_t e = cudaDeviceSynchronize();
        uint64_t h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%s M=128 N=%3d K=16 x%2d: %6llu cycles total, %5.1f cyc/MMA, %6.0f MAC/clk (%s)\n",
               kind == 0 ? "SS" : "TS", N, n, (unsigned long long)h, (double)h / n, 128.0 * N * 16 * n / h,
               cudaGetErrorString(e));
      }
}
