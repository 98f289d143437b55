// Single-thread cost of the synchronisation instructions the kernel-4 issuer executes per
// slot-tile: tcgen05.commit (no MMA pending), mbarrier test_wait on a completed phase,
// tcgen05.fence::after_thread_sync, mbarrier.arrive, and an LDC-dependent branch.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "../paper_2506_22169_b200/csrc/ptx.cuh"
using namespace mbci;
__global__ void __launch_bounds__(128, 1) k(int mode, int n, uint64_t* out) {
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1); ptx::mbar_init(&bar[1], 1); ptx::mbar_init(&bar[2], 1 << 20);
    ptx::fence_mbar_init();
    ptx::mbar_arrive(&bar[1]);   // phase 0 of bar[1] completed
  }
  if (warp == 1) ptx::tmem_alloc(&tslot, 32);
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  if (warp == 1 && ptx::elect_one()) {
    uint32_t acc = 0;
    const uint64_t c0 = clock64();
    for (int i = 0; i < n; ++i) {
      if (mode == 0) ptx::mma_commit(&bar[0]);
      else if (mode == 1) acc += ptx::mbar_test(&bar[1], 0) ? 1 : 0;
      else if (mode == 2) ptx::tc_fence_after();
      else if (mode == 3) ptx::mbar_arrive(&bar[2]);
      else if (mode == 4) { ptx::mma_commit(&bar[0]); acc += ptx::mbar_test(&bar[1], 0) ? 1 : 0; ptx::tc_fence_after(); }
    }
    const uint64_t c1 = clock64();
    out[0] = (c1 - c0) / n;
    out[1] = acc;
  }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 1) { ptx::tc_fence_after(); ptx::tmem_dealloc(tslot, 32); }
}
int main() {
  uint64_t* d; cudaMalloc(&d, 16);
  const char* names[] = {"tcgen05.commit (nothing pending)", "mbarrier.test_wait (done phase)", "tcgen05.fence::after_thread_sync",
                         "mbarrier.arrive", "commit + test_wait + fence"};
  for (int m = 0; m < 5; ++m) {
    k<<<1, 128>>>(m, 1000, d);
    cudaError_t e = cudaDeviceSynchronize();
    uint64_t h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-36s %5llu cycles/iter (%s)\n", names[m], (unsigned long long)h[0], cudaGetErrorString(e));
  }
}
