// How long does the issuing thread take to get past tcgen05.mma / tcgen05.commit?
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "../paper_2506_22169_b200/csrc/ptx.cuh"
using namespace mbci;
__global__ void __launch_bounds__(128, 1) k(int nmma, int ncommit, int nrep, uint64_t* out) {
  __shared__ __align__(1024) uint8_t smA[16384];
  __shared__ __align__(1024) uint8_t smB[16384];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) ptx::mbar_init(&bar[i], 1); ptx::fence_mbar_init(); }
  for (int i = threadIdx.x; i < 4096; i += 128) { ((uint32_t*)smA)[i] = 0; ((uint32_t*)smB)[i] = 0; }
  if (warp == 1) ptx::tmem_alloc(&tslot, 256);
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc = ptx::idesc_f16(0, 0, 0, 128, 64);
  if (warp == 1 && ptx::elect_one()) {
    const uint64_t da = ptx::sdesc_sw128(ptx::smem_u32(smA), 16, 1024);
    const uint64_t db = ptx::sdesc_sw128(ptx::smem_u32(smB), 16, 1024);
    uint64_t t_mma = 0, t_commit = 0, t_total = 0;
    for (int r = 0; r < nrep; ++r) {
      const uint64_t c0 = clock64();
      for (int k = 0; k < nmma; ++k) ptx::mma_ss(tmem, da + 2 * (k & 3), db + 2 * (k & 3), idesc, k > 0);
      const uint64_t c1 = clock64();
      for (int c = 0; c < ncommit; ++c) ptx::mma_commit(&bar[c]);
      const uint64_t c2 = clock64();
      for (int c = 0; c < ncommit; ++c) ptx::mbar_wait(&bar[c], r & 1);
      const uint64_t c3 = clock64();
      t_mma += c1 - c0; t_commit += c2 - c1; t_total += c3 - c0;
    }
    out[0] = t_mma / nrep; out[1] = t_commit / nrep; out[2] = t_total / nrep;
  }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 1) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 256); }
}
int main() {
  uint64_t* d; cudaMalloc(&d, 64);
  for (int nmma : {0, 1, 4, 8, 16})
    for (int nc : {1, 3}) {
      k<<<1, 128>>>(nmma, nc, 200, d);
      cudaError_t e = cudaDeviceSynchronize();
      uint64_t h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
      printf("mma x%2d (128x64x16) + %d commits: issue mma %4llu cyc, issue commits %4llu cyc, until all barriers done %5llu cyc (%s)\n",
             nmma, nc, (unsigned long long)h[0], (unsigned long long)h[1], (unsigned long long)h[2], cudaGetErrorString(e));
    }
}
