// Pure TMA throughput: one thread issues `nload` loads back-to-back into distinct SMEM buffers,
// all completing on one mbarrier; time = first issue .. barrier complete.  L2-resident source.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../paper_2506_22169_b200/csrc/ptx.cuh"
using namespace mbci;
__global__ void __launch_bounds__(32, 1) k_burst(const __grid_constant__ CUtensorMap map, int rows, int nload,
                                                 int reps, uint64_t* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  const uint32_t bytes = 64 * 2 * rows;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); ptx::tma_prefetch(&map); }
  __syncwarp();
  uint64_t best = ~0ull;
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) {
      const uint64_t t0 = ptx::globaltimer();
      ptx::mbar_arrive_expect_tx(&bar, bytes * nload);
      for (int i = 0; i < nload; ++i)
        ptx::tma_load_3d(sm + i * bytes, &map, &bar, 0, ((blockIdx.x * 13 + i * rows) % 4096), (blockIdx.x + r) % 96);
      ptx::mbar_wait(&bar, r & 1);
      const uint64_t t1 = ptx::globaltimer();
      if (t1 - t0 < best) best = t1 - t0;
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = best;
}
int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int nbatch = 96, N = 4096, K = 64;
  void* buf; cudaMalloc(&buf, (size_t)nbatch * N * K * 2); cudaMemset(buf, 0, (size_t)nbatch * N * K * 2);
  uint64_t* d; cudaMalloc(&d, 148 * 8);
  for (int rows : {64, 128, 256}) {
    CUtensorMap map;
    cuuint64_t dims[3] = {K, N, nbatch};
    cuuint64_t str[2] = {K * 2, (cuuint64_t)N * K * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)rows, 1}, es[3] = {1, 1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int bytes = 64 * 2 * rows;
    for (int nload : {1, 2, 4, 8, 16}) {
      if (nload * bytes > 200 * 1024) continue;
      for (int grid : {1, 148}) {
        const int smem = nload * bytes + 1024;
        cudaFuncSetAttribute(k_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_burst<<<grid, 32, smem>>>(map, rows, nload, 20, d);
        cudaError_t e = cudaDeviceSynchronize();
        uint64_t h[148]; cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
        double mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("box %6d B x %2d loads, grid %3d: %7.0f ns total, %6.0f ns/load, %.1f GB/s per SM (%s)\n", bytes, nload,
               grid, mx, mx / nload, (double)bytes * nload / mx, cudaGetErrorString(e));
      }
    }
  }
}
