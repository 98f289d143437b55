// TMA load throughput / latency probe (sm_100a): one producer thread streams 3-D boxes
// {64, rows, 1} (128-B swizzle) from an L2-resident tensor into an S-deep SMEM ring; one
// consumer thread waits each full barrier and releases the slot.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../paper_2506_22169_b200/csrc/ptx.cuh"
using namespace mbci;
__global__ void __launch_bounds__(256, 1) k_tma(const __grid_constant__ CUtensorMap map, int S, int rows, int iters,
                                               int nbatch, int prefetch, uint64_t* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[16], empty[16];
  const uint32_t bytes = 64 * 2 * rows;
  if (threadIdx.x % 64 == 0 && prefetch) ptx::tma_prefetch(&map);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  uint64_t t0 = ptx::globaltimer();
  if (threadIdx.x % 64 == 0) {
    for (int g = 0; g < iters; ++g) {
      const int s = g % S;
      if (g >= S) ptx::mbar_wait(&empty[s], ((g / S) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&full[s], bytes);
      const int b = (blockIdx.x * 7 + g) % nbatch;
      ptx::tma_load_3d(sm + s * bytes, &map, &full[s], 0, (g * rows) % 4096, b);
    }
  } else if (threadIdx.x % 64 == 32) {
    for (int g = 0; g < iters; ++g) {
      const int s = g % S;
      ptx::mbar_wait(&full[s], (g / S) & 1);
      ptx::mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = ptx::globaltimer() - t0;
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
    for (int S : {1, 4}) {
      for (int np : {1, 2, 4}) {
        const int nb = 1;
        const int iters = 512, bytes = 64 * 2 * rows;
        int smem = np * S * bytes + 1024;
        if (smem > 220000) continue;
        cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_tma<<<148, 64 * np, smem>>>(map, S, rows, iters, 96, nb, d);
        k_tma<<<148, 64 * np, smem>>>(map, S, rows, iters, 96, nb, d);
        cudaError_t e = cudaDeviceSynchronize();
        uint64_t h[148]; cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("box 64x%-3d (%5d B) stages=%d producers=%d: %.0f ns/load per producer, %.1f GB/s per SM, %.2f TB/s total (%s)\n",
               rows, bytes, S, np, mx / iters, (double)np * bytes * iters / mx, 148.0 * np * bytes * iters / mx / 1000.0,
               cudaGetErrorString(e));
      }
    }
  }
}
