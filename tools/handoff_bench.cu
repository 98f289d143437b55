// Latency of the pipeline hand-offs the fused kernel uses (sm_100a): mbarrier ping-pong between
// warps, tcgen05.commit -> mbarrier, and a small tcgen05.mma + commit.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "../paper_2506_22169_b200/csrc/ptx.cuh"
using namespace mbci;
#define ROUNDS 2000
__device__ __forceinline__ void wait_plain(uint64_t* bar, uint32_t par) {
  const uint32_t a = ptx::smem_u32(bar);
  while (!ptx::mbar_try_wait(a, par)) {}
}
__device__ __forceinline__ void wait_test(uint64_t* bar, uint32_t par) {
  while (!ptx::mbar_test(bar, par)) {}
}
__device__ int g_wait_mode;
__device__ __forceinline__ void WAIT(uint64_t* bar, uint32_t par, int mode) {
  const int m = mode % 3;
  if (m == 0) ptx::mbar_wait(bar, par);
  else if (m == 1) wait_plain(bar, par);
  else wait_test(bar, par);
}
__global__ void __launch_bounds__(384, 1) k_pingpong(int variant, int mode, uint64_t* out) {
  __shared__ volatile int done_flag;
  __shared__ __align__(1024) uint8_t smA[16384];
  __shared__ __align__(1024) uint8_t smB[16384];
  __shared__ uint64_t bar1, bar2;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar1, variant >= 3 ? 128 : 1);
    ptx::mbar_init(&bar2, 1);
    ptx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) { ((uint32_t*)smA)[i] = 0; ((uint32_t*)smB)[i] = 0; }
  if (threadIdx.x == 0) done_flag = 0;
  if (warp == 5) ptx::tmem_alloc(&tslot, 256);
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc = ptx::idesc_f16(0, 0, 0, 128, 64);
  uint64_t t0 = ptx::globaltimer();
  if (warp < 4) {
    const bool active = variant >= 3 || threadIdx.x == 0;
    if (active) {
      for (int r = 0; r < ROUNDS; ++r) {
        ptx::mbar_arrive(&bar1);
        WAIT(&bar2, r & 1, mode);
      }
    }
  } else if (warp >= 6) {
    // background MUFU/FMA load on every SMSP (like the other slot's softmax)
    if (mode >= 3) {
      float x = threadIdx.x * 1e-3f, y = 0.f;
      while (!done_flag) {
#pragma unroll
        for (int i = 0; i < 64; ++i) { y += ptx::ex2(x); x = fmaf(x, 0.999f, 1e-4f); }
      }
      if (y == 1234.5f) out[0] = 0;
    }
  } else if (warp == 5) {
    if (ptx::elect_one()) {
      for (int r = 0; r < ROUNDS; ++r) {
        WAIT(&bar1, r & 1, mode);
        if (variant == 0 || variant == 3) {
          ptx::mbar_arrive(&bar2);
        } else if (variant == 1 || variant == 4) {
          ptx::tc_fence_after();
          ptx::mma_commit(&bar2);
        } else {
          ptx::tc_fence_after();
          const uint64_t da = ptx::sdesc_sw128(ptx::smem_u32(smA), 16, 1024);
          const uint64_t db = ptx::sdesc_sw128(ptx::smem_u32(smB), 16, 1024);
          for (int k = 0; k < 4; ++k) ptx::mma_ss(tmem, da + 2 * k, db + 2 * k, idesc, k > 0);
          ptx::mma_commit(&bar2);
        }
      }
      done_flag = 1;
    }
  }
  if (warp < 4 && threadIdx.x == 0 && variant < 3) {}
  __syncthreads();
  uint64_t t1 = ptx::globaltimer();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 5) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 256); }
}
int main() {
  uint64_t* d; cudaMalloc(&d, 148 * 8);
  const char* names[] = {"mbar arrive(1 thr) <-> arrive", "arrive(1) <-> tcgen05.commit", "arrive(1) <-> 4x MMA 128x64x16 + commit",
                         "arrive(128 thr) <-> arrive", "arrive(128) <-> commit", "arrive(128) <-> 4x MMA + commit"};
  const char* modes[] = {"mbar_wait(timer)", "try_wait loop", "test_wait spin", "LOADED mbar_wait", "LOADED try_wait", "LOADED test_wait"};
  for (int mode = 0; mode < 6; ++mode)
  for (int v = 0; v < 6; ++v) {
    for (int grid : {148}) {
      k_pingpong<<<grid, 384>>>(v, mode, d);
      k_pingpong<<<grid, 384>>>(v, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      uint64_t h[148]; cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%-18s %-44s grid=%3d  round trip %.1f ns  (%s)\n", modes[mode], names[v], grid, mx / ROUNDS, cudaGetErrorString(e));
    }
  }
}
