// k_simt.cu — instantiations of kernel 1 (chain_simt.cuh, CUDA cores).
#include "kernels.h"

namespace mbci {

const void* simt_fn(int dtype) {
  return dtype == 0 ? (const void*)k_chain_simt<float>
                    : dtype == 1 ? (const void*)k_chain_simt<__half> : (const void*)k_chain_simt<__nv_bfloat16>;
}

cudaError_t launch_simt(int dtype, unsigned grid, int smem, cudaStream_t st, const void* A, const void* B,
                        const void* D, void* E, const SimtParams& sp) {
  if (dtype == 0)
    k_chain_simt<float><<<grid, kSimtThreads, smem, st>>>((const float*)A, (const float*)B, (const float*)D,
                                                           (float*)E, sp);
  else if (dtype == 1)
    k_chain_simt<__half><<<grid, kSimtThreads, smem, st>>>((const __half*)A, (const __half*)B, (const __half*)D,
                                                            (__half*)E, sp);
  else
    k_chain_simt<__nv_bfloat16><<<grid, kSimtThreads, smem, st>>>(
        (const __nv_bfloat16*)A, (const __nv_bfloat16*)B, (const __nv_bfloat16*)D, (__nv_bfloat16*)E, sp);
  return cudaGetLastError();
}

}  // namespace mbci
