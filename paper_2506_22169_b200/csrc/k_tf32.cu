// k_tf32.cu — kernel 7 (chain_tf32.cuh): fp32 chain on tcgen05 (kind::tf32, 3xTF32).
#define MBCI_TF32_KERNEL 1
#include "kernels.h"

namespace mbci {

const void* tf32_fn(bool wide) {
  return wide ? (const void*)k_chain_tf32<TfWide> : (const void*)k_chain_tf32<TfSmall>;
}

cudaError_t launch_tf32(bool wide, unsigned grid, cudaStream_t st, const float* A, const float* B, const float* D,
                        float* E, const Tf32Params& p) {
  if (wide)
    k_chain_tf32<TfWide><<<grid, kTf32Threads, kTf32WideSmem, st>>>(A, B, D, E, p);
  else
    k_chain_tf32<TfSmall><<<grid, kTf32Threads, kTf32Smem, st>>>(A, B, D, E, p);
  return cudaGetLastError();
}

}  // namespace mbci
