// kernels.h — host-side handles of the kernel instantiations.  Each kernel family is
// instantiated in its own translation unit (k_*.cu) so the library builds in parallel; api.cu
// only sees these selector functions and the parameter structs.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "chain_simt.cuh"
#include "chain_tc.cuh"
#include "chain_tc4.cuh"
#include "chain_tf32.cuh"

namespace mbci {

using TcKernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, TcParams);
using Tc4Kernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, Tc4Params);
using Tc5Kernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, Tc4Params);

// kernel 0 (k_tc0.cu)
TcKernel pick_tc(bool bf16, int bn, int kch, int bl, int dch);
// kernel 4 (k_tc4_f16.cu, k_tc4_bf16.cu)
Tc4Kernel pick_tc4_f16(int kch, int bl, int dch, int emu);
Tc4Kernel pick_tc4_bf16(int kch, int bl, int dch, int emu);
inline Tc4Kernel pick_tc4(bool bf16, int kch, int bl, int dch, int emu) {
  return bf16 ? pick_tc4_bf16(kch, bl, dch, emu) : pick_tc4_f16(kch, bl, dch, emu);
}
// kernel 5 (k_tc5_f16.cu, k_tc5_bf16.cu)
Tc5Kernel pick_tc5_f16(int kch, int bl, int emu);
Tc5Kernel pick_tc5_bf16(int kch, int bl, int emu);
inline Tc5Kernel pick_tc5(bool bf16, int kch, int bl, int emu) {
  return bf16 ? pick_tc5_bf16(kch, bl, emu) : pick_tc5_f16(kch, bl, emu);
}
// kernel 6 (k_tc6_f16.cu, k_tc6_bf16.cu): kernel 5's signature
Tc5Kernel pick_tc6_f16(int kch, int bl, int emu);
Tc5Kernel pick_tc6_bf16(int kch, int bl, int emu);
inline Tc5Kernel pick_tc6(bool bf16, int kch, int bl, int emu) {
  return bf16 ? pick_tc6_bf16(kch, bl, emu) : pick_tc6_f16(kch, bl, emu);
}
// kernel 7 (k_tf32.cu): fp32 on tcgen05, 3xTF32; wide = the K, L <= 128 variant (32-key tiles)
const void* tf32_fn(bool wide);
cudaError_t launch_tf32(bool wide, unsigned grid, cudaStream_t st, const float* A, const float* B, const float* D,
                        float* E, const Tf32Params& p);
// kernel 1, CUDA cores (k_simt.cu): dtype 0 f32, 1 f16, 2 bf16
const void* simt_fn(int dtype);
cudaError_t launch_simt(int dtype, unsigned grid, int smem, cudaStream_t st, const void* A, const void* B,
                        const void* D, void* E, const SimtParams& sp);
// split-N merge (k_merge.cu): E = Σ_r w_r E_r over R packed partials [R][rows][L]; vec = 16-byte chunks
cudaError_t launch_merge(int dtype, const void* parts, const float* lse, void* E, int R, int64_t rows, int64_t L,
                         bool softmax, bool vec, int n_sm, cudaStream_t st);

}  // namespace mbci
