// k_tc0.cu — instantiations of kernel 0 (chain_tc.cuh).
#include "kernels.h"

namespace mbci {
namespace {
template <bool BF16, int BN, int KCH, int BL>
TcKernel pick_d(int dch) {
  return dch == 1 ? (TcKernel)k_chain_tc<BF16, BN, KCH, BL, 1> : (TcKernel)k_chain_tc<BF16, BN, KCH, BL, 2>;
}
template <bool BF16, int BN, int KCH>
TcKernel pick_bl(int bl, int dch) {
  return bl == 0 ? pick_d<BF16, BN, KCH, 0>(dch) : pick_d<BF16, BN, KCH, 1>(dch);
}
template <bool BF16, int BN>
TcKernel pick_kch(int kch, int bl, int dch) {
  return kch == 1 ? pick_bl<BF16, BN, 1>(bl, dch) : pick_bl<BF16, BN, 2>(bl, dch);
}
template <bool BF16>
TcKernel pick_bn(int bn, int kch, int bl, int dch) {
  return bn == 64 ? pick_kch<BF16, 64>(kch, bl, dch) : pick_kch<BF16, 128>(kch, bl, dch);
}
}  // namespace

TcKernel pick_tc(bool bf16, int bn, int kch, int bl, int dch) {
  return bf16 ? pick_bn<true>(bn, kch, bl, dch) : pick_bn<false>(bn, kch, bl, dch);
}
}  // namespace mbci
