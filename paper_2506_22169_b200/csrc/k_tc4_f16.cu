// k_tc4_f16.cu — instantiations of kernel 4 (chain_tc4.cuh), f16 inputs.
#include "kernels.h"

namespace mbci {
namespace {
constexpr bool kBF16 = false;
template <int KCH, int BL, int DCH>
Tc4Kernel pick_emu(int emu) {
  constexpr int NSB = DCH == 1 ? 3 : 2;   // three S buffers fit TMEM next to two 64-column O
  switch (emu) {
    case 0: return (Tc4Kernel)k_chain_tc4<kBF16, KCH, BL, DCH, 0, NSB>;
    case 2: return (Tc4Kernel)k_chain_tc4<kBF16, KCH, BL, DCH, 2, NSB>;
    default: return (Tc4Kernel)k_chain_tc4<kBF16, KCH, BL, DCH, 3, NSB>;
  }
}
template <int KCH, int BL>
Tc4Kernel pick_d(int dch, int emu) {
  return dch == 1 ? pick_emu<KCH, BL, 1>(emu) : pick_emu<KCH, BL, 2>(emu);
}
template <int KCH>
Tc4Kernel pick_bl(int bl, int dch, int emu) {
  return bl == 0 ? pick_d<KCH, 0>(dch, emu) : pick_d<KCH, 1>(dch, emu);
}
}  // namespace

Tc4Kernel pick_tc4_f16(int kch, int bl, int dch, int emu) {
  return kch == 1 ? pick_bl<1>(bl, dch, emu) : pick_bl<2>(bl, dch, emu);
}
}  // namespace mbci
