// k_tc5_f16.cu — instantiations of kernel 5 (chain_tc5.cuh), f16 inputs.
#include "kernels.h"
#include "chain_tc5.cuh"

namespace mbci {
namespace {
constexpr bool kBF16 = false;
template <int KCH, int BL>
Tc5Kernel pick_emu(int emu) {
  switch (emu) {
    case -1: return (Tc5Kernel)k_chain_tc5<kBF16, KCH, BL, -1>;   // linear ops
    case 0: return (Tc5Kernel)k_chain_tc5<kBF16, KCH, BL, 0>;
    case 2: return (Tc5Kernel)k_chain_tc5<kBF16, KCH, BL, 2>;
    case 4: return (Tc5Kernel)k_chain_tc5<kBF16, KCH, BL, 4>;
    default: return (Tc5Kernel)k_chain_tc5<kBF16, KCH, BL, 3>;
  }
}
template <int KCH>
Tc5Kernel pick_bl(int bl, int emu) {
  return bl == 0 ? pick_emu<KCH, 0>(emu) : pick_emu<KCH, 1>(emu);
}
}  // namespace

Tc5Kernel pick_tc5_f16(int kch, int bl, int emu) {
  return kch == 1 ? pick_bl<1>(bl, emu) : pick_bl<2>(bl, emu);
}
}  // namespace mbci
