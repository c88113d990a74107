// DMMA Gram backward instances (sk_mma_bwd.cuh).
#include "sk_mma_bwd.cuh"
#include "sk_plan.h"
namespace sk {
BwdFn select_bwd_mma(int DP, int WPC, int& smem_doubles_per_warp, bool dyadic, bool f32) {
  if (f32) {  // FP32 recurrences (order 0, 2-warp CTAs)
    if (dyadic || WPC != 2) return nullptr;
    switch (DP) {
      case 8: smem_doubles_per_warp = MmaBwdCfg<8>::WARP_DOUBLES; return gram_bwd_mma<8, 2, false, float>;
      case 16: smem_doubles_per_warp = MmaBwdCfg<16>::WARP_DOUBLES; return gram_bwd_mma<16, 2, false, float>;
      default: return nullptr;
    }
  }
  switch (DP) {
    case 8:
      smem_doubles_per_warp = MmaBwdCfg<8>::WARP_DOUBLES;
      if (dyadic) return gram_bwd_mma<8, 2, true>;
      return WPC == 2 ? gram_bwd_mma<8, 2> : WPC == 3 ? gram_bwd_mma<8, 3> : gram_bwd_mma<8, 4>;
    case 16:
      smem_doubles_per_warp = MmaBwdCfg<16>::WARP_DOUBLES;
      if (dyadic) return gram_bwd_mma<16, 2, true>;
      return WPC == 2 ? gram_bwd_mma<16, 2> : WPC == 3 ? gram_bwd_mma<16, 3> : gram_bwd_mma<16, 4>;
    default: return nullptr;
  }
}
}  // namespace sk
