// DMMA Gram forward instances (sk_mma_fwd.cuh), one per padded dimension.
#include "sk_mma_fwd.cuh"
#include "sk_plan.h"
namespace sk {
FwdFn select_fwd_mma(int DP, int& smem_per_warp, bool dyadic, bool f32) {
  smem_per_warp = MmaFwdCfg::WARP_BYTES;
#define SK_MMA_PICK(D)                                                               \
  (f32 ? (dyadic ? gram_fwd_mma<D, true, float> : gram_fwd_mma<D, false, float>)    \
       : (dyadic ? gram_fwd_mma<D, true> : gram_fwd_mma<D>))
  switch (DP) {
    case 4: return SK_MMA_PICK(4);
    case 8: return SK_MMA_PICK(8);
    case 16: return SK_MMA_PICK(16);
    case 32: return SK_MMA_PICK(32);
    default: return nullptr;
  }
#undef SK_MMA_PICK
}
}  // namespace sk
