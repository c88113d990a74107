// DMMA Gram forward instances (sk_mma_fwd.cuh), one per padded dimension.
#include "sk_mma_fwd.cuh"
#include "sk_plan.h"
namespace sk {
FwdFn select_fwd_mma(int DP, int& smem_per_warp, bool dyadic) {
  smem_per_warp = MmaFwdCfg::WARP_BYTES;
  switch (DP) {
    case 4: return dyadic ? gram_fwd_mma<4, true> : gram_fwd_mma<4>;
    case 8: return dyadic ? gram_fwd_mma<8, true> : gram_fwd_mma<8>;
    case 16: return dyadic ? gram_fwd_mma<16, true> : gram_fwd_mma<16>;
    case 32: return dyadic ? gram_fwd_mma<32, true> : gram_fwd_mma<32>;
    default: return nullptr;
  }
}
}  // namespace sk
