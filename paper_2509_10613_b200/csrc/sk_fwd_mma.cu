// DMMA Gram forward instances (sk_mma_fwd.cuh), one per padded dimension.
#include "sk_mma_fwd.cuh"
#include "sk_plan.h"
namespace sk {
FwdFn select_fwd_mma(int DP, int& smem_per_warp) {
  smem_per_warp = MmaFwdCfg::WARP_BYTES;
  switch (DP) {
    case 4: return gram_fwd_mma<4>;
    case 8: return gram_fwd_mma<8>;
    case 16: return gram_fwd_mma<16>;
    case 32: return gram_fwd_mma<32>;
    default: return nullptr;
  }
}
}  // namespace sk
