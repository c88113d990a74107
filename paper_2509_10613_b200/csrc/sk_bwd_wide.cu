// Backward kernel instances for the linear kernel at d > 32 (split for parallel builds).
#include "sk_bwd_tables.cuh"
namespace sk {
BwdFn select_bwd_wide(const BwdShape& s, int& smem_doubles) {
  return sk_bwd_select_wide(s, smem_doubles);
}
}  // namespace sk
