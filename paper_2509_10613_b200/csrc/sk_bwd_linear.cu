// Backward kernel instances for static kernel kind LINEAR (split for parallel builds).
#include "sk_bwd_tables.cuh"
namespace sk {
BwdFn select_bwd_linear(const BwdShape& s, int& smem_doubles) {
  return sk_bwd_select<LINEAR>(s, smem_doubles);
}
}  // namespace sk
