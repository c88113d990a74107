// Backward kernel instances for static kernel kind RBF (split for parallel builds).
#include "sk_bwd_tables.cuh"
namespace sk {
BwdFn select_bwd_rbf(const BwdShape& s, int& smem_doubles) {
  return sk_bwd_select<RBF>(s, smem_doubles);
}
}  // namespace sk
