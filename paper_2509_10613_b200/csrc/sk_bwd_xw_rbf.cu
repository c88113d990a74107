// Backward instances, one pair per CTA (few long pairs), RBF kernel.
#include "sk_bwd_tables.cuh"
namespace sk {
BwdFn select_bwd_xw_rbf(const BwdShape& s, int& smem_doubles) {
  return sk_bwd_select_xw<RBF>(s, smem_doubles);
}
}  // namespace sk
