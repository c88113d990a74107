// Backward instances, one pair per CTA (few long pairs), linear kernel.
#include "sk_bwd_tables.cuh"
namespace sk {
BwdFn select_bwd_xw_linear(const BwdShape& s, int& smem_doubles) {
  return sk_bwd_select_xw<LINEAR>(s, smem_doubles);
}
}  // namespace sk
