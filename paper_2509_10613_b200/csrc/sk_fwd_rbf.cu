// Forward kernel instances for static kernel kind RBF (split for parallel builds).
#include "sk_fwd_tables.cuh"
namespace sk {
FwdFn select_fwd_rbf(const FwdShape& s, int& smem) { return sk_fwd_select<RBF>(s, smem); }
}  // namespace sk
