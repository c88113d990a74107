// Forward kernel instances for static kernel kind RBF (split for parallel builds).
#include "sk_fwd_tables.cuh"
namespace sk {
FwdFn select_fwd_rbf(const FwdShape& s) { return sk_fwd_select<RBF>(s); }
}  // namespace sk
