// Forward kernel instances for static kernel kind LINEAR (split for parallel builds).
#include "sk_fwd_tables.cuh"
namespace sk {
FwdFn select_fwd_linear(const FwdShape& s, int& smem) { return sk_fwd_select<LINEAR>(s, smem); }
}  // namespace sk
