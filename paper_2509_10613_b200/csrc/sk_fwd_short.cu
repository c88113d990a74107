// Forward kernel instances for short paths (fewer rows per lane; split for
// parallel builds).
#include "sk_fwd_tables.cuh"
namespace sk {
FwdFn select_fwd_short(const FwdShape& s, int& smem) {
  return s.kind == RBF ? sk_fwd_select_short<RBF>(s, smem) : sk_fwd_select_short<LINEAR>(s, smem);
}
}  // namespace sk
