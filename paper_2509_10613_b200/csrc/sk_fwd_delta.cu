// Forward kernel instances for precomputed-delta solves (solve_goursat facade).
#include "sk_fwd_tables.cuh"
namespace sk {
FwdFn select_fwd_delta(const FwdShape& s, int& smem) {
  FwdFn fn = nullptr;
  sk_fwd_table<DELTA, 4, 8, double>(s, fn, smem);  // delta read per coarse cell; DP unused
  return fn;
}
}  // namespace sk
