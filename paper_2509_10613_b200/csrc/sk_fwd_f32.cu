// Forward kernel instances with FP32 arithmetic (linear static kernel; split
// for parallel builds).  Same wavefront as the fp64 kernels, small-correction
// cell (sk_cell.cuh Coef32).
#include "sk_fwd_tables.cuh"
namespace sk {
FwdFn select_fwd_linear_f32(const FwdShape& s, int& smem) {
  return sk_fwd_select<LINEAR, float>(s, smem);
}
}  // namespace sk
