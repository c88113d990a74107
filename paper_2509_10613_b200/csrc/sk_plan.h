// sk_plan.h -- host-side kernel selection (template instance tables).
#pragma once
#include <cstdlib>

#include "sk_common.cuh"

namespace sk {

using FwdFn = void (*)(Problem, double*, int64_t);

// Shape class chosen on the host for one call.
struct FwdShape {
  int kind;
  int DP;   // 4, 8, 16, 32
  int R;    // fine rows per lane
  int FR;   // fine rows per coarse row inside a lane
  int F;    // fine columns per step
  int G;    // lanes per pair (4 or 32), ignored if XW
  bool XW;  // cross-warp groups: one pair per CTA of W warps
  int W;    // warps per CTA when XW
  bool MMA; // DMMA Gram tile kernel (sk_mma_fwd.cuh): LINEAR, dyadic order 0, DP <= 16
};

using BwdFn = void (*)(Problem, BwdArgs);

struct BwdShape {
  int kind;
  int DP, R, FR, F;  // as FwdShape; lanes per pair 32 NW, CB = 8 / F
  int NW;            // warps per pair (1: one pair per warp; 4, 8: one pair per CTA)
  bool MMA;          // DMMA Gram tile kernel (sk_mma_bwd.cuh): LINEAR, order 0, DP 8/16
  int WPC;           // warps per CTA of the DMMA kernel
};

BwdFn select_bwd_linear(const BwdShape& s, int& smem_doubles);
BwdFn select_bwd_rbf(const BwdShape& s, int& smem_doubles);
BwdFn select_bwd_wide(const BwdShape& s, int& smem_doubles);  // linear, d > 32
BwdFn select_bwd_xw_linear(const BwdShape& s, int& smem_doubles);  // one pair per CTA
BwdFn select_bwd_xw_rbf(const BwdShape& s, int& smem_doubles);
BwdFn select_bwd_mma(int DP, int WPC, int& smem_doubles_per_warp, bool dyadic, bool f32 = false);

// Per-kind instance tables (one translation unit each, compiled in parallel).
FwdFn select_fwd_linear(const FwdShape& s, int& smem);
FwdFn select_fwd_linear_f32(const FwdShape& s, int& smem);  // FP32 arithmetic
FwdFn select_fwd_short(const FwdShape& s, int& smem);       // short paths, fp64
FwdFn select_fwd_rbf(const FwdShape& s, int& smem);
FwdFn select_fwd_delta(const FwdShape& s, int& smem);
FwdFn select_fwd_mma(int DP, int& smem_per_warp, bool dyadic, bool f32);
// few short pairs (sk_small.cu); false when the shape does not apply
bool launch_small_fwd(const double* xr, const double* xc, int64_t B, int64_t LR, int64_t LC,
                      int64_t d, int lamR, int lamC, double scale, double* out, int sms,
                      cudaStream_t st);

inline int rows_per_lane(int DP) {
  switch (DP) {
    case 4: return 8;
    case 8: return 4;
    case 16: return 2;
    default: return 1;
  }
}

// Backward: the reverse sweep keeps dx, gx (RC x DP each) and the gy chain
// (DP) live, so wide paths trade rows per lane for occupancy.
// Backward columns per step (narrow paths amortise per-step overhead) and
// block width in steps (~16 recomputed values per lane, at least one step).
// (measured: S = 2 for d = 8 was slower, 426 vs 366 ms on a 256^2 C5-shaped Gram,
// register pressure; kept as a knob)
constexpr int bwd_steps_cols(int DP, int F) { return (DP <= 8 && F == 1 && false) ? 2 : 1; }
constexpr int bwd_block_steps(int DP, int R, int F, int S) {
  // wide paths: ~8 values per lane so two CTAs of four warps fit in shared memory
  return ((DP >= 16 ? 8 : 16) / (F * R * S)) < 1 ? 1
         : ((DP >= 16 ? 8 : 16) / (F * R * S)) > 8 ? 8
                                                   : (DP >= 16 ? 8 : 16) / (F * R * S);
}

// cross-warp (one pair per CTA) backward: fine cells per lane per block
#ifndef SK_XW_CBV
#define SK_XW_CBV 32  // measured at C2: 16 -> 2.02 ms, 32 -> 1.61 ms, 64 (shared memory) 2.98 ms
#endif
constexpr int bwd_block_steps_xw(int R, int F, int S) {
  return (SK_XW_CBV / (F * R * S)) < 1 ? 1 : (SK_XW_CBV / (F * R * S)) > 8 ? 8 : SK_XW_CBV / (F * R * S);
}

inline int bwd_rows_per_lane(int DP) {
  if (DP != 16) return rows_per_lane(DP);
  const char* e = std::getenv("SK_BWD_R16");  // tuning override (1 or 2)
  return (e && e[0] == '1') ? 1 : 2;  // measured: R=2 beats R=1 (238 vs 411 ms, C3 n=256)
}

}  // namespace sk

