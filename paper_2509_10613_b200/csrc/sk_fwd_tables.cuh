// sk_fwd_tables.cuh -- maps a runtime FwdShape to a forward kernel instance.
#pragma once
#include "sk_forward.cuh"
#include "sk_plan.h"

namespace sk {

template <int KIND, int DP, int R, int FR, int F, typename T>
inline void sk_fwd_leaf(const FwdShape& s, FwdFn& fn, int& smem) {
  if (s.XW) {
    if constexpr (KIND == LINEAR) {
      fn = fwd_kernel<KIND, DP, R, FR, F, 32, true, 2, T>;
      smem = fwd_smem_bytes<KIND, DP, F, 32, true, 2, T>(s.W);
    }
    return;
  }
  if (s.G == 4) {
    // columns per step: amortise per-step overhead without crowding registers
    constexpr int S4 = DP >= 16 ? 1 : 4;
    fn = fwd_kernel<KIND, DP, R, FR, F, 4, false, S4, T>;
    smem = fwd_smem_bytes<KIND, DP, F, 4, false, S4, T>(4);
  } else if (s.G == 32) {
    fn = fwd_kernel<KIND, DP, R, FR, F, 32, false, 2, T>;
    smem = fwd_smem_bytes<KIND, DP, F, 32, false, 2, T>(4);
  }
}

template <int KIND, int DP, int R, int FR, typename T>
inline void sk_fwd_f(const FwdShape& s, FwdFn& fn, int& smem) {
  switch (s.F) {
    case 1: sk_fwd_leaf<KIND, DP, R, FR, 1, T>(s, fn, smem); break;
    case 2: sk_fwd_leaf<KIND, DP, R, FR, 2, T>(s, fn, smem); break;
    case 4: sk_fwd_leaf<KIND, DP, R, FR, 4, T>(s, fn, smem); break;
    default: break;
  }
}

template <int KIND, int DP, int R, typename T>
inline void sk_fwd_table(const FwdShape& s, FwdFn& fn, int& smem) {
  switch (s.FR) {
    case 1: sk_fwd_f<KIND, DP, R, 1, T>(s, fn, smem); break;
    case 2: if constexpr (R >= 2) sk_fwd_f<KIND, DP, R, 2, T>(s, fn, smem); break;
    case 4: if constexpr (R >= 4) sk_fwd_f<KIND, DP, R, 4, T>(s, fn, smem); break;
    case 8: if constexpr (R >= 8) sk_fwd_f<KIND, DP, R, 8, T>(s, fn, smem); break;
    default: break;
  }
}

template <int KIND, typename T = double>
inline FwdFn sk_fwd_select(const FwdShape& s, int& smem) {
  FwdFn fn = nullptr;
  switch (s.DP) {
    case 4: sk_fwd_table<KIND, 4, 8, T>(s, fn, smem); break;
    case 8: sk_fwd_table<KIND, 8, 4, T>(s, fn, smem); break;
    case 16: sk_fwd_table<KIND, 16, 2, T>(s, fn, smem); break;
    case 32: sk_fwd_table<KIND, 32, 1, T>(s, fn, smem); break;
    default: break;
  }
  return fn;
}

}  // namespace sk
