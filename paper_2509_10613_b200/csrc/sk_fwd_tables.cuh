// sk_fwd_tables.cuh -- maps a runtime FwdShape to a forward kernel instance.
#pragma once
#include <type_traits>

#include "sk_forward.cuh"
#include "sk_plan.h"

namespace sk {

template <int KIND, int DP, int R, int FR, int F, typename T, bool XWONLY = false>
inline void sk_fwd_leaf(const FwdShape& s, FwdFn& fn, int& smem) {
  if (XWONLY || s.XW) {
    if constexpr (KIND != DELTA) {
      // up to 8 warps: the 255-register instance (measured at BASELINE config 2:
      // RBF forward 0.57 -> 0.50 ms, the 128-register one spills)
      if (s.W <= 8) fn = fwd_kernel<KIND, DP, R, FR, F, 32, true, 2, T, 256>;
      else fn = fwd_kernel<KIND, DP, R, FR, F, 32, true, 2, T, 512>;
      smem = fwd_smem_bytes<KIND, DP, F, 32, true, 2, T>(s.W);
    }
    return;
  }
  if constexpr (XWONLY) return;
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

template <int KIND, int DP, int R, int FR, typename T, bool XWONLY = false>
inline void sk_fwd_f(const FwdShape& s, FwdFn& fn, int& smem) {
  switch (s.F) {
    case 1: sk_fwd_leaf<KIND, DP, R, FR, 1, T, XWONLY>(s, fn, smem); break;
    case 2: sk_fwd_leaf<KIND, DP, R, FR, 2, T, XWONLY>(s, fn, smem); break;
    case 4: sk_fwd_leaf<KIND, DP, R, FR, 4, T, XWONLY>(s, fn, smem); break;
    default: break;
  }
}

template <int KIND, int DP, int R, typename T, bool XWONLY = false>
inline void sk_fwd_table(const FwdShape& s, FwdFn& fn, int& smem) {
  switch (s.FR) {
    case 1: sk_fwd_f<KIND, DP, R, 1, T, XWONLY>(s, fn, smem); break;
    case 2: if constexpr (R >= 2) sk_fwd_f<KIND, DP, R, 2, T, XWONLY>(s, fn, smem); break;
    case 4: if constexpr (R >= 4) sk_fwd_f<KIND, DP, R, 4, T, XWONLY>(s, fn, smem); break;
    case 8: if constexpr (R >= 8) sk_fwd_f<KIND, DP, R, 8, T, XWONLY>(s, fn, smem); break;
    default: break;
  }
}

template <int KIND, typename T = double>
inline FwdFn sk_fwd_select(const FwdShape& s, int& smem) {
  FwdFn fn = nullptr;
  switch (s.DP) {
    case 4: sk_fwd_table<KIND, 4, 8, T>(s, fn, smem); break;
    case 8:
      // cross-warp pairs taller than one 4-row strip: 8 rows per lane
      if (s.XW && s.R == 8) {
        if constexpr (KIND != DELTA) sk_fwd_table<KIND, 8, 8, T, true>(s, fn, smem);
      } else {
        sk_fwd_table<KIND, 8, 4, T>(s, fn, smem);
      }
      break;
    case 16: sk_fwd_table<KIND, 16, 2, T>(s, fn, smem); break;
    case 32: sk_fwd_table<KIND, 32, 1, T>(s, fn, smem); break;
    default: break;
  }
  return fn;
}

// Short paths (batch, one pair per warp): fewer rows per lane than the
// register-balanced default, so all 32 lanes hold rows and the dependent chain
// per step is short (BASELINE config 1: 63 rows -> R = 2 instead of 8).
template <int KIND, int DP, int R>
inline void sk_fwd_short_table(const FwdShape& s, FwdFn& fn, int& smem) {
  auto leaf = [&](auto fr, auto f) {
    constexpr int FR = decltype(fr)::value, F = decltype(f)::value;
    if constexpr (FR <= R) {
      fn = fwd_kernel<KIND, DP, R, FR, F, 32, false, 2, double>;
      smem = fwd_smem_bytes<KIND, DP, F, 32, false, 2, double>(4);
    }
  };
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  using I4 = std::integral_constant<int, 4>;
  auto by_f = [&](auto fr) {
    switch (s.F) {
      case 1: leaf(fr, I1{}); break;
      case 2: leaf(fr, I2{}); break;
      case 4: leaf(fr, I4{}); break;
      default: break;
    }
  };
  switch (s.FR) {
    case 1: by_f(I1{}); break;
    case 2: by_f(I2{}); break;
    case 4: by_f(I4{}); break;
    default: break;
  }
}

template <int KIND>
inline FwdFn sk_fwd_select_short(const FwdShape& s, int& smem) {
  FwdFn fn = nullptr;
  if (s.G != 32 || s.XW) return nullptr;
  switch (s.DP) {
    case 4:
      if (s.R == 1) sk_fwd_short_table<KIND, 4, 1>(s, fn, smem);
      else if (s.R == 2) sk_fwd_short_table<KIND, 4, 2>(s, fn, smem);
      else if (s.R == 4) sk_fwd_short_table<KIND, 4, 4>(s, fn, smem);
      break;
    case 8:
      if (s.R == 1) sk_fwd_short_table<KIND, 8, 1>(s, fn, smem);
      else if (s.R == 2) sk_fwd_short_table<KIND, 8, 2>(s, fn, smem);
      break;
    case 16:
      if (s.R == 1) sk_fwd_short_table<KIND, 16, 1>(s, fn, smem);
      break;
    default: break;
  }
  return fn;
}

}  // namespace sk
