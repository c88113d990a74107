// sk_bwd_tables.cuh -- maps a runtime BwdShape to a backward kernel instance.
#pragma once
#include <type_traits>

#include "sk_backward.cuh"
#include "sk_plan.h"

namespace sk {

template <int KIND, int DP, int R, int FR, int F, bool WIDE = false>
inline void sk_bwd_leaf(BwdFn& fn, int& smem_doubles) {
  constexpr int S = bwd_steps_cols(DP, F);
  constexpr int CB = bwd_block_steps(DP, R, F, S);
  // LINEAR maps the adjoint in the sweep (FUSED) unless d > 32 (WIDE: stored
  // coarse adjoint, mapped chunk by chunk after the sweep)
  constexpr int MAP = (KIND == LINEAR && !WIDE) ? FUSED : DBUF;
  fn = bwd_kernel<KIND, DP, R, FR, F, CB, MAP, S>;
  smem_doubles = BwdSmem<DP, R, R / FR, F, CB, S>::TOTAL;  // per warp
}

template <int KIND, int DP, int R, int FR>
inline void sk_bwd_f(const BwdShape& s, BwdFn& fn, int& sm) {
  switch (s.F) {
    case 1: sk_bwd_leaf<KIND, DP, R, FR, 1>(fn, sm); break;
    case 2: sk_bwd_leaf<KIND, DP, R, FR, 2>(fn, sm); break;
    case 4: sk_bwd_leaf<KIND, DP, R, FR, 4>(fn, sm); break;
    default: break;
  }
}

template <int KIND, int DP, int R>
inline void sk_bwd_table(const BwdShape& s, BwdFn& fn, int& sm) {
  switch (s.FR) {
    case 1: sk_bwd_f<KIND, DP, R, 1>(s, fn, sm); break;
    case 2: if constexpr (R >= 2) sk_bwd_f<KIND, DP, R, 2>(s, fn, sm); break;
    case 4: if constexpr (R >= 4) sk_bwd_f<KIND, DP, R, 4>(s, fn, sm); break;
    case 8: if constexpr (R >= 8) sk_bwd_f<KIND, DP, R, 8>(s, fn, sm); break;
    default: break;
  }
}

template <int KIND>
inline BwdFn sk_bwd_select(const BwdShape& s, int& smem_doubles) {
  BwdFn fn = nullptr;
  switch (s.DP) {
    case 4: sk_bwd_table<KIND, 4, 8>(s, fn, smem_doubles); break;
    case 8: sk_bwd_table<KIND, 8, 4>(s, fn, smem_doubles); break;
    case 16:
      if (s.R == 1) sk_bwd_table<KIND, 16, 1>(s, fn, smem_doubles);
      else sk_bwd_table<KIND, 16, 2>(s, fn, smem_doubles);
      break;
    case 32: sk_bwd_table<KIND, 32, 1>(s, fn, smem_doubles); break;
    default: break;
  }
  return fn;
}

// Few long pairs (batch): one pair per CTA of NW warps.
template <int KIND, int DP, int R, int FR, int F, int NW>
inline void sk_bwd_leaf_xw(BwdFn& fn, int& smem_doubles) {
  constexpr int S = bwd_steps_cols(DP, F);
  constexpr int CB = bwd_block_steps_xw(R, F, S);
  constexpr int MAP = (KIND == LINEAR) ? FUSED : DBUF;
  fn = bwd_kernel<KIND, DP, R, FR, F, CB, MAP, S, NW>;
  smem_doubles = BwdSmem<DP, R, R / FR, F, CB, S, 32 * NW>::TOTAL;  // per CTA
}

template <int KIND, int DP, int R, int NW>
inline void sk_bwd_table_xw(const BwdShape& s, BwdFn& fn, int& sm) {
  auto by_f = [&](auto fr) {
    constexpr int FR = decltype(fr)::value;
    if constexpr (FR <= R) {
      switch (s.F) {
        case 1: sk_bwd_leaf_xw<KIND, DP, R, FR, 1, NW>(fn, sm); break;
        case 2: sk_bwd_leaf_xw<KIND, DP, R, FR, 2, NW>(fn, sm); break;
        case 4: sk_bwd_leaf_xw<KIND, DP, R, FR, 4, NW>(fn, sm); break;
        default: break;
      }
    }
  };
  switch (s.FR) {
    case 1: by_f(std::integral_constant<int, 1>{}); break;
    case 2: by_f(std::integral_constant<int, 2>{}); break;
    case 4: by_f(std::integral_constant<int, 4>{}); break;
    case 8: by_f(std::integral_constant<int, 8>{}); break;
    default: break;
  }
}

template <int KIND>
inline BwdFn sk_bwd_select_xw(const BwdShape& s, int& smem_doubles) {
  BwdFn fn = nullptr;
  if (s.DP == 4 && s.NW == 4) sk_bwd_table_xw<KIND, 4, 8, 4>(s, fn, smem_doubles);
  else if (s.DP == 4 && s.NW == 8) sk_bwd_table_xw<KIND, 4, 8, 8>(s, fn, smem_doubles);
  else if (s.DP == 8 && s.NW == 4 && s.R == 8) sk_bwd_table_xw<KIND, 8, 8, 4>(s, fn, smem_doubles);
  else if (s.DP == 8 && s.NW == 4) sk_bwd_table_xw<KIND, 8, 4, 4>(s, fn, smem_doubles);
  else if (s.DP == 8 && s.NW == 8) sk_bwd_table_xw<KIND, 8, 4, 8>(s, fn, smem_doubles);
  return fn;
}

// d > 32 (linear kernel): DP = 32 chunks, one row per lane.
inline BwdFn sk_bwd_select_wide(const BwdShape& s, int& smem_doubles) {
  BwdFn fn = nullptr;
  switch (s.F) {
    case 1: sk_bwd_leaf<LINEAR, 32, 1, 1, 1, true>(fn, smem_doubles); break;
    case 2: sk_bwd_leaf<LINEAR, 32, 1, 1, 2, true>(fn, smem_doubles); break;
    case 4: sk_bwd_leaf<LINEAR, 32, 1, 1, 4, true>(fn, smem_doubles); break;
    default: break;
  }
  return fn;
}

}  // namespace sk
