// sk_cell.cuh -- per-cell arithmetic and row/column data helpers shared by the
// forward and backward wavefront kernels.
#pragma once
#include <type_traits>

#include "sk_common.cuh"

namespace sk {

// _kernels.py:286-290: k = (k_up + k_left) * A(p) - k_diag * B(p),
// A = 1 + p/2 + p^2/12, B = 1 - p^2/12 (A, B hoisted per coarse cell).
struct Coef {
  double A, B;
};
__device__ __forceinline__ Coef coef(double p) {
  double q = p * p;
  Coef c;
  c.A = fma(q, 1.0 / 12.0, fma(p, 0.5, 1.0));
  c.B = fma(-q, 1.0 / 12.0, 1.0);
  return c;
}
__device__ __forceinline__ double cell(double up, double left, double diag, const Coef& c) {
  return fma(up + left, c.A, -diag * c.B);
}

// FP32 arithmetic (the fp32 kernels): the cell in
// "small-correction" form.  With u = k_up + k_left,
//   k = u A - k_diag B = (u - k_diag) + (u (p/2 + q) + k_diag q),  q = p^2/12,
// so the O(1) part is one exact-ish difference and the O(p) corrections are
// formed separately: the fp32 rounding of A = 1 + p/2 + ... would otherwise
// swallow p ~ 1e-4 increments (measured 3.8e-3 relative error at BASELINE
// config 2 as written vs 5.9e-5 in this form).
struct Coef32 {
  float Ap, q;  // p/2 + q, p^2/12
};
__device__ __forceinline__ Coef32 coef(float p) {
  Coef32 c;
  c.q = p * p * (1.0f / 12.0f);
  c.Ap = fmaf(p, 0.5f, c.q);
  return c;
}
__device__ __forceinline__ float cell(float up, float left, float diag, const Coef32& c) {
  const float u = up + left;
  return (u - diag) + fmaf(diag, c.q, u * c.Ap);
}
template <typename T>
using CoefOf = typename std::conditional<sizeof(T) == 8, Coef, Coef32>::type;

template <int DP>
__device__ __forceinline__ void load_vec(float (&v)[DP], const float* __restrict__ src) {
  if constexpr (DP % 4 == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int k = 0; k < DP / 4; ++k) {
      float4 t = __ldg(s4 + k);
      v[4 * k] = t.x;
      v[4 * k + 1] = t.y;
      v[4 * k + 2] = t.z;
      v[4 * k + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < DP; ++k) v[k] = __ldg(src + k);
  }
}

template <int DP>
__device__ __forceinline__ float dot(const float (&a)[DP], const float (&b)[DP]) {
  float s = a[0] * b[0];
#pragma unroll
  for (int k = 1; k < DP; ++k) s = fmaf(a[k], b[k], s);
  return s;
}

template <int DP>
__device__ __forceinline__ void load_vec(double (&v)[DP], const double* __restrict__ src) {
  if constexpr (DP % 2 == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int k = 0; k < DP / 2; ++k) {
      double2 t = __ldg(s2 + k);
      v[2 * k] = t.x;
      v[2 * k + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < DP; ++k) v[k] = __ldg(src + k);
  }
}

template <int DP>
__device__ __forceinline__ double dot(const double (&a)[DP], const double (&b)[DP]) {
  // one sequential FMA chain, k = 0..DP-1, starting from 0: exactly what the
  // FP64 tensor-core path computes (mma.m8n8k4.f64 is a sequential fma chain
  // over its k, measured bitwise by tools/dmma_probe.cu), so the DMMA Gram
  // kernels, the batch kernels and the backward recompute agree bitwise
  double s = a[0] * b[0];
#pragma unroll
  for (int k = 1; k < DP; ++k) s = fma(a[k], b[k], s);
  return s;
}

template <int DP>
__device__ __forceinline__ double sqdist(const double (&a)[DP], const double (&b)[DP]) {
  double t = a[0] - b[0];
  double s = t * t;
#pragma unroll
  for (int k = 1; k < DP; ++k) {
    t = a[k] - b[k];
    s = fma(t, t, s);
  }
  return s;
}

// Row-path registers of one lane for one strip (T: arithmetic type; the
// fp32 kernels' path data are float arrays behind the same pointers).
template <int KIND, int DP, int RC, typename T = double>
struct RowRegs {
  static constexpr int NR = (KIND == RBF) ? RC + 1 : RC;
  T v[NR][DP];
};

template <int KIND, int DP, int RC, typename T = double>
__device__ __forceinline__ void load_rows(RowRegs<KIND, DP, RC, T>& rr, const Problem& pb,
                                          int64_t pr, int i0, int ch) {
  constexpr int NR = RowRegs<KIND, DP, RC, T>::NR;
  const int lim = (KIND == RBF) ? pb.M1c + 1 : pb.M1c;
  const T* base = reinterpret_cast<const T*>(pb.R.p);
#pragma unroll
  for (int c = 0; c < NR; ++c) {
    if (i0 + c < lim) {
      load_vec<DP>(rr.v[c], base + pr * pb.R.path_stride + (int64_t)(i0 + c) * pb.dpad + ch * DP);
    } else {
#pragma unroll
      for (int k = 0; k < DP; ++k) rr.v[c][k] = 0.0;
    }
  }
}

// p for the lane's RC coarse rows at coarse column jc (LINEAR / DELTA), or the
// RBF second difference using the K values carried between steps.
template <int KIND, int DP, int RC>
struct ColState {
  double Kold[RC + 1];
  double Knew[RC + 1];
  int have;  // coarse column whose Kold/Knew are held (-1: none)
};

template <int KIND, int DP, int RC>
__device__ __forceinline__ void rbf_column(double (&K)[RC + 1], const RowRegs<KIND, DP, RC>& rr,
                                           const Problem& pb, int64_t pc, int node) {
  double yv[DP];
  load_vec<DP>(yv, pb.C.p + pc * pb.C.path_stride + (int64_t)node * pb.dpad);
#pragma unroll
  for (int c = 0; c <= RC; ++c) K[c] = exp(-sqdist<DP>(rr.v[c], yv) * pb.inv2s2);
}

template <int KIND, int DP, int RC>
__device__ __forceinline__ void coarse_p(double (&p)[RC], RowRegs<KIND, DP, RC>& rr,
                                         ColState<KIND, DP, RC>& cs, const Problem& pb,
                                         int64_t pr, int64_t pc, int64_t pidx, int i0, int jc) {
  if constexpr (KIND == LINEAR) {
    if (pb.nch == 1) {
      double dy[DP];
      load_vec<DP>(dy, pb.C.p + pc * pb.C.path_stride + (int64_t)jc * pb.dpad);
#pragma unroll
      for (int c = 0; c < RC; ++c) p[c] = dot<DP>(rr.v[c], dy);
    } else {
#pragma unroll
      for (int c = 0; c < RC; ++c) p[c] = 0.0;
      for (int ch = 0; ch < pb.nch; ++ch) {
        double dy[DP];
        load_vec<DP>(dy, pb.C.p + pc * pb.C.path_stride + (int64_t)jc * pb.dpad + ch * DP);
        load_rows<KIND, DP, RC>(rr, pb, pr, i0, ch);
#pragma unroll
        for (int c = 0; c < RC; ++c) p[c] += dot<DP>(rr.v[c], dy);
      }
    }
  } else if constexpr (KIND == RBF) {
    if (cs.have != jc) {
      if (cs.have == jc - 1) {
#pragma unroll
        for (int c = 0; c <= RC; ++c) cs.Kold[c] = cs.Knew[c];
      } else {
        rbf_column<KIND, DP, RC>(cs.Kold, rr, pb, pc, jc);
      }
      rbf_column<KIND, DP, RC>(cs.Knew, rr, pb, pc, jc + 1);
      cs.have = jc;
    }
#pragma unroll
    for (int c = 0; c < RC; ++c)
      p[c] = ((cs.Knew[c + 1] - cs.Kold[c + 1]) - (cs.Knew[c] - cs.Kold[c])) * pb.scale;
  } else {  // DELTA
#pragma unroll
    for (int c = 0; c < RC; ++c) {
      int i = i0 + c;
      p[c] = (i < pb.M1c) ? __ldg(pb.delta + pidx * (int64_t)pb.M1c * pb.M2c +
                                  (int64_t)i * pb.M2c + jc) * pb.scale
                          : 0.0;
    }
  }
}


// ------------------------------------------------------------ async copies
// cp.async (LDGSTS) into shared memory; src_bytes = 0 zero-fills (used for
// out-of-range columns so consumers never branch on validity).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
// one element of T (8- or 4-byte copy)
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem, bool valid);
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid);
template <>
__device__ __forceinline__ void cp_async_elem<double>(double* smem, const double* gmem, bool valid) {
  cp_async8(smem, gmem, valid);
}
template <>
__device__ __forceinline__ void cp_async_elem<float>(float* smem, const float* gmem, bool valid) {
  cp_async4(smem, gmem, valid);
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace sk
