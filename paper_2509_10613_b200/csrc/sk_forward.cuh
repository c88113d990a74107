// sk_forward.cuh -- forward Goursat solve as a register-resident skewed wavefront.
//
// Replaces the reference's CPU march (goursat_strip / goursat_batch /
// goursat_gram, /root/reference/pkg/src/sigcore/_kernels.py:293-338, 399-429).
//
// Mapping (B200-first):
//   * a lane group of G lanes solves one pair; lane u owns R consecutive fine
//     rows of a strip of G*R rows and sweeps the columns left->right, one
//     "step" (F fine columns) at a time, lagging lane u-1 by one step.  The
//     three rotating anti-diagonals of the reference become registers: k_left
//     per owned row, the top-row value from lane u-1 arrives by __shfl_up_sync.
//   * G <= 32: 32/G pairs per warp (Gram tiles share the column path, so the
//     per-step column loads are warp broadcasts).  XW: one pair per CTA and
//     G = blockDim.x lanes; lane 31 -> lane 0 of the next warp goes through a
//     double-buffered shared-memory slot with one CTA barrier per step (long
//     pairs, BASELINE config 4).
//   * the increment product delta (kernel.py:60-77) is never materialised: the
//     lane keeps its rows' (pre-scaled) increments in registers and forms
//     <dx_i, dy_j> on the fly per coarse cell; dyadic refinement is on the fly
//     (fine cell (s,t) reads coarse (s-1)>>lam1, (t-1)>>lam2, _kernels.py:325).
//   * the strip's bottom row is handed to the next strip through a per-group
//     row in global memory (L2 resident), in place, exactly like the
//     reference's handoff row.
#pragma once
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

// Row-path registers of one lane for one strip.
template <int KIND, int DP, int RC>
struct RowRegs {
  static constexpr int NR = (KIND == RBF) ? RC + 1 : RC;
  double v[NR][DP];
};

template <int KIND, int DP, int RC>
__device__ __forceinline__ void load_rows(RowRegs<KIND, DP, RC>& rr, const Problem& pb,
                                          int64_t pr, int i0, int ch) {
  constexpr int NR = RowRegs<KIND, DP, RC>::NR;
  const int lim = (KIND == RBF) ? pb.M1c + 1 : pb.M1c;
#pragma unroll
  for (int c = 0; c < NR; ++c) {
    if (i0 + c < lim) {
      load_vec<DP>(rr.v[c], pb.R.p + pr * pb.R.path_stride + (int64_t)(i0 + c) * pb.dpad + ch * DP);
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

// Forward kernel.  Template parameters:
//   KIND  LINEAR / RBF / DELTA
//   DP    padded path dimension held in registers per chunk
//   R     fine rows per lane;  FR = fine rows per coarse row inside a lane
//         (= min(2^lam1, R)), so RC = R / FR coarse rows per lane
//   F     fine columns per step (= min(2^lam2, 4))
//   G     lanes per pair (<= 32); ignored when XW (G = blockDim.x)
//   XW    cross-warp lane groups (one pair per CTA)
template <int KIND, int DP, int R, int FR, int F, int G, bool XW>
__global__ void __launch_bounds__(XW ? 1024 : 128)
fwd_kernel(Problem pb, double* __restrict__ hand, int64_t hand_stride) {
  constexpr int RC = R / FR;
  constexpr int P = XW ? 1 : 32 / G;
  __shared__ double xbuf[XW ? 2 : 1][XW ? 32 : 1][F];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int Grt = XW ? (int)blockDim.x : G;
  const int g = XW ? 0 : lane / G;
  const int u = XW ? (int)threadIdx.x : lane % G;

  const int M1 = pb.M1c << pb.lam1;
  const int M2 = pb.M2c << pb.lam2;
  const int NS = M2 / F;  // steps per strip
  const int H = Grt * R;  // strip height
  const int nstrips = (M1 + H - 1) / H;
  const int last_strip = (M1 - 1) / H;
  const int u_star = ((M1 - 1) % H) / R;
  const int r_star = (M1 - 1) % R;

  const int64_t slot = XW ? (int64_t)blockIdx.x : ((int64_t)blockIdx.x * nw + warp) * P + g;
  double* __restrict__ hrow = hand + slot * hand_stride;

  const int64_t item0 = XW ? blockIdx.x : (int64_t)blockIdx.x * nw + warp;
  const int64_t istep = XW ? gridDim.x : (int64_t)gridDim.x * nw;

  for (int64_t item = item0; item < pb.nitems; item += istep) {
    int64_t pr = 0, pc = 0, oidx = 0, pidx = 0;
    const bool valid = resolve_pair(pb, item, P, g, pr, pc, oidx, pidx);
    if (!valid) { pr = 0; pc = 0; pidx = 0; }

    for (int t = u; t <= M2; t += Grt) hrow[t] = 1.0;
    if (XW) __syncthreads(); else __syncwarp();

    for (int strip = 0; strip < nstrips; ++strip) {
      const int rbase = strip * H + u * R;  // 0-based fine row of the lane's first row
      const int i0 = rbase >> pb.lam1;
      RowRegs<KIND, DP, RC> rr;
      if constexpr (KIND != DELTA) load_rows<KIND, DP, RC>(rr, pb, pr, i0, 0);
      ColState<KIND, DP, RC> cs;
      cs.have = -2;
      double kl[R];
#pragma unroll
      for (int r = 0; r < R; ++r) kl[r] = 1.0;
      double topc = 1.0;
      double bot[F];
#pragma unroll
      for (int f = 0; f < F; ++f) bot[f] = 1.0;

      const int nsteps = NS + Grt - 1;
      for (int tau = 0; tau < nsteps; ++tau) {
        const int jj = tau - u;
        const bool active = (jj >= 0) && (jj < NS);
        double tv[F];
        if constexpr (XW) {
#pragma unroll
          for (int f = 0; f < F; ++f) tv[f] = __shfl_up_sync(0xffffffffu, bot[f], 1);
          if (lane == 0 && warp > 0) {
#pragma unroll
            for (int f = 0; f < F; ++f) tv[f] = xbuf[(tau + 1) & 1][warp - 1][f];
          }
        } else {
#pragma unroll
          for (int f = 0; f < F; ++f) tv[f] = __shfl_up_sync(0xffffffffu, bot[f], 1, G);
        }
        if (u == 0 && active) {
#pragma unroll
          for (int f = 0; f < F; ++f) tv[f] = (strip == 0) ? 1.0 : hrow[jj * F + f + 1];
        }
        if (active) {
          const int jc = (jj * F) >> pb.lam2;
          double p[RC];
          coarse_p<KIND, DP, RC>(p, rr, cs, pb, pr, pc, pidx, i0, jc);
          if constexpr (KIND == LINEAR) {
            if (pb.scale != 1.0) {
#pragma unroll
              for (int c = 0; c < RC; ++c) p[c] *= pb.scale;  // exact: power of two
            }
          }
          Coef cf[RC];
#pragma unroll
          for (int c = 0; c < RC; ++c) cf[c] = coef(p[c]);
#pragma unroll
          for (int f = 0; f < F; ++f) {
            double up = tv[f];
            double dg = (f == 0) ? topc : tv[f - 1];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const double nk = cell(up, kl[r], dg, cf[r / FR]);
              dg = kl[r];
              kl[r] = nk;
              up = nk;
            }
            bot[f] = up;
          }
          topc = tv[F - 1];
          if (u == Grt - 1) {
#pragma unroll
            for (int f = 0; f < F; ++f) hrow[jj * F + f + 1] = bot[f];
          }
          if (strip == last_strip && u == u_star && jj == NS - 1 && valid) {
            double v = kl[0];
#pragma unroll
            for (int r = 1; r < R; ++r)
              if (r == r_star) v = kl[r];
            pb.out[oidx] = v;
          }
        }
        if constexpr (XW) {
          if (lane == 31) {
#pragma unroll
            for (int f = 0; f < F; ++f) xbuf[tau & 1][warp][f] = bot[f];
          }
          __syncthreads();
        }
      }
      if (XW) __syncthreads(); else __syncwarp();
    }
  }
}

}  // namespace sk
