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
//   * G = 4: 8 pairs per warp sharing the column path (Gram tiles); G = 32: one
//     pair per warp; XW: one pair per CTA, G = blockDim.x lanes, lane 31 ->
//     lane 0 of the next warp through a double-buffered shared-memory slot and
//     one CTA barrier per step (long pairs, BASELINE config 4).
//   * column data (increments dy_j or RBF nodes y_{j+1}) and the strip's
//     handoff row stream through a shared-memory ring filled by cp.async PF
//     steps ahead, so no global latency sits on the recurrence;
//   * the increment product delta (kernel.py:60-77) is never materialised: the
//     lane keeps its rows' increments in registers and forms <dx_i, dy_j> for
//     step tau+1 while the recurrence of step tau runs (software pipeline);
//     dyadic refinement is on the fly (fine cell (s,t) reads coarse
//     (s-1)>>lam1, (t-1)>>lam2, _kernels.py:325);
//   * the strip's bottom row is handed to the next strip through a per-group
//     row in global memory (L2 resident), in place, like the reference's
//     handoff row.
#pragma once
#include "sk_cell.cuh"

namespace sk {

template <int KIND, int DP, int F, int P>
struct FwdRec {
  static constexpr int CD = (KIND == DELTA) ? 0 : DP;  // column data doubles
  static constexpr int RAW = CD + P * F;               // + handoff values per group
  static constexpr int REC = (RAW + 1) & ~1;           // 16-byte aligned records
};

template <bool XW, int G>
struct FwdRing {
  static constexpr int PF = 4;
  static constexpr int SLOTS = XW ? 1024 : (G >= 32 ? 64 : 16);
};

// Issue the ring record of step jj: column data of coarse column jc(jj) and
// the handoff values of every group (strip > 0).  Executed by one warp.
template <int KIND, int DP, int F, int P>
__device__ __forceinline__ void fwd_issue(double* ring_slot, const Problem& pb, int64_t pc,
                                          const double* hrow0, int64_t hand_stride, int jj,
                                          int NS, int strip, int lane) {
  using RC_ = FwdRec<KIND, DP, F, P>;
  const bool valid = (jj >= 0) && (jj < NS);
  const int jc = valid ? ((jj * F) >> pb.lam2) : 0;
  if constexpr (RC_::CD > 0) {
    const int node = (KIND == RBF) ? jc + 1 : jc;
    const double* src = pb.C.p + pc * pb.C.path_stride + (int64_t)node * pb.dpad;
    for (int c = lane; c < RC_::CD / 2; c += 32) cp_async16(ring_slot + 2 * c, src + 2 * c, valid);
  }
  for (int e = lane; e < P * F; e += 32) {
    const int g = e / F, f = e % F;
    const double* src = hrow0 + g * hand_stride + (valid ? jj * F + f + 1 : 0);
    cp_async8(ring_slot + RC_::CD + e, src, valid && strip > 0);
  }
  cp_async_commit();
}

// Forward kernel.  Template parameters:
//   KIND  LINEAR / RBF / DELTA
//   DP    padded path dimension held in registers per chunk
//   R     fine rows per lane;  FR = fine rows per coarse row inside a lane
//         (= min(2^lam1, R)), so RC = R / FR coarse rows per lane
//   F     fine columns per step (= min(2^lam2, 4))
//   G     lanes per pair (4 or 32); ignored when XW (G = blockDim.x)
//   XW    cross-warp lane groups (one pair per CTA)
// Every group of a warp must share the column path (Gram tiles / one pair).
template <int KIND, int DP, int R, int FR, int F, int G, bool XW>
__global__ void __launch_bounds__(XW ? 512 : 128)
fwd_kernel(Problem pb, double* __restrict__ hand, int64_t hand_stride) {
  constexpr int RC = R / FR;
  constexpr int P = XW ? 1 : 32 / G;
  using Rec = FwdRec<KIND, DP, F, P>;
  using Rg = FwdRing<XW, G>;
  constexpr int REC = Rec::REC;
  constexpr int SLOTS = Rg::SLOTS;
  constexpr int PF = Rg::PF;
  extern __shared__ double smem_fwd[];
  __shared__ double xbuf[XW ? 2 : 1][XW ? 32 : 1][F];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int Grt = XW ? (int)blockDim.x : G;
  const int g = XW ? 0 : lane / G;
  const int u = XW ? (int)threadIdx.x : lane % G;
  double* ring = XW ? smem_fwd : smem_fwd + (size_t)warp * SLOTS * REC;

  const int M1 = pb.M1c << pb.lam1;
  const int M2 = pb.M2c << pb.lam2;
  const int NS = M2 / F;  // steps per strip
  const int H = Grt * R;  // strip height
  const int nstrips = (M1 + H - 1) / H;
  const int last_strip = (M1 - 1) / H;
  const int u_star = ((M1 - 1) % H) / R;
  const int r_star = (M1 - 1) % R;

  const int64_t slot0 = XW ? (int64_t)blockIdx.x : ((int64_t)blockIdx.x * nw + warp) * P;
  const double* hrow0 = hand + slot0 * hand_stride;  // group g's row: + g * hand_stride
  double* __restrict__ hrow = hand + (slot0 + g) * hand_stride;
  const bool issuer = !XW || warp == 0;

  const int64_t item0 = XW ? blockIdx.x : (int64_t)blockIdx.x * nw + warp;
  const int64_t istep = XW ? gridDim.x : (int64_t)gridDim.x * nw;

  for (int64_t item = item0; item < pb.nitems; item += istep) {
    int64_t pr = 0, pc = 0, oidx = 0, pidx = 0;
    const bool valid = resolve_pair(pb, item, P, g, pr, pc, oidx, pidx);
    if (!valid) pidx = 0;
    {
      // the warp's column path (all groups share it; group 0 always resolves)
      int64_t pr0, oi0, pi0;
      resolve_pair(pb, item, P, 0, pr0, pc, oi0, pi0);
      if (!valid) pr = pr0;
    }

    for (int t = u; t <= M2; t += Grt) hrow[t] = 1.0;
    if (XW) __syncthreads(); else __syncwarp();

    for (int strip = 0; strip < nstrips; ++strip) {
      const int rbase = strip * H + u * R;  // 0-based fine row of the lane's first row
      const int i0 = rbase >> pb.lam1;
      RowRegs<KIND, DP, RC> rr;
      if constexpr (KIND != DELTA) load_rows<KIND, DP, RC>(rr, pb, pr, i0, 0);
      double Kl[RC + 1], Kr[RC + 1];  // RBF: K at node columns jc, jc+1 of the pending step
      int jcur = -1;
      if constexpr (KIND == RBF) {
        double y0[DP];
        load_vec<DP>(y0, pb.C.p + pc * pb.C.path_stride);
#pragma unroll
        for (int c = 0; c <= RC; ++c) Kr[c] = exp(-sqdist<DP>(rr.v[c], y0) * pb.inv2s2);
#pragma unroll
        for (int c = 0; c <= RC; ++c) Kl[c] = Kr[c];
      }
      // prologue: PF records in flight
      if (issuer) {
        for (int q = 0; q < PF; ++q)
          fwd_issue<KIND, DP, F, P>(ring + (q & (SLOTS - 1)) * REC, pb, pc, hrow0, hand_stride, q, NS, strip,
                                    lane);
      }

      // coefficients of the next step (software pipeline)
      auto coefs_for = [&](int jj, Coef (&cf)[RC]) {
        const double* rec = ring + (jj & (SLOTS - 1)) * REC;
        const int jc = (jj * F) >> pb.lam2;
        double p[RC];
        if constexpr (KIND == LINEAR) {
          double dy[DP];
#pragma unroll
          for (int k = 0; k < DP; k += 2) {
            const double2 t2 = *reinterpret_cast<const double2*>(rec + k);
            dy[k] = t2.x;
            dy[k + 1] = t2.y;
          }
          if (DP < 32 || pb.nch == 1) {  // d > 32 only ever selects DP = 32
#pragma unroll
            for (int c = 0; c < RC; ++c) {
              // two partial sums halve the dependent FMA chain
              double s0 = rr.v[c][0] * dy[0], s1 = rr.v[c][1] * dy[1];
#pragma unroll
              for (int k = 2; k < DP; k += 2) {
                s0 = fma(rr.v[c][k], dy[k], s0);
                s1 = fma(rr.v[c][k + 1], dy[k + 1], s1);
              }
              p[c] = (s0 + s1) * pb.scale;
            }
          } else {
            // d > 32: chunked dot products (second chunk onwards from L1)
#pragma unroll
            for (int c = 0; c < RC; ++c) p[c] = dot<DP>(rr.v[c], dy);
            for (int ch = 1; ch < pb.nch; ++ch) {
              double dyc[DP], xc[DP];
              load_vec<DP>(dyc, pb.C.p + pc * pb.C.path_stride + (int64_t)jc * pb.dpad + ch * DP);
#pragma unroll
              for (int c = 0; c < RC; ++c) {
                const int i = i0 + c;
                if (i < pb.M1c) {
                  load_vec<DP>(xc, pb.R.p + pr * pb.R.path_stride + (int64_t)i * pb.dpad + ch * DP);
                  p[c] += dot<DP>(xc, dyc);
                }
              }
            }
#pragma unroll
            for (int c = 0; c < RC; ++c) p[c] *= pb.scale;
          }
        } else if constexpr (KIND == RBF) {
          if (jj >= 0 && jc != jcur) {
            double yv[DP];
#pragma unroll
            for (int k = 0; k < DP; k += 2) {
              const double2 t2 = *reinterpret_cast<const double2*>(rec + k);
              yv[k] = t2.x;
              yv[k + 1] = t2.y;
            }
#pragma unroll
            for (int c = 0; c <= RC; ++c) {
              Kl[c] = Kr[c];
              Kr[c] = exp(-sqdist<DP>(rr.v[c], yv) * pb.inv2s2);
            }
            jcur = jc;
          }
#pragma unroll
          for (int c = 0; c < RC; ++c) p[c] = ((Kr[c + 1] - Kl[c + 1]) - (Kr[c] - Kl[c])) * pb.scale;
        } else {  // DELTA: per-row coarse values straight from global
#pragma unroll
          for (int c = 0; c < RC; ++c) {
            const int i = i0 + c;
            p[c] = (i < pb.M1c && jj >= 0 && jj < NS)
                       ? __ldg(pb.delta + pidx * (int64_t)pb.M1c * pb.M2c + (int64_t)i * pb.M2c + jc) *
                             pb.scale
                       : 0.0;
          }
        }
#pragma unroll
        for (int c = 0; c < RC; ++c) cf[c] = coef(p[c]);
      };

      double kl[R];
#pragma unroll
      for (int r = 0; r < R; ++r) kl[r] = 1.0;
      double topc = 1.0;
      double bot[F];
#pragma unroll
      for (int f = 0; f < F; ++f) bot[f] = 1.0;
      Coef cf[RC];
      if (issuer) cp_async_wait<PF - 1>();
      if (XW) __syncthreads(); else __syncwarp();
      coefs_for(-u, cf);

      const int nsteps = NS + Grt - 1;
      for (int tau = 0; tau < nsteps; ++tau) {
        if (issuer) {
          fwd_issue<KIND, DP, F, P>(ring + ((tau + PF) & (SLOTS - 1)) * REC, pb, pc, hrow0,
                                    hand_stride, tau + PF, NS, strip, lane);
          cp_async_wait<PF - 1>();  // records <= tau + 1 landed
        }
        if (XW) __syncthreads(); else __syncwarp();
        const int jj = tau - u;
        const bool active = (jj >= 0) && (jj < NS);
        Coef cfn[RC];
        coefs_for(jj + 1, cfn);  // independent of this step's recurrence

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
        if (u == 0) {
          const double* rec = ring + (jj & (SLOTS - 1)) * REC + Rec::CD + g * F;
#pragma unroll
          for (int f = 0; f < F; ++f) tv[f] = (strip == 0) ? 1.0 : rec[f];
        }
#pragma unroll
        for (int f = 0; f < F; ++f) {
          double up = tv[f];
          double dg = (f == 0) ? topc : tv[f - 1];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double nk = cell(up, kl[r], dg, cf[r / FR]);
            dg = kl[r];
            kl[r] = active ? nk : kl[r];
            up = nk;
          }
          bot[f] = up;
        }
        if (active) {
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
#pragma unroll
        for (int c = 0; c < RC; ++c) cf[c] = cfn[c];
        if constexpr (XW) {
          if (lane == 31) {
#pragma unroll
            for (int f = 0; f < F; ++f) xbuf[tau & 1][warp][f] = bot[f];
          }
        }
      }
      if (issuer) cp_async_wait<0>();
      if (XW) __syncthreads(); else __syncwarp();
    }
  }
}

// Dynamic shared memory of one fwd_kernel CTA (bytes).
template <int KIND, int DP, int F, int G, bool XW>
constexpr int fwd_smem_bytes(int warps) {
  using Rec = FwdRec<KIND, DP, F, XW ? 1 : 32 / G>;
  return (XW ? 1 : warps) * FwdRing<XW, G>::SLOTS * Rec::REC * (int)sizeof(double);
}

}  // namespace sk
