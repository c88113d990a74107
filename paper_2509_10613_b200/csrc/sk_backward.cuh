// sk_backward.cuh -- exact backward (paper Alg. 4) as a reverse wavefront.
//
// Replaces the reference's goursat_grid + goursat_backward + kernel_backward
// (/root/reference/pkg/src/sigcore/_kernels.py:381-396, 436-466;
//  kernel_grad.py:27-98).  The adjoint recursion is the reference's
//    d1[s,t] = d1[s+1,t] A(p[s+1,t]) + d1[s,t+1] A(p[s,t+1]) - d1[s+1,t+1] B(p[s+1,t+1])
//    d2[coarse(s,t)] += d1[s,t] * ((k[s,t-1] + k[s-1,t]) (1/2 + p/6) + k[s-1,t-1] p/6) * scale
// written in "push" form: every cell forwards a = A*lambda to its upper and left
// neighbours and -b = -B*lambda to its upper-left one.
//
// B200 mapping:
//   * one warp per pair, lane u owns R fine rows of a 32R-row strip;
//   * phase A: the forward wavefront of sk_forward.cuh, which additionally
//     saves every lane's bottom row (row checkpoint, coalesced "diagonal"
//     layout [strip][step][f][lane]) and every lane's R values at staggered
//     block boundaries (column checkpoint);
//   * phase B: strips bottom-up; per block of CB steps every lane recomputes its
//     R x CB*F forward values from its own checkpoints into shared memory (no
//     inter-lane dependency, so all lanes do it at the same time), then sweeps
//     the block right-to-left one step behind lane u+1, receiving lane u+1's
//     top-row messages by __shfl_down_sync;
//   * the coarse adjoint dF/d(delta) is mapped to path space on the fly
//     (FUSED: gx = D dy in registers, gy = D^T dx accumulated down the warp as a
//     shuffle chain) or through a per-pair coarse buffer (DBUF: RBF and large
//     dyadic orders), then telescoped to point gradients (kernel_grad.py:51-60).
//   * nothing proportional to the fine grid is stored per pair beyond the
//     checkpoints (1/R + 1/(CB*F) of the grid).
#pragma once
#include "sk_forward.cuh"

namespace sk {

enum MapMode : int { FUSED = 0, DBUF = 1 };


__device__ __forceinline__ void grad_add(double* p, double v, bool atomic) {
  if (atomic) atomicAdd(p, v);
  else *p += v;
}

// Per-warp shared-memory block store, lane-minor ([idx][32]) for conflict-free access.
template <int R, int RC, int F, int CB>
struct BlockSmem {
  static constexpr int NK = CB * F * R;     // recomputed k values
  static constexpr int NP = CB * RC;        // coarse p values
  static constexpr int NT = CB * F + 1;     // top row (incl. left node)
  static constexpr int NL = R;              // left column
  static constexpr int TOTAL = NK + NP + NT + NL;
};

template <int KIND, int DP, int R, int FR, int F, int CB, int MAP>
__global__ void __launch_bounds__(128)
bwd_kernel(Problem pb, BwdArgs ba) {
  constexpr int RC = R / FR;
  using SM = BlockSmem<R, RC, F, CB>;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  double* sK = smem + (size_t)warp * SM::TOTAL * 32;
  double* sP = sK + SM::NK * 32;
  double* sT = sP + SM::NP * 32;
  double* sL = sT + SM::NT * 32;
#define SK_KB(kap, f, r) sK[(((kap) * F + (f)) * R + (r)) * 32 + lane]
#define SK_PB(kap, c) sP[((kap) * RC + (c)) * 32 + lane]
#define SK_TB(q) sT[(q) * 32 + lane]
#define SK_LB(r) sL[(r) * 32 + lane]

  const int u = lane;
  const int M1 = pb.M1c << pb.lam1;
  const int M2 = pb.M2c << pb.lam2;
  const int NS = M2 / F;          // steps per strip
  const int NT = NS + 31;         // skewed steps per strip
  const int NB = (NT + CB - 1) / CB;
  const int H = 32 * R;
  const int nstrips = (M1 + H - 1) / H;
  const int last_strip = (M1 - 1) / H;
  const int u_star = ((M1 - 1) % H) / R;
  const int r_star = (M1 - 1) % R;
  const int dR = ba.d;

  const int64_t slot = (int64_t)blockIdx.x * nw + warp;
  double* __restrict__ rowck = ba.rowck + slot * ba.rowck_stride;
  double* __restrict__ colck = ba.colck + slot * ba.colck_stride;
  double* __restrict__ hrow = ba.hand + slot * ba.row_stride;
  double* __restrict__ arow = ba.adj + slot * ba.row_stride;
  double* __restrict__ dbuf = (MAP == DBUF) ? ba.dbuf + slot * ba.dbuf_stride : nullptr;
#define SK_ROWCK(strip, tau, f, ln) rowck[(((int64_t)(strip) * NT + (tau)) * F + (f)) * 32 + (ln)]
#define SK_COLCK(strip, blk, r) colck[(((int64_t)(strip) * NB + (blk)) * R + (r)) * 32 + lane]

  for (int64_t item = slot; item < pb.nitems; item += (int64_t)gridDim.x * nw) {
    // ---------------------------------------------------------- resolve pair
    int64_t pr = 0, pc = 0, oidx = 0, pidx = 0;
    const bool valid = resolve_pair(pb, item, 1, 0, pr, pc, oidx, pidx);
    if (!valid) continue;  // warp-uniform
    double wcot = 1.0;
    if (pb.mode == BATCH) {
      if (ba.cot) wcot = ba.cot[item];
    } else {
      int a = pb.r0 + (int)(pidx / pb.n2), b = (int)(pidx % pb.n2);
      wcot = ba.cot[(int64_t)a * pb.n2 + b];
      if (pb.mode == GRAM_SYM && a != b) wcot += ba.cot[(int64_t)b * pb.n2 + a];
    }

    // ------------------------------------------- phase A: forward + checkpoints
    for (int t = u; t <= M2; t += 32) hrow[t] = 1.0;
    __syncwarp();
    double kval = 0.0;
    for (int strip = 0; strip < nstrips; ++strip) {
      const int rbase = strip * H + u * R;
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
      for (int tau = 0; tau < NT; ++tau) {
        if (tau % CB == 0) {
#pragma unroll
          for (int r = 0; r < R; ++r) SK_COLCK(strip, tau / CB, r) = kl[r];
        }
        const int jj = tau - u;
        const bool active = (jj >= 0) && (jj < NS);
        double tv[F];
#pragma unroll
        for (int f = 0; f < F; ++f) tv[f] = __shfl_up_sync(0xffffffffu, bot[f], 1);
        if (u == 0 && active) {
#pragma unroll
          for (int f = 0; f < F; ++f) tv[f] = (strip == 0) ? 1.0 : hrow[jj * F + f + 1];
        }
        if (active) {
          const int jc = (jj * F) >> pb.lam2;
          double p[RC];
          coarse_p<KIND, DP, RC>(p, rr, cs, pb, pr, pc, pidx, i0, jc);
          if constexpr (KIND == LINEAR) {
            if (pb.pscale != 1.0) {
#pragma unroll
              for (int c = 0; c < RC; ++c) p[c] *= pb.pscale;
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
            SK_ROWCK(strip, tau, f, lane) = up;
          }
          topc = tv[F - 1];
          if (u == 31) {
#pragma unroll
            for (int f = 0; f < F; ++f) hrow[jj * F + f + 1] = bot[f];
          }
          if (strip == last_strip && u == u_star && jj == NS - 1) {
            double v = kl[0];
#pragma unroll
            for (int r = 1; r < R; ++r)
              if (r == r_star) v = kl[r];
            kval = v;
          }
        }
      }
      __syncwarp();
    }
    if (ba.values && u == u_star) ba.values[oidx] = kval;

    // ------------------------------------------------ phase B: reverse sweep
    for (int t = u; t <= M2; t += 32) arow[t] = 0.0;
    if constexpr (MAP == DBUF) {
      for (int64_t e = u; e < (int64_t)pb.M1c * pb.M2c; e += 32) dbuf[e] = 0.0;
    }
    // increment-gradient scratch of this pair: rows [M1c][DP], cols [M2c][DP]
    double* __restrict__ gxs = ba.gscr + slot * ba.gscr_stride;
    double* __restrict__ gcs = gxs + (int64_t)pb.M1c * DP;
    if constexpr (MAP == FUSED) {
      for (int64_t e = u; e < (int64_t)(pb.M1c + pb.M2c) * DP; e += 32) gxs[e] = 0.0;
    }
    __syncwarp();
    double* __restrict__ gR = ba.gradR + pr * ba.gR_path;
    double* __restrict__ gC = ba.gradC + pc * ba.gC_path;
    const bool atomic = ba.atomic != 0;

    for (int strip = nstrips - 1; strip >= 0; --strip) {
      const int rbase = strip * H + u * R;
      const int i0 = rbase >> pb.lam1;
      RowRegs<KIND, DP, RC> rr;
      if constexpr (KIND != DELTA) load_rows<KIND, DP, RC>(rr, pb, pr, i0, 0);
      ColState<KIND, DP, RC> cs;
      cs.have = -2;
      double aR[R], bR[R];
#pragma unroll
      for (int r = 0; r < R; ++r) { aR[r] = 0.0; bR[r] = 0.0; }
      double sendm[F];
#pragma unroll
      for (int f = 0; f < F; ++f) sendm[f] = 0.0;
      double gxr[(MAP == FUSED) ? RC : 1][DP];
      double gys[DP];
#pragma unroll
      for (int k = 0; k < DP; ++k) {
        gys[k] = 0.0;
#pragma unroll
        for (int c = 0; c < ((MAP == FUSED) ? RC : 1); ++c) gxr[c][k] = 0.0;
      }

      for (int blk = NB - 1; blk >= 0; --blk) {
        const int jj0 = blk * CB - u;  // lane's first step in this block
        // ---- recompute the block's forward values into shared memory
        {
          double kl[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            kl[r] = SK_COLCK(strip, blk, r);
            SK_LB(r) = kl[r];
          }
          // top row: node columns t = jj0*F + q, q = 0..CB*F
#pragma unroll
          for (int q = 0; q <= CB * F; ++q) {
            const int t = jj0 * F + q;
            double v;
            if (t <= 0 || (strip == 0 && u == 0)) {
              v = 1.0;
            } else if (t > M2) {
              v = 0.0;  // dead columns: keep values finite
            } else {
              const int js = (t - 1) / F, fs = (t - 1) % F;
              v = (u > 0) ? SK_ROWCK(strip, js + u - 1, fs, u - 1)
                          : SK_ROWCK(strip - 1, js + 31, fs, 31);
            }
            SK_TB(q) = v;
          }
          double topc = SK_TB(0);
#pragma unroll
          for (int kap = 0; kap < CB; ++kap) {
            const int jj = jj0 + kap;
            const bool colv = (jj >= 0) && (jj < NS);
            double p[RC];
            if (colv) {
              const int jc = (jj * F) >> pb.lam2;
              coarse_p<KIND, DP, RC>(p, rr, cs, pb, pr, pc, pidx, i0, jc);
              if constexpr (KIND == LINEAR) {
                if (pb.pscale != 1.0) {
#pragma unroll
                  for (int c = 0; c < RC; ++c) p[c] *= pb.pscale;
                }
              }
            } else {
#pragma unroll
              for (int c = 0; c < RC; ++c) p[c] = 0.0;
            }
            Coef cf[RC];
#pragma unroll
            for (int c = 0; c < RC; ++c) {
              SK_PB(kap, c) = p[c];
              cf[c] = coef(p[c]);
            }
#pragma unroll
            for (int f = 0; f < F; ++f) {
              double up = SK_TB(kap * F + f + 1);
              double dg = (f == 0) ? topc : SK_TB(kap * F + f);
#pragma unroll
              for (int r = 0; r < R; ++r) {
                const double nk = cell(up, kl[r], dg, cf[r / FR]);
                dg = kl[r];
                kl[r] = nk;
                up = nk;
                SK_KB(kap, f, r) = nk;
              }
            }
            topc = SK_TB(kap * F + F);
          }
        }
        // ---- reverse sweep over the block, one step per kap
#pragma unroll 1
        for (int kap = CB - 1; kap >= 0; --kap) {
          const int jj = jj0 + kap;
          const bool colv = (jj >= 0) && (jj < NS);
          double recv[F];
#pragma unroll
          for (int f = 0; f < F; ++f) recv[f] = __shfl_down_sync(0xffffffffu, sendm[f], 1);
          double grecv[DP];
          if constexpr (MAP == FUSED) {
#pragma unroll
            for (int k = 0; k < DP; ++k) grecv[k] = __shfl_down_sync(0xffffffffu, gys[k], 1);
          }
          if (u == 31) {
#pragma unroll
            for (int f = 0; f < F; ++f) recv[f] = colv ? arow[jj * F + f + 1] : 0.0;
#pragma unroll
            for (int k = 0; k < DP; ++k) grecv[k] = 0.0;
          }
          double Dp[RC];
#pragma unroll
          for (int c = 0; c < RC; ++c) Dp[c] = 0.0;
          double pk[RC];
          Coef cf[RC];
#pragma unroll
          for (int c = 0; c < RC; ++c) {
            pk[c] = SK_PB(kap, c);
            cf[c] = coef(pk[c]);
          }
#pragma unroll
          for (int f = F - 1; f >= 0; --f) {
            const int t = jj * F + f + 1;
            double m = recv[f];
#pragma unroll
            for (int r = R - 1; r >= 0; --r) {
              const int s = rbase + r + 1;
              const bool live = colv && (s <= M1);
              double lam = aR[r] + m;
              if (s == M1 && t == M2) lam += wcot;
              lam = live ? lam : 0.0;
              const int c = r / FR;
              const double a = cf[c].A * lam;
              const double b = cf[c].B * lam;
              // forward values around the cell (s,t): left, up, up-left
              const double kL = (f > 0) ? SK_KB(kap, f - 1, r)
                                        : (kap > 0 ? SK_KB(kap - 1, F - 1, r) : SK_LB(r));
              const double kU = (r > 0) ? SK_KB(kap, f, r - 1) : SK_TB(kap * F + f + 1);
              const double kD = (r > 0) ? ((f > 0) ? SK_KB(kap, f - 1, r - 1)
                                                   : (kap > 0 ? SK_KB(kap - 1, F - 1, r - 1)
                                                              : SK_LB(r - 1)))
                                        : SK_TB(kap * F + f);
              const double p6 = pk[c] * (1.0 / 6.0);
              const double wv = fma(kL + kU, 0.5 + p6, kD * p6);
              if (live) Dp[c] = fma(lam, wv, Dp[c]);
              m = a - bR[r];
              aR[r] = a;
              bR[r] = b;
            }
            sendm[f] = m;
          }
          if (u == 0 && colv) {
#pragma unroll
            for (int f = 0; f < F; ++f) arow[jj * F + f + 1] = sendm[f];
          }
          const int jc = colv ? ((jj * F) >> pb.lam2) : 0;
#pragma unroll
          for (int c = 0; c < RC; ++c) Dp[c] *= pb.scale;
          if constexpr (MAP == FUSED) {
            // gx_i += D_ij dy_j (row-local);  gy_j += D_ij dx_i (down the warp)
            double dy[DP];
            if (colv) {
              load_vec<DP>(dy, pb.C.p + pc * pb.C.path_stride + (int64_t)jc * pb.dpad);
            } else {
#pragma unroll
              for (int k = 0; k < DP; ++k) dy[k] = 0.0;
            }
#pragma unroll
            for (int k = 0; k < DP; ++k) {
              double g = grecv[k];
#pragma unroll
              for (int c = 0; c < RC; ++c) {
                gxr[c][k] = fma(Dp[c], dy[k], gxr[c][k]);
                g = fma(Dp[c], rr.v[c][k], g);
              }
              gys[k] = g;
            }
            if (u == 0 && colv) {
              // lane 0 holds the strip's column sum: accumulate dF/d(dy_j)
              double2* q = reinterpret_cast<double2*>(gcs + (int64_t)jc * DP);
#pragma unroll
              for (int k = 0; k < DP / 2; ++k) {
                double2 v = q[k];
                v.x += gys[2 * k];
                v.y += gys[2 * k + 1];
                q[k] = v;
              }
            }
          } else {
            // coarse adjoint buffer; lanes sharing a coarse cell write in
            // a fixed order (lane u+1 one step before lane u)
            if (colv) {
#pragma unroll
              for (int c = 0; c < RC; ++c) {
                const int i = i0 + c;
                if (i < pb.M1c) dbuf[(int64_t)i * pb.M2c + jc] += Dp[c];
              }
            }
            __syncwarp();
          }
        }
      }
      if constexpr (MAP == FUSED) {
        // row-side dF/d(dx_i) into the pair's scratch.  A coarse row owned by
        // one lane is stored once; when 2^lam1 > R a coarse row spans lanes
        // (and possibly strips) and the lanes add in a fixed order.
        if (ba.rows_exclusive) {
#pragma unroll
          for (int c = 0; c < RC; ++c) {
            const int i = i0 + c;
            if (i < pb.M1c) {
              double2* q = reinterpret_cast<double2*>(gxs + (int64_t)i * DP);
#pragma unroll
              for (int k = 0; k < DP / 2; ++k) q[k] = make_double2(gxr[c][2 * k], gxr[c][2 * k + 1]);
            }
          }
        } else {
          for (int ln = 31; ln >= 0; --ln) {
            if (u == ln) {
#pragma unroll
              for (int c = 0; c < RC; ++c) {
                const int i = i0 + c;
                if (i < pb.M1c) {
#pragma unroll
                  for (int k = 0; k < DP; ++k) gxs[(int64_t)i * DP + k] += gxr[c][k];
                }
              }
            }
            __syncwarp();
          }
        }
      }
      __syncwarp();
    }

    if constexpr (MAP == FUSED) {
      // telescope increment gradients to point gradients (kernel_grad.py:55-60)
      // and flush once per pair, coalesced across the warp
      __syncwarp();
      for (int64_t e = u; e < (int64_t)(pb.M1c + 1) * dR; e += 32) {
        const int p = (int)(e / dR), k = (int)(e % dR);
        double v = 0.0;
        if (p >= 1) v += gxs[(int64_t)(p - 1) * DP + k];
        if (p < pb.M1c) v -= gxs[(int64_t)p * DP + k];
        grad_add(gR + e, v, atomic);
      }
      for (int64_t e = u; e < (int64_t)(pb.M2c + 1) * dR; e += 32) {
        const int p = (int)(e / dR), k = (int)(e % dR);
        double v = 0.0;
        if (p >= 1) v += gcs[(int64_t)(p - 1) * DP + k];
        if (p < pb.M2c) v -= gcs[(int64_t)p * DP + k];
        grad_add(gC + e, v, atomic);
      }
      __syncwarp();
    }

    if constexpr (MAP == DBUF) {
      __syncwarp();
      const double* D = dbuf;
      if constexpr (KIND == LINEAR) {
        // gx_i = sum_j D_ij dy_j, gy_j = sum_i D_ij dx_i, then telescope
        const double* dxp = pb.R.p + pr * pb.R.path_stride;
        const double* dyp = pb.C.p + pc * pb.C.path_stride;
        // serialised telescoping (deterministic): one lane at a time
        for (int ln = 0; ln < 32; ++ln) {
          if (u == ln) {
            for (int i = u; i < pb.M1c; i += 32) {
              for (int k = 0; k < dR; ++k) {
                double g = 0.0;
                for (int j = 0; j < pb.M2c; ++j)
                  g = fma(D[(int64_t)i * pb.M2c + j], dyp[(int64_t)j * pb.dpad + k], g);
                grad_add(gR + (int64_t)i * dR + k, -g, atomic);
                grad_add(gR + (int64_t)(i + 1) * dR + k, g, atomic);
              }
            }
          }
          __syncwarp();
        }
        for (int ln = 0; ln < 32; ++ln) {
          if (u == ln) {
            for (int j = u; j < pb.M2c; j += 32) {
              for (int k = 0; k < dR; ++k) {
                double g = 0.0;
                for (int i = 0; i < pb.M1c; ++i)
                  g = fma(D[(int64_t)i * pb.M2c + j], dxp[(int64_t)i * pb.dpad + k], g);
                grad_add(gC + (int64_t)j * dR + k, -g, atomic);
                grad_add(gC + (int64_t)(j + 1) * dR + k, g, atomic);
              }
            }
          }
          __syncwarp();
        }
      } else if constexpr (KIND == RBF) {
        // node adjoint G_ij = D[i-1,j-1] - D[i-1,j] - D[i,j-1] + D[i,j] (zero padded);
        // dF/dx_i = sum_j G_ij K_ij (y_j - x_i)/sigma^2,  dF/dy_j = -sum_i (same)
        const double* xp = pb.R.p + pr * pb.R.path_stride;
        const double* yp = pb.C.p + pc * pb.C.path_stride;
        const int L1n = pb.M1c + 1, L2n = pb.M2c + 1;
        auto Dat = [&](int i, int j) -> double {
          return (i >= 0 && j >= 0 && i < pb.M1c && j < pb.M2c) ? D[(int64_t)i * pb.M2c + j] : 0.0;
        };
        for (int i = u; i < L1n; i += 32) {
          for (int k = 0; k < dR; ++k) {
            double acc = 0.0;
            for (int j = 0; j < L2n; ++j) {
              const double G = Dat(i - 1, j - 1) - Dat(i - 1, j) - Dat(i, j - 1) + Dat(i, j);
              if (G == 0.0) continue;
              double s2 = 0.0;
              for (int kk = 0; kk < dR; ++kk) {
                const double t = xp[(int64_t)i * pb.dpad + kk] - yp[(int64_t)j * pb.dpad + kk];
                s2 = fma(t, t, s2);
              }
              const double K = exp(-s2 * pb.inv2s2);
              acc = fma(G * K * pb.invs2, yp[(int64_t)j * pb.dpad + k] - xp[(int64_t)i * pb.dpad + k], acc);
            }
            grad_add(gR + (int64_t)i * dR + k, acc, atomic);
          }
        }
        for (int j = u; j < L2n; j += 32) {
          for (int k = 0; k < dR; ++k) {
            double acc = 0.0;
            for (int i = 0; i < L1n; ++i) {
              const double G = Dat(i - 1, j - 1) - Dat(i - 1, j) - Dat(i, j - 1) + Dat(i, j);
              if (G == 0.0) continue;
              double s2 = 0.0;
              for (int kk = 0; kk < dR; ++kk) {
                const double t = xp[(int64_t)i * pb.dpad + kk] - yp[(int64_t)j * pb.dpad + kk];
                s2 = fma(t, t, s2);
              }
              const double K = exp(-s2 * pb.inv2s2);
              acc = fma(G * K * pb.invs2, xp[(int64_t)i * pb.dpad + k] - yp[(int64_t)j * pb.dpad + k], acc);
            }
            grad_add(gC + (int64_t)j * dR + k, acc, atomic);
          }
        }
      }
      __syncwarp();
    }
  }
#undef SK_KB
#undef SK_PB
#undef SK_TB
#undef SK_LB
#undef SK_ROWCK
#undef SK_COLCK
}

}  // namespace sk
