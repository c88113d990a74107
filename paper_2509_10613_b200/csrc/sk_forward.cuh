// sk_forward.cuh -- forward Goursat solve as a register-resident skewed wavefront.
//
// Replaces the reference's CPU march (goursat_strip / goursat_batch /
// goursat_gram, /root/reference/pkg/src/sigcore/_kernels.py:293-338, 399-429).
//
// Mapping (B200-first):
//   * a lane group of G lanes solves one pair; lane u owns R consecutive fine
//     rows of a strip of G*R rows and sweeps the columns left->right, S
//     columns (S*F fine columns) per step, lagging lane u-1 by one step.  The
//     three rotating anti-diagonals of the reference become registers: k_left
//     per owned row, the top-row values from lane u-1 arrive by __shfl_up_sync.
//   * G = 4: 8 pairs per warp sharing the column path (Gram tiles); G = 32: one
//     pair per warp; XW: one pair per CTA, G = blockDim.x lanes, lane 31 ->
//     lane 0 of the next warp through a double-buffered shared-memory slot and
//     one CTA barrier per step (long pairs, BASELINE config 4).
//   * column data (increments dy_j or RBF nodes y_{j+1}) and the strip's
//     handoff row stream through a shared-memory ring filled by cp.async PF
//     steps ahead, so no global latency sits on the recurrence;
//   * the increment product delta (kernel.py:60-77) is never materialised: the
//     lane keeps its rows' increments in registers (pre-scaled by the exact
//     dyadic factor 2^-(lam1+lam2)) and forms <dx_i, dy_j> per coarse cell;
//     dyadic refinement is on the fly (fine cell (s,t) reads coarse
//     (s-1)>>lam1, (t-1)>>lam2, _kernels.py:325);
//   * the strip's bottom row is handed to the next strip through a per-group
//     row in global memory (L2 resident), in place, like the reference's
//     handoff row.
#pragma once
#include "sk_cell.cuh"

namespace sk {

template <int KIND, int DP, int F, int P, typename T = double>
struct FwdRec {
  static constexpr int VEC = 16 / (int)sizeof(T);      // elements per 16-byte copy
  static constexpr int CD = (KIND == DELTA) ? 0 : DP;  // column data elements
  static constexpr int RAW = CD + P * F;               // + handoff values per group
  static constexpr int REC = (RAW + VEC - 1) & ~(VEC - 1);  // 16-byte aligned records
};

// Ring slots (a power of two) for `lanes` lanes in flight: every lane's step
// plus the PF prefetched steps, S column records each.
__host__ __device__ constexpr int ring_slots(int lanes, int S, int PF) {
  return ((lanes + PF + 1) * S) <= 32 ? 32 : ((lanes + PF + 1) * S) <= 64 ? 64
         : ((lanes + PF + 1) * S) <= 128 ? 128 : ((lanes + PF + 1) * S) <= 256 ? 256
         : ((lanes + PF + 1) * S) <= 512 ? 512 : ((lanes + PF + 1) * S) <= 1024 ? 1024 : 2048;
}

// Cross-warp (XW) pairs: lane 0 of warp w runs SK_XW_LAG steps behind lane 31
// of warp w-1 (instead of one), so the cross-warp hops of SK_XW_LAG steps
// travel together and the CTA meets at a barrier once per SK_XW_LAG steps
// (measured at BASELINE config 2: the per-step barrier was the top stall).
// Costs (LAG-1)(W-1) extra skew steps per strip.
#ifndef SK_XW_LAG
#define SK_XW_LAG 4
#endif
// ring records in flight for an XW CTA of `lanes` lanes: every lane's column,
// the extra inter-warp skew, a LAG-step chunk of drift, LAG + PF - 1 prefetched steps
__host__ __device__ constexpr int xw_ring_slots(int lanes, int S, int PF) {
  return ring_slots(lanes + (SK_XW_LAG - 1) * (lanes / 32) + 2 * SK_XW_LAG, S, PF);
}

// the same pipeline for the one-pair-per-warp / Gram-tile RBF instances:
// measured slower (RBF Gram 256 x 256, L = 128: 3.2 -> 4.6 ms), off
#ifndef SK_RBF_PIPE
#define SK_RBF_PIPE 0
#endif
#ifndef SK_XW_PIPE
#define SK_XW_PIPE 1
#endif
#ifndef SK_FWD_PF
#define SK_FWD_PF 2  // measured: 6 slower at C1 (32.3 vs 29.0 us) and on Gram tiles
#endif

template <bool XW, int G, int S>
struct FwdRing {
  // steps in flight.  Short steps (few rows per lane, e.g. BASELINE config 1:
  // 2 rows) finish long before an L2 / HBM round trip, so lane groups keep
  // more steps of column records in flight; XW CTAs add their LAG chunk
  static constexpr int PF = XW ? 2 : SK_FWD_PF;
  static constexpr int NEED = ((XW ? 512 : G) + PF + 1) * S;
  static constexpr int SLOTS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128
                               : NEED <= 256 ? 256 : NEED <= 512 ? 512 : NEED <= 1024 ? 1024
                                                                                      : 2048;
};

// Issue the ring records of columns [col0, col0 + S): column data of coarse
// column jc(col) and the handoff values of every group (strip > 0).  One warp
// issues; a single commit group per step.
template <int KIND, int DP, int F, int P, int S, typename T = double>
__device__ __forceinline__ void fwd_issue(T* ring, int smask, const Problem& pb, int64_t pc,
                                          const T* hrow0, int64_t hand_stride, int col0,
                                          int NC, int strip, int lane) {
  using Rc = FwdRec<KIND, DP, F, P, T>;
  constexpr int VEC = Rc::VEC;
  constexpr int CH = Rc::CD / VEC;  // 16-byte chunks of column data
  const T* cdata = reinterpret_cast<const T*>(pb.C.p);
  for (int e = lane; e < S * CH; e += 32) {
    const int s = e / CH, c = e % CH;
    const int col = col0 + s;
    const bool valid = (col >= 0) && (col < NC);
    const int jc = valid ? ((col * F) >> pb.lam2) : 0;
    const int node = (KIND == RBF) ? jc + 1 : jc;
    const T* src = cdata + pc * pb.C.path_stride + (int64_t)node * pb.dpad + VEC * c;
    cp_async16(ring + ((col & smask) * Rc::REC) + VEC * c, src, valid);
  }
  if (strip > 0) {
    for (int e = lane; e < S * P * F; e += 32) {
      const int s = e / (P * F), q = e % (P * F);
      const int g = q / F, f = q % F;
      const int col = col0 + s;
      const bool valid = (col >= 0) && (col < NC);
      const T* src = hrow0 + g * hand_stride + (valid ? col * F + f + 1 : 0);
      cp_async_elem<T>(ring + ((col & smask) * Rc::REC) + Rc::CD + q, src, valid);
    }
  }
  cp_async_commit();
}

// Forward kernel.  Template parameters:
//   KIND  LINEAR / RBF / DELTA
//   DP    padded path dimension held in registers per chunk
//   R     fine rows per lane;  FR = fine rows per coarse row inside a lane
//         (= min(2^lam1, R)), so RC = R / FR coarse rows per lane
//   F     fine columns per column record (= min(2^lam2, 4))
//   G     lanes per pair (4 or 32); ignored when XW (G = blockDim.x)
//   XW    cross-warp lane groups (one pair per CTA)
//   S     columns per step
//   T     arithmetic type: double (the reference's fp64 arithmetic) or float
//         (the fp32 kernels: LINEAR only, small-correction cell, path data,
//         handoff rows and outputs are float arrays behind the same pointers)
// Every group of a warp must share the column path (Gram tiles / one pair).
//   XWT   XW CTAs: threads at most (256: 255 registers per thread, up to 8
//         warps; 512: 128 registers, 16 warps for the longest pairs)
template <int KIND, int DP, int R, int FR, int F, int G, bool XW, int S, typename T = double,
          int XWT = 512>
__global__ void __launch_bounds__(XW ? XWT : 128)
fwd_kernel(Problem pb, double* __restrict__ hand_, int64_t hand_stride) {
  constexpr int RC = R / FR;
  constexpr int P = XW ? 1 : 32 / G;
  constexpr int SF = S * F;
  using Rec = FwdRec<KIND, DP, F, P, T>;
  using Rg = FwdRing<XW, G, S>;
  using Cf = CoefOf<T>;
  constexpr int REC = Rec::REC;
  constexpr int SLOTS = Rg::SLOTS;  // per warp (non-XW); XW: sized by the CTA's lanes
  constexpr int PF = Rg::PF;
  static_assert(sizeof(T) == 8 || KIND == LINEAR, "fp32 kernels: linear static kernel only");
  extern __shared__ double smem_fwd_raw[];
  T* smem_fwd = reinterpret_cast<T*>(smem_fwd_raw);
  T* hand = reinterpret_cast<T*>(hand_);
  constexpr int XK = XW ? SK_XW_LAG : 1;  // steps per cross-warp chunk
  __shared__ T xbuf[XW ? 2 * XK : 1][XW ? 16 : 1][SF];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int Grt = XW ? (int)blockDim.x : G;
  const int g = XW ? 0 : lane / G;
  const int u = XW ? (int)threadIdx.x : lane % G;
  T* ring = XW ? smem_fwd : smem_fwd + (size_t)warp * SLOTS * REC;
  const int smask = (XW ? xw_ring_slots((int)blockDim.x, S, PF) : SLOTS) - 1;

  const int M1 = pb.M1c << pb.lam1;
  const int M2 = pb.M2c << pb.lam2;
  const int NC = M2 / F;                 // column records per strip row
  const int NSTEP = (NC + S - 1) / S;    // steps per strip
  const int H = Grt * R;                 // strip height
  const int nstrips = (M1 + H - 1) / H;
  const int last_strip = (M1 - 1) / H;
  const int u_star = ((M1 - 1) % H) / R;
  const int r_star = (M1 - 1) % R;
  const int s_star = (NC - 1) % S;       // sub-step of the last column

  const int64_t slot0 = XW ? (int64_t)blockIdx.x : ((int64_t)blockIdx.x * nw + warp) * P;
  const T* hrow0 = hand + slot0 * hand_stride;  // group g's row: + g * hand_stride
  T* __restrict__ hrow = hand + (slot0 + g) * hand_stride;
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
    T outv = 0;

    for (int t = u; t <= M2; t += Grt) hrow[t] = T(1);
    if (XW) __syncthreads(); else __syncwarp();

    for (int strip = 0; strip < nstrips; ++strip) {
      const int rbase = strip * H + u * R;  // 0-based fine row of the lane's first row
      const int i0 = rbase >> pb.lam1;
      RowRegs<KIND, DP, RC, T> rr;
      if constexpr (KIND != DELTA) load_rows<KIND, DP, RC, T>(rr, pb, pr, i0, 0);
      double Kl[RC + 1], Kr[RC + 1];  // RBF: K at node columns jc, jc+1
      int jcur = -1;
      if constexpr (KIND == RBF) {
        double y0[DP];
        load_vec<DP>(y0, pb.C.p + pc * pb.C.path_stride);
#pragma unroll
        for (int c = 0; c <= RC; ++c) Kr[c] = exp(-sqdist<DP>(rr.v[c], y0) * pb.inv2s2);
#pragma unroll
        for (int c = 0; c <= RC; ++c) Kl[c] = Kr[c];
      }
      // XW: records of LAG + PF - 1 steps ahead, so a whole LAG-step chunk has
      // landed at the chunk's barrier with PF groups still in flight
      constexpr int LOOK = XW ? XK + PF - 1 : PF;
      if (issuer) {
        for (int q = 0; q < LOOK; ++q)
          fwd_issue<KIND, DP, F, P, S, T>(ring, smask, pb, pc, hrow0, hand_stride, q * S, NC,
                                          strip, lane);
      }

      // coefficients of the S columns of step js (reads the ring; no recurrence)
      auto col_coefs = [&](int col, Cf (&cfo)[RC]) {
        {
          const T* rec = ring + (col & smask) * REC;
          T p[RC];
          if constexpr (KIND == LINEAR) {
            T dy[DP];
            if constexpr (sizeof(T) == 8) {
#pragma unroll
              for (int k = 0; k < DP; k += 2) {
                const double2 t2 = *reinterpret_cast<const double2*>(rec + k);
                dy[k] = t2.x;
                dy[k + 1] = t2.y;
              }
            } else {
#pragma unroll
              for (int k = 0; k < DP; k += 4) {
                const float4 t4 = *reinterpret_cast<const float4*>(rec + k);
                dy[k] = t4.x;
                dy[k + 1] = t4.y;
                dy[k + 2] = t4.z;
                dy[k + 3] = t4.w;
              }
            }
#pragma unroll
            for (int c = 0; c < RC; ++c) p[c] = dot<DP>(rr.v[c], dy);
            if (DP == 32 && pb.nch > 1 && col >= 0 && col < NC) {  // d > 32: further chunks
              const int jc = (col * F) >> pb.lam2;
              const T* cdata = reinterpret_cast<const T*>(pb.C.p);
              const T* rdata = reinterpret_cast<const T*>(pb.R.p);
              for (int ch = 1; ch < pb.nch; ++ch) {
                T dyc[DP], xc[DP];
                load_vec<DP>(dyc, cdata + pc * pb.C.path_stride + (int64_t)jc * pb.dpad + ch * DP);
#pragma unroll
                for (int c = 0; c < RC; ++c) {
                  const int i = i0 + c;
                  if (i < pb.M1c) {
                    load_vec<DP>(xc, rdata + pr * pb.R.path_stride + (int64_t)i * pb.dpad + ch * DP);
                    p[c] += dot<DP>(xc, dyc);
                  }
                }
              }
            }
            if (pb.pscale != 1.0) {
#pragma unroll
              for (int c = 0; c < RC; ++c) p[c] *= (T)pb.pscale;
            }
          } else if constexpr (KIND == RBF) {
            const int jc = (col * F) >> pb.lam2;
            if (col >= 0 && col < NC && jc != jcur) {
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
            const int jc = (col * F) >> pb.lam2;
#pragma unroll
            for (int c = 0; c < RC; ++c) {
              const int i = i0 + c;
              p[c] = (i < pb.M1c && col >= 0 && col < NC)
                         ? __ldg(pb.delta + pidx * (int64_t)pb.M1c * pb.M2c + (int64_t)i * pb.M2c +
                                 jc) * pb.scale
                         : 0.0;
            }
          }
#pragma unroll
          for (int c = 0; c < RC; ++c) cfo[c] = coef(p[c]);
        }
      };
      auto step_coefs = [&](int js, Cf (&cfo)[S][RC]) {
#pragma unroll
        for (int s = 0; s < S; ++s) col_coefs(js * S + s, cfo[s]);
      };

      T kl[R];
#pragma unroll
      for (int r = 0; r < R; ++r) kl[r] = T(1);
      T topc = T(1);
      T bot[SF];
#pragma unroll
      for (int q = 0; q < SF; ++q) bot[q] = T(1);
      // wide paths (DP >= 16) pipeline the next step's coefficients behind the
      // recurrence; narrow ones keep the registers for S columns per step
      // (short paths: latency; XW RBF with the 255-register instance: the next
      // step's exps under this step's recurrence instead of on the lane chain,
      // measured at BASELINE config 2: 0.46 -> 0.40 ms; the linear XW forward
      // is faster without it, 0.26 vs 0.30 ms)
      constexpr bool PIPE = XW ? (KIND == RBF && XWT <= 256 && SK_XW_PIPE != 0)
                               : (DP >= 16 || (G == 32 && R <= 2) || (KIND == RBF && SK_RBF_PIPE));
      const int lagw = XW ? (XK - 1) * warp : 0;  // extra skew of this warp (XW)
      Cf cf[S][RC];
      if constexpr (PIPE) {
        if constexpr (XW) {
          if (issuer) cp_async_wait<LOOK - 1>();  // step 0 landed
          __syncthreads();
        } else {
          if (issuer) cp_async_wait<PF - 1>();  // step 0 landed
          __syncwarp();
        }
        step_coefs(-u - lagw, cf);
      }

      const int nsteps = NSTEP + Grt - 1 + (XW ? (XK - 1) * (nw - 1) : 0);
      for (int tau = 0; tau < nsteps; ++tau) {
        if constexpr (XW) {
          // once per chunk: steps tau .. tau + XK - 1 landed, hops of the last
          // chunk visible, the chunk before it consumed
          if (issuer) {
            fwd_issue<KIND, DP, F, P, S, T>(ring, smask, pb, pc, hrow0, hand_stride,
                                            (tau + LOOK) * S, NC, strip, lane);
            if (tau % XK == 0) {
              if constexpr (PIPE) cp_async_wait<PF - 1>();  // ... and step tau + XK (next coefs)
              else cp_async_wait<PF>();
            }
          }
          if (tau % XK == 0) __syncthreads();
        } else {
          if (issuer) {
            fwd_issue<KIND, DP, F, P, S, T>(ring, smask, pb, pc, hrow0, hand_stride,
                                            (tau + PF) * S, NC, strip, lane);
            if constexpr (PIPE) cp_async_wait<PF - 1>();  // steps <= tau + 1 landed
            else cp_async_wait<PF>();                     // step tau landed
          }
          __syncwarp();
        }
        const int js = tau - u - lagw;
        const bool active = (js >= 0) && (js < NSTEP);
        // software pipeline: next step's coefficients overlap this step's recurrence
        Cf cfn[PIPE ? S : 1][RC];
        if constexpr (PIPE) step_coefs(js + 1, cfn);

        T tv[SF];
        if constexpr (XW) {
#pragma unroll
          for (int q = 0; q < SF; ++q) tv[q] = __shfl_up_sync(0xffffffffu, bot[q], 1);
          if (lane == 0 && warp > 0) {
#pragma unroll
            for (int q = 0; q < SF; ++q) tv[q] = xbuf[(tau + XK) % (2 * XK)][warp - 1][q];
          }
        } else {
#pragma unroll
          for (int q = 0; q < SF; ++q) tv[q] = __shfl_up_sync(0xffffffffu, bot[q], 1, G);
        }
        if (active) {
          const int col0 = js * S;
          if (u == 0) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const T* rec = ring + ((col0 + s) & smask) * REC + Rec::CD + g * F;
#pragma unroll
              for (int f = 0; f < F; ++f) tv[s * F + f] = (strip == 0) ? T(1) : rec[f];
            }
          }
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const int col = col0 + s;
            if constexpr (!PIPE) col_coefs(col, cf[s]);
#pragma unroll
            for (int f = 0; f < F; ++f) {
              const int q = s * F + f;
              T up = tv[q];
              T dg = (q == 0) ? topc : tv[q - 1];
#pragma unroll
              for (int r = 0; r < R; ++r) {
                const T nk = cell(up, kl[r], dg, cf[s][r / FR]);
                dg = kl[r];
                kl[r] = nk;
                up = nk;
              }
              bot[q] = up;
            }
            if (s == s_star && col == NC - 1) {
#pragma unroll
              for (int r = 0; r < R; ++r)
                if (r == r_star) outv = kl[r];
            }
          }
          topc = tv[SF - 1];
          if (u == Grt - 1) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
              if (col0 + s < NC) {
#pragma unroll
                for (int f = 0; f < F; ++f) hrow[(col0 + s) * F + f + 1] = bot[s * F + f];
              }
            }
          }
        }
        if constexpr (PIPE) {
#pragma unroll
          for (int s = 0; s < S; ++s)
#pragma unroll
            for (int c = 0; c < RC; ++c) cf[s][c] = cfn[s][(PIPE ? c : 0)];
        }
        if constexpr (XW) {
          if (lane == 31) {
#pragma unroll
            for (int q = 0; q < SF; ++q) xbuf[tau % (2 * XK)][warp][q] = bot[q];
          }
        }
      }
      if (issuer) cp_async_wait<0>();
      if (XW) __syncthreads(); else __syncwarp();
    }
    if (u == u_star && valid) reinterpret_cast<T*>(pb.out)[oidx] = outv;
  }
}

// Dynamic shared memory of one fwd_kernel CTA (bytes).
template <int KIND, int DP, int F, int G, bool XW, int S, typename T = double>
constexpr int fwd_smem_bytes(int warps) {
  using Rec = FwdRec<KIND, DP, F, XW ? 1 : 32 / G, T>;
  return XW ? xw_ring_slots(32 * warps, S, FwdRing<XW, G, S>::PF) * Rec::REC * (int)sizeof(T)
            : warps * FwdRing<XW, G, S>::SLOTS * Rec::REC * (int)sizeof(T);
}

}  // namespace sk
