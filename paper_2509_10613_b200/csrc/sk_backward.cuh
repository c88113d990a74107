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
//   * one warp per pair, lane u owns R fine rows of a 32R-row strip; a "step"
//     is S columns (S*F fine columns) and lane u runs one step behind lane u-1;
//   * phase A: the forward wavefront (as sk_forward.cuh), which additionally
//     saves every lane's bottom row (row checkpoint, coalesced "diagonal"
//     layout [strip][step + lane][fine column][lane]) and every lane's R values
//     at staggered block boundaries (column checkpoint, [strip][blk][r][lane]);
//   * phase B: strips bottom-up; per block of CB steps every lane recomputes
//     its R x CB*S*F forward values from its own checkpoints into shared memory
//     (no inter-lane dependency, so all lanes do it at the same time), then
//     sweeps the block right-to-left one step behind lane u+1, receiving lane
//     u+1's top-row messages by __shfl_down_sync;
//   * column data (dy_j / RBF nodes), the adjoint handoff row from the strip
//     below and the next block's checkpoints stream into shared memory by
//     cp.async while the current block is swept;
//   * the coarse adjoint dF/d(delta) is mapped to path space on the fly
//     (FUSED): gx_i += D_ij dy_j stays in the lane's registers; gy_j += D_ij dx_i
//     is accumulated in a per-warp shared-memory row per column (lanes touch a
//     row one step apart, in a fixed order, so no shuffles and no atomics),
//     seeded by the strips below and finished by lane 0; RBF uses a per-pair
//     coarse buffer (DBUF).  Increment gradients are telescoped to point
//     gradients once per pair (kernel_grad.py:51-60).
//   * Gram gradients go into exact fixed-point accumulators (FixAcc,
//     sk_common.cuh), bitwise independent of the order pairs finish in;
//   * nothing proportional to the fine grid is stored per pair beyond the
//     checkpoints (1/R + 1/(CB*S*F) of the grid).
#pragma once
#include "sk_forward.cuh"

namespace sk {

enum MapMode : int { FUSED = 0, DBUF = 1 };

// Profiling experiments only (default 0): 1 skips the gradient map, 2 the
// reverse sweep, 4 the block recompute.  Results are wrong when set.
#ifndef SK_EXP
#define SK_EXP 0
#endif

// Batch: the pair owns its gradient rows (plain add into the zeroed output);
// Gram: exact fixed-point accumulation (FixAcc, sk_common.cuh).
__device__ __forceinline__ void grad_add(double* g, const FixAcc& f, int64_t e, double v,
                                         bool gram) {
  if (gram) fix_add(f, e, v);
  else g[e] += v;
}

constexpr int pow2_at_least(int n) {
  return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : n <= 512 ? 512
         : n <= 1024 ? 1024 : 2048;
}

// Shared-memory layout (doubles) of one lane group: a warp (NL = 32) or, for
// cross-warp pairs (NW > 1), the whole CTA (NL = 32 NW lanes).
template <int DP, int R, int RC, int F, int CB, int S, int NL = 32>
struct BwdSmem {
  static constexpr int SF = S * F;
  // column ring: power of two when cheap, else the exact need (modulo indexing)
  static constexpr int NEED = (2 * CB + NL) * S;
  static constexpr int SLOTS = (DP >= 16) ? ((NEED + 15) / 16) * 16 : pow2_at_least(NEED);
  static constexpr int REC = ((DP + F) + 1) & ~1;    // column data | handoff/adjoint (F)
  static constexpr int NK = CB * SF * R;             // recomputed k values (x NL lanes)
  static constexpr int NP = CB * S * RC;             // coarse p (then D) values (x NL lanes)
  static constexpr int NTR = CB * SF + 1;            // top row of the block (x NL lanes)
  static constexpr int TS = (CB + 1) * SF * NL;      // top-row checkpoints of the next block
  static constexpr int T0 = ((CB * SF + 1) + 1) & ~1; // lane 0's top row (strip above)
  static constexpr int LS = R * NL;                  // left-column checkpoint
  static constexpr int GS = CB * S * DP;             // last lane's incoming column gradients (x2)
  static constexpr int GROWS = (NL + CB) * S;        // gy accumulator rows (one per column)
  static constexpr int GSTR = DP + 2;                // row stride: conflict-free 16-B accesses
  static constexpr int PS = CB * S * RC * NL;        // coarse p checkpoints of the next block
  static constexpr int XCH = NL > 32 ? 4 * (NL / 32) * SF : 0;  // cross-warp hops (2 x 2 buffers)
  // block values, coarse p and top row: registers when <= 32 values per lane
  // (REGK in bwd_kernel), else per-lane shared-memory columns
  static constexpr int KPT = NK <= 32 ? 0 : NK + NP + NTR;
  // staged block inputs, double-buffered by block parity (the next block's
  // staging is issued before this block's recompute, no barrier between)
  static constexpr int STG = TS + T0 + LS + PS;
  static constexpr int MAIN = SLOTS * REC + KPT * NL + 2 * STG + 2 * GS + GROWS * GSTR + 2 * DP +
                              XCH;
  // RBF node-adjoint epilogue (after the sweep, reuses the region): a band of
  // EH node rows x NL node columns -- D tile (EH+1) x (NL+1), weights EH x
  // (NL+1), the band's row nodes, the chunk's column nodes
  static constexpr int EH = NL >= 128 ? 16 : 8;
  static constexpr int EPI = (EH + 1) * (NL + 1) + EH * (NL + 1) + 2 * EH * DP + NL * DP;
  static constexpr int TOTAL = MAIN > EPI ? MAIN : EPI;
};

//   NW    warps per pair: 1 = one pair per warp (Gram tiles, many pairs); > 1 =
//         one pair per CTA, a single wavefront over NL = 32 NW lanes whose
//         cross-warp hops (lane 31 -> lane 0 of the next warp forward, lane 0
//         -> lane 31 of the previous warp backward) go through shared memory
//         with one CTA barrier per step (few long pairs: BASELINE config 2)
template <int KIND, int DP, int R, int FR, int F, int CB, int MAP, int S, int NW = 1>
__global__ void __launch_bounds__(NW > 1 ? 32 * NW : 128, NW > 1 ? 1 : 2)
bwd_kernel(Problem pb, BwdArgs ba) {
  constexpr int RC = R / FR;
  constexpr int SF = S * F;
  constexpr int NL = 32 * NW;  // lanes per pair
  constexpr bool XW = NW > 1;
  using SM = BwdSmem<DP, R, RC, F, CB, S, NL>;
  constexpr int SLOTS = SM::SLOTS;
  constexpr int REC = SM::REC;
  constexpr int PF = 2;  // steps in flight in phase A
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int u = XW ? (int)threadIdx.x : lane;  // lane of the pair's wavefront
  double* ring = smem + (XW ? 0 : (size_t)warp * SM::TOTAL);
  double* sK = ring + SLOTS * REC;
  double* sP = sK + (SM::KPT ? SM::NK * NL : 0);
  double* sTR = sP + (SM::KPT ? SM::NP * NL : 0);
  double* sSTG = sTR + (SM::KPT ? SM::NTR * NL : 0);  // [2][STG] staged block inputs
  // staging of block parity par: top-row checkpoints, lane 0's top row, left
  // column checkpoint, coarse p
  auto stg_ts = [&](int par) { return sSTG + par * SM::STG; };
  auto stg_t0 = [&](int par) { return sSTG + par * SM::STG + SM::TS; };
  auto stg_ls = [&](int par) { return sSTG + par * SM::STG + SM::TS + SM::T0; };
  auto stg_ps = [&](int par) { return sSTG + par * SM::STG + SM::TS + SM::T0 + SM::LS; };
  double* sGS0 = sSTG + 2 * SM::STG;
  double* sGW = sGS0 + 2 * SM::GS;
  double* sZero = sGW + SM::GROWS * SM::GSTR;  // DP zeros (the last lane's unseeded rows)
  double* sGA = sZero + DP;                    // lane 0's coarse-column sums (2^lam2 > F)
  double* sXA = sGA + DP;                      // XW: [2][NW][SF] forward hops (bottom rows)
  double* sXB = sXA + (XW ? 2 * NW * SF : 0);  // XW: [2][NW][SF] backward hops (messages)
#define SK_BAR()                          \
  do {                                     \
    if constexpr (XW) __syncthreads();     \
    else __syncwarp();                     \
  } while (0)
  for (int k = u; k < DP; k += NL) sZero[k] = 0.0;
  SK_BAR();
  // small blocks (<= 32 recomputed values per lane, e.g. one coarse column of
  // 4 x 4 fine cells): the block's forward values, top row and coarse p live in
  // registers (every index is a compile-time constant after unrolling) instead
  // of the per-lane shared-memory columns
  constexpr bool REGK = SM::NK <= 32;
  double rK[REGK ? SM::NK : 1], rP[REGK ? SM::NP : 1], rT[REGK ? SM::NTR : 1];
  auto kb_ref = [&](int i) -> double& {
    if constexpr (REGK) return rK[i];
    else return sK[i * NL + u];
  };
  auto pb_ref = [&](int i) -> double& {
    if constexpr (REGK) return rP[i];
    else return sP[i * NL + u];
  };
  auto tr_ref = [&](int i) -> double& {
    if constexpr (REGK) return rT[i];
    else return sTR[i * NL + u];
  };
#define SK_TR(q) tr_ref(q)
#define SK_KB(kap, s, f, r) kb_ref((((kap) * S + (s)) * F + (f)) * R + (r))
#define SK_PB(kap, s, c) pb_ref(((kap) * S + (s)) * RC + (c))
#define SK_REC(col)                                                                     \
  (ring + ((SLOTS & (SLOTS - 1)) == 0 ? ((col) & (SLOTS - 1))                              \
                                      : (((col) + 4 * SLOTS) % SLOTS)) * REC)

  const int M1 = pb.M1c << pb.lam1;
  const int M2 = pb.M2c << pb.lam2;
  const int NC = M2 / F;                // columns per strip row
  const int NSTEP = (NC + S - 1) / S;   // steps per strip row
  const int NT = NSTEP + NL - 1;        // skewed steps per strip
  const int NB = (NT + CB - 1) / CB;
  const int H = NL * R;
  const int nstrips = (M1 + H - 1) / H;
  const int last_strip = (M1 - 1) / H;
  const int u_star = ((M1 - 1) % H) / R;
  const int r_star = (M1 - 1) % R;
  const int dR = ba.d;
  const int K2m = (1 << pb.lam2) / F - 1;  // columns per coarse column - 1 (power of 2)
  // LINEAR rows carry the exact dyadic factor: gx needs it on D, gy does not
  const double gxs_scale = (KIND == LINEAR) ? pb.scale : 1.0;

  const int64_t slot = XW ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * nw + warp;
  const int64_t item_step = XW ? (int64_t)gridDim.x : (int64_t)gridDim.x * nw;
  double* __restrict__ rowck = ba.rowck + slot * ba.rowck_stride;
  double* __restrict__ colck = ba.colck + slot * ba.colck_stride;
  double* __restrict__ pck = ba.pck + slot * ba.pck_stride;
  double* __restrict__ hrow = ba.hand + slot * ba.row_stride;
  double* __restrict__ arow = ba.adj + slot * ba.row_stride;
  double* __restrict__ dbuf = (MAP == DBUF) ? ba.dbuf + slot * ba.dbuf_stride : nullptr;
  // LINEAR + DBUF serves d > 32 (several DP-chunks): the increment gradients
  // are formed after the sweep from the stored coarse adjoint, all chunks
  constexpr bool WIDE = (KIND == LINEAR) && (MAP == DBUF);
  const int GW = WIDE ? pb.dpad : DP;  // row length of the increment-gradient scratch
  double* __restrict__ gxs = ba.gscr + slot * ba.gscr_stride;  // [M1c][GW]
  double* __restrict__ gcs = gxs + (int64_t)pb.M1c * GW;       // [M2c][GW]
#define SK_ROWCK(strip, d, q, ln) rowck[(((int64_t)(strip) * NT + (d)) * SF + (q)) * NL + (ln)]

  for (int64_t item = slot; item < pb.nitems; item += item_step) {
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
    const double* cbase = pb.C.p + pc * pb.C.path_stride;  // this pair's column path

    // ring records of columns [c0, c0 + n): column data + F handoff values (no commit)
    auto issue_cols = [&](int c0, int n, const double* hsrc, bool hvalid) {
      constexpr int PER = DP / 2 + F;
      for (int e = u; e < n * PER; e += NL) {
        const int q = e / PER, w = e % PER;
        const int col = c0 + q;
        const bool cv = (col >= 0) && (col < NC);
        double* dst = SK_REC(col);
        if (w < DP / 2) {
          const int jc = cv ? ((col * F) >> pb.lam2) : 0;
          const int node = (KIND == RBF) ? jc + 1 : jc;
          cp_async16(dst + 2 * w, cbase + (int64_t)node * pb.dpad + 2 * w, cv);
        } else {
          const int f = w - DP / 2;
          cp_async8(dst + DP + f, hsrc + (cv ? col * F + f + 1 : 0), cv && hvalid);
        }
      }
    };

    // coefficients of column col from its ring record (RBF carries K across columns)
    double Kl[RC + 1], Kr[RC + 1];
    int jcur = -1;
    auto colcoef = [&](const RowRegs<KIND, DP, RC>& rr, int col, int i0, Coef (&cfo)[RC],
                       double (&po)[RC]) {
      const double* rec = SK_REC(col);
      const bool cv = (col >= 0) && (col < NC);
      double p[RC];
      if constexpr (KIND == LINEAR) {
        double dy[DP];
#pragma unroll
        for (int k = 0; k < DP; k += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(rec + k);
          dy[k] = t2.x;
          dy[k + 1] = t2.y;
        }
#pragma unroll
        for (int c = 0; c < RC; ++c) p[c] = dot<DP>(rr.v[c], dy);
        if (WIDE && pb.nch > 1 && cv) {  // d > 32: further chunks, as the forward
          const int jc = (col * F) >> pb.lam2;
          for (int ch = 1; ch < pb.nch; ++ch) {
            double dyc[DP], xc[DP];
            load_vec<DP>(dyc, cbase + (int64_t)jc * pb.dpad + ch * DP);
#pragma unroll
            for (int c = 0; c < RC; ++c) {
              const int i = i0 + c;
              if (i < pb.M1c) {
                load_vec<DP>(xc, pb.R.p + pr * pb.R.path_stride + (int64_t)i * pb.dpad + ch * DP);
                p[c] += dot<DP>(xc, dyc);
              }
            }
          }
        }
      } else {
        const int jc = (col * F) >> pb.lam2;
        if (cv && jc != jcur) {
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
        for (int c = 0; c < RC; ++c)
          p[c] = cv ? ((Kr[c + 1] - Kl[c + 1]) - (Kr[c] - Kl[c])) * pb.scale : 0.0;
      }
#pragma unroll
      for (int c = 0; c < RC; ++c) {
        cfo[c] = coef(p[c]);
        po[c] = p[c];
      }
    };

    // ------------------------------------------- phase A: forward + checkpoints
    for (int t = u; t <= M2; t += NL) hrow[t] = 1.0;
    SK_BAR();
    double kval = 0.0;
    for (int strip = 0; strip < nstrips; ++strip) {
      const int rbase = strip * H + u * R;
      const int i0 = rbase >> pb.lam1;
      RowRegs<KIND, DP, RC> rr;
      load_rows<KIND, DP, RC>(rr, pb, pr, i0, 0);
      jcur = -1;
      double* __restrict__ rowck_s = rowck + (int64_t)strip * NT * SF * NL + u;
      // coarse p of every column this lane solves: the block recompute reads
      // it back instead of re-forming <dx_i, dy_j> (or the RBF exps)
      double* __restrict__ pck_s = pck + (int64_t)strip * NT * S * RC * NL + u;
      if constexpr (KIND == RBF) {
        double y0[DP];
        load_vec<DP>(y0, cbase);
#pragma unroll
        for (int c = 0; c <= RC; ++c) Kr[c] = exp(-sqdist<DP>(rr.v[c], y0) * pb.inv2s2);
#pragma unroll
        for (int c = 0; c <= RC; ++c) Kl[c] = Kr[c];
      }
      for (int q = 0; q < PF; ++q) {
        issue_cols(q * S, S, hrow, strip > 0);
        cp_async_commit();
      }
      double kl[R];
#pragma unroll
      for (int r = 0; r < R; ++r) kl[r] = 1.0;
      double topc = 1.0;
      double bot[SF];
#pragma unroll
      for (int q = 0; q < SF; ++q) bot[q] = 1.0;
      if constexpr (XW) {  // lane 0 of warp w reads warp w-1's lane 31 from here
        for (int e = u; e < 2 * NW * SF; e += NL) sXA[e] = 1.0;
      }
      for (int tau = 0; tau < NT; ++tau) {
        issue_cols((tau + PF) * S, S, hrow, strip > 0);
        cp_async_commit();
        cp_async_wait<PF>();  // step tau landed
        SK_BAR();
        if (tau % CB == 0) {
          // column checkpoint: values at node column (tau - u) * S * F
#pragma unroll
          for (int r = 0; r < R; ++r)
            colck[(((int64_t)strip * NB + tau / CB) * R + r) * NL + u] = kl[r];
        }
        const int js = tau - u;
        const bool active = (js >= 0) && (js < NSTEP);
        double tv[SF];
#pragma unroll
        for (int q = 0; q < SF; ++q) tv[q] = __shfl_up_sync(0xffffffffu, bot[q], 1);
        if constexpr (XW) {
          if (lane == 0 && warp > 0) {
#pragma unroll
            for (int q = 0; q < SF; ++q) tv[q] = sXA[(((tau + 1) & 1) * NW + warp - 1) * SF + q];
          }
        }
        if (active) {
          if (u == 0) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const double* rec = SK_REC(js * S + s);
#pragma unroll
              for (int f = 0; f < F; ++f) tv[s * F + f] = (strip == 0) ? 1.0 : rec[DP + f];
            }
          }
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const int col = js * S + s;
            Coef cf[RC];
            double pv[RC];
            colcoef(rr, col, i0, cf, pv);
#pragma unroll
            for (int c = 0; c < RC; ++c) pck_s[((tau * S + s) * RC + c) * NL] = pv[c];
#pragma unroll
            for (int f = 0; f < F; ++f) {
              const int q = s * F + f;
              double up = tv[q];
              double dg = (q == 0) ? topc : tv[q - 1];
#pragma unroll
              for (int r = 0; r < R; ++r) {
                const double nk = cell(up, kl[r], dg, cf[r / FR]);
                dg = kl[r];
                kl[r] = nk;
                up = nk;
              }
              bot[q] = up;
              rowck_s[(tau * SF + q) * NL] = up;  // diagonal index = step + writer lane = tau
            }
            if (strip == last_strip && u == u_star && col == NC - 1) {
#pragma unroll
              for (int r = 0; r < R; ++r)
                if (r == r_star) kval = kl[r];
            }
          }
          topc = tv[SF - 1];
          if (u == NL - 1) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const int col = js * S + s;
              if (col < NC) {
#pragma unroll
                for (int f = 0; f < F; ++f) hrow[col * F + f + 1] = bot[s * F + f];
              }
            }
          }
        }
        if constexpr (XW) {
          if (lane == 31 && warp < NW - 1) {
#pragma unroll
            for (int q = 0; q < SF; ++q) sXA[((tau & 1) * NW + warp) * SF + q] = bot[q];
          }
        }
      }
      cp_async_wait<0>();
      SK_BAR();
    }
    if (ba.values && u == u_star) ba.values[oidx] = kval;

    // ------------------------------------------------ phase B: reverse sweep
    for (int t = u; t <= M2; t += NL) arow[t] = 0.0;
    // RBF (and WIDE) coarse adjoint: written once per cell when one (lane,
    // step) covers whole coarse cells, else accumulated into a zeroed buffer
    const bool dbuf_once = MAP == DBUF && ba.rows_exclusive != 0 && K2m == 0;
    if constexpr (MAP == DBUF) {
      if (!dbuf_once)
        for (int64_t e = u; e < (int64_t)pb.M1c * pb.M2c; e += NL) dbuf[e] = 0.0;
    } else {
      for (int64_t e = u; e < (int64_t)pb.M1c * DP; e += NL) gxs[e] = 0.0;
    }
    SK_BAR();
    const bool atomic = ba.atomic != 0;
    double* __restrict__ gR = atomic ? nullptr : ba.gradR + pr * ba.gR_path;
    double* __restrict__ gC = atomic ? nullptr : ba.gradC + pc * ba.gC_path;
    const FixAcc fxR = atomic ? fix_make(ba.accR, ba.metaR) : FixAcc{};
    const FixAcc fxC = atomic ? fix_make(ba.accC, ba.metaC) : FixAcc{};
    const int64_t eR = atomic ? pr * ba.gR_path : 0;  // element offsets into the accumulators
    const int64_t eC = atomic ? pc * ba.gC_path : 0;

    for (int strip = nstrips - 1; strip >= 0; --strip) {
      const int rbase = strip * H + u * R;
      const int i0 = rbase >> pb.lam1;
      const bool seed_lane = strip == last_strip && u == u_star;
      RowRegs<KIND, DP, RC> rr;
      load_rows<KIND, DP, RC>(rr, pb, pr, i0, 0);

      // records + staging of block blk (buffers of parity blk & 1): top-row
      // checkpoints, lane 0's top row, left checkpoint, coarse p (consumed by
      // the recompute) and lane 31's incoming column gradients (the sweep)
      auto issue_block = [&](int blk, bool first) {
        double* sTS = stg_ts(blk & 1);
        double* sT0 = stg_t0(blk & 1);
        double* sLS = stg_ls(blk & 1);
        double* sPS = stg_ps(blk & 1);
        if (first) issue_cols((blk * CB - (NL - 1)) * S, (CB + NL - 1) * S, arow, true);
        else issue_cols((blk * CB - (NL - 1)) * S, CB * S, arow, true);  // the new columns only
        {
          const int dlo = blk * CB - 2;  // rowck[strip][d][q][*], d in [blk*CB-2, blk*CB+CB-2]
          constexpr int NCH = SM::TS / 2;
          constexpr int ROWT = SF * NL / 2;  // 16-byte chunks per diagonal row
          for (int e = u; e < NCH; e += NL) {
            const int row = e / ROWT;  // (CB+1) rows of SF*NL doubles
            const int d = dlo + row;
            const bool v = (d >= 0) && (d < NT);
            cp_async16(sTS + 2 * e,
                       rowck + (((int64_t)strip * NT + (v ? d : 0)) * SF) * NL + 2 * (e % ROWT),
                       v);
          }
        }
        if (strip > 0) {
          // lane 0's top row: nodes t = blk*CB*SF + q, written by strip-1's last lane
          for (int q = u; q <= CB * SF; q += NL) {
            const int t = blk * CB * SF + q;
            const bool v = (t >= 1) && (t <= M2);
            const int js = v ? (t - 1) / SF : 0, qs = v ? (t - 1) % SF : 0;
            cp_async8(sT0 + q, &SK_ROWCK(strip - 1, js + NL - 1, qs, NL - 1), v);
          }
        }
        for (int e = u; e < SM::LS / 2; e += NL)
          cp_async16(sLS + 2 * e, colck + (((int64_t)strip * NB + blk) * R) * NL + 2 * e, true);
        {
          // coarse p: lane u's step js0 + kap sits at diagonal index blk*CB + kap
          constexpr int ROWC = S * RC * NL / 2;  // 16-byte chunks per diagonal row
          for (int e = u; e < CB * ROWC; e += NL) {
            const int d = blk * CB + e / ROWC;
            const bool v = d < NT;
            cp_async16(sPS + 2 * e,
                       pck + ((int64_t)strip * NT + (v ? d : 0)) * S * RC * NL + 2 * (e % ROWC), v);
          }
        }
        if constexpr (MAP == FUSED) {
          double* gs = sGS0 + (blk & 1) * SM::GS;
          for (int e = u; e < CB * S * (DP / 2); e += NL) {
            const int ks = e / (DP / 2), w = e % (DP / 2);
            const int col = (blk * CB - (NL - 1)) * S + ks;  // the last lane's columns
            const bool v = (col >= 0) && (col < NC) && (strip < nstrips - 1);
            const int jc = v ? ((col * F) >> pb.lam2) : 0;
            cp_async16(gs + ks * DP + 2 * w, gcs + (int64_t)jc * DP + 2 * w, v);
          }
        }
        cp_async_commit();
      };

      double aR[R], bR[R];
#pragma unroll
      for (int r = 0; r < R; ++r) { aR[r] = 0.0; bR[r] = 0.0; }
      double sendm[SF];
#pragma unroll
      for (int q = 0; q < SF; ++q) sendm[q] = 0.0;
      double gxr[(MAP == FUSED) ? RC : 1][DP];
#pragma unroll
      for (int k = 0; k < DP; ++k)
#pragma unroll
        for (int c = 0; c < ((MAP == FUSED) ? RC : 1); ++c) gxr[c][k] = 0.0;

      int bstep = 0;  // XW: sweep-step parity of the backward hops
      if constexpr (XW) {
        for (int e = u; e < 2 * NW * SF; e += NL) sXB[e] = 0.0;
      }
      issue_block(NB - 1, true);
      for (int blk = NB - 1; blk >= 0; --blk) {
        cp_async_wait<0>();
        SK_BAR();  // block blk staged; block blk+1's buffers (parity of blk-1) consumed
        const double* sTS = stg_ts(blk & 1);
        const double* sT0 = stg_t0(blk & 1);
        const double* sLS = stg_ls(blk & 1);
        const double* sPS = stg_ps(blk & 1);
        // the next block's staging goes into the other parity's buffers at once
        if (blk > 0) issue_block(blk - 1, false);
        const double* sGS = sGS0 + (blk & 1) * SM::GS;
        const int js0 = blk * CB - u;  // lane's first step in this block
        double kleft[R];
#pragma unroll
        for (int r = 0; r < R; ++r) kleft[r] = sLS[r * NL + u];

        // ---- recompute the block's forward values into shared memory
        if (!(SK_EXP & 4)) {
          // top row at node t = js0*SF + q (q = 0..CB*SF) of this lane's rows
#pragma unroll
          for (int q = 0; q <= CB * SF; ++q) {
            const int t = js0 * SF + q;
            double v;
            if (t <= 0 || (strip == 0 && u == 0)) {
              v = 1.0;
            } else if (t > M2) {
              v = 0.0;  // dead columns: keep values finite
            } else if (u == 0) {
              v = sT0[q];
            } else {
              const int d = (t - 1) / SF + u - 1 - (blk * CB - 2);
              v = sTS[(d * SF + (t - 1) % SF) * NL + (u - 1)];
            }
            SK_TR(q) = v;
          }
          double kl[R];
#pragma unroll
          for (int r = 0; r < R; ++r) kl[r] = kleft[r];
          double topc = SK_TR(0);
#pragma unroll
          for (int kap = 0; kap < CB; ++kap) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const int col = (js0 + kap) * S + s;
              Coef cf[RC];
              {
                const bool cv = (col >= 0) && (col < NC);
#pragma unroll
                for (int c = 0; c < RC; ++c) {
                  const double p = cv ? sPS[((kap * S + s) * RC + c) * NL + u] : 0.0;
                  SK_PB(kap, s, c) = p;
                  cf[c] = coef(p);
                }
              }
#pragma unroll
              for (int f = 0; f < F; ++f) {
                const int q = (kap * S + s) * F + f;
                double up = SK_TR(q + 1);
                double dg = (q == 0) ? topc : SK_TR(q);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                  const double nk = cell(up, kl[r], dg, cf[r / FR]);
                  dg = kl[r];
                  kl[r] = nk;
                  up = nk;
                  SK_KB(kap, s, f, r) = nk;
                }
              }
            }
          }
        }
        if constexpr (SM::KPT != 0) SK_BAR();  // shared-memory block values visible

        // ---- reverse sweep over the block, one step per kap
#pragma unroll
        for (int kap = CB - 1; kap >= 0 && !(SK_EXP & 2); --kap) {
          const int js = js0 + kap;
          double recv[SF];
#pragma unroll
          for (int q = 0; q < SF; ++q) recv[q] = __shfl_down_sync(0xffffffffu, sendm[q], 1);
          if constexpr (XW) {
            if (lane == 31 && warp < NW - 1) {
#pragma unroll
              for (int q = 0; q < SF; ++q)
                recv[q] = sXB[(((bstep + 1) & 1) * NW + warp + 1) * SF + q];
            }
          }
          if (u == NL - 1) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const int col = js * S + s;
              const bool cv = (col >= 0) && (col < NC);
              const double* rec = SK_REC(col);
#pragma unroll
              for (int f = 0; f < F; ++f) recv[s * F + f] = cv ? rec[DP + f] : 0.0;
            }
          }
#pragma unroll
          for (int s = S - 1; s >= 0; --s) {
            const int jj = js * S + s;  // column
            const bool colv = (jj >= 0) && (jj < NC);
            const double* rec = SK_REC(jj);
            // the seed dF/dk(M1, M2) = cot enters as the final cell's "message
            // from the right" (exactly 0 there: right of it every cell is dead),
            // once per step instead of a test per cell: (0 + cot) + m == (0 + m) + cot
            if (seed_lane && jj == NC - 1) {
#pragma unroll
              for (int r = 0; r < R; ++r)
                if (r == r_star) aR[r] += wcot;
            }
            double Dp[RC];
#pragma unroll
            for (int c = 0; c < RC; ++c) Dp[c] = 0.0;
            double pk[RC];
            Coef cf[RC];
#pragma unroll
            for (int c = 0; c < RC; ++c) {
              pk[c] = SK_PB(kap, s, c);
              cf[c] = coef(pk[c]);
            }
#pragma unroll
            for (int f = F - 1; f >= 0; --f) {
              const int q = s * F + f;                 // fine column within the step
              const int qb = (kap * S + s) * F + f;    // fine column within the block
              double m = recv[q];
              // no masks: dead rows (> M1) and columns (>= NC) lie below / right
              // of the seeded final cell and their p is finite (zero-filled
              // rows and records), so their adjoint is exactly 0; columns < 0
              // only feed cells further left, and their D is never consumed
#pragma unroll
              for (int r = R - 1; r >= 0; --r) {
                const double lam = aR[r] + m;
                const int c = r / FR;
                const double a = cf[c].A * lam;
                const double b = cf[c].B * lam;
                // forward values around the cell: left, up, up-left
                const double kL = (qb > 0) ? kb_ref((qb - 1) * R + r) : kleft[r];
                const double kU = (r > 0) ? kb_ref(qb * R + r - 1) : SK_TR(qb + 1);
                const double kD = (r > 0) ? ((qb > 0) ? kb_ref((qb - 1) * R + r - 1)
                                                      : kleft[r - 1])
                                          : SK_TR(qb);
                const double p6 = pk[c] * (1.0 / 6.0);
                const double wv = fma(kL + kU, 0.5 + p6, kD * p6);
                Dp[c] = fma(lam, wv, Dp[c]);
                m = a - bR[r];
                aR[r] = a;
                bR[r] = b;
              }
              sendm[q] = m;
            }
            if (u == 0 && colv) {
#pragma unroll
              for (int f = 0; f < F; ++f) arow[jj * F + f + 1] = sendm[s * F + f];
            }
            const int jc = colv ? ((jj * F) >> pb.lam2) : 0;
            if constexpr (MAP == FUSED && !(SK_EXP & 1)) {
              // gx_i += D_ij dy_j (row-local registers; D carries the dyadic factor)
              double Dg[RC];
#pragma unroll
              for (int c = 0; c < RC; ++c) Dg[c] = Dp[c] * gxs_scale;
#pragma unroll
              for (int k = 0; k < DP; k += 2) {
                const double2 t2 = *reinterpret_cast<const double2*>(rec + k);
#pragma unroll
                for (int c = 0; c < RC; ++c) {
                  gxr[c][k] = fma(Dg[c], t2.x, gxr[c][k]);
                  gxr[c][k + 1] = fma(Dg[c], t2.y, gxr[c][k + 1]);
                }
              }
              // gy_j += D_ij dx_i into the column's shared row (rows carry the
              // dyadic factor already).  Lanes touch a row one step apart (u+1
              // before u); lane 31 starts it (seeded by the strips below at the
              // coarse column's first column), lane 0 finishes it.
              if (colv) {
                double* row = sGW + (jj % SM::GROWS) * SM::GSTR;
                const bool seed = ((jj + 1) & K2m) == 0;
                const double* src = (u == NL - 1) ? (seed ? (sGS + ((kap * S + s) * DP)) : sZero) : row;
#pragma unroll
                for (int k = 0; k < DP; k += 2) {
                  double2 v = *reinterpret_cast<const double2*>(src + k);
#pragma unroll
                  for (int c = 0; c < RC; ++c) {
                    v.x = fma(Dp[c], rr.v[c][k], v.x);
                    v.y = fma(Dp[c], rr.v[c][k + 1], v.y);
                  }
                  *reinterpret_cast<double2*>(row + k) = v;
                }
                if (u == 0) {
                  double2* dst = reinterpret_cast<double2*>(gcs + (int64_t)jc * DP);
                  if (K2m == 0) {  // one column per coarse column
#pragma unroll
                    for (int k = 0; k < DP; k += 2) dst[k / 2] = *reinterpret_cast<const double2*>(row + k);
                  } else {  // several: lane 0 sums them (reverse order), emits at the last
                    const bool last = (jj & K2m) == 0;
#pragma unroll
                    for (int k = 0; k < DP; ++k) {
                      const double a = (seed ? 0.0 : sGA[k]) + row[k];
                      sGA[k] = a;
                      if (last) gcs[(int64_t)jc * DP + k] = a;
                    }
                  }
                }
              }
            } else if constexpr (MAP == DBUF) {
              // RBF: coarse adjoint, kept per block in shared memory (p is dead)
#pragma unroll
              for (int c = 0; c < RC; ++c) SK_PB(kap, s, c) = colv ? Dp[c] * pb.scale : 0.0;
            }
          }
          if constexpr (XW) {
            if (lane == 0 && warp > 0) {
#pragma unroll
              for (int q = 0; q < SF; ++q) sXB[((bstep & 1) * NW + warp) * SF + q] = sendm[q];
            }
          }
          ++bstep;
          SK_BAR();
        }
        if constexpr (MAP == DBUF) {
          // flush the block's coarse adjoint; lanes sharing coarse rows go in
          // order.  When one (lane, step) covers whole coarse cells (rows
          // exclusive, F = 2^lam2) every cell is written exactly once: plain
          // stores (no read-modify-write), bitwise the same as 0 + v.
          const bool excl = ba.rows_exclusive != 0;
          if (dbuf_once) {
#pragma unroll
            for (int kap = CB - 1; kap >= 0; --kap) {
#pragma unroll
              for (int s = S - 1; s >= 0; --s) {
                const int jj = (js0 + kap) * S + s;
                if (jj >= 0 && jj < NC) {
                  const int jc = (jj * F) >> pb.lam2;
#pragma unroll
                  for (int c = 0; c < RC; ++c) {
                    const int i = i0 + c;
                    if (i < pb.M1c) dbuf[(int64_t)i * pb.M2c + jc] = SK_PB(kap, s, c);
                  }
                }
              }
            }
          }
          for (int ln = (excl ? 0 : NL - 1) - (dbuf_once ? NL : 0); ln >= 0; --ln) {
            if (excl || u == ln) {
#pragma unroll
              for (int kap = CB - 1; kap >= 0; --kap) {
#pragma unroll
                for (int s = S - 1; s >= 0; --s) {
                  const int jj = (js0 + kap) * S + s;
                  if (jj >= 0 && jj < NC) {
                    const int jc = (jj * F) >> pb.lam2;
#pragma unroll
                    for (int c = 0; c < RC; ++c) {
                      const int i = i0 + c;
                      if (i < pb.M1c) dbuf[(int64_t)i * pb.M2c + jc] += SK_PB(kap, s, c);
                    }
                  }
                }
              }
            }
            if (!excl) SK_BAR();
          }
        }
        // (no barrier: the next block starts with one)
      }
      cp_async_wait<0>();
      SK_BAR();
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
          for (int ln = NL - 1; ln >= 0; --ln) {
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
            SK_BAR();
          }
        }
      }
      SK_BAR();
    }

    if constexpr (MAP == FUSED) {
      // telescope increment gradients to point gradients (kernel_grad.py:55-60)
      // and flush once per pair, coalesced across the warp
      SK_BAR();
      for (int64_t e = u; e < (int64_t)(pb.M1c + 1) * dR; e += NL) {
        const int p = (int)(e / dR), k = (int)(e % dR);
        double v = 0.0;
        if (p >= 1) v += gxs[(int64_t)(p - 1) * DP + k];
        if (p < pb.M1c) v -= gxs[(int64_t)p * DP + k];
        grad_add(gR, fxR, eR + e, v, atomic);
      }
      for (int64_t e = u; e < (int64_t)(pb.M2c + 1) * dR; e += NL) {
        const int p = (int)(e / dR), k = (int)(e % dR);
        double v = 0.0;
        if (p >= 1) v += gcs[(int64_t)(p - 1) * DP + k];
        if (p < pb.M2c) v -= gcs[(int64_t)p * DP + k];
        grad_add(gC, fxC, eC + e, v, atomic);
      }
      SK_BAR();
    } else if constexpr (WIDE) {
      // d > 32: gx_i = sum_j D_ij dy_j, gy_j = sum_i D_ij dx_i (kernel_grad.py:53-54)
      // from the stored coarse adjoint D (dbuf, carries the dyadic factor), one
      // 32-wide chunk of components at a time, then telescoped as above
      SK_BAR();
      const double* D = dbuf;
      const double* xp = pb.R.p + pr * pb.R.path_stride;  // rows carry the dyadic factor
      const double unscale = 1.0 / pb.scale;               // exact (power of two)
      for (int ch = 0; ch < pb.nch; ++ch) {
        for (int i = u; i < pb.M1c; i += NL) {
          double acc[DP];
#pragma unroll
          for (int k = 0; k < DP; ++k) acc[k] = 0.0;
          for (int j = 0; j < pb.M2c; ++j) {
            const double w = D[(int64_t)i * pb.M2c + j];
            double yj[DP];
            load_vec<DP>(yj, cbase + (int64_t)j * pb.dpad + ch * DP);
#pragma unroll
            for (int k = 0; k < DP; ++k) acc[k] = fma(w, yj[k], acc[k]);
          }
#pragma unroll
          for (int k = 0; k < DP; ++k) gxs[(int64_t)i * GW + ch * DP + k] = acc[k];
        }
        for (int j = u; j < pb.M2c; j += NL) {
          double acc[DP];
#pragma unroll
          for (int k = 0; k < DP; ++k) acc[k] = 0.0;
          for (int i = 0; i < pb.M1c; ++i) {
            const double w = D[(int64_t)i * pb.M2c + j];
            double xi[DP];
            load_vec<DP>(xi, xp + (int64_t)i * pb.dpad + ch * DP);
#pragma unroll
            for (int k = 0; k < DP; ++k) acc[k] = fma(w, xi[k], acc[k]);
          }
#pragma unroll
          for (int k = 0; k < DP; ++k) gcs[(int64_t)j * GW + ch * DP + k] = acc[k] * unscale;
        }
      }
      SK_BAR();
      for (int64_t e = u; e < (int64_t)(pb.M1c + 1) * dR; e += NL) {
        const int p = (int)(e / dR), k = (int)(e % dR);
        double v = 0.0;
        if (p >= 1) v += gxs[(int64_t)(p - 1) * GW + k];
        if (p < pb.M1c) v -= gxs[(int64_t)p * GW + k];
        grad_add(gR, fxR, eR + e, v, atomic);
      }
      for (int64_t e = u; e < (int64_t)(pb.M2c + 1) * dR; e += NL) {
        const int p = (int)(e / dR), k = (int)(e % dR);
        double v = 0.0;
        if (p >= 1) v += gcs[(int64_t)(p - 1) * GW + k];
        if (p < pb.M2c) v -= gcs[(int64_t)p * GW + k];
        grad_add(gC, fxC, eC + e, v, atomic);
      }
      SK_BAR();
    } else {
      // RBF node adjoint G_ij = D[i-1,j-1] - D[i-1,j] - D[i,j-1] + D[i,j] (zero
      // padded); with W_ij = G_ij K_ij / sigma^2 (one distance, one exp per
      // node pair): dF/dx_i = sum_j W_ij (y_j - x_i), dF/dy_j = sum_i W_ij (x_i - y_j).
      // Chunks of NL node columns (lane u owns column j0 + u and its dF/dy_j
      // chain), bands of EH node rows staged in shared memory (D tile, row
      // nodes); W of the band goes to shared memory and the band's dF/dx
      // chains (row, component) continue over the chunk's columns.  Both sums
      // run in ascending index order, as a per-(i, j) loop would.
      constexpr int EH = SM::EH, TW = NL + 1;
      SK_BAR();
      const double* D = dbuf;
      const double* xp = pb.R.p + pr * pb.R.path_stride;
      const double* yp = cbase;
      const int L1n = pb.M1c + 1, L2n = pb.M2c + 1;
      const int nchunk = (L2n + NL - 1) / NL;
      double* sDt = smem + (XW ? 0 : (size_t)warp * SM::TOTAL);  // [EH+1][TW]
      double* sW = sDt + (EH + 1) * TW;                             // [EH][TW]
      double* sXb0 = sW + EH * TW;                                  // [2][EH][DP]
      double* sYc = sXb0 + 2 * EH * DP;                             // [NL][DP]
      double* gxa = gxs;  // [L1n][DP] dF/dx chains between column chunks
      for (int ch = 0; ch < nchunk; ++ch) {
        const int j0 = ch * NL, j = j0 + u;
        const bool jv = j < L2n;
        const int ncol = min(NL, L2n - j0);
        double yj[DP], gy[DP];
#pragma unroll
        for (int k = 0; k < DP; ++k) {
          yj[k] = jv ? yp[(int64_t)j * pb.dpad + k] : 0.0;
          gy[k] = 0.0;
          sYc[u * DP + k] = yj[k];
        }
        // band staging by cp.async (zero-filled outside the grid): the D tile
        // and the band's row nodes; the next band's is issued under the
        // current band's dF/dx pass (the D tile is dead by then)
        auto stage_band = [&](int i0, double* sXb) {
          for (int e = u; e < (EH + 1) * TW; e += NL) {
            const int rr = e / TW, cc = e % TW;
            const int i = i0 - 1 + rr, jd = j0 - 1 + cc;
            const bool v = i >= 0 && jd >= 0 && i < pb.M1c && jd < pb.M2c;
            cp_async8(sDt + e, D + (v ? (int64_t)i * pb.M2c + jd : 0), v);
          }
          for (int e = u; e < EH * DP; e += NL) {
            const int i = i0 + e / DP;
            const bool v = i < L1n;
            cp_async8(sXb + e, xp + (v ? (int64_t)i * pb.dpad + (e % DP) : 0), v);
          }
          cp_async_commit();
        };
        SK_BAR();  // the previous chunk's band buffers consumed
        stage_band(0, sXb0);
        for (int i0 = 0, bb = 0; i0 < L1n; i0 += EH, bb ^= 1) {
          double* sXb = sXb0 + bb * EH * DP;
          cp_async_wait<0>();
          SK_BAR();  // band staged, the previous band's W consumed
#pragma unroll 2
          for (int r = 0; r < EH; ++r) {
            const double G = sDt[r * TW + u] - sDt[r * TW + u + 1] - sDt[(r + 1) * TW + u] +
                             sDt[(r + 1) * TW + u + 1];
            double w = 0.0;
            if (G != 0.0 && jv && i0 + r < L1n) {
              double s2 = 0.0;  // padded components are 0 on both sides: exact no-ops
#pragma unroll
              for (int kk = 0; kk < DP; ++kk) {
                const double t = sXb[r * DP + kk] - yj[kk];
                s2 = fma(t, t, s2);
              }
              w = G * exp(-s2 * pb.inv2s2) * pb.invs2;
#pragma unroll
              for (int k = 0; k < DP; ++k) gy[k] = fma(w, sXb[r * DP + k] - yj[k], gy[k]);
            }
            sW[r * TW + u] = w;
          }
          SK_BAR();
          if (i0 + EH < L1n) stage_band(i0 + EH, sXb0 + (bb ^ 1) * EH * DP);
          // dF/dx chains of the band's rows over the chunk's columns
          for (int e = u; e < EH * dR; e += NL) {
            const int r = e / dR, k = e % dR, i = i0 + r;
            if (i >= L1n) continue;
            double acc = ch == 0 ? 0.0 : gxa[(int64_t)i * DP + k];
            const double xk = sXb[r * DP + k];
            for (int c = 0; c < ncol; ++c) {
              const double w = sW[r * TW + c];
              if (w != 0.0) acc = fma(w, sYc[c * DP + k] - xk, acc);
            }
            if (ch == nchunk - 1) grad_add(gR, fxR, eR + (int64_t)i * dR + k, acc, atomic);
            else gxa[(int64_t)i * DP + k] = acc;
          }
        }
        if (jv) {
#pragma unroll
          for (int k = 0; k < DP; ++k)
            if (k < dR) grad_add(gC, fxC, eC + (int64_t)j * dR + k, gy[k], atomic);
        }
        SK_BAR();  // sYc reused by the next chunk
      }
      SK_BAR();
    }
  }
#undef SK_KB
#undef SK_PB
#undef SK_REC
#undef SK_TR
#undef SK_ROWCK
#undef SK_BAR
}

}  // namespace sk
