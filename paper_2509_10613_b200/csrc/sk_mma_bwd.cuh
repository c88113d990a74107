// sk_mma_bwd.cuh -- Gram backward (paper Alg. 4, the exact adjoint of the
// solver) with every dense contraction on the FP64 tensor cores (DMMA).
//
// Replaces goursat_grid + goursat_backward + the gradient map of
// kernel_backward (/root/reference/pkg/src/sigcore/_kernels.py:381-396,
// 436-466; kernel_grad.py:27-61) for linear-kernel Gram tiles at dyadic
// order 0 (BASELINE configs C3, C5).  The adjoint recursion is the
// reference's, in push form (see sk_backward.cuh):
//    d1[s,t] = d1[s+1,t] A(p[s+1,t]) + d1[s,t+1] A(p[s,t+1]) - d1[s+1,t+1] B(p[s+1,t+1])
//    D[s,t]  = d1[s,t] ((k[s,t-1] + k[s-1,t]) (1/2 + p/6) + k[s-1,t-1] p/6)
//    gx_i = sum_j D_ij dy_j,  gy_j = sum_i D_ij dx_i          (kernel_grad.py:53-54)
//
// Work per fine cell: p = <dx_i, dy_j> twice (forward checkpoint pass and the
// block recompute), gx and gy: 4d FMAs, all on DMMA; the recurrences (forward
// 7 DP ops, adjoint ~15, recompute 7) on the FMA pipe.  In r01 the FMA-pipe-only
// backward was issue/latency bound at ~10 % of the FP64 roofline.
//
// Mapping (one warp = one Gram tile of 8 pairs (a0+g, b), lane = 4g + u;
// 2-warp CTAs, 4 CTAs = 8 warps per SM, bounded by 255 registers and ~28 KB
// of shared memory per warp):
//   phase A  forward wavefront as sk_mma_fwd.cuh (lane u owns rows 2u, 2u+1 of
//            each 8-row strip, skew 1 column per lane; p tiles two ahead in a
//            4-slot ring that borrows the idle D ring), plus checkpoints: every
//            lane's bottom row, diagonal layout rowck[strip][step][8u+g] (one
//            coalesced 256-B store per step), and every lane's two values at
//            its block boundaries colck[strip][blk][lane].  The strip's top row
//            and the p tiles' dY rows stream through cp.async rings 3-4
//            iterations ahead.  Value + gradient calls also write G here;
//   phase B  strips bottom-up, blocks of 8 lane-relative columns right-to-left
//            (lane u's block blk = columns 8blk-u .. 8blk-u+7):
//            1. each lane recomputes its 2 x 8 forward values in registers from
//               its own checkpoints (staged one block ahead by lane-private
//               cp.async) and p from a 2-slot DMMA tile ring;
//            2. reverse sweep of the block, lane u one column behind lane u+1,
//               adjoint messages by __shfl_down_sync; D per cell into a
//               2-tile shared ring [column][row];
//            3. p tile blk-2 into the dead slot, then, tile blk's D being
//               complete for all 64 rows: gx += D dY (DMMA, accumulators in
//               registers for the strip) and gy = D^T dX (DMMA over the 64 rows
//               of the tile, dX staged in shared memory), added to the column
//               path's scratch.
//   Shared tiles are unpadded with XOR swizzles (psw / dsw / xsw): every
//   fragment store and load is bank-conflict-free.
//   Increment gradients are telescoped to point gradients (rows: per strip
//   from registers; columns: once per tile from the scratch) and flushed into
//   exact fixed-point accumulators (FixAcc, sk_common.cuh: integer atomics, so
//   the result is bitwise independent of tile order), kernel_grad.py:55-60.
#pragma once
#include <type_traits>

#include "sk_mma_fwd.cuh"

namespace sk {

// 1: the gx map of block blk + 1 (32 DMMAs at DP = 16) is issued inside block
// blk's reverse sweep, to fill the sweep chain's latency bubbles (same
// accumulation order: bitwise equal -- measured slower: C3 fp64 1175 -> 1208
// ms, FP32 1106 -> 1122 ms); 0 (default): after the sweep, with gy
#ifndef SK_GX_DEFER
#define SK_GX_DEFER 0
#endif

// 1: the adjoint message to lane u-1 as one FMA of the received one (+3 DP ops
// per column, shorter lane chain); 0: the chain as written (measured faster)
#ifndef SK_AFFINE_MSG
#define SK_AFFINE_MSG 0
#endif

template <int K>
struct Frag {
  double v[K];
};

template <int DP>
struct MmaBwdCfg {
  static constexpr int KS = DP / 4;            // k-steps of a p tile
  static constexpr int NN = DP / 8;            // 8-wide component tiles (gx, gy)
  // shared-memory tiles are unpadded; XOR swizzles (psw / dsw / xsw below)
  // keep every fragment store and load conflict-free
  static constexpr int PSTR = 32;              // double2 per p-tile column
  static constexpr int PTILE = 8 * PSTR;       // double2 per p tile
  static constexpr int DSTR = 64;              // doubles per D column (64 rows)
  static constexpr int DTILE = 8 * DSTR;
  static constexpr int XSTR = DP;              // doubles per staged dX row
  // block-input staging (cp.async, lane-private, double buffered): 9 top-row
  // values + 2 left values per lane, 8 strip-below messages per lane group
  // + the block's column checkpoints of all 32 lanes' previous bottom value
  static constexpr int STG = 11 * 32 + 8 * 8 + 32;
  static constexpr int WARP_DOUBLES = 2 * PTILE * 2 + 2 * DTILE + 64 * XSTR + STG;
};

//   DY  dyadic orders > 0 (runtime lam1 / lam2: coarse p tiles, coarse rows /
//       columns of the operands, fine -> coarse sums before the telescoping);
//       false: order 0 at compile time (C3, C5), no index shifts
//   TR  the recurrences' arithmetic type: double, or float for the FP32
//       backward (forward, recompute and adjoint on the FP32 pipe in the
//       small-correction forms of sk_cell.cuh; p, gx, gy stay on DMMA with
//       exact fp64 operands; checkpoints keep their fp64 slots, exact)
template <int DP, int WPC, bool DY = false, typename TR = double>
__global__ void __launch_bounds__(32 * WPC, 1)
gram_bwd_mma(Problem pb, BwdArgs ba) {
  constexpr bool F32 = std::is_same<TR, float>::value;
  using Cf = MmaBwdCfg<DP>;
  constexpr int KS = Cf::KS, NN = Cf::NN, PSTR = Cf::PSTR, DSTR = Cf::DSTR, XSTR = Cf::XSTR;
  extern __shared__ double smem_mb[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, u = lane & 3;
  double* wsm = smem_mb + (size_t)warp * Cf::WARP_DOUBLES;
  double2* __restrict__ sP = reinterpret_cast<double2*>(wsm);  // 2 p tiles
  double* __restrict__ sD = wsm + 2 * Cf::PTILE * 2;            // 2 D tiles
  double* __restrict__ sX = sD + 2 * Cf::DTILE;                  // [64][XSTR]
  double* __restrict__ sS = sX + 64 * XSTR;                      // [STG] staging
  // swizzles: p tile slot of wavefront lane wl in column col; D row in column
  // col; dX component k of staged row R
  auto psw = [](int col, int wl) { return wl ^ (4 * (col & 1)); };
  auto dsw = [](int col, int row) { return row ^ (4 * (col & 3)); };
  auto xsw = [](int R, int k) { return k ^ (DP == 16 ? 4 * (R & 3) : 4 * ((R >> 1) & 1)); };
  for (int e = lane; e < Cf::WARP_DOUBLES; e += 32) wsm[e] = 0.0;
  __syncwarp();

  const int lamR = DY ? pb.lam1 : 0, lamC = DY ? pb.lam2 : 0;
  const int LCm = (1 << lamC) - 1;
  const int M1c = pb.M1c, M2c = pb.M2c;
  const int M1 = M1c << lamR, NC = M2c << lamC;  // fine rows / columns
  const int nstrips = (M1 + 7) >> 3;
  const int NT8 = (NC + 3 + 7) >> 3;
  const int TRS = 8 * (NT8 + 5);  // doubles per strip top row (per pair)
  const int u_star = ((M1 - 1) & 7) >> 1, r_star = (M1 - 1) & 1;  // lane/row of the final cell
  const int64_t slot = (int64_t)blockIdx.x * WPC + warp;
  // strip top rows trow[strip][pair g][TRS] (= lane u = 3's bottom row of the
  // strip above, written in phase A, read by lane u = 0 in both phases)
  double* __restrict__ trows = ba.rowck + slot * ba.rowck_stride + (int64_t)g * TRS;
  // the lane's bottom value one column before its block boundary,
  // colck2[strip][blk][lane] (with colck: lane u-1's inputs to lane u's recompute)
  double* __restrict__ colck2 = ba.pck + slot * ba.pck_stride;
  double2* __restrict__ colck = reinterpret_cast<double2*>(ba.colck + slot * ba.colck_stride);
  double* __restrict__ arow = ba.adj + (slot * 8 + g) * ba.row_stride;
  double* __restrict__ gcs = ba.gscr + slot * ba.gscr_stride;  // column gradients [8*NT8][DP]
  // read-modified-written once per strip and block: keep it in L2
  const unsigned long long pol_keep = l2_evict_last_policy();
  const FixAcc fxR = fix_make(ba.accR, ba.metaR), fxC = fix_make(ba.accC, ba.metaC);
  double* __restrict__ rs = ba.rsum + slot * ba.rsum_stride;  // [8][M1][DP]

  for (int64_t sitem = slot; sitem < pb.nitems; sitem += (int64_t)gridDim.x * WPC) {
  int ab, chunk;
  super_item(pb, sitem, ab, chunk);
  const int a0 = pb.r0 + 8 * ab;
  const int bbeg = max(chunk * SK_SUPER_B, pb.mode == GRAM_SYM ? a0 : 0);
  const int bend = min(pb.mode == GRAM_CROSS ? pb.c1 : pb.n2, (chunk + 1) * SK_SUPER_B);
  for (int b = bbeg; b < bend; ++b) {
    const bool first_tile = b == bbeg;
    const int a = a0 + g;
    const bool valid = a < pb.r1 && !(pb.mode == GRAM_SYM && a > b);
    double wcot = 0.0;
    if (valid) {
      wcot = ba.cot[(int64_t)a * pb.n2 + b];
      if (pb.mode == GRAM_SYM && a != b) wcot += ba.cot[(int64_t)b * pb.n2 + a];
    }
    const double* __restrict__ cpath = pb.C.p + (int64_t)b * pb.C.path_stride;

    // the strip's dX (8 pairs x 8 rows) staged in shared memory: B operand of
    // the p tiles (row 8h + lane/4, component 4kk + lane%4) and of gy
    // (row 4kk + lane%4, component 8n + lane/4); both reads are conflict-free
    auto stage_x = [&](int strip) {
      for (int e = lane; e < 64 * (DP / 2); e += 32) {
        const int R = e / (DP / 2), k2 = e % (DP / 2);
        const int h = R >> 3, row = strip * 8 + (R & 7);
        const int ah = min(a0 + h, pb.r1 - 1);
        double2 v = make_double2(0.0, 0.0);
        if (row < M1)
          v = __ldg(reinterpret_cast<const double2*>(pb.R.p + (int64_t)ah * pb.R.path_stride +
                                                     (int64_t)(row >> lamR) * DP) + k2);
        *reinterpret_cast<double2*>(sX + R * XSTR + xsw(R, 2 * k2)) = v;
      }
    };
    auto loadA = [&](int T, double (&af)[KS]) {  // dY[col 8T + lane/4][4kk + lane%4], coarse tile T
      const int col = 8 * T + g;
      const double* cp = cpath + (int64_t)col * DP + u;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) af[kk] = (col >= 0 && col < M2c) ? __ldg(cp + 4 * kk) : 0.0;
    };
    auto ptile = [&](double2* ring, int slotT, int h, const double (&af)[KS]) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk)
        dmma(c0, c1, af[kk], sX[(8 * h + g) * XSTR + xsw(8 * h + g, 4 * kk + u)]);
      ring[(slotT * 8 + g) * PSTR + psw(g, 4 * h + u)] = make_double2(c0, c1);
    };
    // phase A keeps the B fragments in registers (phase B's state is not live
    // then); phase B reads them from the staged strip
    auto ptile_r = [&](double2* ring, int slotT, int h, const double (&af)[KS],
                       const double (&bf)[8][KS]) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) dmma(c0, c1, af[kk], bf[h][kk]);
      ring[(slotT * 8 + g) * PSTR + psw(g, 4 * h + u)] = make_double2(c0, c1);
    };

    // ------------------------------------------------ phase A: forward + checkpoints
    TR kval = 0;  // the pair's kernel value (fused value + gradient calls)
    // B fragments: dX of pair h, row 8 strip + lane/4, component 4kk + lane%4;
    // the next strip's are loaded one strip ahead
    double bfn[8][KS];
    auto load_bf = [&](int strip, double (&b)[8][KS]) {
      const int row = strip * 8 + g;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const int ah = min(a0 + h, pb.r1 - 1);
        const double* rp = pb.R.p + (int64_t)ah * pb.R.path_stride + (int64_t)(row >> lamR) * DP + u;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) b[h][kk] = (row < M1) ? __ldg(rp + 4 * kk) : 0.0;
      }
    };
    // (measured: the prefetch pays for d = 8, costs registers for d = 16)
    constexpr bool PFB = DP <= 8;
    if (PFB) load_bf(0, bfn);
    for (int strip = 0; strip < ((ba.exp & 2) ? 0 : nstrips); ++strip) {
      __syncwarp();
      const double* __restrict__ trow_cur = trows + (int64_t)strip * 8 * TRS;
      double* __restrict__ trow_next = trows + (int64_t)(strip + 1) * 8 * TRS;
      double bf[8][KS];
      if constexpr (PFB) {
#pragma unroll
        for (int h = 0; h < 8; ++h)
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) bf[h][kk] = bfn[h][kk];
        if (strip + 1 < nstrips) load_bf(strip + 1, bfn);
      } else {
        load_bf(strip, bf);
      }
      // phase A ring: 4 tiles, slots 0-1 in sP and 2-3 in the (idle) D region
      auto aslot = [&](int t) -> double2* {
        return ((t & 2) ? reinterpret_cast<double2*>(sD) : sP);
      };
      Frag<KS> af;
      loadA(0, af.v);
#pragma unroll
      for (int h = 0; h < 8; ++h) ptile_r(aslot(0), 0, h, af.v, bf);
      loadA(1, af.v);
#pragma unroll
      for (int h = 0; h < 8; ++h) ptile_r(aslot(1), 1, h, af.v, bf);
      // Two input streams go through shared rings HPD iterations ahead (the
      // checkpoint stores push them out of L2): the strip's top row (lane u = 0,
      // written by the strip above; in the idle dX area) and the dY rows of the
      // p tiles (A operand; in the idle staging area for d = 8, after the top
      // row ring for d = 16).  One cp.async group per iteration carries both.
      constexpr int HPD = (DP == 16) ? 3 : 4;
      constexpr int RA = HPD + 1;  // A ring depth (iterations)
      double* __restrict__ sH = sX;  // [8 iterations][8 pairs][8 columns]
      double* __restrict__ sA = (DP == 16) ? sX + 512 : sS;  // [RA][8 columns][DP]
      static_assert(DP != 16 || 512 + RA * 8 * DP <= 64 * XSTR, "A ring must fit after the top row ring");
      static_assert(DP == 16 || RA * 8 * DP <= Cf::STG, "A ring must fit in the staging area");
      auto issue_in = [&](int T) {  // top row of iteration T, dY of tile T+2
        if (strip > 0 && u == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            cp_async16(sH + (T & 7) * 64 + g * 8 + 2 * q, trow_cur + 8 * T + 2 * q, true);
        }
        if ((T & LCm) == 0) {  // coarse tile (T >> lamC) + 2 is formed at iteration T
          const int t = (T >> lamC) + 2;
#pragma unroll
          for (int e = lane; e < 8 * DP / 2; e += 32) {
            const int col = 8 * t + e / (DP / 2), q = e % (DP / 2);
            const bool v = col < M2c;
            cp_async16(sA + ((t % RA) * 8 + e / (DP / 2)) * DP + 2 * q,
                       cpath + (int64_t)(v ? col : 0) * DP + 2 * q, v);
          }
        }
        cp_async_commit();
      };
#pragma unroll
      for (int T = 0; T < HPD; ++T) issue_in(T);
      // checkpoint rows keep lane (g, u) at position 8u + g, so lane u = 3's
      // values (the strip handoff) are one contiguous 64-B quarter row
      double2* __restrict__ cck = colck + (int64_t)strip * NT8 * 32 + lane;
      double* __restrict__ cck2 = colck2 + (int64_t)strip * NT8 * 32 + lane;
      TR kl0 = 1, kl1 = 1, topc = 1, bot = 1;
      TR bprev = 1;  // the lane's bottom value one column before kl1
      const bool last = strip == nstrips - 1;
      __syncwarp();
      // one 8-step iteration; EDGE iterations hold columns outside [0, NC)
      // acur: A operand of tile T+2 (loaded two iterations ago); the buffer is
      // refilled with tile T+4's after this iteration's DMMAs
      auto iterA = [&](auto edge, int T) {
        constexpr bool EDGE = decltype(edge)::value;
        issue_in(T + HPD);
        cp_async_wait<HPD>();  // this iteration's top row and tile T+2's dY landed
        __syncwarp();          // (the dY ring is shared by the warp)
        TR hcur[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) hcur[m] = (strip > 0) ? (TR)sH[(T & 7) * 64 + g * 8 + m] : TR(1);
        const bool newtile = (T & LCm) == 0;  // (always at order 0)
        const int Tc = T >> lamC;             // coarse tile of this iteration
        double acur[KS];  // A operand of coarse tile Tc+2: dY[col 8(Tc+2) + lane/4][4kk + lane%4]
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) acur[kk] = sA[(((Tc + 2) % RA) * 8 + g) * DP + 4 * kk + u];
        // checkpoints are read back only after the whole item's forward: for
        // d = 16 stream them past L2 (evict-first; measured +0.5 %, -2.5 % at d = 8)
        // values at node column 8T - u (and the bottom one a column before):
        // read back only after the item's forward, so stream them past L2
        __stcs(cck + (int64_t)T * 32, make_double2(kl0, kl1));
        __stcs(cck2 + (int64_t)T * 32, (double)bprev);
        double2* __restrict__ r0 = aslot(T);
        double2* __restrict__ r1 = aslot(T - 1);
        const int s0 = T & 1, s1 = (T - 1) & 1;  // slot within the ring half
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          if (newtile) ptile_r(aslot(Tc + 2), (Tc + 2) & 1, m, acur, bf);  // pair m, under the recurrence
          const int c = 8 * T + m - u;
          double2 pv;
          if constexpr (DY) {  // coarse column of fine column c, its tile in the 4-slot ring
            const int jc = c >> lamC, tj = jc >> 3;
            pv = aslot(tj)[(((tj & 1) * 8) + (jc & 7)) * PSTR + psw(jc, lane)];
          } else {
            const int sl = (m - u < 0) ? s1 : s0;
            pv = ((m - u < 0) ? r1 : r0)[(sl * 8 + ((m - u) & 7)) * PSTR + psw(m - u, lane)];
          }
          TR tv = __shfl_up_sync(0xffffffffu, bot, 1, 4);
          if (u == 0) tv = hcur[m];
          if (!EDGE || (c >= 0 && c < NC)) {
            const CoefOf<TR> c0 = coef((TR)pv.x), c1 = coef((TR)pv.y);
            const TR k0 = cell(tv, kl0, topc, c0);
            const TR k1 = cell(k0, kl1, kl0, c1);
            topc = tv;
            kl0 = k0;
            bprev = kl1;
            kl1 = k1;
            bot = k1;
            if (u == 3 && !last) trow_next[c] = k1;
            if (EDGE && last && u == u_star && c == NC - 1) kval = r_star ? k1 : k0;
          }
        }
        __syncwarp();  // tile T+2 visible, tile T-1 dead
      };
      for (int T = 0; T < NT8; ++T) {
        if (T == 0 || 8 * T + 8 > NC) iterA(std::true_type{}, T);
        else iterA(std::false_type{}, T);
      }
      cp_async_wait<0>();
    }

    if (ba.values && valid && u == u_star && !(ba.exp & 2))
      ba.values[(int64_t)(a - pb.r0) * pb.ldo + (b - pb.c0)] = (double)kval;

    // ------------------------------------------------ phase B: reverse sweep
    for (int e = lane; e < 8 * NT8 * DP; e += 32) gcs[e] = 0.0;
    for (int strip = nstrips - 1; strip >= ((ba.exp & 1) ? nstrips : 0); --strip) {
      __syncwarp();
      stage_x(strip);
      __syncwarp();
      const int rb = strip * 8 + 2 * u;  // lane's first fine row (0-based)
      const bool fin0 = (rb == M1 - 1), fin1 = (rb + 1 == M1 - 1);
      const double* __restrict__ trow_cur = trows + (int64_t)strip * 8 * TRS;
      const double2* __restrict__ cck0 = colck + (int64_t)strip * NT8 * 32;
      const double* __restrict__ cck20 = colck2 + (int64_t)strip * NT8 * 32;
      const bool below = strip < nstrips - 1;

      // block inputs staged by cp.async one block ahead: lane u = 0's top row
      // tv[i] = node column 8blk+i of the strip's top row (i = 0..8), every
      // lane's two values at its node column 8blk-u and its bottom value a
      // column before (lane u > 0 starts its recompute from lane u-1's), and
      // (lane u = 3) the adjoint messages of the strip below at columns
      // 8blk-3 .. 8blk+4, which arow holds at index column + 3
      auto stage_block = [&](int blk) {
        double* st = sS;
        if (u == 0) {
#pragma unroll
          for (int i = 0; i < 9; ++i)
            cp_async8(st + i * 32 + lane, trow_cur + max(8 * blk - 1 + i, 0), strip > 0);
        }
        cp_async16(st + 9 * 32 + 2 * lane, cck0 + (int64_t)blk * 32 + lane, true);
        cp_async8(st + 11 * 32 + 64 + lane, cck20 + (int64_t)blk * 32 + lane, true);
        if (u == 3) {
#pragma unroll
          for (int i = 0; i < 8; i += 2)
            cp_async16(st + 11 * 32 + g * 8 + i, arow + 8 * blk + i, below);
        }
        cp_async_commit();
      };
      auto loadGX = [&](int T, double (&gb)[2][NN]) {  // dY[col 8T + 4kk + lane%4][8n + lane/4]
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int col = 8 * T + 4 * kk + u;  // fine column; its coarse dY
#pragma unroll
          for (int n = 0; n < NN; ++n)
            gb[kk][n] = (col >= 0 && col < NC) ? __ldg(cpath + (int64_t)(col >> lamC) * DP + 8 * n + g)
                                               : 0.0;
        }
      };

      double gx[8][NN][2];
#pragma unroll
      for (int h = 0; h < 8; ++h)
#pragma unroll
        for (int n = 0; n < NN; ++n) gx[h][n][0] = gx[h][n][1] = 0.0;
      {
        // coarse tiles of the last block and the one before (order 0: blocks)
        const int Tl = (NT8 - 1) >> lamC;
        double af[KS];
        loadA(Tl, af);
#pragma unroll
        for (int h = 0; h < 8; ++h) ptile(sP, Tl & 1, h, af);
        loadA(Tl - 1, af);
#pragma unroll
        for (int h = 0; h < 8; ++h) ptile(sP, (Tl - 1) & 1, h, af);
      }
      stage_block(NT8 - 1);
      double aR0 = 0.0, aR1 = 0.0, bR0 = 0.0, bR1 = 0.0, sendm = 0.0;
      // F32: the right neighbours' adjoints and A / B corrections, and the
      // two-part message (main, correction) to lane u-1
      float lR0 = 0.f, lR1 = 0.f, aC0 = 0.f, aC1 = 0.f, bC0 = 0.f, bC1 = 0.f, sM = 0.f, sC = 0.f;

      // gx += D dY for one k-half and four pairs of tile t (D slot t & 1)
      double gbp[2][NN];  // SK_GX_DEFER: tile blk + 1's gx B operand, mapped in blk's sweep
      auto gx_part = [&](int t, const double (&gbx)[2][NN], int kk, int h0) {
        const double* __restrict__ Dx = sD + (t & 1) * Cf::DTILE;
#pragma unroll
        for (int h = h0; h < h0 + 4; ++h) {
          const double av_ = Dx[(4 * kk + u) * DSTR + dsw(u, 8 * h + g)];
#pragma unroll
          for (int n = 0; n < NN; ++n) dmma(gx[h][n][0], gx[h][n][1], av_, gbx[kk][n]);
        }
      };
      // one block; EDGE blocks hold columns outside [0, NC) or the final cell
      auto blockB = [&](auto edge, int blk) {
        constexpr bool EDGE = decltype(edge)::value;
        double af[KS], gb[2][NN];
        // coarse tile Tc - 2 is formed after the sweep of Tc's leftmost block
        const bool lefttile = (blk & LCm) == 0;  // (always at order 0)
        const int Tcb = blk >> lamC;
        loadA(Tcb - 2, af);
        loadGX(blk, gb);      // gx B operand of tile blk
        cp_async_wait<0>();
        __syncwarp();         // staged inputs, p tiles blk and blk-1 visible
        const double* st = sS;
        double2 gco[NN];  // column-gradient scratch of tile blk, read early
#pragma unroll
        for (int n = 0; n < NN; ++n)
          gco[n] = ld_l2hint(reinterpret_cast<const double2*>(gcs + (int64_t)(8 * blk + g) * DP + 8 * n + 2 * u),
                             pol_keep);
        // the row above the lane: lane u = 0 from the strip's top row; lane
        // u > 0 starts from lane u-1's checkpoints (node columns 8blk-u,
        // 8blk-u+1) and receives the rest from lane u-1's recompute below
        TR tv[9];
        if (u == 0) {
#pragma unroll
          for (int i = 0; i < 9; ++i) {
            const TR v = (strip == 0) ? TR(1) : (TR)st[i * 32 + lane];
            if constexpr (EDGE) {
              const int cc = 8 * blk + i;
              tv[i] = (cc <= 0) ? TR(1) : (cc > NC ? TR(0) : v);
            } else {
              tv[i] = v;
            }
          }
        } else {
          tv[0] = (TR)st[11 * 32 + 64 + lane - 1];
          tv[1] = (TR)st[9 * 32 + 2 * (lane - 1) + 1];
#pragma unroll
          for (int i = 2; i < 9; ++i) tv[i] = TR(0);
        }
        const double2 kleft2 = *reinterpret_cast<const double2*>(st + 9 * 32 + 2 * lane);
        const TR kleftx = (TR)kleft2.x, klefty = (TR)kleft2.y;
        // lane u = 3: adjoint messages of the strip below (F32: a float2
        // (main, correction) in each fp64 slot)
        double av[8];
        float2 avf[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if constexpr (F32) {
            avf[i] = *reinterpret_cast<const float2*>(st + 11 * 32 + g * 8 + i);
            if (EDGE && 8 * blk - 3 + i < 0) avf[i] = make_float2(0.f, 0.f);
          } else {
            av[i] = st[11 * 32 + g * 8 + i];
            if (EDGE && 8 * blk - 3 + i < 0) av[i] = 0.0;  // left of column 0: never written
          }
        }
        // refill the staging records for block blk-1 (lanes read lane u-1's)
        __syncwarp();
        if (blk > 0) stage_block(blk - 1);

        // ---- 1. recompute the lane's 2 x 8 forward values (registers): the
        // skewed wavefront of phase A over the block (lane u-1's bottom row
        // arrives by shuffle one step ahead), bitwise phase A's values
        TR K0[8], K1[8];
        {
          TR k0 = kleftx, k1 = klefty;
#pragma unroll
          for (int kap = 0; kap < 8; ++kap) {
            if (kap > 0) {
              const TR sh = __shfl_up_sync(0xffffffffu, k1, 1, 4);
              if (u > 0) tv[kap + 1] = sh;
            }
            const int c = 8 * blk - u + kap;
            const int jc = c >> lamC;  // coarse column
            double2 pv = sP[((((jc >> 3) & 1) * 8) + (jc & 7)) * PSTR + psw(jc, lane)];
            if (EDGE && (c < 0 || c >= NC)) pv = make_double2(0.0, 0.0);
            const CoefOf<TR> c0 = coef((TR)pv.x), c1 = coef((TR)pv.y);
            const TR n0 = cell(tv[kap + 1], k0, tv[kap], c0);
            const TR n1 = cell(n0, k1, k0, c1);
            k0 = n0;
            k1 = n1;
            K0[kap] = n0;
            K1[kap] = n1;
          }
        }


        // ---- 2. reverse sweep, lane u one column behind lane u+1.  Dead rows
        // (>= M1) and columns (>= NC) lie below / right of the seeded final
        // cell, so their adjoint is exactly 0 without masking; columns < 0
        // (block 0) only feed D slots that are never consumed.
#pragma unroll
        for (int kap = 7; kap >= 0; --kap) {
          if (SK_GX_DEFER && kap >= 4 && blk + 1 < NT8 && !(ba.exp & 4))
            gx_part(blk + 1, gbp, (7 - kap) >> 1, ((7 - kap) & 1) * 4);
          // tile blk+1's D is read (above) before this sweep stores tile
          // blk-1's columns into the same slot (lanes u > kap, kap <= 2)
          if (SK_GX_DEFER && kap == 3) __syncwarp();
          const int c = 8 * blk - u + kap;
          const int jc = c >> lamC;
          double2 pv = sP[((((jc >> 3) & 1) * 8) + (jc & 7)) * PSTR + psw(jc, lane)];
          if (EDGE && (c < 0 || c >= NC)) pv = make_double2(0.0, 0.0);
          TR lam1, lam0;
          if constexpr (F32) {
            // small-correction adjoint (A = 1 + Ap, B = 1 - q): every cell's
            // pushes split into an O(lambda) main part and an O(p lambda)
            // correction, summed separately (the fp32 rounding of A, B would
            // otherwise swallow the p ~ 1e-3 terms); the message to lane u-1
            // is (lam0 - lamR0, a0 + bR0): below-push + diagonal-push of the
            // row above's cell
            float rM = __shfl_down_sync(0xffffffffu, sM, 1, 4);
            float rC = __shfl_down_sync(0xffffffffu, sC, 1, 4);
            if (u == 3) {
              rM = avf[kap].x;
              rC = avf[kap].y;
            }
            const Coef32 c0 = coef((float)pv.x), c1 = coef((float)pv.y);
            float m1 = lR1 + rM;
            if (EDGE && fin1 && c == NC - 1) m1 += (float)wcot;
            lam1 = m1 + (aC1 + rC);
            const float a1 = lam1 * c1.Ap;
            float m0 = lR0 + (lam1 - lR1);
            if (EDGE && fin0 && c == NC - 1) m0 += (float)wcot;
            lam0 = m0 + (aC0 + (a1 + bC1));
            const float a0 = lam0 * c0.Ap;
            sM = lam0 - lR0;
            sC = a0 + bC0;
            lR1 = lam1;
            aC1 = a1;
            bC1 = lam1 * c1.q;
            lR0 = lam0;
            aC0 = a0;
            bC0 = lam0 * c0.q;
          } else {
          double recv = __shfl_down_sync(0xffffffffu, sendm, 1, 4);
          if (u == 3) recv = av[kap];
          const Coef c0 = coef(pv.x), c1 = coef(pv.y);
          if constexpr (EDGE || SK_AFFINE_MSG == 0) {
            // rows 1 then 0, the message chain as written (final-cell seed here)
            lam1 = aR1 + recv;
            if (EDGE && fin1 && c == NC - 1) lam1 += wcot;
            lam0 = aR0 + (c1.A * lam1 - bR1);
            if (EDGE && fin0 && c == NC - 1) lam0 += wcot;
            sendm = c0.A * lam0 - bR0;
          } else {
            // the message to lane u-1 is affine in recv: one FMA on the
            // lane-to-lane critical path instead of six dependent operations
            const double R0 = aR0 + fma(c1.A, aR1, -bR1);  // lam0 - A1 recv
            const double P = c0.A * c1.A, Q = fma(c0.A, R0, -bR0);
            sendm = fma(P, recv, Q);
            lam1 = aR1 + recv;
            lam0 = fma(c1.A, recv, R0);
          }
          aR1 = c1.A * lam1;
          bR1 = c1.B * lam1;
          aR0 = c0.A * lam0;
          bR0 = c0.B * lam0;
          }
          const TR kL1 = kap > 0 ? K1[kap - 1] : klefty;
          const TR kD1 = kap > 0 ? K0[kap - 1] : kleftx;
          const TR p61 = (TR)pv.y * TR(1.0 / 6.0);
          const TR D1 = lam1 * fma(kL1 + K0[kap], TR(0.5) + p61, kD1 * p61);
          const TR kL0 = kap > 0 ? K0[kap - 1] : kleftx;
          const TR p60 = (TR)pv.x * TR(1.0 / 6.0);
          const TR D0 = lam0 * fma(kL0 + tv[kap + 1], TR(0.5) + p60, tv[kap] * p60);
          // columns outside [0, NC) store exact zeros: their slots are read by
          // the tile maps as dead columns later (x 0 dY), so no garbage (e.g.
          // the never-written adjoint messages left of column 0) may reach them
          const bool cdead = EDGE && (c < 0 || c >= NC);
          *reinterpret_cast<double2*>(sD + ((c >> 3) & 1) * Cf::DTILE + (c & 7) * DSTR +
                                      dsw(c, 2 * lane)) =
              cdead ? make_double2(0.0, 0.0) : make_double2((double)D0, (double)D1);
          if (u == 0 && (!EDGE || c >= 0)) {
            if constexpr (F32) *reinterpret_cast<float2*>(arow + c + 3) = make_float2(sM, sC);
            else arow[c + 3] = sendm;
          }
        }
        __syncwarp();  // tile blk's D complete, p tile blk dead

        // ---- 3. p tile blk-2 into tile blk's slot (its latency hides under the
        // maps), then the gradient maps on tile blk
#pragma unroll
        for (int h = 0; h < 8 && !(ba.exp & 8) && lefttile; h += 8) {
          // all 8 pairs' chains side by side, k-step outermost (same per-chain
          // order as ptile, so the values are unchanged)
          double c[8][2];
#pragma unroll
          for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
#pragma unroll
          for (int kk = 0; kk < KS; ++kk)
#pragma unroll
            for (int q = 0; q < 8; ++q)
              dmma(c[q][0], c[q][1], af[kk], sX[(8 * q + g) * XSTR + xsw(8 * q + g, 4 * kk + u)]);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            sP[(((Tcb & 1) * 8 + g) * PSTR) + psw(g, 4 * q + u)] = make_double2(c[q][0], c[q][1]);
        }
        const double* __restrict__ Dt = sD + (blk & 1) * Cf::DTILE;
        if (!(ba.exp & 4)) {
        if (!SK_GX_DEFER) {
#pragma unroll
          for (int q = 0; q < 4; ++q) gx_part(blk, gb, q >> 1, (q & 1) * 4);
        }
        // gy = D^T dX over the tile's 64 rows: four independent DMMA chains per
        // component tile, all chains side by side (fixed order: deterministic)
        {
          double c[NN][4][2];
#pragma unroll
          for (int n = 0; n < NN; ++n)
#pragma unroll
            for (int j = 0; j < 4; ++j) c[n][j][0] = c[n][j][1] = 0.0;
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) {
            const double a_ = Dt[g * DSTR + dsw(g, 4 * kk + u)];
#pragma unroll
            for (int n = 0; n < NN; ++n)
              dmma(c[n][kk & 3][0], c[n][kk & 3][1], a_,
                   sX[(4 * kk + u) * XSTR + xsw(4 * kk + u, 8 * n + g)]);
          }
#pragma unroll
          for (int n = 0; n < NN; ++n)
            st_l2hint(reinterpret_cast<double2*>(gcs + (int64_t)(8 * blk + g) * DP + 8 * n + 2 * u),
                      make_double2(gco[n].x + ((c[n][0][0] + c[n][1][0]) + (c[n][2][0] + c[n][3][0])),
                                   gco[n].y + ((c[n][0][1] + c[n][1][1]) + (c[n][2][1] + c[n][3][1]))),
                      pol_keep);
        }
        }
        if (SK_GX_DEFER) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
#pragma unroll
            for (int n = 0; n < NN; ++n) gbp[kk][n] = gb[kk][n];
        }
        __syncwarp();
      };
      for (int blk = NT8 - 1; blk >= 0; --blk) {
        if (blk == 0 || 8 * blk + 8 >= NC) blockB(std::true_type{}, blk);
        else blockB(std::false_type{}, blk);
      }
      if (SK_GX_DEFER && !(ba.exp & 4)) {  // block 0's gx map (D slot 0 is intact)
#pragma unroll
        for (int q = 0; q < 4; ++q) gx_part(0, gbp, q >> 1, (q & 1) * 4);
      }

      // row-side increment gradients of the strip into the super-item's sums
      // (b ascending; flushed once per super-item below)
      const int rho = strip * 8 + g;
      if (rho < M1) {
#pragma unroll
        for (int h = 0; h < 8; ++h) {
#pragma unroll
          for (int n = 0; n < NN; ++n) {
            double2* q = reinterpret_cast<double2*>(rs + ((int64_t)h * M1 + rho) * DP + 8 * n + 2 * u);
            double2 v = make_double2(gx[h][n][0], gx[h][n][1]);
            if constexpr (DY) {  // dY is unscaled: dp/d(dx) carries the dyadic factor (exact)
              v.x *= pb.scale;
              v.y *= pb.scale;
            }
            if (!first_tile) {
              const double2 o = *q;
              v = make_double2(o.x + v.x, o.y + v.y);
            }
            *q = v;
          }
        }
      }
    }
    __syncwarp();

    // column-side gradient (summed over the tile's pairs and strips), telescoped
    {
      const int dR = ba.d;
      const int64_t gC = (int64_t)b * ba.gC_path;
      // (dyadic: the fine columns of a coarse column summed first, ascending)
      auto csum = [&](int j, int k) {
        double a = gcs[(int64_t)(j << lamC) * DP + k];
        for (int c = (j << lamC) + 1; c < ((j + 1) << lamC); ++c) a += gcs[(int64_t)c * DP + k];
        return a;
      };
      for (int e = lane; e < (M2c + 1) * dR; e += 32) {
        const int p = e / dR, k = e % dR;
        double v = 0.0;
        if (p >= 1) v += csum(p - 1, k);
        if (p < M2c) v -= csum(p, k);
        fix_add(fxC, gC + e, v);
      }
    }
    __syncwarp();
  }  // tiles of the super-item
  // row-side gradients of the super-item's 8 paths, telescoped to points
  // (kernel_grad.py:55-60: point r gets g[r-1] - g[r]) and flushed once
  {
    const int dR = ba.d;
    for (int h = 0; h < 8; ++h) {
      const int ah = a0 + h;
      if (ah >= pb.r1 || bbeg >= bend) continue;  // warp-uniform
      const double* rh = rs + (int64_t)h * M1 * DP;
      const int64_t gp = (int64_t)ah * ba.gR_path;
      auto rsumc = [&](int i, int k) {  // fine rows of coarse row i, ascending
        double a = rh[(int64_t)(i << lamR) * DP + k];
        for (int r = (i << lamR) + 1; r < ((i + 1) << lamR); ++r) a += rh[(int64_t)r * DP + k];
        return a;
      };
      for (int e = lane; e < (M1c + 1) * dR; e += 32) {
        const int p = e / dR, k = e % dR;
        double v = 0.0;
        if (p >= 1) v += rsumc(p - 1, k);
        if (p < M1c) v -= rsumc(p, k);
        fix_add(fxR, gp + e, v);
      }
    }
    __syncwarp();
  }
  }  // super-items
}

}  // namespace sk
