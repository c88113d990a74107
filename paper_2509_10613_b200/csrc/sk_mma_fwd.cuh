// sk_mma_fwd.cuh -- Gram forward with the increment products on the FP64
// tensor cores (DMMA) and the Goursat recurrence on the FP64 FMA pipe.
//
// Replaces goursat_gram (/root/reference/pkg/src/sigcore/_kernels.py:408-429)
// for the linear static kernel at dyadic order 0 (the BASELINE Gram configs
// C3 and C5).  The reference forms delta = dx[a] @ dyt[b] per pair with BLAS
// (_kernels.py:426) and marches it in strips (_kernels.py:293-338).
//
// Why DMMA: on B200 mma.m8n8k4.f64 runs at the DFMA rate on the same pipe
// (tools/dmma_probe.cu: 1.85e13 FMA/s either way), so it does not raise the
// FP64 ceiling -- but one DMMA issues 256 FMAs, so the d FMAs per cell of
// <dx_i, dy_j> stop competing with the recurrence for issue slots.  The
// forward kernels of r01 were issue/latency bound at 24-36 % of the pipe with
// ~87 instructions per cell for 23 FP64 operations (profiles/r01_*).
//
// Mapping (one warp = one Gram tile of 8 pairs (a0+g, b), g = lane / 4):
//   * lane (g, u = lane % 4) owns fine rows 2u, 2u+1 of pair g's 8-row strip
//     and runs one column behind lane u-1 (skewed register wavefront, top
//     values by __shfl_up_sync within the 4-lane group);
//   * increment products come in 8-column tiles: p^T(8 cols x 8 rows of pair h)
//     = dY(8 x DP) . dX_h^T(DP x 8), DP/4 DMMAs per pair h.  The dX fragments of
//     the strip stay in registers (B operand, lane holds row lane/4, k lane%4),
//     the dY fragments stream from global one tile ahead;
//   * the mma groupID (lane / 4) is the tile column and the C fragment holds
//     rows 2(lane%4), 2(lane%4)+1, i.e. exactly a wavefront lane's two rows:
//     fragments go through a 4-tile shared-memory ring as one 16-byte store
//     and come back as one 16-byte load per lane and column (conflict-free);
//   * tile T+2 is computed during the 8 steps of tile T (one pair h per step),
//     so the tensor-core work is spread evenly under the recurrence;
//   * the strip's bottom row goes to the next strip through a per-pair row in
//     global memory (L2), prefetched 8 columns ahead by lane u = 0.
// p is formed as ONE sequential FMA chain over k (the DMMA's own order), the
// same as sk_cell.cuh dot(), so these values are bitwise those of the batch
// kernels.
#pragma once
#include <type_traits>

#include "sk_cell.cuh"

namespace sk {

// D += A * B for one m8n8k4 f64 tile (A: 8x4 row, lane holds A[lane/4][lane%4];
// B: 4x8 col, lane holds B[lane%4][lane/4]; C/D: lane holds C[lane/4][2(lane%4)+{0,1}]).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

struct MmaFwdCfg {
  static constexpr int PSTR = 36;             // double2 per tile column: 32 lanes + 4 (bank spread)
  static constexpr int TILE = 8 * PSTR;       // double2 per tile
  static constexpr int RING = 4;              // tiles in flight per warp
  static constexpr int WARP_BYTES = RING * TILE * 16;
  static constexpr int THREADS = 128;
};

//   DY  dyadic orders > 0 (runtime lam1 / lam2); false: order 0 at compile
//       time, so the order-0 instance (C3, C5) carries no index shifts
//   TR  the recurrence's arithmetic type: double, or float for the FP32
//       kernels (p from the fp64 DMMA, rounded once to float; the cell in the
//       small-correction form of sk_cell.cuh Coef32); the handoff rows and
//       the output are TR
template <int DP, bool DY = false, typename TR = double>
__global__ void __launch_bounds__(MmaFwdCfg::THREADS, DP >= 32 ? 2 : 3)
gram_fwd_mma(Problem pb, double* __restrict__ hand, int64_t hand_stride) {
  constexpr int KS = DP / 4;
  constexpr int PSTR = MmaFwdCfg::PSTR;
  extern __shared__ double2 smem_mf[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, u = lane & 3;
  double2* __restrict__ sP = smem_mf + (size_t)warp * MmaFwdCfg::RING * MmaFwdCfg::TILE;

  // dyadic orders (round 2): fine rows / columns, coarse = fine >> lam.  The
  // p tiles are coarse (8 coarse columns); their B operand row r is the coarse
  // row of the strip's fine row r, so the C fragment of lane (g, u) still holds
  // p of the lane's two fine rows (duplicated coarse rows cost redundant DMMA
  // work, no layout change); a coarse tile spans 8 << lam2 fine columns and is
  // formed during the first 8-column iteration of the tile two ahead.
  const int lamR = DY ? pb.lam1 : 0, lamC = DY ? pb.lam2 : 0;
  const int M1 = pb.M1c << lamR, NC = pb.M2c << lamC;  // fine rows / columns
  const int M2c = pb.M2c;
  const int LCm = (1 << lamC) - 1;
  const int nstrips = (M1 + 7) >> 3;
  const int NT8 = (NC + 3 + 7) >> 3;  // 8-step iterations per strip (skew 3)
  const int u_star = ((M1 - 1) & 7) >> 1, r_star = (M1 - 1) & 1;
  const int64_t slot = (int64_t)blockIdx.x * nw + warp;
  TR* __restrict__ hrow = reinterpret_cast<TR*>(hand) + (slot * 8 + g) * hand_stride;
  // two consecutive handoff values (8- or 16-byte aligned: m even)
  auto load2 = [](const TR* p, TR& a, TR& b) {
    if constexpr (sizeof(TR) == 8) {
      const double2 t = *reinterpret_cast<const double2*>(p);
      a = t.x;
      b = t.y;
    } else {
      const float2 t = *reinterpret_cast<const float2*>(p);
      a = t.x;
      b = t.y;
    }
  };

  for (int64_t item = slot; item < pb.nitems; item += (int64_t)gridDim.x * nw) {
    int a0, b;
    gram_item(pb, item, 8, a0, b);
    const int a = a0 + g;
    const bool valid = a < pb.r1 && !(pb.mode == GRAM_SYM && a > b);
    const double* __restrict__ cpath = pb.C.p + (int64_t)b * pb.C.path_stride;
    TR kval = 0;

    for (int strip = 0; strip < nstrips; ++strip) {
      __syncwarp();  // previous strip's handoff row and ring reads are done
      // B fragments: dX of pair h, row strip*8 + lane/4, component 4kk + lane%4
      double bf[8][KS];
      {
        const int row = strip * 8 + g;    // fine row
        const int crow = row >> lamR;      // its coarse row
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int ah = min(a0 + h, pb.r1 - 1);
          const double* rp = pb.R.p + (int64_t)ah * pb.R.path_stride + (int64_t)crow * DP + u;
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) bf[h][kk] = (row < M1) ? __ldg(rp + 4 * kk) : 0.0;
        }
      }
      auto loadA = [&](int T, double (&af)[KS]) {  // coarse tile T: coarse columns 8T + g
        const int col = 8 * T + g;
        const double* cp = cpath + (int64_t)col * DP + u;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) af[kk] = (col < M2c) ? __ldg(cp + 4 * kk) : 0.0;
      };
      auto tile = [&](int T, int h, const double (&af)[KS]) {
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) dmma(c0, c1, af[kk], bf[h][kk]);
        sP[((T & 3) * 8 + g) * PSTR + 4 * h + u] = make_double2(c0, c1);
      };
      double af[KS], an[KS];
      loadA(0, af);
#pragma unroll
      for (int h = 0; h < 8; ++h) tile(0, h, af);
      loadA(1, af);
#pragma unroll
      for (int h = 0; h < 8; ++h) tile(1, h, af);
      loadA(2, af);
      TR hcur[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) hcur[m] = TR(1);
      if (strip > 0 && u == 0) {
#pragma unroll
        for (int m = 0; m < 8; m += 2) {
          load2(hrow + m, hcur[m], hcur[m + 1]);
        }
      }
      __syncwarp();
      // p of fine column c: coarse column jc = c >> lamC, tile jc >> 3 (c < 0:
      // arithmetic shift keeps the skewed lanes' dead columns in tile -1)
      auto pslot = [&](int c) {
        const int jc = c >> lamC;
        return (((jc >> 3) & 3) * 8 + (jc & 7)) * PSTR + lane;
      };
      double2 pcur = sP[pslot(0 - u)];
      TR kl0 = 1, kl1 = 1, topc = 1, bot = 1;
      const bool last = strip == nstrips - 1;

      // one 8-step iteration; EDGE iterations hold columns outside [0, NC) or
      // the final column (the only ones that need range checks)
      auto iter = [&](auto edge, int T) {
        constexpr bool EDGE = decltype(edge)::value;
        // coarse tile Tc + 2 is formed in the first fine iteration of tile Tc
        const bool newtile = (T & LCm) == 0;
        const int Tc = T >> lamC;
        if (newtile) loadA(Tc + 3, an);
        TR hnxt[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) hnxt[m] = TR(1);
        if (strip > 0 && u == 0) {
#pragma unroll
          for (int m = 0; m < 8; m += 2) {
            load2(hrow + 8 * (T + 1) + m, hnxt[m], hnxt[m + 1]);
          }
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          if (newtile) tile(Tc + 2, m, af);
          const int c = 8 * T + m - u;  // this lane's (fine) column
          const double2 pv = pcur;
          pcur = sP[pslot(c + 1)];
          TR tv = __shfl_up_sync(0xffffffffu, bot, 1, 4);
          if (u == 0) tv = hcur[m];
          if (!EDGE || (c >= 0 && c < NC)) {
            const CoefOf<TR> c0 = coef((TR)pv.x), c1 = coef((TR)pv.y);
            const TR k0 = cell(tv, kl0, topc, c0);
            const TR k1 = cell(k0, kl1, kl0, c1);
            topc = tv;
            kl0 = k0;
            kl1 = k1;
            bot = k1;
            if (u == 3 && !last) hrow[c] = k1;
            if (EDGE && last && u == u_star && c == NC - 1) kval = r_star ? k1 : k0;
          }
        }
        if (newtile) {
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) af[kk] = an[kk];
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) hcur[m] = hnxt[m];
        __syncwarp();  // tile T+2 visible; tile T-2's slot free
      };
      for (int T = 0; T < NT8; ++T) {
        if (T == 0 || 8 * T + 8 >= NC) iter(std::true_type{}, T);
        else iter(std::false_type{}, T);
      }
    }
    if (valid && u == u_star) reinterpret_cast<TR*>(pb.out)[(int64_t)(a - pb.r0) * pb.ldo + b] = kval;
  }
}

}  // namespace sk
