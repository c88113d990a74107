// sk_small.cu -- forward for few short pairs (BASELINE config 1: 32 pairs,
// L = 64, d = 4): the latency regime, where one pair's wavefront is the whole
// cost of a call.
//
// The general batch kernel streams column records through a cp.async ring and
// forms p = <dx_i, dy_j> and A(p), B(p) inside the wavefront step, so each of
// its ~60-90 dependent steps pays a dot product, the coefficients and the
// ring bookkeeping on the critical path (measured 28 us per C1 call on an
// otherwise idle GPU).  Here one CTA solves one pair in two phases:
//   1. the pair's increments (the same subtraction and exact dyadic scale as
//      the prep kernel, kernel.py:74-75) and the coefficient tile
//      A, B (p_ij) for every coarse cell go to shared memory -- independent
//      work, four warps, independent chains (dot in the sequential FMA order of
//      sk_cell.cuh, so p, A, B and the values are bitwise the other kernels');
//   2. one warp runs the skewed register wavefront (lane u owns fine rows 2u+1, 2u+2, one
//      column behind lane u-1, bottom values by __shfl_up_sync) reads A, B
//      from the tile: two cells per step on the critical path.
// No workspace, no prep launch.  Linear static kernel, no transform, up to 64
// fine rows on the longer axis (the tile then holds at most 64 x 64 coarse
// cells); reference: _kernels.py:286-338 (cell, strip recurrence).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "sk_cell.cuh"
#include "sk_plan.h"

namespace sk {

template <int DP>
__global__ void __launch_bounds__(128)
small_fwd_kernel(const double* __restrict__ xr, const double* __restrict__ xc, int64_t B,
                 int LR, int LC, int d, int lamR, int lamC, double scale,
                 double* __restrict__ out) {
  extern __shared__ double smem_small[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int M1c = LR - 1, M2c = LC - 1;
  const int M1 = M1c << lamR, M2 = M2c << lamC;
  double* __restrict__ dyc = smem_small;                                  // [M2c][DP]
  double2* __restrict__ ab = reinterpret_cast<double2*>(dyc + M2c * DP);  // [M2c][M1c]
  const int u_star = (M1 - 1) >> 1, r_star = (M1 - 1) & 1;
#ifdef SK_SMALL_CLOCKS
  long long c0_ = clock64(), c1_ = 0, c2_ = 0, c3_ = 0;
#endif
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    const double* xp = xr + b * (int64_t)LR * d;
    const double* yp = xc + b * (int64_t)LC * d;
    __syncthreads();  // the previous pair's tile is consumed
    for (int e = tid; e < M2c * DP; e += blockDim.x) {
      const int j = e / DP, k = e % DP;
      dyc[e] = (k < d) ? (yp[(j + 1) * d + k] - yp[j * d + k]) * 1.0 : 0.0;
    }
    // 1. coefficient tile, all four warps: thread owns coarse row tid % 64
    //    and every second coarse column from tid / 64, two columns per
    //    iteration (independent dot / coef chains)
    double dx[DP];
    const int i = tid & 63, jp = tid >> 6;
    const bool iv = i < M1c;
#pragma unroll
    for (int k = 0; k < DP; ++k)
      dx[k] = (iv && k < d) ? (xp[(i + 1) * d + k] - xp[i * d + k]) * scale : 0.0;
    __syncthreads();
#ifdef SK_SMALL_CLOCKS
    c1_ = clock64();
#endif
    if (iv) {
      for (int j = jp; j < M2c; j += 4) {
        const int j1 = min(j + 2, M2c - 1);
        double dy0[DP], dy1[DP];
#pragma unroll
        for (int k = 0; k < DP; ++k) {
          dy0[k] = dyc[j * DP + k];
          dy1[k] = dyc[j1 * DP + k];
        }
        const Coef c0 = coef(dot<DP>(dx, dy0)), c1 = coef(dot<DP>(dx, dy1));
        ab[j * M1c + i] = make_double2(c0.A, c0.B);
        ab[j1 * M1c + i] = make_double2(c1.A, c1.B);
      }
    }
    __syncthreads();
#ifdef SK_SMALL_CLOCKS
    c2_ = clock64();
#endif
    // 2. wavefront (warp 0): lane u, fine rows s0 = 2u+1, s1 = 2u+2 (1-based),
    //    column t = tau - u + 1 at step tau; row 0 and column 0 are the boundary
    if (tid < 32) {
      const int i0 = min((2 * lane) >> lamR, M1c - 1), i1 = min((2 * lane + 1) >> lamR, M1c - 1);
      // branch-free steps (inactive lanes compute and discard), the next
      // step's coefficients loaded one step ahead: the lane chain is the
      // shuffle and four dependent FP64 operations per step (measured: 180 ->
      // 123 cycles per step; two columns per step measured 203)
      double kl0 = 1.0, kl1 = 1.0, topc = 1.0, bot = 1.0;
      const int nsteps = M2 + 31;
      auto coefs_at = [&](int t, double2& a0, double2& a1) {
        const int jc = min(max(t - 1, 0), M2 - 1) >> lamC;
        a0 = ab[jc * M1c + i0];
        a1 = ab[jc * M1c + i1];
      };
      double2 n0, n1;
      coefs_at(1 - lane, n0, n1);
#pragma unroll 2
      for (int tau = 0; tau < nsteps; ++tau) {
        const int t = tau - lane + 1;
        const double2 c0 = n0, c1 = n1;
        coefs_at(t + 1, n0, n1);
        double top = __shfl_up_sync(0xffffffffu, bot, 1);
        if (lane == 0) top = 1.0;
        const double k0 = cell(top, kl0, topc, Coef{c0.x, c0.y});
        const double k1 = cell(k0, kl1, kl0, Coef{c1.x, c1.y});
        const bool act = t >= 1 && t <= M2;
        topc = act ? top : topc;
        kl0 = act ? k0 : kl0;
        kl1 = act ? k1 : kl1;
        bot = act ? k1 : bot;
      }
      // column M2 is the lane's last: its row values are the final ones
      if (lane == u_star) out[b] = r_star ? kl1 : kl0;
    }
  }
#ifdef SK_SMALL_CLOCKS
  c3_ = clock64();
  if (tid == 0 && blockIdx.x == 0) printf("small_fwd cycles: load %lld, tile %lld, wave %lld\n", c1_ - c0_, c2_ - c1_, c3_ - c2_);
#endif
}

// dynamic shared memory of the tile (bytes)
static int small_smem(int DP, int64_t M1c, int64_t M2c) {
  return (int)(M2c * DP * sizeof(double) + M2c * M1c * 2 * sizeof(double));
}

// Launches the small-pair forward when it applies (returns false otherwise):
// rows = the longer fine axis (oriented by the caller), DP <= 32 single chunk.
bool launch_small_fwd(const double* xr, const double* xc, int64_t B, int64_t LR, int64_t LC,
                      int64_t d, int lamR, int lamC, double scale, double* out, int sms,
                      cudaStream_t st) {
  const int64_t M1 = (LR - 1) << lamR, M2 = (LC - 1) << lamC;
  if (M1 > 64 || M2 > 64 || d > 32 || B < 1) return false;
  const int DP = d <= 4 ? 4 : d <= 8 ? 8 : d <= 16 ? 16 : 32;
  const int smem = small_smem(DP, LR - 1, LC - 1);
  const void* fn = DP == 4    ? (const void*)small_fwd_kernel<4>
                   : DP == 8  ? (const void*)small_fwd_kernel<8>
                   : DP == 16 ? (const void*)small_fwd_kernel<16>
                              : (const void*)small_fwd_kernel<32>;
  static bool opted[64][4] = {};  // per device and instance
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    (void)cudaGetLastError();
    dev = 0;
  }
  const int slot = DP == 4 ? 0 : DP == 8 ? 1 : DP == 16 ? 2 : 3;
  if (!opted[dev][slot]) {
    // the largest tile (64 x 64 coarse cells + 64 rows of DP) fits under this
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024) !=
        cudaSuccess) {
      (void)cudaGetLastError();
      return false;
    }
    opted[dev][slot] = true;
  }
  const unsigned grid = (unsigned)std::min<int64_t>(B, (int64_t)sms * 4);
  const int Li = (int)LR, Lc = (int)LC, di = (int)d;
  switch (DP) {
    case 4: small_fwd_kernel<4><<<grid, 128, smem, st>>>(xr, xc, B, Li, Lc, di, lamR, lamC, scale, out); break;
    case 8: small_fwd_kernel<8><<<grid, 128, smem, st>>>(xr, xc, B, Li, Lc, di, lamR, lamC, scale, out); break;
    case 16: small_fwd_kernel<16><<<grid, 128, smem, st>>>(xr, xc, B, Li, Lc, di, lamR, lamC, scale, out); break;
    default: small_fwd_kernel<32><<<grid, 128, smem, st>>>(xr, xc, B, Li, Lc, di, lamR, lamC, scale, out); break;
  }
  return true;
}

}  // namespace sk
