// sk_signature.cu -- truncated signatures of piecewise-linear paths, forward
// and backward, on sm_100a (pySigLib's other hot path).
//
// Reference: /root/reference/pkg/src/sigcore/signature.py:104-121 (signature),
// signature_grad.py:20-53 (signature_backward), _kernels.py:26-279 (exp_into,
// chen_update_inplace, horner_sig_path, sig_backward_path).  Layout as the
// reference (tensors.py:1-40): levels 1..N back to back, level k holds d^k
// coefficients in row-major multi-index order, level 0 (= 1) implicit.
//
// Forward (sig_fwd_kernel).  The Horner update of level k reads only the
// entries of the levels below k with the SAME leading indices, so the tensor
// splits into independent "rows": a thread owns one row of the top level
// (prefix i1..i_{N-1}, its d entries in registers) plus the chain of lower-level
// entries along its prefix S_1[i1], S_2[i1 i2], ..., S_{N-1}[i1..i_{N-1}] (also
// registers; shared chain entries are recomputed identically by every thread
// that needs them).  No shared state, no barriers, no atomics; the increments
// of the path stream through a shared-memory ring.  Every multiply and add is
// issued separately (no FMA contraction) in the reference's order
// (_kernels.py:124-150: acc = z_i1 / k; acc = ((acc + S_j) / (k - j)) z_ij;
// S_k += (acc + S_{k-1}) z_ik), so the result is bitwise the reference's.
//
// Backward (sig_bwd_kernel).  The reference's time-reversed deconstruction
// (_kernels.py:182-266): per segment, peel it off the prefix signature
// (prefix <- prefix (x) exp(-z)), form the segment exponential E = exp(z), the
// adjoint of C = A (x) E w.r.t. E (left contraction with A) and w.r.t. A
// (right contraction with E), then reverse the exp recurrence for dF/dz.  The
// contractions couple the whole tensor, so one CTA owns one path: the four
// tensors live in the workspace (L2), each phase is parallel over output
// entries with CTA barriers between dependent phases; long reductions are split
// into fixed chunks combined in a fixed order (deterministic, not bitwise the
// reference's serial order).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/sigkernel.h"

namespace sk {

int set_error(int code, const char* msg);

constexpr int kSigMaxDepth = 16;
constexpr int kSigStage = 32;  // increments per staged chunk

// offsets[k] = sum_{j=1..k} d^j (offsets[0] = 0); false if too large
static bool sig_offsets(int64_t d, int depth, int64_t (&off)[kSigMaxDepth + 1]) {
  off[0] = 0;
  int64_t p = 1;
  for (int k = 1; k <= depth; ++k) {
    if (p > (int64_t(1) << 40) / d) return false;
    p *= d;
    off[k] = off[k - 1] + p;
  }
  return true;
}

struct SigGeom {
  int d, N;
  int64_t off[kSigMaxDepth + 1];
  int64_t pw[kSigMaxDepth + 1];  // d^k
};

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

// ------------------------------------------------------------------ increments
// Increments of the (optionally transformed) path in the reference's
// fused_increments layout (transforms.py:91-120): [B][M'][d'].
__global__ void sig_prep_kernel(const double* __restrict__ x, const double* __restrict__ times,
                                int64_t B, int64_t L, int64_t d, int tf, double* __restrict__ inc) {
  const int64_t Me = tf == 2 ? 2 * (L - 1) : L - 1;
  const int64_t de = tf == 1 ? d + 1 : tf == 2 ? 2 * d : d;
  const int64_t total = B * Me * de;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e % de, r = (e / de) % Me, p = e / (de * Me);
    const double* xp = x + p * L * d;
    double v = 0.0;
    if (tf == 0) {
      v = xp[(r + 1) * d + k] - xp[r * d + k];
    } else if (tf == 1) {
      if (k < d) {
        v = xp[(r + 1) * d + k] - xp[r * d + k];
      } else if (times) {
        v = times[r + 1] - times[r];
      } else {  // numpy.linspace(0, 1, L) (transforms.py:30-34)
        const double t1 = (r + 1 == L - 1) ? 1.0 : (double)(r + 1) * (1.0 / (double)(L - 1));
        const double t0 = (double)r * (1.0 / (double)(L - 1));
        v = t1 - t0;
      }
    } else {  // lead-lag: (dX_i, 0) then (0, dX_i)
      const int64_t i = r >> 1;
      if ((r & 1) == 0 && k < d) v = xp[(i + 1) * d + k] - xp[i * d + k];
      else if ((r & 1) == 1 && k >= d) v = xp[(i + 1) * d + (k - d)] - xp[i * d + (k - d)];
    }
    inc[e] = v;
  }
}

// -------------------------------------------------------------------- forward
// One thread = one top-level row of one path.  DM: register capacity for d
// (d <= DM), NM: capacity for the depth (N <= NM).
__constant__ double c_inv[kSigMaxDepth + 1] = {
    0.0,       1.0,       1.0 / 2,  1.0 / 3,  1.0 / 4,  1.0 / 5,  1.0 / 6,  1.0 / 7, 1.0 / 8,
    1.0 / 9,   1.0 / 10,  1.0 / 11, 1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16};

template <int DM, int NM>
__global__ void __launch_bounds__(256)
sig_fwd_kernel(const double* __restrict__ inc, int64_t B, int64_t M, SigGeom g,
               int64_t rows, int64_t ctas_per_path, double* __restrict__ out,
               int64_t out_stride) {
  __shared__ __align__(16) double sZ[2][kSigStage][DM];
  const int d = g.d, N = g.N;
  const int64_t path = blockIdx.x / ctas_per_path;
  const int64_t row = (blockIdx.x % ctas_per_path) * blockDim.x + threadIdx.x;
  const bool live = row < rows;
  const int64_t total = g.off[N];
  // prefix indices of the row (most significant first): idx[1..N-1]
  int idx[NM];
  {
    int64_t r = live ? row : 0;
#pragma unroll
    for (int j = NM - 1; j >= 1; --j) {
      if (j <= N - 1) {
        idx[j] = (int)(r % d);
        r /= d;
      } else {
        idx[j] = 0;
      }
    }
    idx[0] = 0;
  }
  double top[DM], c[NM];
#pragma unroll
  for (int j = 0; j < DM; ++j) top[j] = 0.0;
#pragma unroll
  for (int j = 0; j < NM; ++j) c[j] = 0.0;

  const double* src = inc + path * M * d;
  auto stage = [&](int buf, int64_t s0) {
    const int n = (int)lmin((int64_t)kSigStage, M - s0) * d;
    for (int e = threadIdx.x; e < n; e += blockDim.x)
      sZ[buf][e / d][e % d] = __ldg(src + s0 * d + e);
  };
  if (M > 0) stage(0, 0);
  __syncthreads();
  for (int64_t s0 = 0, chunk = 0; s0 < M; s0 += kSigStage, ++chunk) {
    const int buf = (int)(chunk & 1);
    if (s0 + kSigStage < M) stage(buf ^ 1, s0 + kSigStage);  // next chunk under this one
    const int n = (int)lmin((int64_t)kSigStage, M - s0);
    for (int s = 0; s < n; ++s) {
      double z[DM];
      bool nz = false;
#pragma unroll
      for (int j = 0; j < DM; ++j) {
        z[j] = j < d ? sZ[buf][s][j] : 0.0;
        nz |= (j < d) && (z[j] != 0.0);
      }
      if (!nz) continue;  // identity update: bit-exact no-op (_kernels.py:107-112)
      double zi[NM];      // z at the row's prefix indices
#pragma unroll
      for (int j = 1; j < NM; ++j) zi[j] = sZ[buf][s][idx[j]];
      zi[0] = 0.0;
      if (N == 1) {
#pragma unroll
        for (int j = 0; j < DM; ++j) top[j] = add(top[j], z[j]);
        continue;
      }
      // level N (the row's d entries), from the old chain
      {
        double acc = mul(zi[1], c_inv[N]);
#pragma unroll
        for (int j = 1; j < NM - 1; ++j)
          if (j <= N - 2) acc = mul(mul(add(acc, c[j]), c_inv[N - j]), zi[j + 1]);
        double a = c[0];
#pragma unroll
        for (int j = 1; j < NM; ++j)
          if (j == N - 1) a = add(acc, c[j]);
#pragma unroll
        for (int j = 0; j < DM; ++j) top[j] = add(top[j], mul(a, z[j]));
      }
      // chain levels N-1 .. 2 (each from the old lower levels), then level 1
#pragma unroll
      for (int k = NM - 1; k >= 2; --k) {
        if (k <= N - 1) {
          double acc = mul(zi[1], c_inv[k]);
#pragma unroll
          for (int j = 1; j < NM - 1; ++j)
            if (j <= k - 2) acc = mul(mul(add(acc, c[j]), c_inv[k - j]), zi[j + 1]);
          c[k] = add(c[k], mul(add(acc, c[k - 1]), zi[k]));
        }
      }
      c[1] = add(c[1], zi[1]);
    }
    __syncthreads();  // next chunk staged; this one free
  }
  if (!live) return;
  double* o = out + path * out_stride;
  if (N == 1) {
#pragma unroll
    for (int j = 0; j < DM; ++j)
      if (j < d) o[j] = top[j];
    return;
  }
#pragma unroll
  for (int j = 0; j < DM; ++j)
    if (j < d) o[g.off[N - 1] + row * d + j] = top[j];
  // chain entries: written by the row whose remaining indices are all zero
  int64_t pre = row;
  bool zero_tail = true;
#pragma unroll
  for (int k = NM - 1; k >= 1; --k) {
    if (k <= N - 1) {
      // level k entry = prefix of length k: row / d^(N-1-k); owner iff idx[k+1..N-1] == 0
      if (zero_tail) o[g.off[k - 1] + pre] = c[k];
      zero_tail = zero_tail && (idx[k] == 0);
      pre /= d;
    }
  }
}

// ------------------------------------------------------------------- backward
// Deterministic CTA-wide contractions (fixed chunking and combine order).
// out[c] += sum_r a[r] * M[r*C + c]
__device__ void cta_vecmat(double* __restrict__ out, const double* __restrict__ a,
                           const double* __restrict__ Mx, int64_t R, int64_t C,
                           double* __restrict__ part) {
  const int T = blockDim.x, t = threadIdx.x;
  if (C >= T / 4 || R <= 4) {
    for (int64_t cc = t; cc < C; cc += T) {
      double acc = out[cc];
#pragma unroll 8
      for (int64_t r = 0; r < R; ++r) acc = add(acc, mul(a[r], Mx[r * C + cc]));
      out[cc] = acc;
    }
    __syncthreads();
    return;
  }
  const int64_t Q = lmin((int64_t)T / C, R);
  const int64_t Rc = (R + Q - 1) / Q;
  if (t < Q * C) {
    const int64_t cc = t % C, q = t / C;
    double acc = 0.0;
    const int64_t r1 = lmin(R, (q + 1) * Rc);
#pragma unroll 8
    for (int64_t r = q * Rc; r < r1; ++r) acc = add(acc, mul(a[r], Mx[r * C + cc]));
    part[q * C + cc] = acc;
  }
  __syncthreads();
  for (int64_t cc = t; cc < C; cc += T) {
    double acc = out[cc];
    for (int64_t q = 0; q < Q; ++q) acc = add(acc, part[q * C + cc]);
    out[cc] = acc;
  }
  __syncthreads();
}

// out[r] += sum_c M[r*C + c] * v[c]   (the dot formed first, then added)
__device__ void cta_matvec(double* __restrict__ out, const double* __restrict__ Mx,
                           const double* __restrict__ v, int64_t R, int64_t C,
                           double* __restrict__ part) {
  const int T = blockDim.x, t = threadIdx.x;
  if (R >= T / 4 || C <= 4) {
    for (int64_t r = t; r < R; r += T) {
      double acc = 0.0;
#pragma unroll 8
      for (int64_t cc = 0; cc < C; ++cc) acc = add(acc, mul(Mx[r * C + cc], v[cc]));
      out[r] = add(out[r], acc);
    }
    __syncthreads();
    return;
  }
  const int64_t Q = lmin((int64_t)T / R, C);
  const int64_t Cc = (C + Q - 1) / Q;
  if (t < Q * R) {
    const int64_t r = t % R, q = t / R;
    double acc = 0.0;
    const int64_t c1 = lmin(C, (q + 1) * Cc);
#pragma unroll 8
    for (int64_t cc = q * Cc; cc < c1; ++cc) acc = add(acc, mul(Mx[r * C + cc], v[cc]));
    part[q * R + r] = acc;
  }
  __syncthreads();
  for (int64_t r = t; r < R; r += T) {
    double acc = 0.0;
    for (int64_t q = 0; q < Q; ++q) acc = add(acc, part[q * R + r]);
    out[r] = add(out[r], acc);
  }
  __syncthreads();
}

// E = exp(zs) with zs = sign * z: level m entry J = ((z_j1 (1/2)) z_j2 (1/3)) ...
// exactly as exp_into (_kernels.py:26-42)
// Level by level: entry J of level m is level m-1's entry J / d (its leading
// digits) times 1/m times z of its last digit -- the very operations of the
// digit loop, so every value is bitwise unchanged, at one multiply pair per
// entry instead of m (the per-digit 64-bit divisions were the kernel's top cost).
// 32-bit indices: the planner's (d, N) range keeps every level below 2^24 entries.
__device__ void cta_exp(double* __restrict__ E, const double* __restrict__ z, double sign,
                        const SigGeom& g) {
  const unsigned d = (unsigned)g.d;
  const int N = g.N;
  for (unsigned J = threadIdx.x; J < d; J += blockDim.x) E[J] = sign * z[J];
  __syncthreads();
  for (int m = 2; m <= N; ++m) {
    const unsigned n = (unsigned)g.pw[m];
    const double* __restrict__ prev = E + g.off[m - 2];
    double* __restrict__ cur = E + g.off[m - 1];
    const double im = c_inv[m];
    for (unsigned J = threadIdx.x; J < n; J += blockDim.x)
      cur[J] = mul(mul(prev[J / d], im), sign * z[J % d]);
    __syncthreads();
  }
}

// One CTA per path: the reverse walk of sig_backward_path (_kernels.py:182-266).
// W: per-path workspace [SIG | SB | EB | EX] (4 x total); SIG enters as the
// full signature, SB as the cotangent.  gout: [M][d] increment gradients.
// ONCHIP: the four tensors live in shared memory (4 x total doubles fit, e.g.
// d = 4, N = 6: 175 KB); SIG and SB are copied in once, every per-segment sweep
// then stays on chip (the global walk is L2 / DRAM latency bound).  Same
// operations in the same order: bitwise the global-memory walk.
template <bool ONCHIP>
__global__ void __launch_bounds__(512)
sig_bwd_kernel(const double* __restrict__ inc, int64_t M, SigGeom g, double* __restrict__ work,
               int64_t wstride, double* __restrict__ gout) {
  extern __shared__ double sm_sig[];
  const int d = g.d, N = g.N;
  const int64_t total = g.off[N];
  double* z = sm_sig;                     // [d]
  double* gz = z + 32;                    // [d] increment gradient of the step
  double* part = gz + 32;                 // [blockDim]
  const int64_t path = blockIdx.x;
  double* SIG = work + path * wstride;
  if constexpr (ONCHIP) {
    double* t4 = part + ((blockDim.x + 1) & ~1u);
    for (int64_t t = threadIdx.x; t < 2 * total; t += blockDim.x) t4[t] = SIG[t];
    SIG = t4;
    __syncthreads();
  }
  double* SB = SIG + total;
  double* EB = SB + total;
  double* EX = EB + total;
  const double* src = inc + path * M * d;
  double* go = gout + path * M * d;

  for (int64_t step = M - 1; step >= 0; --step) {
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      z[j] = src[step * d + j];
      gz[j] = 0.0;
    }
    __syncthreads();
    // ---- peel the segment off the prefix: SIG <- SIG (x) exp(-z)
    if (step > 0) {
      cta_exp(EX, z, -1.0, g);
      for (int k = N; k >= 1; --k) {  // top-down: level k reads the old lower levels
        const int64_t n = g.pw[k];
        // level k (written) and the levels below / EX (read) do not overlap
        double* __restrict__ dst = SIG + g.off[k - 1];
        const double* __restrict__ low = SIG;
        const double* __restrict__ ex = EX;
#pragma unroll 4
        for (int64_t I = threadIdx.x; I < n; I += blockDim.x) {
          double v = dst[I];
          for (int i = 1; i < k; ++i) {
            const unsigned pk = (unsigned)g.pw[k - i];
            const unsigned head = (unsigned)I / pk, tail = (unsigned)I % pk;
            v = add(v, mul(low[g.off[i - 1] + head], ex[g.off[k - i - 1] + tail]));
          }
          dst[I] = add(v, ex[g.off[k - 1] + I]);
        }
        __syncthreads();
      }
    } else {
      for (int64_t t = threadIdx.x; t < total; t += blockDim.x) SIG[t] = 0.0;
      __syncthreads();
    }
    // ---- the segment exponential E = exp(z)
    cta_exp(EX, z, 1.0, g);
    // ---- EB = adjoint w.r.t. E: EB_m = SB_m + sum_{k>m} A_{k-m}^T SB_k.  The
    // top level has no correction (EB_N = SB_N, and SB_N is never updated), so
    // it is read from SB below and only the lower levels are copied
    for (int64_t t = threadIdx.x; t < g.off[N - 1]; t += blockDim.x) EB[t] = SB[t];
    __syncthreads();
    for (int m = 1; m < N; ++m)
      for (int k = m + 1; k <= N; ++k)
        cta_vecmat(EB + g.off[m - 1], SIG + g.off[k - m - 1], SB + g.off[k - 1], g.pw[k - m],
                   g.pw[m], part);
    // ---- SB = adjoint w.r.t. the prefix: SB_i += sum_{k>i} SB_k . E_{k-i}
    if (step > 0) {
      for (int i = 1; i < N; ++i)
        for (int k = i + 1; k <= N; ++k)
          cta_matvec(SB + g.off[i - 1], SB + g.off[k - 1], EX + g.off[k - i - 1], g.pw[i],
                     g.pw[k - i], part);
    }
    // ---- reverse the exp recurrence E_m = (E_{m-1} / m) (x) z (_kernels.py:252-266)
    for (int m = N; m >= 2; --m) {
      const double im = c_inv[m];
      const int64_t rows = g.pw[m - 1];
      const double* Em1 = EX + g.off[m - 2];
      double* Bm = (m == N ? SB : EB) + g.off[m - 1];
      double* Bm1 = EB + g.off[m - 2];
      // g[j] += sum_rows E_{m-1}[row] * (Bm[row, j] / m)   (chunked, fixed order)
      {
        const int T = blockDim.x, t = threadIdx.x;
        const int64_t Q = lmax((int64_t)1, lmin((int64_t)(T / d), rows));
        const int64_t Rc = (rows + Q - 1) / Q;
        if (t < Q * d) {
          const int j = t % d;
          const int64_t q = t / d;
          double acc = 0.0;
          const int64_t r1 = lmin(rows, (q + 1) * Rc);
#pragma unroll 8
          for (int64_t r = q * Rc; r < r1; ++r) acc = add(acc, mul(Em1[r], mul(Bm[r * d + j], im)));
          part[q * d + j] = acc;
        }
        __syncthreads();
        if (t < d) {
          double acc = gz[t];
          for (int64_t q = 0; q < Q; ++q) acc = add(acc, part[q * d + t]);
          gz[t] = acc;
        }
      }
      // Bm1[row] += sum_j (Bm[row, j] / m) z_j
      for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < d; ++j) acc = add(acc, mul(mul(Bm[r * d + j], im), z[j]));
        Bm1[r] = add(Bm1[r], acc);
      }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < d; j += blockDim.x)
      go[step * d + j] = add(gz[j], (N == 1 ? SB : EB)[j]);
    __syncthreads();
  }
}

// Telescope increment gradients to (transformed-)point gradients
// (signature_grad.py:45-48), then the transform adjoint (transforms.py:69-90).
__global__ void sig_points_kernel(const double* __restrict__ g, int64_t B, int64_t M, int64_t de,
                                  int64_t L, int64_t d, int tf, double* __restrict__ grad) {
  const int64_t total = B * L * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e % d, i = (e / d) % L, p = e / (d * L);
    const double* gp = g + p * M * de;
    // transformed-point gradient at point q, component cc
    auto pt = [&](int64_t q, int64_t cc) -> double {
      double v = 0.0;  // grad_eff[:, :-1] -= g ; grad_eff[:, 1:] += g
      if (q < M) v -= gp[q * de + cc];
      if (q >= 1) v += gp[(q - 1) * de + cc];
      return v;
    };
    double v;
    if (tf == 2) {
      v = pt(2 * i, c) + pt(2 * i, d + c);
      if (i < L - 1) v += pt(2 * i + 1, d + c);
      if (i >= 1) v += pt(2 * i - 1, c);
    } else {
      v = pt(i, c);
    }
    grad[e] = v;
  }
}

// ----------------------------------------------------------------- planning
struct SigPlan {
  SigGeom g;
  int64_t M, de, total, rows;
  int DM, NM;
};

static int sig_plan(SigPlan& p, int64_t L, int64_t d, int depth, int tf) {
  if (L < 2) return set_error(SK_INVALID_ARGUMENT, "signature needs at least 2 points");
  if (d < 1) return set_error(SK_INVALID_ARGUMENT, "path dimension must be >= 1");
  if (depth < 1) return set_error(SK_INVALID_ARGUMENT, "depth must be >= 1");
  if (tf < 0 || tf > 2) return set_error(SK_INVALID_ARGUMENT, "unknown path transform");
  p.M = tf == 2 ? 2 * (L - 1) : L - 1;
  p.de = tf == 1 ? d + 1 : tf == 2 ? 2 * d : d;
  const int de = (int)p.de;
  // register capacity per thread: (DM, NM) instances
  if (de <= 2 && depth <= 16) { p.DM = 2; p.NM = 16; }
  else if (de <= 4 && depth <= 10) { p.DM = 4; p.NM = 10; }
  else if (de <= 8 && depth <= 8) { p.DM = 8; p.NM = 8; }
  else if (de <= 16 && depth <= 6) { p.DM = 16; p.NM = 6; }
  else if (de <= 32 && depth <= 4) { p.DM = 32; p.NM = 4; }
  else return set_error(SK_INVALID_ARGUMENT, "signature: (dimension, depth) beyond the supported "
                                             "range (d'<=2 & N<=16, 4 & 10, 8 & 8, 16 & 6, 32 & 4)");
  int64_t off[kSigMaxDepth + 1];
  if (!sig_offsets(p.de, depth, off)) return set_error(SK_INVALID_ARGUMENT, "signature too large");
  p.g.d = de;
  p.g.N = depth;
  int64_t pw = 1;
  for (int k = 0; k <= kSigMaxDepth; ++k) {
    p.g.off[k] = k <= depth ? off[k] : off[depth];
    p.g.pw[k] = pw;
    if (k < depth) pw *= de;
  }
  p.total = off[depth];
  p.rows = depth == 1 ? 1 : p.g.pw[depth - 1];
  return SK_OK;
}

template <int DM, int NM>
static void launch_fwd(const SigPlan& p, const double* inc, int64_t B, double* out,
                       int64_t out_stride, cudaStream_t st) {
  const int threads = (int)std::min<int64_t>(256, ((p.rows + 31) / 32) * 32);
  const int64_t cpp = (p.rows + threads - 1) / threads;
  sig_fwd_kernel<DM, NM><<<(unsigned)(B * cpp), threads, 0, st>>>(inc, B, p.M, p.g, p.rows, cpp,
                                                                    out, out_stride);
}

static int sig_forward_impl(const SigPlan& p, const double* inc, int64_t B, double* out,
                            cudaStream_t st, int64_t out_stride = -1) {
  if (B <= 0) return SK_OK;
  if (out_stride < 0) out_stride = p.total;
  switch (p.DM) {
    case 2: launch_fwd<2, 16>(p, inc, B, out, out_stride, st); break;
    case 4: launch_fwd<4, 10>(p, inc, B, out, out_stride, st); break;
    case 8: launch_fwd<8, 8>(p, inc, B, out, out_stride, st); break;
    case 16: launch_fwd<16, 6>(p, inc, B, out, out_stride, st); break;
    default: launch_fwd<32, 4>(p, inc, B, out, out_stride, st); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SK_CUDA_ERROR, cudaGetErrorString(e));
  return SK_OK;
}

static size_t align256(size_t v) { return (v + 255) / 256 * 256; }

}  // namespace sk

using namespace sk;

extern "C" {

int64_t sk_signature_length(int64_t d, int depth) {
  int64_t off[kSigMaxDepth + 1];
  if (d < 1 || depth < 1 || depth > kSigMaxDepth || !sig_offsets(d, depth, off)) return 0;
  return off[depth];
}

size_t sk_signature_workspace_bytes(int64_t B, int64_t L, int64_t d, int depth, int transform) {
  SigPlan p;
  if (B < 0 || sig_plan(p, L, d, depth, transform)) return 0;
  return align256((size_t)B * p.M * p.de * sizeof(double));
}

int sk_signature(const double* x, const double* times, int64_t B, int64_t L, int64_t d, int depth,
                 int transform, double* out, void* ws, size_t ws_bytes, void* stream) {
  SigPlan p;
  if (B < 0) return set_error(SK_INVALID_ARGUMENT, "negative batch");
  if (int rc = sig_plan(p, L, d, depth, transform)) return rc;
  if (B == 0) return SK_OK;
  const size_t need = align256((size_t)B * p.M * p.de * sizeof(double));
  if (ws_bytes < need) return set_error(SK_INVALID_ARGUMENT, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  double* inc = static_cast<double*>(ws);
  const int64_t n = B * p.M * p.de;
  sig_prep_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(
      x, times, B, L, d, transform, inc);
  return sig_forward_impl(p, inc, B, out, st);
}

size_t sk_signature_backward_workspace_bytes(int64_t B, int64_t L, int64_t d, int depth,
                                             int transform) {
  SigPlan p;
  if (B < 0 || sig_plan(p, L, d, depth, transform)) return 0;
  const size_t inc = align256((size_t)B * p.M * p.de * sizeof(double));
  const size_t work = align256((size_t)B * 4 * p.total * sizeof(double));
  return 2 * inc + work;
}

int sk_signature_backward(const double* x, const double* times, int64_t B, int64_t L, int64_t d,
                          int depth, int transform, const double* cot, double* grad, void* ws,
                          size_t ws_bytes, void* stream) {
  SigPlan p;
  if (B < 0) return set_error(SK_INVALID_ARGUMENT, "negative batch");
  if (int rc = sig_plan(p, L, d, depth, transform)) return rc;
  if (B == 0) return SK_OK;
  if (!cot || !grad) return set_error(SK_INVALID_ARGUMENT, "cotangent / gradient buffer missing");
  const size_t incb = align256((size_t)B * p.M * p.de * sizeof(double));
  const size_t workb = align256((size_t)B * 4 * p.total * sizeof(double));
  if (ws_bytes < 2 * incb + workb) return set_error(SK_INVALID_ARGUMENT, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* base = static_cast<char*>(ws);
  double* inc = reinterpret_cast<double*>(base);
  double* gin = reinterpret_cast<double*>(base + incb);
  double* work = reinterpret_cast<double*>(base + 2 * incb);
  const int64_t n = B * p.M * p.de;
  sig_prep_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(
      x, times, B, L, d, transform, inc);
  // per path [SIG | SB | EB | EX]: SIG = the full signature (the walk's start,
  // horner_sig_path, _kernels.py:199-201), SB = the cotangent
  const int64_t wstride = 4 * p.total;
  if (int rc = sig_forward_impl(p, inc, B, work, st, wstride)) return rc;
  {
    cudaError_t e = cudaMemcpy2DAsync(work + p.total, wstride * sizeof(double), cot,
                                      p.total * sizeof(double), p.total * sizeof(double), B,
                                      cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return set_error(SK_CUDA_ERROR, cudaGetErrorString(e));
  }
  const int threads = 512;
  const size_t smem = (64 + threads) * sizeof(double);
  const size_t smem_on = smem + 4 * (size_t)p.total * sizeof(double);
  static bool opted[64] = {};
  int dev = 0;
  (void)cudaGetDevice(&dev);
  bool onchip = smem_on <= 227 * 1024 && dev >= 0 && dev < 64;
  if (onchip && !opted[dev]) {
    if (cudaFuncSetAttribute(sig_bwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024) == cudaSuccess)
      opted[dev] = true;
    else
      (void)cudaGetLastError();
  }
  onchip = onchip && opted[dev];
  if (onchip)
    sig_bwd_kernel<true><<<(unsigned)B, threads, smem_on, st>>>(inc, p.M, p.g, work, wstride, gin);
  else
    sig_bwd_kernel<false><<<(unsigned)B, threads, smem, st>>>(inc, p.M, p.g, work, wstride, gin);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SK_CUDA_ERROR, cudaGetErrorString(e));
  const int64_t np = B * L * d;
  sig_points_kernel<<<(unsigned)std::min<int64_t>((np + 255) / 256, 4096), 256, 0, st>>>(
      gin, B, p.M, p.de, L, d, transform, grad);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SK_CUDA_ERROR, cudaGetErrorString(e));
  return SK_OK;
}

}  // extern "C"
