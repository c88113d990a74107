// sk_capi.cu -- extern "C" boundary (include/sigkernel.h) and host planning.
//
// The planning mirrors the reference's dispatch (kernel.py:125-180):
//   * orientation: the longer fine axis goes on the grid rows (kernel.py:137-140,
//     164-170), so results are bit-identical under x<->y swap;
//   * symmetric Gram: upper triangle only, then mirrored (kernel.py:177-179).
// Everything runs on the caller's stream; no allocation happens here
// (the reference's "caller buffers only" contract, _kernels.py:9-10).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/sigkernel.h"
#include "sk_backward.cuh"
#include "sk_plan.h"

namespace sk {

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
// error reporting for the other translation units (sk_signature.cu)
int set_error(int code, const char* msg) { return fail(code, msg); }

#define SK_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(SK_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------ host caches
// Planning runs on every call (the workspace query and the launch), so every
// driver query it needs is cached per device: SM count, memory budget, the
// dynamic-shared-memory opt-in and the occupancy of each kernel instance.
static std::mutex g_mu;
static constexpr int kMaxDev = 64;

static int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return dev < kMaxDev ? dev : 0;
}

static int device_sms() {
  static int cache[kMaxDev] = {0};
  const int dev = current_device();
  if (cache[dev] > 0) return cache[dev];
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return 148;
  }
  cache[dev] = sms > 0 ? sms : 148;
  return cache[dev];
}

// Blocks of `fn` resident per SM at (threads, smem); opts the kernel into
// `smem` bytes of dynamic shared memory first (once per device and size).
static int occupancy(const void* fn, int threads, int smem) {
  struct Key {
    const void* fn;
    int threads, smem, dev;
    bool operator==(const Key& o) const {
      return fn == o.fn && threads == o.threads && smem == o.smem && dev == o.dev;
    }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.fn) ^ ((size_t)k.threads << 20) ^ ((size_t)k.smem << 32) ^
             (size_t)k.dev;
    }
  };
  static std::unordered_map<Key, int, Hash> cache;
  const Key key{fn, threads, smem, current_device()};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  // (always: static shared memory counts against the 48 KB default too)
  if (smem > 0 &&
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    (void)cudaGetLastError();
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess ||
      occ < 1) {
    (void)cudaGetLastError();
    occ = 1;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  cache[key] = occ;
  return occ;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Budget for the backward's per-slot workspace (checkpoints grow with L^2 / 8
// per in-flight tile): half the device memory, or SK_WS_BUDGET_GB.  Long paths
// get fewer slots (fewer resident warps) instead of an allocation failure.
static double ws_budget_bytes() {
  static const double env_gb = [] {
    const char* e = std::getenv("SK_WS_BUDGET_GB");
    return (e && e[0]) ? std::atof(e) : 0.0;
  }();
  if (env_gb > 0) return env_gb * 1e9;
  static double cache[kMaxDev] = {0};
  const int dev = current_device();
  if (cache[dev] > 0) return cache[dev];
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
    (void)cudaGetLastError();
    return 64e9;
  }
  cache[dev] = 0.5 * (double)tot;
  return cache[dev];
}

// Shrinks the grid so that slots * per_slot_bytes fits the budget.
static void cap_slots(int64_t& blocks, int64_t& slots, int warps, double per_slot_bytes) {
  const double budget = ws_budget_bytes();
  if ((double)slots * per_slot_bytes <= budget) return;
  blocks = std::max<int64_t>(1, (int64_t)(budget / (per_slot_bytes * warps)));
  slots = blocks * warps;
}

// ---------------------------------------------------------------- prep kernels
// Path transforms (pySigLib's time augmentation and lead-lag; reference
// transforms.py:37-120), applied inside the preparation launch: the kernels
// read transformed increments (linear kernel; the reference's
// fused_increments, transforms.py:91-120) or transformed nodes (RBF) built
// straight from the raw points, so no transformed path is ever materialised.
enum Transform : int { TF_NONE = 0, TF_TIME = 1, TF_LEADLAG = 2 };
__host__ __device__ inline int64_t eff_len(int64_t L, int tf) { return tf == TF_LEADLAG ? 2 * L - 1 : L; }
__host__ __device__ inline int64_t eff_dim(int64_t d, int tf) {
  return tf == TF_TIME ? d + 1 : tf == TF_LEADLAG ? 2 * d : d;
}
// numpy.linspace(0, 1, L)[i] as the reference computes it (default_times,
// transforms.py:30-34): i * (1 / (L - 1)), the last point exactly 1
__device__ inline double time_point(int64_t i, int64_t L) {
  if (L <= 1) return 0.0;
  return i == L - 1 ? 1.0 : (double)i * (1.0 / (double)(L - 1));
}

template <typename T, typename TO = T>
struct PrepSide {
  const T* x;
  int64_t n, L;  // raw points per path
  double scale;
  TO* out;       // (TO = double for float inputs of the FP32-recurrence DMMA forward)
};
// Both sides of a call in ONE launch (rows side, then the columns side):
// increments (kernel.py:74-75 np.diff, scaled by the exact dyadic factor,
// zero-padded to dpad) for the linear kernel, padded nodes for RBF, each of
// the transformed path when tf != TF_NONE (bitwise the np.diff of the
// materialised transform: the same subtractions, and exact zeros).
template <typename T, typename TO = T>
__global__ void prep_sides(PrepSide<T, TO> s0, PrepSide<T, TO> s1, int nsides, int rbf, int tf,
                           int64_t d, int dpad) {
  const int64_t per0 = rbf ? eff_len(s0.L, tf) : eff_len(s0.L, tf) - 1;
  const int64_t per1 = rbf ? eff_len(s1.L, tf) : eff_len(s1.L, tf) - 1;
  const int64_t rows0 = s0.n * per0;
  const int64_t rows1 = nsides > 1 ? s1.n * per1 : 0;
  const int64_t total = (rows0 + rows1) * dpad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rowg = e / dpad, k = e % dpad;
    const bool first = rowg < rows0;
    const PrepSide<T, TO>& sd = first ? s0 : s1;
    const int64_t row = first ? rowg : rowg - rows0;
    const int64_t per = first ? per0 : per1;
    const int64_t p = row / per, r = row % per;
    const T* xp = sd.x + p * sd.L * d;
    TO v = 0;  // (computed in TO: the identity for TO == T)
    if (rbf) {  // node r of the transformed path
      if (tf == TF_NONE) {
        if (k < d) v = (TO)xp[r * d + k];
      } else if (tf == TF_TIME) {
        if (k < d) v = (TO)xp[r * d + k];
        else if (k == d) v = (TO)time_point(r, sd.L);
      } else {  // lead-lag: Z[2i] = (X[i], X[i]), Z[2i+1] = (X[i+1], X[i])
        if (k < d) v = (TO)xp[((r + 1) >> 1) * d + k];
        else if (k < 2 * d) v = (TO)xp[(r >> 1) * d + (k - d)];
      }
    } else {  // increment r of the transformed path
      if (tf == TF_NONE) {
        if (k < d) v = ((TO)xp[(r + 1) * d + k] - (TO)xp[r * d + k]) * (TO)sd.scale;
      } else if (tf == TF_TIME) {
        if (k < d) v = ((TO)xp[(r + 1) * d + k] - (TO)xp[r * d + k]) * (TO)sd.scale;
        else if (k == d) v = ((TO)time_point(r + 1, sd.L) - (TO)time_point(r, sd.L)) * (TO)sd.scale;
      } else {  // lead-lag: (dX_i, 0), then (0, dX_i)
        const int64_t i = r >> 1;
        const bool lead = (r & 1) == 0;
        if (lead && k < d) v = ((TO)xp[(i + 1) * d + k] - (TO)xp[i * d + k]) * (TO)sd.scale;
        else if (!lead && k >= d && k < 2 * d)
          v = ((TO)xp[(i + 1) * d + (k - d)] - (TO)xp[i * d + (k - d)]) * (TO)sd.scale;
      }
    }
    sd.out[row * dpad + k] = v;
  }
}

// Adjoint of a transform on point gradients (reference transform_adjoint,
// transforms.py:69-90, same addition order): g_t (n, L', d') -> grad (n, L, d);
// grad = value, or grad += value.
__global__ void transform_adjoint_kernel(const double* __restrict__ gt, int64_t n, int64_t L,
                                         int64_t d, int tf, double* __restrict__ grad,
                                         int accumulate) {
  const int64_t Le = eff_len(L, tf), de = eff_dim(d, tf);
  const int64_t total = n * L * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e % d, i = (e / d) % L, p = e / (d * L);
    const double* g = gt + p * Le * de;
    double v;
    if (tf == TF_LEADLAG) {  // out = lead[0::2] + lag[0::2]; [:-1] += lag[1::2]; [1:] += lead[1::2]
      v = g[(2 * i) * de + c] + g[(2 * i) * de + d + c];
      if (i < L - 1) v += g[(2 * i + 1) * de + d + c];
      if (i >= 1) v += g[(2 * i - 1) * de + c];
    } else {  // time augmentation drops the time column
      v = g[i * de + c];
    }
    grad[e] = accumulate ? grad[e] + v : v;
  }
}

// Mirror the solved upper triangle into the lower one (kernel.py:177-179),
// restricted to rows [r0, r1) (out holds those rows, leading dim ldo).
template <typename T = double>
__global__ void mirror_upper(T* __restrict__ out, int64_t ldo, int r0, int r1) {
  int64_t span = r1 - r0;
  int64_t total = span * span;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = e / span, b = e % span;  // relative
    if (b < a) out[a * ldo + (b + r0)] = out[b * ldo + (a + r0)];
  }
}

// Full fine grid of one delta (store_grid=True facade path, goursat_grid
// _kernels.py:381-396).  One warp; lane u owns fine rows u, u+32, ... and the
// columns are swept as a skewed wavefront with a shared-memory row buffer.
// Used only for the small grids the reference's API returns to the caller.
__global__ void grid_kernel(const double* __restrict__ delta, int r1, int r2, int lam1,
                            int lam2, double scale, double* __restrict__ grid) {
  const int m1 = r1 << lam1, m2 = r2 << lam2;
  const int w = m2 + 1;
  for (int t = threadIdx.x; t <= m2; t += blockDim.x) grid[t] = 1.0;
  for (int s = threadIdx.x; s <= m1; s += blockDim.x) grid[(int64_t)s * w] = 1.0;
  __syncthreads();
  // anti-diagonal sweep: cells with s + t = dd are independent
  for (int dd = 2; dd <= m1 + m2; ++dd) {
    int slo = max(1, dd - m2), shi = min(m1, dd - 1);
    for (int s = slo + threadIdx.x; s <= shi; s += blockDim.x) {
      int t = dd - s;
      double p = delta[(int64_t)((s - 1) >> lam1) * r2 + ((t - 1) >> lam2)] * scale;
      Coef c = coef(p);
      grid[(int64_t)s * w + t] = cell(grid[(int64_t)(s - 1) * w + t],
                                      grid[(int64_t)s * w + t - 1],
                                      grid[(int64_t)(s - 1) * w + t - 1], c);
    }
    __syncthreads();
  }
}

// ------------------------------------------- exact Gram-gradient accumulators
// Accumulator blob (sk_grad_acc_bytes): [meta: 8 x u64][elements x 4 x u64],
// see FixAcc in sk_common.cuh.
constexpr int64_t kAccMeta = 8;

static size_t acc_bytes(int64_t n, int64_t L, int64_t d) {
  return (size_t)(kAccMeta + n * L * d * 4) * sizeof(unsigned long long);
}

__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}

// meta[0] = max|cot| (bit pattern), meta[2] = nscale; up to two metas.
__global__ void fix_init_kernel(const double* __restrict__ cot, int64_t count, double nscale,
                                unsigned long long* meta_a, unsigned long long* meta_b) {
  unsigned long long m = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    m = umax64(m, (unsigned long long)__double_as_longlong(fabs(cot[e])));
  for (int o = 16; o > 0; o >>= 1) m = umax64(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) {
    atomicMax(meta_a, m);
    if (meta_b) atomicMax(meta_b, m);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    meta_a[2] = (unsigned long long)__double_as_longlong(nscale);
    if (meta_b) meta_b[2] = (unsigned long long)__double_as_longlong(nscale);
  }
}

// grad (+)= value of the accumulated limbs; NaN everywhere if the overflow
// flag is set.  The limbs are carry-normalised first, so the value is a
// function of the exact integer sum only (tests/fixpt_ref.py restates it).
__global__ void fix_finalize_kernel(const unsigned long long* __restrict__ blob, int64_t nelem,
                                    double* __restrict__ grad, int accumulate) {
  const unsigned long long* meta = blob;
  const long long* acc = reinterpret_cast<const long long*>(blob + kAccMeta);
  const int E = fix_anchor(__longlong_as_double((long long)meta[0]),
                           __longlong_as_double((long long)meta[2]));
  const bool bad = meta[1] != 0;
  const double u3 = ldexp(1.0, E - 42), u2 = ldexp(1.0, E - 84), u1 = ldexp(1.0, E - 126),
               u0 = ldexp(1.0, E - 168);
  constexpr long long M = (1ll << 42) - 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nelem;
       e += (int64_t)gridDim.x * blockDim.x) {
    const longlong2 lo = reinterpret_cast<const longlong2*>(acc)[2 * e];
    const longlong2 hi = reinterpret_cast<const longlong2*>(acc)[2 * e + 1];
    long long a0 = lo.x, a1 = lo.y, a2 = hi.x, a3 = hi.y;
    auto normalize = [&]() {
      a1 += a0 >> 42;
      a0 &= M;
      a2 += a1 >> 42;
      a1 &= M;
      a3 += a2 >> 42;
      a2 &= M;
    };
    normalize();
    // magnitude first (all four digits non-negative: no cancellation in the
    // fp64 sum), then the sign
    const bool neg = a3 < 0;
    if (neg) {
      a0 = -a0;
      a1 = -a1;
      a2 = -a2;
      a3 = -a3;
      normalize();
    }
    double v = (double)a3 * u3 + ((double)a2 * u2 + ((double)a1 * u1 + (double)a0 * u0));
    if (neg) v = -v;
    if (bad) v = __longlong_as_double(0x7ff8000000000000ll);
    grad[e] = accumulate ? grad[e] + v : v;
  }
}

static int acc_init(unsigned long long* blob_a, unsigned long long* blob_b, size_t bytes_a,
                    size_t bytes_b, const double* cot, int64_t n1, int64_t n2, bool sym,
                    cudaStream_t st) {
  SK_CUDA(cudaMemsetAsync(blob_a, 0, bytes_a, st));
  if (blob_b) SK_CUDA(cudaMemsetAsync(blob_b, 0, bytes_b, st));
  const int64_t count = n1 * n2;
  const double nscale = (double)std::max(n1, n2) * (sym ? 2.0 : 1.0);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 1024));
  fix_init_kernel<<<blocks, 256, 0, st>>>(cot, count, nscale, blob_a, blob_b);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

static int acc_finalize(const unsigned long long* blob, int64_t nelem, double* grad,
                        bool accumulate, cudaStream_t st) {
  if (nelem <= 0) return SK_OK;
  const int blocks = (int)std::min<int64_t>((nelem + 255) / 256, 8 * 148);
  fix_finalize_kernel<<<blocks, 256, 0, st>>>(blob, nelem, grad, accumulate ? 1 : 0);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

// ------------------------------------------------------------------- planning
struct Geometry {
  // oriented problem (rows = longer fine axis)
  int64_t nR, nC;  // path counts on rows / cols side
  int64_t LR, LC;  // points per row / col path
  int lamR, lamC;
  bool swap;
};

static int pick_dp(int64_t d, int& nch) {
  int DP = d <= 4 ? 4 : d <= 8 ? 8 : d <= 16 ? 16 : 32;
  nch = (int)((d + DP - 1) / DP);
  return DP;
}

struct FwdPlan {
  FwdShape shape;
  FwdFn fn = nullptr;
  int threads = 128;
  int64_t blocks = 0;
  int64_t slots = 0;
  int64_t hand_stride = 0;
  int64_t nitems = 0;
  int P = 1;
  int smem_bytes = 0;
};

// Chooses lanes-per-pair and the persistent grid.  `gram` marks tiles whose
// groups share the column path.
static int plan_forward(FwdPlan& pl, int kind, int64_t d, int lamR, int lamC, int64_t M1c,
                        int64_t M2c, int64_t npairs, bool gram, int mode, int n2, int r0,
                        int r1, bool f32 = false) {
  int nch = 1;
  FwdShape s{};
  s.kind = kind;
  s.DP = (kind == DELTA) ? 4 : pick_dp(d, nch);
  s.R = (kind == DELTA) ? 8 : rows_per_lane(s.DP);
  s.FR = std::min(1 << std::min(lamR, 3), s.R);
  s.F = std::min(1 << std::min(lamC, 2), 4);
  const int64_t M1 = M1c << lamR;
  const int sms = device_sms();
  const int64_t target_lanes = (int64_t)sms * 512;
  const int64_t lanes_per_pair = (M1 + s.R - 1) / s.R;
  s.XW = false;
  s.W = 1;
  // G = 4 packs 8 pairs per warp and needs them to share the column path
  // (Gram tiles); batches use one pair per warp, or per CTA when long pairs
  // are too few to fill the GPU.
  if (gram) {
    s.G = (npairs * 4 >= target_lanes || lanes_per_pair <= 8) ? 4 : 32;
  } else if (npairs * 32 >= target_lanes || lanes_per_pair <= 64 || kind == DELTA || s.DP > 8) {
    // (the XW column ring spans 512 lanes of records: DP > 8 would not fit)
    s.G = 32;
  } else {
    // few long pairs (BASELINE configs 2, 4): one pair per CTA of W warps, a
    // single wavefront over 32W lanes (cross-warp hops through shared memory)
    static const int wmax = [] {
      const char* e = std::getenv("SK_FWD_XW_WMAX");  // tuning knob
      const int v = (e && e[0]) ? std::atoi(e) : 16;
      return v >= 2 && v <= 16 ? v : 16;
    }();
    // widen until the GPU is full or one strip covers the pair (measured at
    // BASELINE config 2: one 8-warp strip 0.60 ms vs two 4-warp strips 0.70 ms)
    // DP = 8 pairs taller than 512 fine rows: 8 rows per lane, half the lanes
    // (C2: RBF 0.60 -> 0.56 ms, linear 0.35 -> 0.28 ms)
    static const int xr = [] {
      const char* e = std::getenv("SK_FWD_XW_R");  // tuning knob: 4 or 8 rows per lane (DP = 8)
      return (e && e[0] == '8') ? 8 : (e && e[0] == '4') ? 4 : 0;
    }();
    int64_t lanes = lanes_per_pair;
    if ((xr ? xr == 8 : M1 > 512) && s.DP == 8 && !f32) {
      s.R = 8;
      s.FR = std::min(1 << std::min(lamR, 3), s.R);
      lanes = (M1 + s.R - 1) / s.R;
    }
    int W = 2;
    while (W < wmax && npairs * 32 * W < target_lanes && 32 * W < lanes) W *= 2;
    static const int wforce = [] {
      const char* e = std::getenv("SK_FWD_XW_W");  // tuning knob: force the CTA width
      const int v = (e && e[0]) ? std::atoi(e) : 0;
      return (v == 2 || v == 4 || v == 8 || v == 16) ? v : 0;
    }();
    if (wforce) W = wforce;
    s.XW = true;
    s.W = W;
    s.G = 32 * W;
  }
  // short batch paths: the fewest rows per lane that still cover the pair
  // with one warp (all lanes busy, short dependent chain per step)
  bool short_r = false;
  if (!gram && !s.XW && s.G == 32 && kind != DELTA && !f32 && nch == 1 && M1 < 32 * s.R) {
    int r = 1;
    while (32 * r < M1) r *= 2;
    if (r < s.R) {
      s.R = r;
      s.FR = std::min(s.FR, r);
      short_r = true;
    }
  }
  // Gram tiles of the linear kernel (any dyadic order): increment products on
  // the FP64 tensor cores (sk_mma_fwd.cuh).  SK_NO_MMA=1 keeps the r01 kernels.
  // (measured, n = 256-512 Grams: DMMA wins for DP >= 16 at any order --
  // lambda 1: d = 16 11.5 -> 4.8 ms, d = 32 41 -> 7.3 ms; lambda 2, d = 16 6.8
  // -> 4.2 ms -- and for DP = 8 at order 0; the FMA-pipe kernel wins for
  // DP = 4 (d = 4, lambda 0: 8.4 vs 13.4 ms) and for DP = 8 at order > 0)
  // FP32 arithmetic (float recurrence, fp64 DMMA p): DP >= 16 only (C3 shape
  // 404 -> 189 ms; at DP = 8 the FP32 FMA-pipe kernel is faster, 185 vs 340 ms)
  const bool mma_shape = s.DP >= 16 || (s.DP == 8 && lamR + lamC == 0 && !f32);
  s.MMA = gram && kind == LINEAR && nch == 1 && s.DP <= 32 && mma_shape &&
          !(std::getenv("SK_NO_MMA") && std::getenv("SK_NO_MMA")[0] == '1');
  if (s.MMA) {
    int per_warp = 0;
    FwdFn fn = select_fwd_mma(s.DP, per_warp, lamR + lamC > 0, f32);
    if (!fn) return fail(SK_INVALID_ARGUMENT, "no DMMA forward instance for this shape");
    pl.shape = s;
    pl.fn = fn;
    const char* fw = std::getenv("SK_FWD_WPC");  // warps per CTA (tuning knob)
    const int fwpc = (fw && (fw[0] == '1' || fw[0] == '4')) ? fw[0] - '0' : 2;  // measured: 2 >= 4
    pl.threads = 32 * fwpc;
    pl.P = 8;
    pl.smem_bytes = per_warp * fwpc;
    pl.nitems = gram_items(mode, n2, r0, r1, pl.P);
    const int occ = occupancy((const void*)fn, pl.threads, pl.smem_bytes);
    pl.blocks = std::max<int64_t>(1, std::min<int64_t>((pl.nitems + fwpc - 1) / fwpc, (int64_t)occ * sms));
    pl.slots = pl.blocks * fwpc * pl.P;
    // lane u = 0 prefetches the handoff row 8 columns ahead of an 8-step tile
    // loop (fine columns)
    pl.hand_stride = 8 * (((M2c << lamC) + 10) / 8 + 2);
    return SK_OK;
  }
  int smem = 0;
  FwdFn fn = f32              ? (kind == LINEAR ? select_fwd_linear_f32(s, smem) : nullptr)
             : short_r        ? select_fwd_short(s, smem)
             : kind == LINEAR ? select_fwd_linear(s, smem)
             : kind == RBF    ? select_fwd_rbf(s, smem)
                              : select_fwd_delta(s, smem);
  if (!fn) return fail(SK_INVALID_ARGUMENT, "no forward kernel instance for this shape");
  pl.shape = s;
  pl.fn = fn;
  pl.smem_bytes = smem;
  pl.P = s.XW ? 1 : 32 / s.G;
  if (mode == BATCH) pl.nitems = (npairs + pl.P - 1) / pl.P;
  else pl.nitems = gram_items(mode, n2, r0, r1, pl.P);
  // few work items: smaller CTAs spread them over all SMs (each SM has its own
  // FP64 pipe); e.g. BASELINE config 1 (32 pairs) used 8 SMs with 4-warp CTAs
  const int fw_warps = (int)std::min<int64_t>(4, std::max<int64_t>(1, ceil_div(pl.nitems, sms)));
  pl.threads = s.XW ? 32 * s.W : 32 * fw_warps;
  const int warps = pl.threads / 32;
  const int occ = occupancy((const void*)fn, pl.threads, smem);
  int64_t want = s.XW ? pl.nitems : (pl.nitems + warps - 1) / warps;
  pl.blocks = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)occ * sms));
  pl.slots = s.XW ? pl.blocks : pl.blocks * warps * pl.P;
  pl.hand_stride = (int64_t)align_up((size_t)((M2c << lamC) + 1), 4);
  (void)nch;
  if (std::getenv("SK_DEBUG_PLAN")) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, (const void*)fn);
    std::fprintf(stderr, "plan_forward: XW %d W %d G %d R %d DP %d threads %d smem %d occ %d blocks %lld "
                 "static %zu maxdyn %d regs %d\n", (int)s.XW, s.W, s.G, s.R, s.DP, pl.threads, smem, occ,
                 (long long)pl.blocks, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.numRegs);
  }
  return SK_OK;
}

static size_t prep_elems(int kind, int64_t n, int64_t L, int dpad) {
  return kind == RBF ? (size_t)n * L * dpad : (size_t)n * (L - 1) * dpad;
}

// Prepares the rows side (scaled by `scale`) and, unless `share`, the columns
// side, in one launch (T: the arithmetic type of the kernels that read them).
// LR, LC, d: RAW points / dimension (the prepared arrays hold the transformed path)
template <typename T, typename TO = T>
static void launch_prep(int kind, const T* xr, int64_t nR, int64_t LR, const T* xc, int64_t nC,
                        int64_t LC, bool share, int64_t d, int dpad, TO* outR, TO* outC,
                        cudaStream_t st, double scale, int tf = TF_NONE) {
  const size_t total = prep_elems(kind, nR, eff_len(LR, tf), dpad) +
                       (share ? 0 : prep_elems(kind, nC, eff_len(LC, tf), dpad));
  if (total == 0) return;
  const int blocks = (int)std::min<size_t>((total + 255) / 256, 4096);
  PrepSide<T, TO> s0{xr, nR, LR, scale, outR}, s1{xc, nC, LC, 1.0, outC};
  prep_sides<T, TO><<<blocks, 256, 0, st>>>(s0, s1, share ? 1 : 2, kind == RBF ? 1 : 0, tf, d,
                                            dpad);
}

static int launch_transform_adjoint(const double* gt, int64_t n, int64_t L, int64_t d, int tf,
                                    double* grad, bool accumulate, cudaStream_t st) {
  const int64_t total = n * L * d;
  if (total <= 0) return SK_OK;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
  transform_adjoint_kernel<<<blocks, 256, 0, st>>>(gt, n, L, d, tf, grad, accumulate ? 1 : 0);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

static int validate(int64_t L1, int64_t L2, int64_t d, int lam1, int lam2, int kind,
                    double sigma) {
  if (L1 < 2 || L2 < 2) return fail(SK_INVALID_ARGUMENT, "paths need at least 2 points");
  if (d < 1) return fail(SK_INVALID_ARGUMENT, "path dimension must be >= 1");
  if (lam1 < 0 || lam2 < 0) return fail(SK_INVALID_ARGUMENT, "dyadic orders must be >= 0");
  if (lam1 > 16 || lam2 > 16) return fail(SK_INVALID_ARGUMENT, "dyadic order > 16 unsupported");
  if (kind != SK_STATIC_LINEAR && kind != SK_STATIC_RBF)
    return fail(SK_INVALID_ARGUMENT, "unknown static kernel");
  if (kind == SK_STATIC_RBF && !(sigma > 0.0))
    return fail(SK_INVALID_ARGUMENT, "RBF sigma must be > 0");
  if (((L1 - 1) << lam1) >= (int64_t)1 << 30 || ((L2 - 1) << lam2) >= (int64_t)1 << 30)
    return fail(SK_INVALID_ARGUMENT, "fine grid too large");
  return SK_OK;
}

static Problem base_problem(int kind, int64_t d, int lamR, int lamC, int64_t LR, int64_t LC,
                            double sigma) {
  Problem pb{};
  int nch = 1;
  int DP = pick_dp(d, nch);
  pb.kind = kind;
  pb.dpad = DP * nch;
  pb.nch = nch;
  pb.M1c = (int)(LR - 1);
  pb.M2c = (int)(LC - 1);
  pb.lam1 = lamR;
  pb.lam2 = lamC;
  pb.scale = std::ldexp(1.0, -(lamR + lamC));
  pb.pscale = pb.scale;
  pb.inv2s2 = kind == RBF ? 1.0 / (2.0 * sigma * sigma) : 0.0;
  pb.invs2 = kind == RBF ? 1.0 / (sigma * sigma) : 0.0;
  return pb;
}

// Workspace layout for forward calls: [prep rows][prep cols][handoff rows].
struct FwdLayout {
  size_t prepR = 0, prepC = 0, hand = 0, total = 0;
};

// esz: the recurrence's element size (handoff rows); pesz: the prepared paths'
// (8 for the DMMA kernels' fp64 operands, also under FP32 arithmetic)
static FwdLayout fwd_layout(const FwdPlan& pl, int kind, int64_t nR, int64_t LR, int64_t nC,
                            int64_t LC, int dpad, bool shared_paths, size_t esz = sizeof(double),
                            size_t pesz = 0) {
  FwdLayout lo;
  if (pesz == 0) pesz = esz;
  lo.prepR = align_up(prep_elems(kind, nR, LR, dpad) * pesz, 256);
  lo.prepC = shared_paths ? 0 : align_up(prep_elems(kind, nC, LC, dpad) * pesz, 256);
  lo.hand = align_up((size_t)pl.slots * pl.hand_stride * esz, 256);
  lo.total = lo.prepR + lo.prepC + lo.hand;
  return lo;
}

static Geometry orient(int64_t n1, int64_t n2, int64_t L1, int64_t L2, int lam1, int lam2) {
  Geometry g;
  int64_t m1 = (L1 - 1) << lam1, m2 = (L2 - 1) << lam2;
  g.swap = m2 > m1;
  g.nR = g.swap ? n2 : n1;
  g.nC = g.swap ? n1 : n2;
  g.LR = g.swap ? L2 : L1;
  g.LC = g.swap ? L1 : L2;
  g.lamR = g.swap ? lam2 : lam1;
  g.lamC = g.swap ? lam1 : lam2;
  return g;
}

// f32: FP32 arithmetic kernels (linear static kernel): x, y, out are float
// arrays; otherwise double.
static int forward_impl(const void* x, const void* y, int64_t n1, int64_t n2, int64_t L1,
                        int64_t L2, int64_t d, int lam1, int lam2, int kind, double sigma,
                        int mode, int64_t r0, int64_t r1, void* out, void* ws,
                        size_t ws_bytes, cudaStream_t st, size_t* query, bool f32 = false,
                        int tf = TF_NONE) {
  if (int rc = validate(L1, L2, d, lam1, lam2, kind, sigma)) return rc;
  if (tf < TF_NONE || tf > TF_LEADLAG) return fail(SK_INVALID_ARGUMENT, "unknown path transform");
  // the kernels solve the transformed paths (raw L1, L2, d only for the prep)
  const int64_t L1r = L1, L2r = L2, dr = d;
  L1 = eff_len(L1, tf);
  L2 = eff_len(L2, tf);
  d = eff_dim(d, tf);
  if (f32 && kind != LINEAR)
    return fail(SK_INVALID_ARGUMENT, "FP32 arithmetic supports the linear static kernel only");
  const size_t esz = f32 ? sizeof(float) : sizeof(double);
  const bool sym = mode == GRAM_SYM;
  Geometry g = orient(n1, n2, L1, L2, lam1, lam2);
  Problem pb = base_problem(kind, d, g.lamR, g.lamC, g.LR, g.LC, sigma);
  pb.mode = mode;
  pb.n1 = (int)n1;
  pb.n2 = (int)n2;
  pb.r0 = (int)r0;
  pb.r1 = (int)r1;
  pb.c0 = 0;
  pb.c1 = (int)n2;
  pb.swap = g.swap ? 1 : 0;
  pb.npairs = mode == BATCH ? n1 : 0;
  pb.ldo = n2;
  FwdPlan pl;
  const int64_t npairs = mode == BATCH ? n1 : (r1 - r0) * n2;
  // few short pairs (BASELINE config 1): one warp per pair from a shared
  // coefficient tile, no workspace, no prep launch (sk_small.cu)
  static const bool no_small = std::getenv("SK_NO_SMALL") && std::getenv("SK_NO_SMALL")[0] == '1';
  if (!no_small && mode == BATCH && kind == LINEAR && !f32 && tf == TF_NONE &&
      npairs <= 4 * (int64_t)device_sms() && pb.M1c << g.lamR <= 64 &&
      pb.M2c << g.lamC <= 64 && d <= 32) {
    if (query) {
      *query = 0;
      return SK_OK;
    }
    const double* xr = static_cast<const double*>(g.swap ? y : x);
    const double* xc = static_cast<const double*>(g.swap ? x : y);
    if (launch_small_fwd(xr, xc, n1, g.LR, g.LC, d, g.lamR, g.lamC, pb.scale,
                         static_cast<double*>(out), device_sms(), st)) {
      SK_CUDA(cudaGetLastError());
      return SK_OK;
    }
    return fail(SK_CUDA_ERROR, "small-pair forward could not be launched");
  }
  if (int rc = plan_forward(pl, kind, d, g.lamR, g.lamC, pb.M1c, pb.M2c, npairs,
                            mode != BATCH && !(mode == GRAM_CROSS && g.swap), mode, (int)n2,
                            (int)r0, (int)r1, f32))
    return rc;
  // LINEAR: the exact dyadic factor 2^-(lamR+lamC) is folded into the row
  // increments, so the kernel forms p without a multiply; a symmetric Gram then
  // needs a separate (unscaled) column copy when the factor is not 1.
  const bool fold = kind == LINEAR;
  const bool share = sym && !(fold && pb.scale != 1.0);
  // FP32 arithmetic on the DMMA Gram forward: fp64 operands (exact increments
  // of the float points), float recurrence
  const bool f32mma = f32 && pl.shape.MMA;
  FwdLayout lo = fwd_layout(pl, kind, g.nR, g.LR, g.nC, g.LC, pb.dpad, share, esz,
                            f32mma ? sizeof(double) : esz);
  if (query) {
    *query = lo.total;
    return SK_OK;
  }
  if (npairs <= 0 || pl.nitems == 0) return SK_OK;
  if (ws_bytes < lo.total)
    return fail(SK_INVALID_ARGUMENT, "workspace too small: need " + std::to_string(lo.total) +
                                         " bytes, got " + std::to_string(ws_bytes));
  char* base = static_cast<char*>(ws);
  char* prepR = base;
  char* prepC = share ? prepR : base + lo.prepR;
  double* hand = reinterpret_cast<double*>(base + lo.prepR + lo.prepC);
  const void* xr = g.swap ? y : x;
  const void* xc = g.swap ? x : y;
  if (f32mma)
    launch_prep<float, double>(kind, (const float*)xr, g.nR, g.swap ? L2r : L1r, (const float*)xc,
                               g.nC, g.swap ? L1r : L2r, share, dr, pb.dpad, (double*)prepR,
                               (double*)prepC, st, fold ? pb.scale : 1.0, tf);
  else if (f32)
    launch_prep<float>(kind, (const float*)xr, g.nR, g.swap ? L2r : L1r, (const float*)xc, g.nC,
                       g.swap ? L1r : L2r, share, dr, pb.dpad, (float*)prepR, (float*)prepC, st,
                       fold ? pb.scale : 1.0, tf);
  else
    launch_prep<double>(kind, (const double*)xr, g.nR, g.swap ? L2r : L1r, (const double*)xc, g.nC,
                        g.swap ? L1r : L2r, share, dr, pb.dpad, (double*)prepR, (double*)prepC,
                        st, fold ? pb.scale : 1.0, tf);
  if (fold) pb.pscale = 1.0;
  pb.R.p = reinterpret_cast<const double*>(prepR);
  pb.R.rows = (int)(g.LR - 1);
  pb.R.path_stride = (kind == RBF ? g.LR : g.LR - 1) * pb.dpad;
  pb.C.p = reinterpret_cast<const double*>(prepC);
  pb.C.rows = (int)(g.LC - 1);
  pb.C.path_stride = (kind == RBF ? g.LC : g.LC - 1) * pb.dpad;
  pb.nitems = pl.nitems;
  pb.out = static_cast<double*>(out);
  pl.fn<<<(unsigned)pl.blocks, pl.threads, pl.smem_bytes, st>>>(pb, hand, pl.hand_stride);
  SK_CUDA(cudaGetLastError());
  if (sym) {
    int64_t span = r1 - r0;
    int blocks = (int)std::min<int64_t>((span * span + 255) / 256, 4096);
    if (span > 1) {
      if (f32) mirror_upper<float><<<blocks, 256, 0, st>>>((float*)out, n2, (int)r0, (int)r1);
      else mirror_upper<double><<<blocks, 256, 0, st>>>((double*)out, n2, (int)r0, (int)r1);
    }
    SK_CUDA(cudaGetLastError());
  }
  return SK_OK;
}

}  // namespace sk

using namespace sk;

extern "C" {

int sk_abi_version(void) { return SK_ABI_VERSION; }
const char* sk_last_error(void) { return g_err.c_str(); }
int sk_device_sms(void) { return device_sms(); }

size_t sk_forward_batch_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d, int lam1,
                                        int lam2, int static_kernel) {
  size_t q = 0;
  if (forward_impl(nullptr, nullptr, B, B, L1, L2, d, lam1, lam2, static_kernel, 1.0, BATCH, 0,
                   B, nullptr, nullptr, 0, nullptr, &q))
    return 0;
  return q;
}

int sk_forward_batch(const double* x, const double* y, int64_t B, int64_t L1, int64_t L2,
                     int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                     double* out, void* ws, size_t ws_bytes, void* stream) {
  if (B < 0) return fail(SK_INVALID_ARGUMENT, "negative batch");
  return forward_impl(x, y, B, B, L1, L2, d, lam1, lam2, static_kernel, sigma, BATCH, 0, B, out,
                      ws, ws_bytes, (cudaStream_t)stream, nullptr);
}

size_t sk_forward_gram_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                       int64_t d, int lam1, int lam2, int static_kernel,
                                       int symmetric) {
  size_t q = 0;
  if (forward_impl(nullptr, nullptr, n1, n2, L1, L2, d, lam1, lam2, static_kernel, 1.0,
                   symmetric ? GRAM_SYM : GRAM_CROSS, 0, n1, nullptr, nullptr, 0, nullptr, &q))
    return 0;
  return q;
}

int sk_forward_gram(const double* x, const double* y, int64_t n1, int64_t n2, int64_t L1,
                    int64_t L2, int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                    int64_t row_begin, int64_t row_end, double* out, void* ws, size_t ws_bytes,
                    void* stream) {
  const bool sym = (y == nullptr);
  if (sym && (n2 != n1 || L2 != L1))
    return fail(SK_INVALID_ARGUMENT, "symmetric Gram needs n2 == n1 and L2 == L1");
  if (row_begin < 0 || row_end > n1 || row_begin > row_end)
    return fail(SK_INVALID_ARGUMENT, "row range out of bounds");
  return forward_impl(x, sym ? x : y, n1, n2, L1, L2, d, lam1, lam2, static_kernel, sigma,
                      sym ? GRAM_SYM : GRAM_CROSS, row_begin, row_end, out, ws, ws_bytes,
                      (cudaStream_t)stream, nullptr);
}

size_t sk_forward_batch_f32_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d,
                                            int lam1, int lam2, int transform) {
  size_t q = 0;
  if (forward_impl(nullptr, nullptr, B, B, L1, L2, d, lam1, lam2, LINEAR, 1.0, BATCH, 0, B,
                   nullptr, nullptr, 0, nullptr, &q, true, transform))
    return 0;
  return q;
}

int sk_forward_batch_f32(const float* x, const float* y, int64_t B, int64_t L1, int64_t L2,
                         int64_t d, int lam1, int lam2, int transform, float* out, void* ws,
                         size_t ws_bytes, void* stream) {
  if (B < 0) return fail(SK_INVALID_ARGUMENT, "negative batch");
  return forward_impl(x, y, B, B, L1, L2, d, lam1, lam2, LINEAR, 1.0, BATCH, 0, B, out, ws,
                      ws_bytes, (cudaStream_t)stream, nullptr, true, transform);
}

size_t sk_forward_gram_f32_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                           int64_t d, int lam1, int lam2, int symmetric,
                                           int transform) {
  size_t q = 0;
  if (forward_impl(nullptr, nullptr, n1, n2, L1, L2, d, lam1, lam2, LINEAR, 1.0,
                   symmetric ? GRAM_SYM : GRAM_CROSS, 0, n1, nullptr, nullptr, 0, nullptr, &q,
                   true, transform))
    return 0;
  return q;
}

int sk_forward_gram_f32(const float* x, const float* y, int64_t n1, int64_t n2, int64_t L1,
                        int64_t L2, int64_t d, int lam1, int lam2, int transform,
                        int64_t row_begin, int64_t row_end, float* out, void* ws, size_t ws_bytes,
                        void* stream) {
  const bool sym = (y == nullptr);
  if (sym && (n2 != n1 || L2 != L1))
    return fail(SK_INVALID_ARGUMENT, "symmetric Gram needs n2 == n1 and L2 == L1");
  if (row_begin < 0 || row_end > n1 || row_begin > row_end)
    return fail(SK_INVALID_ARGUMENT, "row range out of bounds");
  return forward_impl(x, sym ? x : y, n1, n2, L1, L2, d, lam1, lam2, LINEAR, 1.0,
                      sym ? GRAM_SYM : GRAM_CROSS, row_begin, row_end, out, ws, ws_bytes,
                      (cudaStream_t)stream, nullptr, true, transform);
}

// ---- path transforms (time augmentation / lead-lag) applied inside the call
size_t sk_forward_batch_tf_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d,
                                           int lam1, int lam2, int static_kernel, int transform) {
  size_t q = 0;
  if (forward_impl(nullptr, nullptr, B, B, L1, L2, d, lam1, lam2, static_kernel, 1.0, BATCH, 0,
                   B, nullptr, nullptr, 0, nullptr, &q, false, transform))
    return 0;
  return q;
}

int sk_forward_batch_tf(const double* x, const double* y, int64_t B, int64_t L1, int64_t L2,
                        int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                        int transform, double* out, void* ws, size_t ws_bytes, void* stream) {
  if (B < 0) return fail(SK_INVALID_ARGUMENT, "negative batch");
  return forward_impl(x, y, B, B, L1, L2, d, lam1, lam2, static_kernel, sigma, BATCH, 0, B, out,
                      ws, ws_bytes, (cudaStream_t)stream, nullptr, false, transform);
}

size_t sk_forward_gram_tf_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                          int64_t d, int lam1, int lam2, int static_kernel,
                                          int symmetric, int transform) {
  size_t q = 0;
  if (forward_impl(nullptr, nullptr, n1, n2, L1, L2, d, lam1, lam2, static_kernel, 1.0,
                   symmetric ? GRAM_SYM : GRAM_CROSS, 0, n1, nullptr, nullptr, 0, nullptr, &q,
                   false, transform))
    return 0;
  return q;
}

int sk_forward_gram_tf(const double* x, const double* y, int64_t n1, int64_t n2, int64_t L1,
                       int64_t L2, int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                       int transform, int64_t row_begin, int64_t row_end, double* out, void* ws,
                       size_t ws_bytes, void* stream) {
  const bool sym = (y == nullptr);
  if (sym && (n2 != n1 || L2 != L1))
    return fail(SK_INVALID_ARGUMENT, "symmetric Gram needs n2 == n1 and L2 == L1");
  if (row_begin < 0 || row_end > n1 || row_begin > row_end)
    return fail(SK_INVALID_ARGUMENT, "row range out of bounds");
  return forward_impl(x, sym ? x : y, n1, n2, L1, L2, d, lam1, lam2, static_kernel, sigma,
                      sym ? GRAM_SYM : GRAM_CROSS, row_begin, row_end, out, ws, ws_bytes,
                      (cudaStream_t)stream, nullptr, false, transform);
}

int sk_transform_adjoint(const double* g_t, int64_t n, int64_t L, int64_t d, int transform,
                         double* grad, int accumulate, void* stream) {
  if (n < 0 || L < 1 || d < 1 || !g_t || !grad) return fail(SK_INVALID_ARGUMENT, "bad arguments");
  if (transform < TF_NONE || transform > TF_LEADLAG)
    return fail(SK_INVALID_ARGUMENT, "unknown path transform");
  if (transform == TF_NONE) {
    if (accumulate) return fail(SK_INVALID_ARGUMENT, "identity transform: nothing to map");
    SK_CUDA(cudaMemcpyAsync(grad, g_t, sizeof(double) * n * L * d, cudaMemcpyDeviceToDevice,
                            (cudaStream_t)stream));
    return SK_OK;
  }
  return launch_transform_adjoint(g_t, n, L, d, transform, grad, accumulate != 0,
                                  (cudaStream_t)stream);
}

static int solve_delta_impl(const double* delta, int64_t B, int64_t r1, int64_t r2, int lam1,
                            int lam2, double* out, void* ws, size_t ws_bytes,
                            cudaStream_t st, size_t* query) {
  if (r1 < 1 || r2 < 1) return fail(SK_INVALID_ARGUMENT, "increment matrix must be non-empty");
  if (lam1 < 0 || lam2 < 0 || lam1 > 16 || lam2 > 16)
    return fail(SK_INVALID_ARGUMENT, "dyadic orders must be in [0, 16]");
  // delta is solved un-transposed: rows = delta rows (kernel.py:106-110 grid
  // orientation; the strip path transposes but is bitwise equal, test_kernel.py:65-71)
  Problem pb = base_problem(DELTA, 4, lam1, lam2, r1 + 1, r2 + 1, 1.0);
  pb.mode = BATCH;
  pb.npairs = B;
  pb.delta = delta;
  FwdPlan pl;
  if (int rc = plan_forward(pl, DELTA, 4, lam1, lam2, r1, r2, B, false, BATCH, 0, 0, 0))
    return rc;
  size_t need = align_up((size_t)pl.slots * pl.hand_stride * sizeof(double), 256);
  if (query) {
    *query = need;
    return SK_OK;
  }
  if (B == 0) return SK_OK;
  if (ws_bytes < need) return fail(SK_INVALID_ARGUMENT, "workspace too small");
  pb.nitems = pl.nitems;
  pb.out = out;
  pl.fn<<<(unsigned)pl.blocks, pl.threads, pl.smem_bytes, st>>>(
      pb, static_cast<double*>(ws), pl.hand_stride);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

size_t sk_solve_delta_workspace_bytes(int64_t B, int64_t r1, int64_t r2, int lam1, int lam2) {
  size_t q = 0;
  if (solve_delta_impl(nullptr, B, r1, r2, lam1, lam2, nullptr, nullptr, 0, nullptr, &q))
    return 0;
  return q;
}

int sk_solve_delta(const double* delta, int64_t B, int64_t r1, int64_t r2, int lam1, int lam2,
                   double* out, void* ws, size_t ws_bytes, void* stream) {
  return solve_delta_impl(delta, B, r1, r2, lam1, lam2, out, ws, ws_bytes,
                          (cudaStream_t)stream, nullptr);
}

int sk_solve_delta_grid(const double* delta, int64_t r1, int64_t r2, int lam1, int lam2,
                        double* grid, void* stream) {
  if (r1 < 1 || r2 < 1) return fail(SK_INVALID_ARGUMENT, "increment matrix must be non-empty");
  if (lam1 < 0 || lam2 < 0 || lam1 > 16 || lam2 > 16)
    return fail(SK_INVALID_ARGUMENT, "dyadic orders must be in [0, 16]");
  grid_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(delta, (int)r1, (int)r2, lam1, lam2,
                                                    std::ldexp(1.0, -(lam1 + lam2)), grid);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

}  // extern "C"


// ====================================================================== backward
namespace sk {

struct BwdPlan {
  BwdShape shape;
  BwdFn fn = nullptr;
  int smem_bytes = 0;
  int threads = 128;
  int64_t blocks = 0, slots = 0, nitems = 0;
  int64_t rowck_stride = 0, colck_stride = 0, pck_stride = 0, row_stride = 0, dbuf_stride = 0, gscr_stride = 0,
          rsum_stride = 0;
};

static int plan_backward(BwdPlan& pl, int kind, int64_t d, int lamR, int lamC, int64_t M1c,
                         int64_t M2c, int mode, int64_t npairs, int n2, int r0, int r1,
                         bool shared_cols, bool f32 = false, int c0 = 0, int c1 = -1) {
  int nch = 1;
  BwdShape s{};
  s.kind = kind;
  s.DP = pick_dp(d, nch);
  const bool wide = nch > 1;  // d > 32: DP-chunks, adjoint mapped after the sweep
  // Gram tiles of the linear kernel at dyadic order 0: DMMA backward
  // (sk_mma_bwd.cuh).  SK_NO_MMA=1 keeps the r01 kernels.
  // (d <= 4 runs the DP = 8 instance on zero-padded increments: the padding
  // adds exact zeros to every FMA chain, so p is bitwise unchanged)
  // dyadic orders > 0: the DY instance (coarse p tiles) only on request
  // (SK_MMA_DY=1, read per plan like SK_NO_MMA): its gradient maps run per
  // fine cell where the FMA-pipe backward sums D per coarse cell first, and it
  // measured no faster (n = 256 Grams, lambda 1: d = 16 30.3 vs 30.0 ms,
  // d = 8 23.6 vs 14.8 ms; lambda 2, d = 16: 28.1 vs 25.8 ms)
  const char* mdy = std::getenv("SK_MMA_DY");
  const bool dy = lamR + lamC > 0;
  const bool dy_ok = mdy && mdy[0] == '1';
  s.MMA = shared_cols && kind == LINEAR && (!dy || dy_ok) && s.DP <= 16 && !wide &&
          !(std::getenv("SK_NO_MMA") && std::getenv("SK_NO_MMA")[0] == '1');
  // FP32 backward: the DMMA Gram instance at order 0 only (d <= 16)
  if (f32 && !(shared_cols && kind == LINEAR && !dy && s.DP <= 16 && !wide))
    return fail(SK_INVALID_ARGUMENT,
                "FP32 backward supports linear Gram tiles at dyadic order 0 with d <= 16");
  if (f32) s.MMA = true;
  if (s.MMA) {
    if (s.DP == 4) s.DP = 8;
    const char* w = std::getenv("SK_BWD_WPC");
    s.WPC = (w && (w[0] == '3' || w[0] == '4') && !f32) ? w[0] - '0' : 2;  // measured: 2 >= 4 > 3
    int per_warp = 0;
    BwdFn fn = select_bwd_mma(s.DP, s.WPC, per_warp, dy, f32);
    if (!fn) return fail(SK_INVALID_ARGUMENT, "no DMMA backward instance for this shape");
    pl.shape = s;
    pl.fn = fn;
    pl.threads = 32 * s.WPC;
    pl.smem_bytes = per_warp * (int)sizeof(double) * s.WPC;
    pl.nitems = super_items(mode, n2, r0, r1, c0, c1);
    const int sms = device_sms();
    const int occ = occupancy((const void*)fn, pl.threads, pl.smem_bytes);
    pl.blocks = std::max<int64_t>(1, std::min<int64_t>((pl.nitems + s.WPC - 1) / s.WPC,
                                                       (int64_t)occ * sms));
    pl.slots = pl.blocks * s.WPC;
    // (fine rows / columns: the strips and blocks are fine-grid ones)
    const int64_t M1f = M1c << lamR, M2f = M2c << lamC;
    const int64_t nstrips = (M1f + 7) / 8, NT8 = (M2f + 10) / 8;
    // rowck: the strips' top rows [strip][8 pairs][8 (NT8 + 5)]; colck: every
    // lane's two values per block (double2); pck: its bottom value a column
    // before (sk_mma_bwd.cuh)
    pl.rowck_stride = nstrips * 8 * 8 * (NT8 + 5);
    pl.colck_stride = nstrips * NT8 * 32 * 2;
    pl.pck_stride = nstrips * NT8 * 32;
    // per pair, 8 pairs per slot: the adjoint row sits at column + 3 and the
    // handoff row is prefetched 4 iterations (32 columns) ahead
    pl.row_stride = 8 * (NT8 + 5);
    pl.dbuf_stride = 0;
    pl.gscr_stride = 8 * NT8 * s.DP;
    pl.rsum_stride = 8 * M1f * s.DP;
    cap_slots(pl.blocks, pl.slots, s.WPC,
              8.0 * (pl.rowck_stride + pl.colck_stride + pl.pck_stride + pl.gscr_stride +
                     pl.rsum_stride + 16 * pl.row_stride));
    return SK_OK;
  }
  s.R = bwd_rows_per_lane(s.DP);
  s.FR = std::min(1 << std::min(lamR, 3), s.R);
  s.F = std::min(1 << std::min(lamC, 2), 4);
  s.NW = 1;
  const int sms = device_sms();
  {
    // few long pairs (BASELINE config 2: 256 pairs of 1020 fine rows): one pair
    // per CTA of NW = 4 warps (measured at config 2: RBF 9.18 ms with one pair
    // per warp, 3.29 ms at NW = 4, 3.93 ms at NW = 8 (one strip, longer skew))
    const int64_t M1 = M1c << lamR;
    const int64_t lanes_per_pair = (M1 + s.R - 1) / s.R;
    static const int nw_force = [] {
      const char* e = std::getenv("SK_BWD_XW_NW");  // tuning knob: 1 (off), 4 or 8
      const int v = (e && e[0]) ? std::atoi(e) : 0;
      return (v == 1 || v == 4 || v == 8) ? v : 0;
    }();
    if (mode == BATCH && !wide && s.DP <= 8 && npairs * 32 < (int64_t)sms * 512 &&
        lanes_per_pair > 64) {
      s.NW = 4;
      if (nw_force) s.NW = nw_force;
      // pairs taller than one 4-row strip: 8 rows per lane, one strip (C2:
      // RBF backward 1.62 -> 1.39 ms, linear 1.35 -> 1.03 ms)
      static const int r_force = [] {
        const char* e = std::getenv("SK_BWD_XW_R");  // tuning knob: 4 or 8 (DP = 8, NW = 4)
        return (e && e[0] == '4') ? 4 : (e && e[0] == '8') ? 8 : 0;
      }();
      const bool r8 = r_force ? r_force == 8 : M1 > 32 * s.NW * s.R;
      if (r8 && s.DP == 8 && s.NW == 4) {
        s.R = 8;
        s.FR = std::min(1 << std::min(lamR, 3), s.R);
      }
    }
  }
  int smd = 0;
  BwdFn fn = s.NW > 1 ? (kind == RBF ? select_bwd_xw_rbf(s, smd) : select_bwd_xw_linear(s, smd))
             : kind == RBF ? select_bwd_rbf(s, smd)
             : wide        ? select_bwd_wide(s, smd)
                           : select_bwd_linear(s, smd);
  if (!fn) return fail(SK_INVALID_ARGUMENT, "no backward kernel instance for this shape");
  pl.shape = s;
  pl.fn = fn;
  pl.nitems = mode == BATCH ? npairs : gram_items(mode, n2, r0, r1, 1, false);
  const int NL = 32 * s.NW;  // lanes per pair
  int warps = 1;             // lane groups (pairs in flight) per CTA
  if (s.NW > 1) {
    pl.threads = NL;
    pl.smem_bytes = smd * (int)sizeof(double);
  } else {
    // few pairs: smaller CTAs spread them over all SMs
    pl.threads = 32 * (int)std::min<int64_t>(4, std::max<int64_t>(1, ceil_div(pl.nitems, sms)));
    warps = pl.threads / 32;
    pl.smem_bytes = smd * (int)sizeof(double) * warps;
  }
  const int occ = occupancy((const void*)fn, pl.threads, pl.smem_bytes);
  pl.blocks = std::max<int64_t>(1, std::min<int64_t>((pl.nitems + warps - 1) / warps,
                                                     (int64_t)occ * sms));
  pl.slots = pl.blocks * warps;
  const int64_t M1 = M1c << lamR, M2 = M2c << lamC;
  const int64_t Sc = bwd_steps_cols(s.DP, s.F), NC = M2 / s.F, NSTEP = (NC + Sc - 1) / Sc,
                NT = NSTEP + NL - 1,
                CB = s.NW > 1 ? bwd_block_steps_xw(s.R, s.F, (int)Sc)
                              : bwd_block_steps(s.DP, s.R, s.F, (int)Sc),
                NB = (NT + CB - 1) / CB;
  const int64_t nstrips = (M1 + NL * s.R - 1) / (NL * s.R);
  pl.rowck_stride = (int64_t)align_up((size_t)(nstrips * NT * Sc * s.F * NL), 32);
  pl.colck_stride = (int64_t)align_up((size_t)(nstrips * NB * s.R * NL), 32);
  pl.pck_stride = (int64_t)align_up((size_t)(nstrips * NT * Sc * (s.R / s.FR) * NL), 32);
  pl.row_stride = (int64_t)align_up((size_t)(M2 + 1), 32);
  pl.dbuf_stride = (kind == RBF || wide) ? (int64_t)align_up((size_t)(M1c * M2c), 32) : 0;
  // LINEAR: increment-gradient scratch; RBF: the epilogue's dF/dx chains [M1c+1][DP]
  pl.gscr_stride = kind == LINEAR ? (int64_t)align_up((size_t)((M1c + M2c) * s.DP * nch), 32)
                                  : (int64_t)align_up((size_t)((M1c + 1) * s.DP), 32);
  cap_slots(pl.blocks, pl.slots, warps,
            8.0 * (pl.rowck_stride + pl.colck_stride + pl.pck_stride + pl.dbuf_stride +
                   pl.gscr_stride + 2 * pl.row_stride));
  return SK_OK;
}

struct BwdLayout {
  size_t prepR = 0, prepC = 0, rowck = 0, colck = 0, pck = 0, rows = 0, dbuf = 0, gscr = 0,
         rsum = 0, accx = 0, accy = 0, total = 0;
};

// Gram gradients go through exact accumulators: the caller's (acc_x / acc_y,
// sk_backward_gram_acc) or, when those are NULL, per-call ones in the
// workspace that are finalised into grad_x / grad_y (+=) at the end.
static int backward_impl(const double* x, const double* y, int64_t n1, int64_t n2, int64_t L1,
                         int64_t L2, int64_t d, int lam1, int lam2, int kind, double sigma,
                         int mode, int64_t r0, int64_t r1, const double* cot, double* values,
                         double* grad_x, double* grad_y, void* ws, size_t ws_bytes,
                         cudaStream_t st, size_t* query, void* acc_x = nullptr,
                         void* acc_y = nullptr, int tf = TF_NONE, bool f32 = false,
                         int64_t c0 = 0, int64_t c1 = -1) {
  if (int rc = validate(L1, L2, d, lam1, lam2, kind, sigma)) return rc;
  if (tf < TF_NONE || tf > TF_LEADLAG) return fail(SK_INVALID_ARGUMENT, "unknown path transform");
  // the kernels solve the transformed paths; their point gradients (transformed
  // space) are mapped back by the transform's adjoint at the end
  const int64_t L1r = L1, L2r = L2, dr = d;
  L1 = eff_len(L1, tf);
  L2 = eff_len(L2, tf);
  d = eff_dim(d, tf);
  const bool sym = mode == GRAM_SYM;
  Geometry g = orient(n1, n2, L1, L2, lam1, lam2);
  Problem pb = base_problem(kind, d, g.lamR, g.lamC, g.LR, g.LC, sigma);
  pb.mode = mode;
  pb.n1 = (int)n1;
  pb.n2 = (int)n2;
  pb.r0 = (int)r0;
  pb.r1 = (int)r1;
  // column range (GRAM_CROSS on the DMMA backward; the values buffer is then
  // (r1 - r0) x (c1 - c0))
  if (c1 < 0) c1 = n2;
  if (c0 < 0 || c1 > n2 || c0 > c1 || c0 % SK_SUPER_B != 0 || ((c0 != 0 || c1 != n2) && mode != GRAM_CROSS))
    return fail(SK_INVALID_ARGUMENT, "column range must be 8-aligned, in bounds, cross Gram only");
  pb.c0 = (int)c0;
  pb.c1 = (int)c1;
  pb.swap = g.swap ? 1 : 0;
  pb.npairs = mode == BATCH ? n1 : 0;
  pb.ldo = c1 - c0;
  // row-block-major tiles (gram_item_amajor) keep the row accumulators in L2 but put
  // hundreds of warps on the same few paths (atomic contention): measured 1.29 s vs
  // 1.25 s per C3 step with the column-major order, so it stays off
  pb.amajor = 0;
  BwdPlan pl;
  const int64_t npairs = mode == BATCH ? n1 : (r1 - r0) * (c1 - c0);
  if (int rc = plan_backward(pl, kind, d, g.lamR, g.lamC, pb.M1c, pb.M2c, mode, npairs,
                             (int)n2, (int)r0, (int)r1,
                             mode != BATCH && !(mode == GRAM_CROSS && g.swap), f32, (int)c0,
                             (int)c1))
    return rc;
  if ((c0 != 0 || c1 != n2) && !pl.shape.MMA)
    return fail(SK_INVALID_ARGUMENT, "column ranges need the DMMA Gram backward (linear, dyadic "
                                     "order 0, d <= 16, x paths not shorter than y)");
  if (pl.shape.MMA) pb.dpad = pl.shape.DP;  // d <= 4: padded to the DP = 8 instance
  BwdLayout lo;
  lo.prepR = align_up(prep_elems(kind, g.nR, g.LR, pb.dpad) * sizeof(double), 256);
  // LINEAR rows carry the exact dyadic factor (as in the forward); a symmetric
  // Gram then needs an unscaled column copy when the factor is not 1
  const bool fold = kind == LINEAR;
  const bool share = sym && !(fold && pb.scale != 1.0);
  lo.prepC = share ? 0 : align_up(prep_elems(kind, g.nC, g.LC, pb.dpad) * sizeof(double), 256);
  lo.rowck = align_up((size_t)pl.slots * pl.rowck_stride * sizeof(double), 256);
  lo.colck = align_up((size_t)pl.slots * pl.colck_stride * sizeof(double), 256);
  lo.pck = align_up((size_t)pl.slots * pl.pck_stride * sizeof(double), 256);
  const int64_t row_slots = pl.slots * (pl.shape.MMA ? 8 : 1);  // DMMA: one row per pair of a tile
  lo.rows = align_up((size_t)row_slots * pl.row_stride * 2 * sizeof(double), 256);
  lo.dbuf = align_up((size_t)pl.slots * pl.dbuf_stride * sizeof(double), 256);
  lo.gscr = align_up((size_t)pl.slots * pl.gscr_stride * sizeof(double), 256);
  lo.rsum = align_up((size_t)pl.slots * pl.rsum_stride * sizeof(double), 256);
  const bool gram = mode != BATCH;
  const bool own_acc = gram && acc_x == nullptr;
  lo.accx = own_acc ? align_up(acc_bytes(n1, L1, d), 256) : 0;
  lo.accy = (own_acc && !sym) ? align_up(acc_bytes(n2, L2, d), 256) : 0;
  // transformed-space point gradients (mapped to the raw paths at the end)
  const bool tgrad = tf != TF_NONE && (own_acc || !gram);
  const size_t gtx = tgrad ? align_up((size_t)n1 * L1 * d * sizeof(double), 256) : 0;
  const size_t gty = (tgrad && !sym) ? align_up((size_t)n2 * L2 * d * sizeof(double), 256) : 0;
  lo.total = lo.prepR + lo.prepC + lo.rowck + lo.colck + lo.pck + lo.rows + lo.dbuf + lo.gscr +
             lo.rsum + lo.accx + lo.accy + gtx + gty;
  if (query) {
    *query = lo.total;
    return SK_OK;
  }
  if (mode == BATCH) {
    // batch gradients are written (not accumulated): zero them first
    if (grad_x) SK_CUDA(cudaMemsetAsync(grad_x, 0, sizeof(double) * n1 * L1r * dr, st));
    if (grad_y) SK_CUDA(cudaMemsetAsync(grad_y, 0, sizeof(double) * n2 * L2r * dr, st));
  }
  if (npairs <= 0 || pl.nitems == 0) return SK_OK;
  if (ws_bytes < lo.total)
    return fail(SK_INVALID_ARGUMENT, "workspace too small: need " + std::to_string(lo.total) +
                                         " bytes, got " + std::to_string(ws_bytes));
  if (own_acc || !gram) {
    if (!grad_x || (!sym && !grad_y)) return fail(SK_INVALID_ARGUMENT, "gradient buffers missing");
  } else if (!sym && !acc_y) {
    return fail(SK_INVALID_ARGUMENT, "cross Gram needs both accumulators");
  }
  char* base = static_cast<char*>(ws);
  double* prepR = reinterpret_cast<double*>(base);
  double* prepC = share ? prepR : reinterpret_cast<double*>(base + lo.prepR);
  char* p = base + lo.prepR + lo.prepC;
  BwdArgs ba{};
  ba.rowck = reinterpret_cast<double*>(p);
  ba.rowck_stride = pl.rowck_stride;
  p += lo.rowck;
  ba.colck = reinterpret_cast<double*>(p);
  ba.colck_stride = pl.colck_stride;
  p += lo.colck;
  ba.pck = reinterpret_cast<double*>(p);
  ba.pck_stride = pl.pck_stride;
  p += lo.pck;
  ba.hand = reinterpret_cast<double*>(p);
  ba.adj = ba.hand + row_slots * pl.row_stride;
  ba.row_stride = pl.row_stride;
  p += lo.rows;
  ba.dbuf = reinterpret_cast<double*>(p);
  ba.dbuf_stride = pl.dbuf_stride;
  p += lo.dbuf;
  ba.gscr = reinterpret_cast<double*>(p);
  ba.gscr_stride = pl.gscr_stride;
  p += lo.gscr;
  ba.rsum = reinterpret_cast<double*>(p);
  ba.rsum_stride = pl.rsum_stride;
  p += lo.rsum;
  unsigned long long* blob_x = static_cast<unsigned long long*>(acc_x);
  unsigned long long* blob_y = static_cast<unsigned long long*>(acc_y);
  if (own_acc) {
    blob_x = reinterpret_cast<unsigned long long*>(p);
    p += lo.accx;
    blob_y = sym ? nullptr : reinterpret_cast<unsigned long long*>(p);
    p += lo.accy;
    if (int rc = acc_init(blob_x, blob_y, acc_bytes(n1, L1, d), acc_bytes(n2, L2, d), cot, n1, n2,
                          sym, st))
      return rc;
  }
  if (sym) blob_y = blob_x;
  double* user_gx = grad_x;
  double* user_gy = grad_y;
  if (tgrad) {  // the kernels write / finalise into transformed-space buffers
    grad_x = reinterpret_cast<double*>(p);
    p += gtx;
    grad_y = sym ? nullptr : reinterpret_cast<double*>(p);
    p += gty;
    if (!gram) {
      SK_CUDA(cudaMemsetAsync(grad_x, 0, sizeof(double) * n1 * L1 * d, st));
      SK_CUDA(cudaMemsetAsync(grad_y, 0, sizeof(double) * n2 * L2 * d, st));
    }
  }
  ba.rows_exclusive = (1 << g.lamR) <= pl.shape.R ? 1 : 0;
  const double* xr = g.swap ? y : x;
  const double* xc = g.swap ? x : y;
  launch_prep<double>(kind, xr, g.nR, g.swap ? L2r : L1r, xc, g.nC, g.swap ? L1r : L2r, share, dr,
                      pb.dpad, prepR, prepC, st, fold ? pb.scale : 1.0, tf);
  if (fold) pb.pscale = 1.0;
  pb.R.p = prepR;
  pb.R.rows = (int)(g.LR - 1);
  pb.R.path_stride = (kind == RBF ? g.LR : g.LR - 1) * pb.dpad;
  pb.C.p = prepC;
  pb.C.rows = (int)(g.LC - 1);
  pb.C.path_stride = (kind == RBF ? g.LC : g.LC - 1) * pb.dpad;
  pb.nitems = pl.nitems;
  pb.out = values;
  // GRAM_SYM keeps (rows, cols) = (X_a, X_b): both sides land in grad_x
  double* gx_rows = sym ? grad_x : (g.swap ? grad_y : grad_x);
  double* gx_cols = sym ? grad_x : (g.swap ? grad_x : grad_y);
  ba.gradR = gx_rows;
  ba.gradC = gx_cols;
  if (gram) {
    unsigned long long* br = g.swap && !sym ? blob_y : blob_x;
    unsigned long long* bc = g.swap && !sym ? blob_x : blob_y;
    ba.metaR = br;
    ba.metaC = bc;
    ba.accR = br + kAccMeta;
    ba.accC = bc + kAccMeta;
  }
  ba.gR_path = g.LR * d;
  ba.gC_path = g.LC * d;
  ba.d = (int)d;
  ba.atomic = mode == BATCH ? 0 : 1;
  ba.cot = cot;
  ba.values = values;
#ifdef SK_PROFILING
  // profiling experiments (tools/build_variant.sh -DSK_PROFILING): skip phases
  ba.exp = std::getenv("SK_EXP") ? std::atoi(std::getenv("SK_EXP")) : 0;
#else
  ba.exp = 0;  // release builds never read SK_EXP (it would corrupt results)
#endif
  pl.fn<<<(unsigned)pl.blocks, pl.threads, pl.smem_bytes, st>>>(pb, ba);
  SK_CUDA(cudaGetLastError());
  if (own_acc) {
    if (int rc = acc_finalize(blob_x, n1 * L1 * d, grad_x, !tgrad, st)) return rc;
    if (!sym)
      if (int rc = acc_finalize(blob_y, n2 * L2 * d, grad_y, !tgrad, st)) return rc;
  }
  if (tgrad) {  // batch: written; Gram: accumulated (+=) like the plain call
    if (int rc = launch_transform_adjoint(grad_x, n1, L1r, dr, tf, user_gx, gram, st)) return rc;
    if (!sym)
      if (int rc = launch_transform_adjoint(grad_y, n2, L2r, dr, tf, user_gy, gram, st)) return rc;
  }
  return SK_OK;
}

}  // namespace sk

extern "C" {

size_t sk_backward_batch_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d,
                                         int lam1, int lam2, int static_kernel) {
  size_t q = 0;
  if (backward_impl(nullptr, nullptr, B, B, L1, L2, d, lam1, lam2, static_kernel, 1.0, BATCH, 0,
                    B, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, &q))
    return 0;
  return q;
}

int sk_backward_batch(const double* x, const double* y, int64_t B, int64_t L1, int64_t L2,
                      int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                      const double* cot, double* values, double* grad_x, double* grad_y,
                      void* ws, size_t ws_bytes, void* stream) {
  if (B < 0) return fail(SK_INVALID_ARGUMENT, "negative batch");
  return backward_impl(x, y, B, B, L1, L2, d, lam1, lam2, static_kernel, sigma, BATCH, 0, B, cot,
                       values, grad_x, grad_y, ws, ws_bytes, (cudaStream_t)stream, nullptr);
}

size_t sk_backward_gram_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                        int64_t d, int lam1, int lam2, int static_kernel,
                                        int symmetric) {
  size_t q = 0;
  if (backward_impl(nullptr, nullptr, n1, n2, L1, L2, d, lam1, lam2, static_kernel, 1.0,
                    symmetric ? GRAM_SYM : GRAM_CROSS, 0, n1, nullptr, nullptr, nullptr,
                    nullptr, nullptr, 0, nullptr, &q))
    return 0;
  return q;
}

int sk_value_and_grad_gram(const double* x, const double* y, int64_t n1, int64_t n2,
                           int64_t L1, int64_t L2, int64_t d, int lam1, int lam2,
                           int static_kernel, double sigma, int64_t row_begin, int64_t row_end,
                           const double* cot, double* values, double* grad_x, double* grad_y,
                           void* ws, size_t ws_bytes, void* stream) {
  const bool sym = (y == nullptr);
  if (sym && (n2 != n1 || L2 != L1))
    return fail(SK_INVALID_ARGUMENT, "symmetric Gram needs n2 == n1 and L2 == L1");
  if (row_begin < 0 || row_end > n1 || row_begin > row_end)
    return fail(SK_INVALID_ARGUMENT, "row range out of bounds");
  if (!cot) return fail(SK_INVALID_ARGUMENT, "Gram backward needs the cotangent matrix");
  if (!values) return fail(SK_INVALID_ARGUMENT, "values buffer missing");
  if (int rc = backward_impl(x, sym ? x : y, n1, n2, L1, L2, d, lam1, lam2, static_kernel, sigma,
                             sym ? GRAM_SYM : GRAM_CROSS, row_begin, row_end, cot, values,
                             grad_x, grad_y, ws, ws_bytes, (cudaStream_t)stream, nullptr))
    return rc;
  const int64_t span = row_end - row_begin;
  if (sym && span > 1) {
    int blocks = (int)std::min<int64_t>((span * span + 255) / 256, 4096);
    mirror_upper<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(values, n2, (int)row_begin,
                                                           (int)row_end);
    SK_CUDA(cudaGetLastError());
  }
  return SK_OK;
}

int sk_backward_gram(const double* x, const double* y, int64_t n1, int64_t n2, int64_t L1,
                     int64_t L2, int64_t d, int lam1, int lam2, int static_kernel,
                     double sigma, int64_t row_begin, int64_t row_end, const double* cot,
                     double* grad_x, double* grad_y, void* ws, size_t ws_bytes, void* stream) {
  const bool sym = (y == nullptr);
  if (sym && (n2 != n1 || L2 != L1))
    return fail(SK_INVALID_ARGUMENT, "symmetric Gram needs n2 == n1 and L2 == L1");
  if (row_begin < 0 || row_end > n1 || row_begin > row_end)
    return fail(SK_INVALID_ARGUMENT, "row range out of bounds");
  if (!cot) return fail(SK_INVALID_ARGUMENT, "Gram backward needs the cotangent matrix");
  return backward_impl(x, sym ? x : y, n1, n2, L1, L2, d, lam1, lam2, static_kernel, sigma,
                       sym ? GRAM_SYM : GRAM_CROSS, row_begin, row_end, cot, nullptr, grad_x,
                       grad_y, ws, ws_bytes, (cudaStream_t)stream, nullptr);
}

size_t sk_backward_batch_tf_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d,
                                            int lam1, int lam2, int static_kernel, int transform) {
  size_t q = 0;
  if (backward_impl(nullptr, nullptr, B, B, L1, L2, d, lam1, lam2, static_kernel, 1.0, BATCH, 0,
                    B, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, &q, nullptr,
                    nullptr, transform))
    return 0;
  return q;
}

int sk_backward_batch_tf(const double* x, const double* y, int64_t B, int64_t L1, int64_t L2,
                         int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                         int transform, const double* cot, double* values, double* grad_x,
                         double* grad_y, void* ws, size_t ws_bytes, void* stream) {
  if (B < 0) return fail(SK_INVALID_ARGUMENT, "negative batch");
  return backward_impl(x, y, B, B, L1, L2, d, lam1, lam2, static_kernel, sigma, BATCH, 0, B, cot,
                       values, grad_x, grad_y, ws, ws_bytes, (cudaStream_t)stream, nullptr,
                       nullptr, nullptr, transform);
}

size_t sk_backward_gram_tf_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                           int64_t d, int lam1, int lam2, int static_kernel,
                                           int symmetric, int transform) {
  size_t q = 0;
  if (backward_impl(nullptr, nullptr, n1, n2, L1, L2, d, lam1, lam2, static_kernel, 1.0,
                    symmetric ? GRAM_SYM : GRAM_CROSS, 0, n1, nullptr, nullptr, nullptr,
                    nullptr, nullptr, 0, nullptr, &q, nullptr, nullptr, transform))
    return 0;
  return q;
}

int sk_backward_gram_tf(const double* x, const double* y, int64_t n1, int64_t n2, int64_t L1,
                        int64_t L2, int64_t d, int lam1, int lam2, int static_kernel,
                        double sigma, int transform, int64_t row_begin, int64_t row_end,
                        const double* cot, double* values, double* grad_x, double* grad_y,
                        void* ws, size_t ws_bytes, void* stream) {
  const bool sym = (y == nullptr);
  if (sym && (n2 != n1 || L2 != L1))
    return fail(SK_INVALID_ARGUMENT, "symmetric Gram needs n2 == n1 and L2 == L1");
  if (row_begin < 0 || row_end > n1 || row_begin > row_end)
    return fail(SK_INVALID_ARGUMENT, "row range out of bounds");
  if (!cot) return fail(SK_INVALID_ARGUMENT, "Gram backward needs the cotangent matrix");
  if (int rc = backward_impl(x, sym ? x : y, n1, n2, L1, L2, d, lam1, lam2, static_kernel, sigma,
                             sym ? GRAM_SYM : GRAM_CROSS, row_begin, row_end, cot, values,
                             grad_x, grad_y, ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr,
                             nullptr, transform))
    return rc;
  const int64_t span = row_end - row_begin;
  if (values && sym && span > 1) {
    int blocks = (int)std::min<int64_t>((span * span + 255) / 256, 4096);
    mirror_upper<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(values, n2, (int)row_begin,
                                                                   (int)row_end);
    SK_CUDA(cudaGetLastError());
  }
  return SK_OK;
}

size_t sk_backward_gram_acc_tf_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                               int64_t d, int lam1, int lam2, int static_kernel,
                                               int symmetric, int transform) {
  size_t q = 0;
  char dummy = 0;  // non-NULL accumulator: the workspace holds no accumulators
  if (backward_impl(nullptr, nullptr, n1, n2, L1, L2, d, lam1, lam2, static_kernel, 1.0,
                    symmetric ? GRAM_SYM : GRAM_CROSS, 0, n1, nullptr, nullptr, nullptr,
                    nullptr, nullptr, 0, nullptr, &q, &dummy, &dummy, transform))
    return 0;
  return q;
}

int sk_backward_gram_acc_tf(const double* x, const double* y, int64_t n1, int64_t n2,
                            int64_t L1, int64_t L2, int64_t d, int lam1, int lam2,
                            int static_kernel, double sigma, int transform, int64_t row_begin,
                            int64_t row_end, const double* cot, double* values, void* acc_x,
                            void* acc_y, void* ws, size_t ws_bytes, void* stream) {
  const bool sym = (y == nullptr);
  if (sym && (n2 != n1 || L2 != L1))
    return fail(SK_INVALID_ARGUMENT, "symmetric Gram needs n2 == n1 and L2 == L1");
  if (row_begin < 0 || row_end > n1 || row_begin > row_end)
    return fail(SK_INVALID_ARGUMENT, "row range out of bounds");
  if (!cot) return fail(SK_INVALID_ARGUMENT, "Gram backward needs the cotangent matrix");
  if (!acc_x) return fail(SK_INVALID_ARGUMENT, "accumulator missing");
  if (int rc = backward_impl(x, sym ? x : y, n1, n2, L1, L2, d, lam1, lam2, static_kernel, sigma,
                             sym ? GRAM_SYM : GRAM_CROSS, row_begin, row_end, cot, values,
                             nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream, nullptr,
                             acc_x, acc_y, transform))
    return rc;
  const int64_t span = row_end - row_begin;
  if (values && sym && span > 1) {
    int blocks = (int)std::min<int64_t>((span * span + 255) / 256, 4096);
    mirror_upper<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(values, n2, (int)row_begin,
                                                                   (int)row_end);
    SK_CUDA(cudaGetLastError());
  }
  return SK_OK;
}

size_t sk_grad_acc_bytes(int64_t n, int64_t L, int64_t d) {
  if (n < 0 || L < 0 || d < 0) return 0;
  return acc_bytes(n, L, d);
}

int sk_grad_acc_init(void* acc, int64_t n, int64_t L, int64_t d, const double* cot, int64_t n1,
                     int64_t n2, int symmetric, void* stream) {
  if (!acc || n < 0 || L < 0 || d < 0 || n1 < 0 || n2 < 0)
    return fail(SK_INVALID_ARGUMENT, "bad accumulator arguments");
  if (n1 * n2 > 0 && !cot) return fail(SK_INVALID_ARGUMENT, "cotangent missing");
  return acc_init(static_cast<unsigned long long*>(acc), nullptr, acc_bytes(n, L, d), 0, cot, n1,
                  n2, symmetric != 0, (cudaStream_t)stream);
}

int sk_grad_acc_finalize(const void* acc, int64_t n, int64_t L, int64_t d, double* grad,
                         int accumulate, void* stream) {
  if (!acc || !grad || n < 0 || L < 0 || d < 0)
    return fail(SK_INVALID_ARGUMENT, "bad accumulator arguments");
  return acc_finalize(static_cast<const unsigned long long*>(acc), n * L * d, grad,
                      accumulate != 0, (cudaStream_t)stream);
}

int sk_backward_gram_acc(const double* x, const double* y, int64_t n1, int64_t n2, int64_t L1,
                         int64_t L2, int64_t d, int lam1, int lam2, int static_kernel,
                         double sigma, int64_t row_begin, int64_t row_end, const double* cot,
                         double* values, void* acc_x, void* acc_y, void* ws, size_t ws_bytes,
                         void* stream) {
  return sk_backward_gram_acc_tf(x, y, n1, n2, L1, L2, d, lam1, lam2, static_kernel, sigma,
                                 TF_NONE, row_begin, row_end, cot, values, acc_x, acc_y, ws,
                                 ws_bytes, stream);
}

size_t sk_backward_gram_acc_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                            int64_t d, int lam1, int lam2, int static_kernel,
                                            int symmetric) {
  return sk_backward_gram_acc_tf_workspace_bytes(n1, n2, L1, L2, d, lam1, lam2, static_kernel,
                                                 symmetric, TF_NONE);
}

int sk_backward_gram_acc_cols(const double* x, const double* y, int64_t n1, int64_t n2,
                              int64_t L1, int64_t L2, int64_t d, int lam1, int lam2,
                              int transform, int64_t row_begin, int64_t row_end,
                              int64_t col_begin, int64_t col_end, const double* cot,
                              double* values, void* acc_x, void* acc_y, void* ws,
                              size_t ws_bytes, void* stream) {
  if (!y) return fail(SK_INVALID_ARGUMENT, "column ranges are for cross Grams (y != NULL)");
  if (row_begin < 0 || row_end > n1 || row_begin > row_end)
    return fail(SK_INVALID_ARGUMENT, "row range out of bounds");
  if (!cot) return fail(SK_INVALID_ARGUMENT, "Gram backward needs the cotangent matrix");
  if (!acc_x || !acc_y) return fail(SK_INVALID_ARGUMENT, "accumulators missing");
  return backward_impl(x, y, n1, n2, L1, L2, d, lam1, lam2, LINEAR, 1.0, GRAM_CROSS, row_begin,
                       row_end, cot, values, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream,
                       nullptr, acc_x, acc_y, transform, false, col_begin, col_end);
}

size_t sk_backward_gram_acc_f32_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                                int64_t d, int lam1, int lam2, int symmetric) {
  size_t q = 0;
  char dummy = 0;
  if (backward_impl(nullptr, nullptr, n1, n2, L1, L2, d, lam1, lam2, LINEAR, 1.0,
                    symmetric ? GRAM_SYM : GRAM_CROSS, 0, n1, nullptr, nullptr, nullptr,
                    nullptr, nullptr, 0, nullptr, &q, &dummy, &dummy, TF_NONE, true))
    return 0;
  return q;
}

int sk_backward_gram_acc_f32(const double* x, const double* y, int64_t n1, int64_t n2,
                             int64_t L1, int64_t L2, int64_t d, int lam1, int lam2,
                             int64_t row_begin, int64_t row_end, const double* cot,
                             double* values, void* acc_x, void* acc_y, void* ws,
                             size_t ws_bytes, void* stream) {
  const bool sym = (y == nullptr);
  if (sym && (n2 != n1 || L2 != L1))
    return fail(SK_INVALID_ARGUMENT, "symmetric Gram needs n2 == n1 and L2 == L1");
  if (row_begin < 0 || row_end > n1 || row_begin > row_end)
    return fail(SK_INVALID_ARGUMENT, "row range out of bounds");
  if (!cot) return fail(SK_INVALID_ARGUMENT, "Gram backward needs the cotangent matrix");
  if (!acc_x) return fail(SK_INVALID_ARGUMENT, "accumulator missing");
  if (int rc = backward_impl(x, sym ? x : y, n1, n2, L1, L2, d, lam1, lam2, LINEAR, 1.0,
                             sym ? GRAM_SYM : GRAM_CROSS, row_begin, row_end, cot, values,
                             nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream, nullptr,
                             acc_x, acc_y, TF_NONE, true))
    return rc;
  const int64_t span = row_end - row_begin;
  if (values && sym && span > 1) {
    int blocks = (int)std::min<int64_t>((span * span + 255) / 256, 4096);
    mirror_upper<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(values, n2, (int)row_begin,
                                                                   (int)row_end);
    SK_CUDA(cudaGetLastError());
  }
  return SK_OK;
}

}  // extern "C"

// ================================================================ peak probe
// Independent DFMA chains (8 per thread, 8 warps per CTA, 8 CTAs per SM):
// the FP64 FMA-pipe issue rate that bench.py divides by (the roofline of
// this path).  Timed by the caller with CUDA events.
namespace sk {
__global__ void dfma_probe_kernel(double* out, double a, double b, int iters) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
}  // namespace sk

extern "C" size_t sk_dfma_probe_scratch_bytes(void) {
  return (size_t)device_sms() * 8 * 256 * sizeof(double);
}

extern "C" int sk_dfma_probe(double* scratch, int iters, double* fma_count, void* stream) {
  const int blocks = device_sms() * 8, threads = 256;
  dfma_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(scratch, 0.999, 1e-3, iters);
  SK_CUDA(cudaGetLastError());
  if (fma_count) *fma_count = (double)blocks * threads * (double)iters * 32.0;
  return SK_OK;
}

// Mirror the upper triangle of an (n x n) matrix into its lower triangle
// (kernel.py:177-179); used after the sharded Gram all-gather.
extern "C" int sk_mirror_upper(double* g, int64_t n, int64_t ld, void* stream) {
  if (n < 0 || ld < n) return fail(SK_INVALID_ARGUMENT, "bad matrix shape");
  if (n < 2) return SK_OK;
  int blocks = (int)std::min<int64_t>((n * n + 255) / 256, 4096);
  mirror_upper<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(g, ld, 0, (int)n);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}
