// sk_common.cuh -- shared definitions for the sm_100a signature-kernel path.
//
// Terminology (follows the reference, /root/reference/pkg/src/sigcore):
//   pair        one (x, y) path pair; batch entry or Gram entry
//   coarse cell data cell (i, j) of the increment matrix delta (kernel.py:60-77)
//   fine cell   dyadically refined cell; coarse cell (i, j) holds 2^lam1 x 2^lam2
//               fine cells that all read delta[i, j] * 2^-(lam1+lam2)
//               (_kernels.py:325)
//   strip       G*R consecutive fine rows solved by one lane group (the
//               reference's "strip of 32", _kernels.py:293-338, here spread over
//               G lanes, R rows each, exchanged by warp shuffles)
//   handoff row bottom row of a strip, initial condition of the next strip
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sk {

enum Kind : int { LINEAR = 0, RBF = 1, DELTA = 2 };

// Pair-to-work mapping modes.
enum Mode : int { BATCH = 0, GRAM_CROSS = 1, GRAM_SYM = 2 };

struct PathData {
  // LINEAR: scaled increments  [n][rows][DP*nch]   (zero padded in k)
  // RBF:    nodes              [n][rows+1][DP*nch] (zero padded in k)
  // DELTA:  unused (delta given per pair)
  const double* p;
  int64_t path_stride;  // elements between consecutive paths
  int rows;             // coarse rows (increments) of each path
};

struct Problem {
  PathData R;  // path on the grid rows (fine rows = R.rows << lam1)
  PathData C;  // path on the grid columns
  const double* delta;  // DELTA kind: [npairs][M1c][M2c]
  int kind;
  int dpad;      // DP * nch (row length of PathData arrays)
  int nch;       // number of DP-chunks of the dimension
  int M1c, M2c;  // coarse rows / cols of every pair
  int lam1, lam2;
  double scale;   // 2^-(lam1+lam2): dyadic factor of every coarse p (exact: power of two)
  double pscale;  // factor still to apply to LINEAR p (1 when folded into the row data)
  double inv2s2;  // RBF: 1/(2 sigma^2)
  double invs2;   // RBF: 1/sigma^2
  // pair mapping
  int mode;
  int64_t nitems;  // work items (each holds P = pairs per item groups)
  int64_t npairs;  // BATCH: number of pairs
  int n1, n2;      // Gram sizes (X count, Y count)
  int r0, r1;      // Gram: X rows [r0, r1) handled by this call
  int c0, c1;      // GRAM_CROSS, DMMA backward: Y columns [c0, c1) (c0 % 8 == 0; 0, n2 = all)
  int swap;        // grid rows are the Y path (fine-axis orientation rule)
  int amajor;      // Gram backward: items enumerated row-block major (see gram_item)
  // output
  double* out;
  int64_t ldo;
};

// Backward scratch and outputs (see sk_backward.cuh).
struct BwdArgs {
  // per-slot scratch
  double* rowck;
  int64_t rowck_stride;
  double* colck;
  int64_t colck_stride;
  double* pck;  // coarse p per solved column ([strip][step + lane][s][c][lane])
  int64_t pck_stride;
  double* hand;  // forward handoff rows
  double* adj;   // reverse handoff rows (messages between strips)
  int64_t row_stride;
  double* dbuf;  // DBUF: per-slot coarse adjoint [M1c][M2c]
  int64_t dbuf_stride;
  double* gscr;  // FUSED: per-slot increment gradients [M1c + M2c][DP]
  int64_t gscr_stride;
  double* rsum;  // DMMA Gram: per-slot row-side increment gradients of a super-item [8][M1c][DP]
  int64_t rsum_stride;
  int rows_exclusive;  // 2^lam1 <= R: every coarse row belongs to one lane
  // outputs (point gradients, real dimension d)
  double* gradR;  // BATCH: gradient of the grid-row path set
  double* gradC;  // BATCH: gradient of the grid-column path set
  // GRAM: exact fixed-point accumulators of the row / column path sets
  // ([path][L][d][4] int64) and their metadata (see FixAcc)
  unsigned long long* accR;
  unsigned long long* accC;
  unsigned long long* metaR;
  unsigned long long* metaC;
  int64_t gR_path, gC_path;  // elements per path (L * d)
  int d;
  int atomic;  // Gram: accumulate into accR / accC (several pairs share a path)
  const double* cot;  // BATCH: [npairs] (nullptr = ones); GRAM: [n1][n2]
  double* values;     // BATCH: optional kernel values
  int exp;            // profiling experiments (env SK_EXP, default 0): 1 skips phase B,
                      // 2 skips phase A, 4 the gradient maps, 8 the phase-B p tiles of
                      // the DMMA backward -- results are wrong when set
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// Exact (order-independent) accumulation of Gram gradients.
//
// A Gram gradient element receives one contribution per Gram tile that
// touches its path, from many warps and -- when sharded -- many GPUs.  fp64
// atomics make the result depend on arrival order; the reference contract is
// that no floating-point reduction order may vary (/root/reference/SPEC.md:261,
// pkg/tests/test_kernel.py:156-171).  Here every contribution v is converted
// exactly (no rounding except below the lowest limb) to a signed fixed-point
// number with four 42-bit chunks relative to a per-call anchor 2^E, and the
// chunks are added into four int64 limbs with integer atomics.  Integer
// addition is associative, so the sums -- and the fp64 value made from them --
// are bitwise identical for any schedule, any row-block split and any number of
// GPUs (the limbs of several ranks are summed as integers).
//
//   element layout: acc[elem][4] (limb 3 = top chunk, unit 2^(E-42); limb k
//   unit 2^(E-42(4-k))), 32 bytes = one sector per element;
//   anchor: E = exponent of (nscale * max|cot|) + 64, nscale = max(n1, n2)
//   (x2 symmetric) -- every gradient element is a sum of at most that many
//   cotangent-weighted pair gradients, so E sits ~64 bits above realistic
//   magnitudes and the lowest limb resolves 2^-104 of the bound;
//   a contribution with |v| >= 2^(E+2) (or inf/NaN) sets the overflow flag and
//   the finalize step writes NaN (never a silent wrong value).
// meta[0]: max|cot| bit pattern (atomicMax; non-negative doubles order like
// their bits), meta[1]: flags, meta[2]: nscale (double bits).
// L2 residency hints (sm_80+ cache-policy operands): scratch that one warp
// re-reads many times (the DMMA backward's column-gradient rows) is marked
// evict-last so the streaming checkpoint traffic does not push it to HBM.
__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_l2hint(const double2* a, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_l2hint(double2* a, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;"
               :: "l"(a), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

struct FixAcc {
  unsigned long long* acc;  // [elements][4]
  unsigned long long* meta;
  double s3;                // 2^(42 - E): contribution -> top-chunk units
};

__host__ __device__ inline int fix_anchor(double maxc, double nscale) {
  const double m = maxc * nscale;
  if (!(m > 0.0) || !(m < 1e300)) return 0;
  int e = 0;
  (void)frexp(m, &e);  // m < 2^e
  e += 64;
  return e < -900 ? -900 : (e > 960 ? 960 : e);
}

__device__ __forceinline__ FixAcc fix_make(unsigned long long* acc, unsigned long long* meta) {
  FixAcc f;
  f.acc = acc;
  f.meta = meta;
  const int E = fix_anchor(__longlong_as_double((long long)meta[0]),
                           __longlong_as_double((long long)meta[2]));
  f.s3 = ldexp(1.0, 42 - E);
  return f;
}

__device__ __forceinline__ void fix_add(const FixAcc& f, int64_t elem, double v) {
  if (v == 0.0) return;  // adds nothing (keeps padded / dead lanes off the atomics)
  double x = v * f.s3;
  if (!(fabs(x) < 0x1p44)) {  // overflow, inf or NaN: flagged, finalize writes NaN
    atomicOr(f.meta + 1, 1ull);
    return;
  }
  // exact splits: each step removes the integer part and shifts the (exact)
  // remainder up by 42 bits; only the last chunk is rounded
  const double c3 = trunc(x);
  x = (x - c3) * 0x1p42;
  const double c2 = trunc(x);
  x = (x - c2) * 0x1p42;
  const double c1 = trunc(x);
  x = (x - c1) * 0x1p42;
  const double c0 = rint(x);
  unsigned long long* p = f.acc + elem * 4;
  atomicAdd(p + 3, (unsigned long long)(long long)c3);
  atomicAdd(p + 2, (unsigned long long)(long long)c2);
  atomicAdd(p + 1, (unsigned long long)(long long)c1);
  atomicAdd(p + 0, (unsigned long long)(long long)c0);
}

// Work item -> (a0, b): the item covers pairs (a0 + g, b), g < P.
// GRAM_CROSS: a-blocks of P rows of [r0, r1) x all b.
// GRAM_SYM:   only pairs a <= b (upper triangle, _kernels.py:421-425).
//   b in [r0, r1-1): a-blocks over [r0, b+1)   (triangle part)
//   b in [r1-1, n2): a-blocks over [r0, r1)     (rectangle part)
// Row-block-major enumeration (Gram backward): the tiles of one row block
// (a0 fixed, b ascending) are consecutive items, so the warps in flight share
// a few row blocks and the row-side gradient accumulators they update stay in
// L2.  SYM: block ab (a0 = r0 + P ab) holds tiles b in [a0, n2).
__host__ __device__ inline int64_t amajor_prefix(int64_t ab, int64_t W, int P) {
  return ab * W - (int64_t)P * (ab * (ab - 1) / 2);  // sum_{i<ab} (W - P i)
}
__device__ inline void gram_item_amajor(const Problem& pb, int64_t item, int P, int& a0, int& b) {
  if (pb.mode == GRAM_CROSS) {
    a0 = pb.r0 + (int)(item / pb.n2) * P;
    b = (int)(item % pb.n2);
    return;
  }
  const int64_t W = pb.n2 - pb.r0;
  // largest ab with prefix(ab) <= item: P/2 ab^2 - (W + P/2) ab + item >= 0 side
  const double hp = 0.5 * P, bq = W + hp;
  double disc = bq * bq - 4.0 * hp * (double)item;
  int64_t ab = (int64_t)((bq - sqrt(disc > 0 ? disc : 0.0)) / (2.0 * hp));
  if (ab < 0) ab = 0;
  while (amajor_prefix(ab + 1, W, P) <= item) ++ab;
  while (ab > 0 && amajor_prefix(ab, W, P) > item) --ab;
  a0 = pb.r0 + (int)(ab * P);
  b = a0 + (int)(item - amajor_prefix(ab, W, P));
}

__device__ inline void gram_item(const Problem& pb, int64_t item, int P, int& a0, int& b) {
  if (pb.amajor) {
    gram_item_amajor(pb, item, P, a0, b);
    return;
  }
  int span = pb.r1 - pb.r0;
  if (pb.mode == GRAM_CROSS) {
    int64_t nblk = ceil_div(span, P);
    b = (int)(item % pb.n2);
    a0 = pb.r0 + (int)(item / pb.n2) * P;
    (void)nblk;
    return;
  }
  // triangle part: b' = b - r0 in [0, span-1), count(b') = b'/P + 1
  // S(b') = b' + P*q(q-1)/2 + r*q with b' = qP + r;  S(qP) = P q(q+1)/2
  int64_t tri_items;
  {
    int64_t nb = span - 1;  // b' in [0, nb)
    int64_t q = nb / P, r = nb % P;
    tri_items = nb + (int64_t)P * (q * (q - 1) / 2) + r * q;
    if (nb <= 0) tri_items = 0;
  }
  if (item < tri_items) {
    // largest q with P q(q+1)/2 <= item
    double fq = (sqrt(8.0 * (double)item / P + 1.0) - 1.0) * 0.5;
    int64_t q = (int64_t)fq;
    while ((int64_t)P * (q + 1) * (q + 2) / 2 <= item) ++q;
    while (q > 0 && (int64_t)P * q * (q + 1) / 2 > item) --q;
    int64_t off = item - (int64_t)P * q * (q + 1) / 2;
    int64_t rr = off / (q + 1), blk = off % (q + 1);
    b = pb.r0 + (int)(q * P + rr);
    a0 = pb.r0 + (int)(blk * P);
    return;
  }
  int64_t rem = item - tri_items;
  int64_t nblk = ceil_div(span, P);
  b = pb.r1 - 1 + (int)(rem / nblk);
  a0 = pb.r0 + (int)(rem % nblk) * P;
}

// DMMA Gram backward work items ("super-items"): one 8-path row block a0 and
// one canonical chunk of SK_SUPER_B consecutive column paths b (absolute
// chunk index b / SK_SUPER_B).  The row-side gradients of the chunk's tiles
// are summed in fp64 in b order inside the item and flushed once, so the
// result does not depend on how rows are split across calls / GPUs (the
// chunks and row blocks are the same in every split aligned to 8 rows).
#define SK_SUPER_B 8
// (GRAM_CROSS: the chunks of the column range [c0, c1), c0 a multiple of
// SK_SUPER_B, so a column split sees the same chunks as the whole call)
__host__ __device__ inline int64_t super_chunks(int mode, int n2, int r0, int ab, int c0 = 0,
                                                int c1 = -1) {
  if (mode == GRAM_CROSS)
    return (int64_t)((c1 < 0 ? n2 : c1) + SK_SUPER_B - 1) / SK_SUPER_B - c0 / SK_SUPER_B;
  return (int64_t)((n2 - 1) / SK_SUPER_B) - (r0 + 8 * ab) / SK_SUPER_B + 1;
}
__host__ inline int64_t super_items(int mode, int n2, int r0, int r1, int c0 = 0, int c1 = -1) {
  const int nblk = (r1 - r0 + 7) / 8;
  if (r1 <= r0) return 0;
  if (mode == GRAM_CROSS) return (int64_t)nblk * super_chunks(mode, n2, r0, 0, c0, c1);
  int64_t n = 0;
  for (int ab = 0; ab < nblk; ++ab) n += super_chunks(mode, n2, r0, ab);
  return n;
}
__device__ inline void super_item(const Problem& pb, int64_t s, int& ab, int& ch) {
  if (pb.mode == GRAM_CROSS) {
    const int64_t nc = super_chunks(pb.mode, pb.n2, pb.r0, 0, pb.c0, pb.c1);
    ab = (int)(s / nc);
    ch = pb.c0 / SK_SUPER_B + (int)(s % nc);
    return;
  }
  const int nblk = (pb.r1 - pb.r0 + 7) / 8;
  int64_t acc = 0;
  for (ab = 0; ab < nblk; ++ab) {
    const int64_t nc = super_chunks(pb.mode, pb.n2, pb.r0, ab);
    if (s < acc + nc) {
      ch = (pb.r0 + 8 * ab) / SK_SUPER_B + (int)(s - acc);
      return;
    }
    acc += nc;
  }
  ab = nblk;
  ch = 0;
}

__host__ inline int64_t gram_items(int mode, int n2, int r0, int r1, int P, bool amajor = false) {
  int64_t span = r1 - r0;
  if (span <= 0) return 0;
  if (amajor) {
    const int64_t nblk = ceil_div(span, P);
    return mode == GRAM_CROSS ? nblk * n2 : amajor_prefix(nblk, (int64_t)n2 - r0, P);
  }
  int64_t nblk = ceil_div(span, P);
  if (mode == GRAM_CROSS) return nblk * n2;
  int64_t nb = span - 1;
  int64_t q = nb / P, r = nb % P;
  int64_t tri = nb > 0 ? nb + (int64_t)P * (q * (q - 1) / 2) + r * q : 0;
  return tri + nblk * (int64_t)(n2 - (r1 - 1));
}

// Resolve a group's pair: returns false when the lane group has no pair.
// pr/pc: path indices on the grid rows / columns; oidx: output element.
__device__ inline bool resolve_pair(const Problem& pb, int64_t item, int P, int g,
                                    int64_t& pr, int64_t& pc, int64_t& oidx, int64_t& pidx) {
  if (pb.mode == BATCH) {
    int64_t p = item * P + g;
    if (p >= pb.npairs) return false;
    pr = p; pc = p; oidx = p; pidx = p;
    return true;
  }
  int a0, b;
  gram_item(pb, item, P, a0, b);
  int a = a0 + g;
  if (a >= pb.r1) return false;
  if (pb.mode == GRAM_SYM && a > b) return false;
  // GRAM_SYM keeps (rows, cols) = (X_a, X_b) even when the dyadic orders are
  // swapped: the reference transposes, mirrors, and transposes back
  // (kernel.py:164-180), which lands on solve(rows=X_a, cols=X_b) for a <= b.
  const bool sw = pb.swap && pb.mode == GRAM_CROSS;
  pr = sw ? b : a;
  pc = sw ? a : b;
  oidx = (int64_t)(a - pb.r0) * pb.ldo + b;
  pidx = (int64_t)(a - pb.r0) * pb.n2 + b;
  return true;
}

}  // namespace sk
