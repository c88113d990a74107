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
  int swap;        // grid rows are the Y path (fine-axis orientation rule)
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
  int rows_exclusive;  // 2^lam1 <= R: every coarse row belongs to one lane
  // outputs (point gradients, real dimension d)
  double* gradR;  // gradient of the grid-row path set
  double* gradC;  // gradient of the grid-column path set
  int64_t gR_path, gC_path;  // elements per path (L * d)
  int d;
  int atomic;  // accumulate with atomics (Gram: several pairs share a path)
  const double* cot;  // BATCH: [npairs] (nullptr = ones); GRAM: [n1][n2]
  double* values;     // BATCH: optional kernel values
  int exp;            // profiling experiments (env SK_EXP, default 0): 1 skips phase B,
                      // 2 skips phase A, 4 the gradient maps, 8 the phase-B p tiles of
                      // the DMMA backward -- results are wrong when set
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Work item -> (a0, b): the item covers pairs (a0 + g, b), g < P.
// GRAM_CROSS: a-blocks of P rows of [r0, r1) x all b.
// GRAM_SYM:   only pairs a <= b (upper triangle, _kernels.py:421-425).
//   b in [r0, r1-1): a-blocks over [r0, b+1)   (triangle part)
//   b in [r1-1, n2): a-blocks over [r0, r1)     (rectangle part)
__device__ inline void gram_item(const Problem& pb, int64_t item, int P, int& a0, int& b) {
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

__host__ inline int64_t gram_items(int mode, int n2, int r0, int r1, int P) {
  int64_t span = r1 - r0;
  if (span <= 0) return 0;
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
