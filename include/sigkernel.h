/*
 * sigkernel.h -- C ABI of the B200 (sm_100a) signature-kernel hot path.
 *
 * Drop-in boundary for the reference's kernel entry points.  The reference
 * (sigcore 0.1.0) binds its solver through numba functions that take
 * caller-allocated buffers and never allocate (/root/reference/pkg/src/sigcore/
 * _kernels.py:9-12); this ABI keeps that contract with device pointers:
 *
 *   sk_forward_batch   replaces kernel.py:125-148   (kernel_batch  -> goursat_batch,
 *                                                    _kernels.py:399-405)
 *   sk_forward_gram    replaces kernel.py:151-180   (kernel_gram   -> goursat_gram,
 *                                                    _kernels.py:408-429), plus a
 *                                                    row range for sharding
 *   sk_solve_delta     replaces kernel.py:94-122    (solve_goursat on a given delta,
 *                                                    goursat_strip/_grid)
 *   sk_solve_delta_grid                             (store_grid=True path,
 *                                                    _kernels.py:381-396)
 *   sk_backward_batch  replaces kernel_grad.py:64-98 (kernel_batch_backward ->
 *                                                    goursat_grid + goursat_backward,
 *                                                    _kernels.py:436-466, plus the
 *                                                    dF/d(delta) -> dF/dx mapping of
 *                                                    kernel_grad.py:51-60)
 *   sk_backward_gram   (no reference counterpart: Gram backward composed from
 *                       kernel_backward per pair)
 *   sk_value_and_grad_gram  the same, also returning the Gram entries (as
 *                       kernel_batch_backward returns values, kernel_grad.py:64-98)
 *   sk_backward_gram_acc + sk_grad_acc_*  the Gram backward into exact
 *                       accumulators (split- and GPU-count-invariant gradients)
 *
 * Conventions
 *   - every array pointer is DEVICE memory, C-contiguous float64, borrowed for
 *     the duration of the call; outputs and the workspace are caller-allocated
 *     (size the workspace with the matching *_workspace_bytes query);
 *   - paths are (n, L, d) row-major; L >= 2;
 *   - static_kernel: SK_STATIC_LINEAR (<a,b>, the reference's increment_gram)
 *     or SK_STATIC_RBF (exp(-|a-b|^2 / (2 sigma^2)); no reference counterpart);
 *   - work is enqueued on `stream` (a cudaStream_t, NULL = legacy default) and
 *     the call returns without synchronising;
 *   - return value: SK_OK, or an error code whose message sk_last_error()
 *     returns (thread-local).  SK_INVALID_ARGUMENT / SK_INVALID_STATE map to
 *     the reference's InvalidArgument(ValueError) / InvalidState(RuntimeError)
 *     (errors.py:4-12).  Non-finite values are never trapped: overflow
 *     propagates as inf, NaN as NaN (kernel.py:97-99).
 */
#ifndef SIGKERNEL_H
#define SIGKERNEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_ABI_VERSION 1

enum {
  SK_OK = 0,
  SK_INVALID_ARGUMENT = 1,
  SK_INVALID_STATE = 2,
  SK_CUDA_ERROR = 3
};

enum { SK_STATIC_LINEAR = 0, SK_STATIC_RBF = 1 };

int sk_abi_version(void);
const char *sk_last_error(void);
/* number of SMs of the current device (the persistent-grid size basis) */
int sk_device_sms(void);

/* FP64 roofline probe: enqueues independent DFMA chains on all SMs; the
 * caller times it with CUDA events and divides *fma_count by the duration
 * (bench.py's roofline denominator).  scratch: sk_dfma_probe_scratch_bytes(). */
size_t sk_dfma_probe_scratch_bytes(void);
int sk_dfma_probe(double *scratch, int iters, double *fma_count, void *stream);

/* ---- forward ----------------------------------------------------------- */

size_t sk_forward_batch_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d,
                                        int lam1, int lam2, int static_kernel);
/* out[b] = k(x_b, y_b);  x (B,L1,d), y (B,L2,d), out (B,) */
int sk_forward_batch(const double *x, const double *y, int64_t B, int64_t L1, int64_t L2,
                     int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                     double *out, void *workspace, size_t workspace_bytes, void *stream);

size_t sk_forward_gram_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                       int64_t d, int lam1, int lam2, int static_kernel,
                                       int symmetric);
/* out[a - row_begin, b] = k(x_a, y_b) for a in [row_begin, row_end), b < n2.
 * y == NULL means y is x (symmetric): only pairs a <= b are solved and the
 * in-range part of the lower triangle is mirrored (kernel.py:177-179);
 * entries with a > b outside the row range are left untouched. */
int sk_forward_gram(const double *x, const double *y, int64_t n1, int64_t n2, int64_t L1,
                    int64_t L2, int64_t d, int lam1, int lam2, int static_kernel,
                    double sigma, int64_t row_begin, int64_t row_end, double *out,
                    void *workspace, size_t workspace_bytes, void *stream);

/* FP32 arithmetic (linear static kernel): float32 paths in, float32 values out.
 * Same wavefront as the fp64 kernels with the cell in small-correction form
 * k = (u - k_diag) + (u (p/2 + q) + k_diag q), u = k_up + k_left, q = p^2/12
 * (fp32 rounding of A = 1 + p/2 + ... would swallow small p).  Accuracy vs
 * the fp64 reference: ~1e-5..6e-5 relative up to ~1000 fine cells per axis,
 * growing ~linearly with the axis length (BASELINE config 4: ~1e-3); the
 * reference's own float32 path keeps fp64 arithmetic (kernel.py:36-38), which
 * the fp64 entry points reproduce.  Symmetric Gram: y == NULL. */
size_t sk_forward_batch_f32_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d,
                                            int lam1, int lam2, int transform);
int sk_forward_batch_f32(const float *x, const float *y, int64_t B, int64_t L1, int64_t L2,
                         int64_t d, int lam1, int lam2, int transform, float *out,
                         void *workspace, size_t workspace_bytes, void *stream);
size_t sk_forward_gram_f32_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                           int64_t d, int lam1, int lam2, int symmetric,
                                           int transform);
int sk_forward_gram_f32(const float *x, const float *y, int64_t n1, int64_t n2, int64_t L1,
                        int64_t L2, int64_t d, int lam1, int lam2, int transform,
                        int64_t row_begin, int64_t row_end, float *out, void *workspace,
                        size_t workspace_bytes, void *stream);

size_t sk_solve_delta_workspace_bytes(int64_t B, int64_t r1, int64_t r2, int lam1, int lam2);
/* out[b] = solve_goursat(delta_b) for delta (B, r1, r2) */
int sk_solve_delta(const double *delta, int64_t B, int64_t r1, int64_t r2, int lam1,
                   int lam2, double *out, void *workspace, size_t workspace_bytes,
                   void *stream);
/* full fine grid ((r1<<lam1)+1, (r2<<lam2)+1) of one delta (B = 1) */
int sk_solve_delta_grid(const double *delta, int64_t r1, int64_t r2, int lam1, int lam2,
                        double *grid, void *stream);

/* mirror the upper triangle of an (n, n) row-major matrix (leading dim ld)
 * into the lower one; used to assemble a sharded symmetric Gram. */
int sk_mirror_upper(double *g, int64_t n, int64_t ld, void *stream);

/* ---- backward ---------------------------------------------------------- */

size_t sk_backward_batch_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d,
                                         int lam1, int lam2, int static_kernel);
/* grad_x = sum_b cot[b] dk(x_b,y_b)/dx_b, grad_y likewise; values (B,) optional
 * (NULL to skip).  cot == NULL means ones (kernel_grad.py:81-82). */
int sk_backward_batch(const double *x, const double *y, int64_t B, int64_t L1, int64_t L2,
                      int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                      const double *cot, double *values, double *grad_x, double *grad_y,
                      void *workspace, size_t workspace_bytes, void *stream);

size_t sk_backward_gram_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                        int64_t d, int lam1, int lam2, int static_kernel,
                                        int symmetric);
/* F = sum_{a, b} cot[a, b] G[a, b] restricted to the pairs this call solves
 * (rows a in [row_begin, row_end); symmetric: pairs a <= b, weighted by
 * cot[a,b] + cot[b,a] because G mirrors the upper triangle).  cot is the FULL
 * (n1, n2) cotangent.  grad_x += dF/dx, grad_y += dF/dy (grad_y unused when
 * y == NULL: both sides land in grad_x).  Inside the call the pair
 * contributions are summed EXACTLY (integer fixed-point limbs, see
 * sk_grad_acc_* below), so the result is bitwise reproducible run to run and
 * independent of the launch geometry (reference contract: no reduction order
 * may vary, tests/test_kernel.py:156-171).  For
 * results that are also bitwise independent of how the rows are split across
 * calls or GPUs, use sk_backward_gram_acc.  The batch backward (no shared
 * paths) writes each pair's gradient exclusively. */
int sk_backward_gram(const double *x, const double *y, int64_t n1, int64_t n2, int64_t L1,
                     int64_t L2, int64_t d, int lam1, int lam2, int static_kernel,
                     double sigma, int64_t row_begin, int64_t row_end, const double *cot,
                     double *grad_x, double *grad_y, void *workspace, size_t workspace_bytes,
                     void *stream);

/* Fused value + gradient of a Gram block: the backward above, plus the Gram
 * entries G[a - row_begin, b] it solves anyway on its forward pass, written to
 * `values` (leading dimension n2; symmetric: the solved upper triangle of the
 * [row_begin, row_end) square is mirrored, entries b < row_begin are left
 * untouched).  This is the Gram counterpart of the reference's
 * kernel_batch_backward, which returns the values with the gradients
 * (kernel_grad.py:64-98); it saves the separate forward solve of
 * sk_forward_gram when both are needed.  Uses the backward's workspace. */
int sk_value_and_grad_gram(const double *x, const double *y, int64_t n1, int64_t n2,
                           int64_t L1, int64_t L2, int64_t d, int lam1, int lam2,
                           int static_kernel, double sigma, int64_t row_begin, int64_t row_end,
                           const double *cot, double *values, double *grad_x, double *grad_y,
                           void *workspace, size_t workspace_bytes, void *stream);

/* ---- path transforms inside the call ------------------------------------
 * pySigLib's path transforms (reference transforms.py:37-120) applied to both
 * path sets by the kernels' input preparation: the solver reads the
 * transformed increments (linear kernel; the reference's fused_increments,
 * transforms.py:91-120) or transformed nodes (RBF) built straight from the
 * raw points, and the backward maps the transformed-path gradients back with
 * the transform's adjoint (transforms.py:69-90).  x, y, grad_x, grad_y keep
 * the RAW shapes (n, L, d); transform == SK_TRANSFORM_NONE is the plain call.
 *   time augmentation: (L, d) -> (L, d+1), time grid numpy.linspace(0, 1, L)
 *   lead-lag:          (L, d) -> (2L-1, 2d), Z[2k] = (X[k], X[k]),
 *                      Z[2k+1] = (X[k+1], X[k]) */
enum { SK_TRANSFORM_NONE = 0, SK_TRANSFORM_TIME_AUGMENT = 1, SK_TRANSFORM_LEAD_LAG = 2 };

size_t sk_forward_batch_tf_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d,
                                           int lam1, int lam2, int static_kernel, int transform);
int sk_forward_batch_tf(const double *x, const double *y, int64_t B, int64_t L1, int64_t L2,
                        int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                        int transform, double *out, void *workspace, size_t workspace_bytes,
                        void *stream);
size_t sk_forward_gram_tf_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                          int64_t d, int lam1, int lam2, int static_kernel,
                                          int symmetric, int transform);
int sk_forward_gram_tf(const double *x, const double *y, int64_t n1, int64_t n2, int64_t L1,
                       int64_t L2, int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                       int transform, int64_t row_begin, int64_t row_end, double *out,
                       void *workspace, size_t workspace_bytes, void *stream);
size_t sk_backward_batch_tf_workspace_bytes(int64_t B, int64_t L1, int64_t L2, int64_t d,
                                            int lam1, int lam2, int static_kernel, int transform);
int sk_backward_batch_tf(const double *x, const double *y, int64_t B, int64_t L1, int64_t L2,
                         int64_t d, int lam1, int lam2, int static_kernel, double sigma,
                         int transform, const double *cot, double *values, double *grad_x,
                         double *grad_y, void *workspace, size_t workspace_bytes, void *stream);
size_t sk_backward_gram_tf_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                           int64_t d, int lam1, int lam2, int static_kernel,
                                           int symmetric, int transform);
/* sk_backward_gram (values == NULL) or sk_value_and_grad_gram (values != NULL) */
int sk_backward_gram_tf(const double *x, const double *y, int64_t n1, int64_t n2, int64_t L1,
                        int64_t L2, int64_t d, int lam1, int lam2, int static_kernel,
                        double sigma, int transform, int64_t row_begin, int64_t row_end,
                        const double *cot, double *values, double *grad_x, double *grad_y,
                        void *workspace, size_t workspace_bytes, void *stream);
/* gradient of the transformed paths g_t (n, L', d') -> raw (n, L, d): grad = or += */
int sk_transform_adjoint(const double *g_t, int64_t n, int64_t L, int64_t d, int transform,
                         double *grad, int accumulate, void *stream);

/* ---- exact Gram-gradient accumulators ------------------------------------
 * A gradient of n paths (L, d) accumulated as fixed-point int64 limbs:
 * blob = [8 x int64 metadata][n*L*d x 4 x int64 limbs].  Contributions are
 * added with integer atomics, so the sum is exact and independent of order;
 * blobs of several calls/ranks combine by adding the limbs as integers
 * (e.g. NCCL all-reduce SUM on int64) and taking the MAX of the metadata.
 * The anchor (scale) is fixed at init from max|cot| and max(n1, n2): every
 * call and rank feeding one gradient must init with the same full cotangent.
 * A contribution beyond the accumulator's range (~2^66 x n x max|cot|) or a
 * non-finite one sets a flag and the finalize step returns NaN. */
size_t sk_grad_acc_bytes(int64_t n, int64_t L, int64_t d);
int sk_grad_acc_init(void *acc, int64_t n, int64_t L, int64_t d, const double *cot, int64_t n1,
                     int64_t n2, int symmetric, void *stream);
/* grad = value (accumulate == 0) or grad += value */
int sk_grad_acc_finalize(const void *acc, int64_t n, int64_t L, int64_t d, double *grad,
                         int accumulate, void *stream);

size_t sk_backward_gram_acc_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                            int64_t d, int lam1, int lam2, int static_kernel,
                                            int symmetric);
/* sk_backward_gram / sk_value_and_grad_gram into caller accumulators: adds the
 * gradient of the pairs with rows in [row_begin, row_end) to acc_x (and acc_y;
 * NULL when y == NULL).  values (nullable) receives the Gram entries as in
 * sk_value_and_grad_gram. */
int sk_backward_gram_acc(const double *x, const double *y, int64_t n1, int64_t n2, int64_t L1,
                         int64_t L2, int64_t d, int lam1, int lam2, int static_kernel,
                         double sigma, int64_t row_begin, int64_t row_end, const double *cot,
                         double *values, void *acc_x, void *acc_y, void *workspace,
                         size_t workspace_bytes, void *stream);
/* the same on transformed paths: the accumulators hold the TRANSFORMED-path
 * gradient (sk_grad_acc_bytes(n, L', d')); map it back after finalising with
 * sk_transform_adjoint */
size_t sk_backward_gram_acc_tf_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                               int64_t d, int lam1, int lam2, int static_kernel,
                                               int symmetric, int transform);
int sk_backward_gram_acc_tf(const double *x, const double *y, int64_t n1, int64_t n2,
                            int64_t L1, int64_t L2, int64_t d, int lam1, int lam2,
                            int static_kernel, double sigma, int transform, int64_t row_begin,
                            int64_t row_end, const double *cot, double *values, void *acc_x,
                            void *acc_y, void *workspace, size_t workspace_bytes, void *stream);
/* sk_backward_gram_acc_tf for the cross-Gram pairs with rows in
 * [row_begin, row_end) AND columns in [col_begin, col_end) (col_begin a
 * multiple of 8): a column split sees the same DMMA work items as the whole
 * call, so its accumulated gradients are bitwise the whole call's.  Linear
 * static kernel on the DMMA backward only (dyadic order 0, d <= 16, x's fine
 * axis not shorter than y's), else SK_INVALID_ARGUMENT.  values (nullable):
 * (row_end - row_begin) x (col_end - col_begin).  The torch layer uses it to
 * solve cross Grams whose y paths are longer as G^T with the row range of G
 * as the column range of G^T.  Workspace: sk_backward_gram_acc_tf_workspace_bytes. */
int sk_backward_gram_acc_cols(const double *x, const double *y, int64_t n1, int64_t n2,
                              int64_t L1, int64_t L2, int64_t d, int lam1, int lam2,
                              int transform, int64_t row_begin, int64_t row_end,
                              int64_t col_begin, int64_t col_end, const double *cot,
                              double *values, void *acc_x, void *acc_y, void *workspace,
                              size_t workspace_bytes, void *stream);
/* FP32-arithmetic Gram backward (linear static kernel, dyadic order 0,
 * d <= 16, cross Grams with L2 <= L1): sk_backward_gram_acc with the forward, recompute and adjoint
 * recurrences in float (small-correction forms) and
 * p = <dx, dy>, gx, gy on the FP64 tensor cores.  x / y are the fp64 copies of
 * float32 points (exact); values (nullable) are the float recurrence's
 * results widened to double.  Other shapes: SK_INVALID_ARGUMENT. */
size_t sk_backward_gram_acc_f32_workspace_bytes(int64_t n1, int64_t n2, int64_t L1, int64_t L2,
                                                int64_t d, int lam1, int lam2, int symmetric);
int sk_backward_gram_acc_f32(const double *x, const double *y, int64_t n1, int64_t n2,
                             int64_t L1, int64_t L2, int64_t d, int lam1, int lam2,
                             int64_t row_begin, int64_t row_end, const double *cot,
                             double *values, void *acc_x, void *acc_y, void *workspace,
                             size_t workspace_bytes, void *stream);

/* ---- truncated signatures ------------------------------------------------
 * Replaces sigcore's signature (signature.py:104-121) and signature_backward
 * (signature_grad.py:20-53).  out (B, sk_signature_length(d', depth)): levels
 * 1..depth back to back, row-major multi-indices (tensors.py layout); d' is
 * the transformed dimension (d, d+1 time-augmented, 2d lead-lag).  times:
 * optional (L,) time grid for the time augmentation (NULL = linspace(0, 1, L),
 * reference PathBatch.times).  The forward issues the reference's Horner
 * operations in the reference's order without FMA contraction (bitwise the
 * reference's values); the backward is the reference's time-reversed
 * deconstruction with deterministic, chunked reductions.  Supported
 * (d', depth): d' <= 2 & depth <= 16, 4 & 10, 8 & 8, 16 & 6, 32 & 4. */
int64_t sk_signature_length(int64_t d, int depth);
size_t sk_signature_workspace_bytes(int64_t B, int64_t L, int64_t d, int depth, int transform);
int sk_signature(const double *x, const double *times, int64_t B, int64_t L, int64_t d,
                 int depth, int transform, double *out, void *workspace, size_t workspace_bytes,
                 void *stream);
size_t sk_signature_backward_workspace_bytes(int64_t B, int64_t L, int64_t d, int depth,
                                             int transform);
/* grad (B, L, d) = dF/dx for cot = dF/d(signature) (B, length); raw path shape */
int sk_signature_backward(const double *x, const double *times, int64_t B, int64_t L, int64_t d,
                          int depth, int transform, const double *cot, double *grad,
                          void *workspace, size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SIGKERNEL_H */
