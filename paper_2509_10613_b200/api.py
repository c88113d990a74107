"""pySigLib-style torch API: sig_kernel / sig_kernel_gram with autograd.

    k = sig_kernel(x, y, dyadic_order=1)                  # (B,)
    G = sig_kernel_gram(X, dyadic_order=(0, 1),
                        static_kernel=RBFKernel(0.5))     # (n, n)
    loss = (G * C).sum(); loss.backward()

Forward and backward both run hand-written sm_100a kernels through the C ABI
(include/sigkernel.h).  The backward is the paper's exact scheme
(differentiate the solver, Alg. 4 / reference kernel_grad.py), done
as a reverse wavefront that recomputes forward values from checkpoints
instead of storing the full PDE grid.

dtype rule (reference kernel.py:36-38, _kernels.py:325): float32 inputs are
solved in float64 arithmetic and the result is returned as float32, exactly
like the reference's "fp32 storage, fp64 math" path.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops
from .errors import InvalidArgument


@dataclass(frozen=True)
class LinearKernel:
    """Static kernel <a, b> (the reference's increment_gram, kernel.py:60-77)."""
    kind: str = "linear"


@dataclass(frozen=True)
class RBFKernel:
    """Static kernel exp(-|a - b|^2 / (2 sigma^2)) (no reference counterpart;
    convention documented in DESIGN.md)."""
    sigma: float = 1.0
    kind: str = "rbf"

    def __post_init__(self):
        if not self.sigma > 0:
            raise InvalidArgument("RBF sigma must be > 0")


def _orders(dyadic_order):
    if isinstance(dyadic_order, (tuple, list)):
        if len(dyadic_order) != 2:
            raise InvalidArgument("dyadic_order must be an int or a pair (lam1, lam2)")
        l1, l2 = int(dyadic_order[0]), int(dyadic_order[1])
    else:
        l1 = l2 = int(dyadic_order)
    if l1 < 0 or l2 < 0:
        raise InvalidArgument("dyadic orders must be >= 0")
    return l1, l2


def _batched(t, name):
    if not isinstance(t, torch.Tensor):
        raise InvalidArgument(f"{name} must be a torch tensor")
    if t.dim() == 2:
        return t.unsqueeze(0), True
    if t.dim() != 3:
        raise InvalidArgument(f"{name} must be (L, d) or (B, L, d), got shape {tuple(t.shape)}")
    return t, False


class _SigKernelFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, y, l1, l2, kind, sigma, tf):
        ctx.save_for_backward(x, y)
        ctx.cfg = (l1, l2, kind, sigma, tf)
        return ops.forward_batch(x, y, l1, l2, kind, sigma, tf)

    @staticmethod
    def backward(ctx, cot):
        x, y = ctx.saved_tensors
        l1, l2, kind, sigma, tf = ctx.cfg
        _, gx, gy = ops.backward_batch(x, y, l1, l2, kind, sigma, cot, transform=tf)
        return (gx if ctx.needs_input_grad[0] else None,
                gy if ctx.needs_input_grad[1] else None, None, None, None, None, None)


class _SigKernelGramFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, y, l1, l2, kind, sigma, tf):
        sym = y is None
        ctx.sym = sym
        ctx.cfg = (l1, l2, kind, sigma, tf)
        ctx.save_for_backward(x) if sym else ctx.save_for_backward(x, y)
        return ops.forward_gram(x, y, l1, l2, kind, sigma, transform=tf)

    @staticmethod
    def backward(ctx, cot):
        l1, l2, kind, sigma, tf = ctx.cfg
        if ctx.sym:
            (x,) = ctx.saved_tensors
            gx, _ = ops.backward_gram(x, None, l1, l2, kind, sigma, cot, transform=tf)
            return gx, None, None, None, None, None, None
        x, y = ctx.saved_tensors
        gx, gy = ops.backward_gram(x, y, l1, l2, kind, sigma, cot, transform=tf)
        return (gx if ctx.needs_input_grad[0] else None,
                gy if ctx.needs_input_grad[1] else None, None, None, None, None, None)


class _SigKernelF32Fn(torch.autograd.Function):
    """FP32-arithmetic forward; the backward is the exact fp64 one (as the
    reference's kernel_backward forces float64, kernel_grad.py:20)."""

    @staticmethod
    def forward(ctx, x, y, l1, l2, tf):
        ctx.save_for_backward(x, y)
        ctx.cfg = (l1, l2, tf)
        return ops.forward_batch_f32(x, y, l1, l2, tf)

    @staticmethod
    def backward(ctx, cot):
        x, y = ctx.saved_tensors
        l1, l2, tf = ctx.cfg
        _, gx, gy = ops.backward_batch(x.double(), y.double(), l1, l2, 0, 1.0, cot.double(),
                                       transform=tf)
        return (gx.to(x.dtype) if ctx.needs_input_grad[0] else None,
                gy.to(y.dtype) if ctx.needs_input_grad[1] else None, None, None, None)


class _SigKernelGramF32Fn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, y, l1, l2, tf):
        ctx.sym = y is None
        ctx.cfg = (l1, l2, tf)
        ctx.save_for_backward(x) if ctx.sym else ctx.save_for_backward(x, y)
        return ops.forward_gram_f32(x, y, l1, l2, transform=tf)

    @staticmethod
    def backward(ctx, cot):
        l1, l2, tf = ctx.cfg
        # FP32-arithmetic backward where it exists (linear Gram tiles, order 0,
        # d <= 16: sk_backward_gram_acc_f32), else the fp64 backward
        sv = ctx.saved_tensors
        f32 = ops.f32_backward_supported(l1, l2, sv[0].shape[2], tf, sv[0].shape[1],
                                         sv[-1].shape[1])
        if ctx.sym:
            (x,) = ctx.saved_tensors
            if f32:
                _, gx, _ = ops.value_and_grad_gram_f32(x, None, cot)
            else:
                gx, _ = ops.backward_gram(x.double(), None, l1, l2, 0, 1.0, cot.double(),
                                          transform=tf)
            return gx.to(x.dtype), None, None, None, None
        x, y = ctx.saved_tensors
        if f32:
            _, gx, gy = ops.value_and_grad_gram_f32(x, y, cot)
        else:
            gx, gy = ops.backward_gram(x.double(), y.double(), l1, l2, 0, 1.0, cot.double(),
                                       transform=tf)
        return (gx.to(x.dtype) if ctx.needs_input_grad[0] else None,
                gy.to(y.dtype) if ctx.needs_input_grad[1] else None, None, None, None)


PRECISIONS = ("fp64", "fp32")


def _precision(precision, kind):
    if precision not in PRECISIONS:
        raise InvalidArgument(f"precision must be one of {PRECISIONS}, got {precision!r}")
    if precision == "fp32" and kind != 0:
        # the RBF second difference K11 - K10 - K01 + K00 cancels catastrophically
        # in fp32 (increments ~1e-4 of K): fp32 arithmetic is linear-only
        raise InvalidArgument("precision='fp32' supports the linear static kernel only")
    return precision == "fp32"


def _needs_graph(*ts) -> bool:
    return torch.is_grad_enabled() and any(t is not None and t.requires_grad for t in ts)


def _prep(t, name):
    if not t.is_cuda:
        raise InvalidArgument(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_floating_point():
        t = t.to(torch.float64)  # reference integer-dtype bug not reproduced
    return t


TRANSFORMS = (None, "time_augment", "lead_lag")


def path_transform(x: torch.Tensor, kind):
    """Materialised time augmentation / lead-lag of a (B, L, d) batch (reference
    transforms.py:37-66), for users who want the transformed points.

    time_augment: (B, L, d) -> (B, L, d+1), last coordinate the uniform time grid
    on [0, 1]; lead_lag: (B, L, d) -> (B, 2L-1, 2d) with Z[2k] = (X[k], X[k]),
    Z[2k+1] = (X[k+1], X[k]).  The kernels do NOT go through this: sig_kernel /
    sig_kernel_gram(transform=...) build the transformed increments inside the
    kernels' input preparation (sk_capi.cu prep_sides) and map gradients back
    with the transform's adjoint."""
    if kind is None:
        return x
    if kind == "time_augment":
        B, L, _ = x.shape
        # numpy.linspace's arithmetic (i * (1/(L-1)), last point exactly 1), as the reference
        t = torch.arange(L, dtype=torch.float64, device=x.device)
        if L > 1:
            t = t * (1.0 / (L - 1))
            t[-1] = 1.0
        t = t.to(x.dtype)
        return torch.cat([x, t.view(1, L, 1).expand(B, L, 1)], dim=2)
    if kind == "lead_lag":
        B, L, d = x.shape
        lead = torch.stack([x, torch.cat([x[:, 1:], x[:, -1:]], 1)], 2).reshape(B, 2 * L, d)
        lag = torch.stack([x, x], 2).reshape(B, 2 * L, d)
        return torch.cat([lead, lag], dim=2)[:, : 2 * L - 1]
    raise InvalidArgument(f"unknown transform {kind!r}, expected one of {TRANSFORMS}")


def _tf(transform):
    if transform not in TRANSFORMS:
        raise InvalidArgument(f"unknown transform {transform!r}, expected one of {TRANSFORMS}")
    return ops.transform_code(transform)


def sig_kernel(x, y, dyadic_order=0, static_kernel=None, transform=None, precision="fp64"):
    """k(x_b, y_b) for aligned batches (B, L1, d), (B, L2, d) -> (B,).

    A pair of (L, d) paths returns a 0-d tensor.  `transform` ("time_augment" or
    "lead_lag", pySigLib's path transforms) is applied to both paths inside the
    kernels (transformed increments built from the raw points; gradients come
    back for the raw points).
    precision: "fp64" (default; the reference's arithmetic -- float32 inputs are
    solved in float64, kernel.py:36-38) or "fp32" (FP32-arithmetic kernels,
    linear static kernel, float32 result; within ~1e-4 of fp64 up to a few
    thousand fine cells per axis; gradients from the fp64
    backward)."""
    x, sq = _batched(_prep(x, "x"), "x")
    y, _ = _batched(_prep(y, "y"), "y")
    tf = _tf(transform)
    l1, l2 = _orders(dyadic_order)
    kind, sigma = ops.static_kind(static_kernel)
    if _precision(precision, kind):
        k = _SigKernelF32Fn.apply(x.to(torch.float32), y.to(torch.float32), l1, l2, tf)
        return k[0] if sq else k
    out_dtype = torch.promote_types(x.dtype, y.dtype)
    if _needs_graph(x, y):
        k = _SigKernelFn.apply(x.to(torch.float64), y.to(torch.float64), l1, l2, kind, sigma, tf)
    else:  # nothing to differentiate: skip the autograd node (small-call latency)
        k = ops.forward_batch(x, y, l1, l2, kind, sigma, tf)
    k = k.to(out_dtype)
    return k[0] if sq else k


def sig_kernel_gram(x, y=None, dyadic_order=0, static_kernel=None, transform=None,
                    precision="fp64"):
    """Gram matrix G[a, b] = k(x_a, y_b) -> (n1, n2).

    y None (or y is x) -> symmetric: only a <= b is solved and the result is
    mirrored, hence exactly symmetric (reference kernel.py:151-180).
    transform, precision: as sig_kernel; with precision="fp32" the gradient of
    a linear Gram at dyadic order 0 with d <= 16 (no transform) comes from the
    FP32-arithmetic backward (sk_backward_gram_acc_f32), other shapes from the
    fp64 backward."""
    sym = y is None or y is x
    x, _ = _batched(_prep(x, "x"), "x")
    tf = _tf(transform)
    l1, l2 = _orders(dyadic_order)
    kind, sigma = ops.static_kind(static_kernel)
    if _precision(precision, kind):
        if sym:
            return _SigKernelGramF32Fn.apply(x.to(torch.float32), None, l1, l2, tf)
        y, _ = _batched(_prep(y, "y"), "y")
        return _SigKernelGramF32Fn.apply(x.to(torch.float32), y.to(torch.float32), l1, l2, tf)
    if sym:
        if _needs_graph(x):
            G = _SigKernelGramFn.apply(x.to(torch.float64), None, l1, l2, kind, sigma, tf)
        else:
            G = ops.forward_gram(x, None, l1, l2, kind, sigma, transform=tf)
        return G.to(x.dtype)
    y, _ = _batched(_prep(y, "y"), "y")
    out_dtype = torch.promote_types(x.dtype, y.dtype)
    if _needs_graph(x, y):
        G = _SigKernelGramFn.apply(x.to(torch.float64), y.to(torch.float64), l1, l2, kind, sigma,
                                   tf)
    else:
        G = ops.forward_gram(x, y, l1, l2, kind, sigma, transform=tf)
    return G.to(out_dtype)


def sig_kernel_value_and_grad(x, y, cotangent=None, dyadic_order=0, static_kernel=None,
                              transform=None):
    """k(x_b, y_b) and the gradients of F = sum_b cotangent[b] k(x_b, y_b) in ONE
    pass: returns (k, dF/dx, dF/dy).  cotangent None = ones.

    The torch form of the reference's kernel_batch_backward, which returns the
    values with the gradients from one call (kernel_grad.py:64-98): the
    backward's own forward solve (phase A) writes k, so no separate forward
    runs.  Not an autograd op -- use sig_kernel for autograd graphs.  Outputs
    follow promote_types(x.dtype, y.dtype); a pair of (L, d) paths gives a 0-d k."""
    x, sq = _batched(_prep(x, "x"), "x")
    y, _ = _batched(_prep(y, "y"), "y")
    out_dtype = torch.promote_types(x.dtype, y.dtype)
    l1, l2 = _orders(dyadic_order)
    kind, sigma = ops.static_kind(static_kernel)
    cot = None if cotangent is None else torch.as_tensor(cotangent, device=x.device).reshape(-1)
    k, gx, gy = ops.backward_batch(x.detach().to(torch.float64), y.detach().to(torch.float64),
                                   l1, l2, kind, sigma, cot, want_values=True,
                                   transform=_tf(transform))
    k, gx, gy = k.to(out_dtype), gx.to(out_dtype), gy.to(out_dtype)
    if sq:
        return k[0], gx[0], gy[0]
    return k, gx, gy


def sig_kernel_gram_value_and_grad(x, y=None, cotangent=None, dyadic_order=0, static_kernel=None,
                                   transform=None, precision="fp64"):
    """Gram matrix and its gradient in ONE fused pass: returns (G, dF/dx, dF/dy)
    for F = sum_ab cotangent[a, b] G[a, b] (cotangent None = ones, the reference
    default kernel_grad.py:81-82); dF/dy is None when y is None (symmetric: both
    slots land in dF/dx).

    This is the Gram counterpart of the reference's kernel_batch_backward, which
    returns values and gradients from one call (kernel_grad.py:64-98): the
    backward's own forward solve produces G, so no separate forward runs.
    Not an autograd op -- use sig_kernel_gram for autograd graphs.
    precision="fp32": FP32-arithmetic recurrences (linear kernel, dyadic order
    0, d <= 16, no transform); G and the gradients come back as float32."""
    sym = y is None or y is x
    x, _ = _batched(_prep(x, "x"), "x")
    l1, l2 = _orders(dyadic_order)
    kind, sigma = ops.static_kind(static_kernel)
    if _precision(precision, kind):
        xf = x.detach().to(torch.float32)
        yf = None if sym else _batched(_prep(y, "y"), "y")[0].detach().to(torch.float32)
        if not ops.f32_backward_supported(l1, l2, x.shape[2], _tf(transform), xf.shape[1],
                                          (xf if yf is None else yf).shape[1]):
            raise InvalidArgument("precision='fp32' value and gradient: linear kernel, dyadic "
                                  "order 0, d <= 16, no transform, y no longer than x")
        n1, n2 = xf.shape[0], (xf if sym else yf).shape[0]
        if cotangent is None:
            cotangent = torch.ones((n1, n2), dtype=torch.float64, device=xf.device)
        G, gx, gy = ops.value_and_grad_gram_f32(xf, yf, cotangent)
        return (G.to(torch.float32), gx.to(torch.float32),
                None if gy is None else gy.to(torch.float32))
    xd = x.detach().to(torch.float64)
    yd = None
    if not sym:
        yd, _ = _batched(_prep(y, "y"), "y")
        yd = yd.detach().to(torch.float64)
    n1, n2 = xd.shape[0], (xd if sym else yd).shape[0]
    if cotangent is None:
        cotangent = torch.ones((n1, n2), dtype=torch.float64, device=xd.device)
    G, gx, gy = ops.value_and_grad_gram(xd, yd, l1, l2, kind, sigma, cotangent,
                                        transform=_tf(transform))
    return G, gx, gy


def sig_mmd(x, y, dyadic_order=0, static_kernel=None):
    """Biased squared maximum mean discrepancy between the path sets x (n, L1, d)
    and y (m, L2, d) under the signature kernel:
        MMD^2 = mean(K_xx) + mean(K_yy) - 2 mean(K_xy),
    differentiable through sig_kernel_gram (a loss built on
    the Gram hot path)."""
    kxx = sig_kernel_gram(x, None, dyadic_order, static_kernel)
    kyy = sig_kernel_gram(y, None, dyadic_order, static_kernel)
    kxy = sig_kernel_gram(x, y, dyadic_order, static_kernel)
    return kxx.mean() + kyy.mean() - 2.0 * kxy.mean()


def sig_mmd_value_and_grad(x, y, dyadic_order=0, static_kernel=None):
    """sig_mmd and its gradients (dMMD/dx, dMMD/dy) from three fused value +
    gradient Gram passes (the cotangents of a mean are constants, so no
    separate forward solve runs).  Not an autograd op.  Values and gradients
    come back in promote_types(x.dtype, y.dtype), like sig_mmd."""
    x, _ = _batched(_prep(x, "x"), "x")
    y, _ = _batched(_prep(y, "y"), "y")
    out_dtype = torch.promote_types(x.dtype, y.dtype)
    n, m = x.shape[0], y.shape[0]
    dev = x.device
    xd = x.detach().to(torch.float64)
    # the cross term must be a cross Gram even when y is x (a symmetric call
    # would fold both gradient slots into dF/dx and return no dF/dy)
    yd = y.detach().to(torch.float64)
    if yd.data_ptr() == xd.data_ptr():
        yd = yd.clone()
    cxx = torch.full((n, n), 1.0 / (n * n), dtype=torch.float64, device=dev)
    cyy = torch.full((m, m), 1.0 / (m * m), dtype=torch.float64, device=dev)
    cxy = torch.full((n, m), -2.0 / (n * m), dtype=torch.float64, device=dev)
    kxx, gxx, _ = sig_kernel_gram_value_and_grad(xd, None, cxx, dyadic_order, static_kernel)
    kyy, gyy, _ = sig_kernel_gram_value_and_grad(yd, None, cyy, dyadic_order, static_kernel)
    kxy, gx, gy = sig_kernel_gram_value_and_grad(xd, yd, cxy, dyadic_order, static_kernel)
    mmd = kxx.mean() + kyy.mean() - 2.0 * kxy.mean()
    return mmd.to(out_dtype), (gxx + gx).to(out_dtype), (gyy + gy).to(out_dtype)
