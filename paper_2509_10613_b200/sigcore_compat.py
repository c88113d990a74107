"""Drop-in facade with the reference's kernel API (sigcore 0.1.0).

Same names, signatures, exceptions and dtype rules as
/root/reference/pkg/src/sigcore/kernel.py and kernel_grad.py, so code (and
the reference's own kernel tests) written against sigcore can switch to the
B200 path by importing this module instead:

    from paper_2509_10613_b200 import sigcore_compat as sc
    sc.kernel_batch(x, y, sc.KernelConfig(1, 1))

numpy arrays in, new numpy arrays out (the caller owns them), exactly like the
reference; every solve runs on the GPU (current CUDA device) through the C ABI.
`threads` is accepted for signature compatibility and ignored (results never
depended on it); `strip_width` likewise has no GPU meaning.

Divergence (documented): integer-dtype paths are cast to float64 instead of
reproducing the reference's integer-buffer bug.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import InvalidArgument, InvalidState

from .signatures import (PathBatch, SigOptions, TensorShape, sig_tensor_shape,  # noqa: E402
                        tensor_shape)
from .signatures import signature_backward_np as signature_backward  # noqa: E402
from .signatures import signature_np as signature  # noqa: E402

from .sgt_io import FormatError, read_array, write_array  # noqa: E402

__all__ = ["KernelConfig", "SolveResult", "InvalidArgument", "InvalidState", "FormatError",
           "read_array", "write_array", "transform", "transform_adjoint", "fused_increments",
           "effective_dim", "effective_length", "default_times", "increment_gram",
           "fine_cells", "solve_workspace_elements", "solve_goursat", "kernel_batch",
           "kernel_gram", "kernel_backward", "kernel_batch_backward",
           # truncated signatures (reference signature.py, signature_grad.py, tensors.py)
           "signature", "signature_backward", "SigOptions", "PathBatch", "TensorShape",
           "tensor_shape", "sig_tensor_shape"]


@dataclass(frozen=True)
class KernelConfig:
    """Per-axis dyadic refinement orders, strip width, grid retention (kernel.py:21-38)."""

    dyadic_x: int = 0
    dyadic_y: int = 0
    strip_width: int = 32
    store_grid: bool = False

    def __post_init__(self):
        if self.dyadic_x < 0 or self.dyadic_y < 0:
            raise InvalidArgument("dyadic orders must be >= 0")
        if self.strip_width < 1:
            raise InvalidArgument("strip width must be >= 1")

    @property
    def scale(self) -> float:
        return 2.0 ** -(self.dyadic_x + self.dyadic_y)


@dataclass
class SolveResult:
    """Kernel value, plus the full fine-resolution grid when retained (kernel.py:41-46)."""

    value: float
    grid: np.ndarray | None = None


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _dtype_of(*arrays):
    dt = np.result_type(*[a.dtype for a in arrays])
    return dt if np.issubdtype(dt, np.floating) else np.dtype(np.float64)


def _as_paths(x, name):
    x = np.ascontiguousarray(x)
    if x.ndim == 2:
        x = x[None]
    if x.ndim != 3:
        raise InvalidArgument(f"{name} must be (L, d) or (B, L, d), got shape {x.shape}")
    if x.shape[1] < 2:
        raise InvalidArgument(f"{name} needs at least 2 points per path")
    return x


def _cuda(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device=_device())


def increment_gram(x, y) -> np.ndarray:
    """Materialised increment products (kernel.py:60-77).  The B200 solvers never
    form this matrix; it is provided for API compatibility (one batched DGEMM)."""
    x = np.asarray(x)
    squeeze = x.ndim == 2
    x = _as_paths(x, "x")
    y = _as_paths(y, "y")
    if x.shape[0] != y.shape[0]:
        raise InvalidArgument(f"batch sizes differ: {x.shape[0]} vs {y.shape[0]}")
    if x.shape[2] != y.shape[2]:
        raise InvalidArgument(f"path dimensions differ: {x.shape[2]} vs {y.shape[2]}")
    dt = _dtype_of(x, y)
    dx = torch.diff(_cuda(x), dim=1)
    dy = torch.diff(_cuda(y), dim=1)
    delta = torch.matmul(dx, dy.transpose(1, 2)).cpu().numpy().astype(dt, copy=False)
    return delta[0] if squeeze else delta


def fine_cells(delta_shape, cfg: KernelConfig) -> tuple[int, int]:
    """kernel.py:80-82."""
    return (delta_shape[0] << cfg.dyadic_x, delta_shape[1] << cfg.dyadic_y)


def solve_workspace_elements(delta_shape, cfg: KernelConfig) -> int:
    """kernel.py:85-91 (the reference's gridless CPU march; reported for API
    compatibility -- the GPU solve keeps its wavefront in registers)."""
    m1, m2 = fine_cells(delta_shape, cfg)
    if m2 > m1:
        m1, m2 = m2, m1
    return 3 * (min(cfg.strip_width, m1) + 1) + (m2 + 1)


def solve_goursat(delta, cfg: KernelConfig) -> SolveResult:
    """One PDE solve over a given coarse increment matrix (kernel.py:94-122)."""
    delta = np.asarray(delta)
    if delta.ndim != 2 or delta.shape[0] < 1 or delta.shape[1] < 1:
        raise InvalidArgument(f"increment matrix must be 2-d and non-empty, "
                              f"got shape {delta.shape}")
    dt = _dtype_of(delta)
    d = _cuda(delta)
    if cfg.store_grid:
        grid = ops.solve_delta_grid(d, cfg.dyadic_x, cfg.dyadic_y).cpu().numpy()
        return SolveResult(float(grid[-1, -1]), grid.astype(dt, copy=False))
    v = ops.solve_delta(d[None], cfg.dyadic_x, cfg.dyadic_y)
    return SolveResult(float(v.item()))


def kernel_batch(x, y, cfg: KernelConfig = KernelConfig(), threads: int | None = None):
    """Pairwise k(x_b, y_b) for aligned batches (kernel.py:125-148)."""
    x = _as_paths(x, "x")
    y = _as_paths(y, "y")
    if x.shape[0] != y.shape[0]:
        raise InvalidArgument(f"batch sizes differ: {x.shape[0]} vs {y.shape[0]}")
    if x.shape[2] != y.shape[2]:
        raise InvalidArgument(f"path dimensions differ: {x.shape[2]} vs {y.shape[2]}")
    dt = _dtype_of(x, y)
    out = ops.forward_batch(_cuda(x), _cuda(y), cfg.dyadic_x, cfg.dyadic_y, 0, 1.0)
    return out.cpu().numpy().astype(dt, copy=False)


def kernel_gram(x, y=None, cfg: KernelConfig = KernelConfig(), threads: int | None = None):
    """Gram matrix G[a, b] = k(x_a, y_b) (kernel.py:151-180); exactly symmetric
    when y is x (or omitted)."""
    symmetric = y is None or y is x
    x = _as_paths(x, "x")
    yy = x if symmetric else _as_paths(y, "y")
    if x.shape[2] != yy.shape[2]:
        raise InvalidArgument(f"path dimensions differ: {x.shape[2]} vs {yy.shape[2]}")
    dt = _dtype_of(x, yy)
    G = ops.forward_gram(_cuda(x), None if symmetric else _cuda(yy), cfg.dyadic_x,
                         cfg.dyadic_y, 0, 1.0)
    return G.cpu().numpy().astype(dt, copy=False)


def _one_pair(x, name):
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if x.ndim != 2 or x.shape[0] < 2:
        raise InvalidArgument(f"{name} must be a single (L, d) path with L >= 2, "
                              f"got shape {x.shape}")
    return x


def kernel_backward(x, y, cfg: KernelConfig, forward: SolveResult, cot: float = 1.0):
    """Gradients of cot * k(x, y) w.r.t. both paths (kernel_grad.py:27-61).

    The reference differentiates through a stored forward grid; the B200
    backward recomputes the forward values it needs from checkpoints, so the
    grid is only validated (presence and shape, same errors as the reference)."""
    x = _one_pair(x, "x")
    y = _one_pair(y, "y")
    if x.shape[1] != y.shape[1]:
        raise InvalidArgument(f"path dimensions differ: {x.shape[1]} vs {y.shape[1]}")
    if forward.grid is None:
        raise InvalidState("kernel_backward needs a forward solve with store_grid=True")
    m1, m2 = fine_cells((x.shape[0] - 1, y.shape[0] - 1), cfg)
    if forward.grid.shape != (m1 + 1, m2 + 1):
        raise InvalidArgument(
            f"forward grid shape {forward.grid.shape} does not match "
            f"({m1 + 1}, {m2 + 1}) for this config")
    _, gx, gy = ops.backward_batch(_cuda(x[None]), _cuda(y[None]), cfg.dyadic_x, cfg.dyadic_y,
                                   0, 1.0, _cuda(np.array([float(cot)])))
    return gx[0].cpu().numpy(), gy[0].cpu().numpy()


def kernel_batch_backward(x, y, cfg: KernelConfig, cot=None, threads: int | None = None):
    """Values and gradients for aligned batches (kernel_grad.py:64-98)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    y = np.ascontiguousarray(np.asarray(y, dtype=np.float64))
    squeeze = x.ndim == 2
    if x.ndim == 2:
        x = x[None]
    if y.ndim == 2:
        y = y[None]
    if x.shape[0] != y.shape[0]:
        raise InvalidArgument(f"batch sizes differ: {x.shape[0]} vs {y.shape[0]}")
    if cot is None:
        cot = np.ones(x.shape[0])
    cot = np.atleast_1d(np.asarray(cot, dtype=np.float64))
    if cot.shape != (x.shape[0],):
        raise InvalidArgument(f"cotangent has shape {cot.shape}, "
                              f"expected ({x.shape[0]},)")
    x = _as_paths(x, "x")
    y = _as_paths(y, "y")
    vals, gx, gy = ops.backward_batch(_cuda(x), _cuda(y), cfg.dyadic_x, cfg.dyadic_y, 0, 1.0,
                                      _cuda(cot), want_values=True)
    vals, gx, gy = vals.cpu().numpy(), gx.cpu().numpy(), gy.cpu().numpy()
    if squeeze:
        return vals[0], gx[0], gy[0]
    return vals, gx, gy


# ------------------------------------------------------------ path transforms
# The reference's numpy transform utilities (transforms.py:30-135) with the
# same names, shapes, dtypes and errors; the work runs on the GPU (torch ops
# for the index bookkeeping, the C-ABI adjoint kernel for transform_adjoint).
# The kernels themselves never need them: sig_kernel(..., transform=...) builds
# the transformed increments inside the kernels' input preparation.
TRANSFORM_KINDS = ("time_augment", "lead_lag")


def _check_kind(kind):
    if kind not in TRANSFORM_KINDS:
        raise InvalidArgument(f"unknown transform kind {kind!r}, expected one of {TRANSFORM_KINDS}")


def _as_3d_np(data, name="path batch"):
    data = np.asarray(data)
    if data.ndim == 2:
        return data[None], True
    if data.ndim != 3:
        raise InvalidArgument(f"{name} must be (L, d) or (B, L, d), got shape {data.shape}")
    return data, False


def default_times(length: int, dtype=np.float64) -> np.ndarray:
    """Uniform time grid on [0, 1] (numpy.linspace); a single point sits at 0."""
    if length == 1:
        return np.zeros(1, dtype=dtype)
    return np.linspace(0.0, 1.0, length, dtype=dtype)


def _times_t(times, length, dtype, dev):
    t = default_times(length, dtype) if times is None else np.asarray(times, dtype=dtype)
    if t.shape != (length,):
        raise InvalidArgument(f"time grid has shape {t.shape}, expected ({length},)")
    return torch.as_tensor(t, device=dev)


def transform(batch, kind: str, times=None):
    """transforms.py:37-63: time_augment (B, L, d) -> (B, L, d+1), lead_lag ->
    (B, 2L-1, 2d) with Z[2k] = (X[k], X[k]), Z[2k+1] = (X[k+1], X[k])."""
    _check_kind(kind)
    data, squeeze = _as_3d_np(batch)
    b, length, d = data.shape
    if length < 1:
        raise InvalidArgument("transform needs at least one point")
    dev = _device()
    x = torch.as_tensor(np.ascontiguousarray(data), device=dev)
    if kind == "time_augment":
        t = _times_t(times, length, data.dtype, dev)
        out = torch.cat([x, t.view(1, length, 1).expand(b, length, 1)], dim=2)
    else:
        out = torch.empty((b, 2 * length - 1, 2 * d), dtype=x.dtype, device=dev)
        out[:, 0::2, :d] = x
        out[:, 0::2, d:] = x
        out[:, 1::2, :d] = x[:, 1:]
        out[:, 1::2, d:] = x[:, :-1]
    out = out.cpu().numpy()
    return out[0] if squeeze else out


def transform_adjoint(grad_out, kind: str):
    """transforms.py:66-88 through the C-ABI adjoint kernel (sk_transform_adjoint,
    the same addition order): the time column gets no gradient; each lead-lag
    point sums the gradients of every slot that reads it."""
    _check_kind(kind)
    g, squeeze = _as_3d_np(grad_out, "gradient batch")
    b, length, dim = g.shape
    if kind == "time_augment":
        if dim < 2:
            raise InvalidArgument("time-augmented gradient needs at least 2 coordinates")
        L, d = length, dim - 1
    else:
        if dim % 2 != 0 or length % 2 != 1:
            raise InvalidArgument(
                f"lead-lag gradient must be (B, 2L-1, 2d), got shape {g.shape}")
        L, d = (length + 1) // 2, dim // 2
    out_dtype = g.dtype
    gt = torch.as_tensor(np.ascontiguousarray(g, dtype=np.float64), device=_device())
    out = ops.transform_adjoint(gt, L, d, kind).cpu().numpy().astype(out_dtype, copy=False)
    return out[0] if squeeze else out


def fused_increments(batch, kind: str | None = None, times=None):
    """transforms.py:91-120: the increments of the transformed path built from
    the input points (none: (B, L-1, d); time_augment: (B, L-1, d+1); lead_lag:
    (B, 2L-2, 2d), alternating (dX_k, 0) and (0, dX_k))."""
    data, squeeze = _as_3d_np(batch)
    b, length, d = data.shape
    if length < 1:
        raise InvalidArgument("increments need at least one point")
    dev = _device()
    x = torch.as_tensor(np.ascontiguousarray(data), device=dev)
    dx = x[:, 1:] - x[:, :-1]
    if kind is None or kind == "none":
        out = dx
    elif kind == "time_augment":
        t = _times_t(times, length, data.dtype, dev)
        out = torch.cat([dx, (t[1:] - t[:-1]).view(1, length - 1, 1).expand(b, length - 1, 1)],
                        dim=2)
    elif kind == "lead_lag":
        out = torch.zeros((b, 2 * length - 2, 2 * d), dtype=x.dtype, device=dev)
        out[:, 0::2, :d] = dx
        out[:, 1::2, d:] = dx
    else:
        _check_kind(kind)
    out = out.cpu().numpy()
    return out[0] if squeeze else out


def effective_dim(d: int, kind) -> int:
    """transforms.py:123-128."""
    if kind is None or kind == "none":
        return d
    _check_kind(kind)
    return d + 1 if kind == "time_augment" else 2 * d


def effective_length(length: int, kind) -> int:
    """transforms.py:131-135."""
    return 2 * length - 1 if kind == "lead_lag" else length
