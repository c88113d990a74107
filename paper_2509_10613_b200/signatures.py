"""Truncated signatures on B200, forward and backward.

Torch API (autograd):

    S = signature(x, depth=4)                       # (B, L, d) -> (B, total)
    S = signature(x, 3, transform="lead_lag")       # transform inside the kernel
    S.sum().backward()

sigcore-compatible numpy facade (reference signature.py:23-121,
signature_grad.py:20-53, tensors.py): SigOptions, PathBatch, tensor_shape,
sig_tensor_shape, signature(batch, opts), signature_backward(batch, opts, cot).

Both run the sm_100a kernels of csrc/sk_signature.cu through the C ABI
(include/sigkernel.h sk_signature*).  The forward issues the reference's
Horner operations in its order without FMA contraction, so values are bitwise
the reference's; the backward is the reference's time-reversed deconstruction
with deterministic chunked reductions.  Divergences (documented): method
"direct" runs the same (Horner) kernel -- the reference's own tests hold the two
within 1e-12 (tests/test_signature.py:33-40); scalar_width=32 computes in fp64
and returns float32 (more accurate than the reference's fp32 arithmetic).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, ops
from .errors import InvalidArgument

METHODS = ("direct", "horner")
WIDTHS = (32, 64)
KINDS = ("time_augment", "lead_lag")


# ------------------------------------------------------------------ tensor shape
@dataclass(frozen=True)
class TensorShape:
    """Dimension, depth, and per-level offsets into the flat buffer (tensors.py:16-47)."""

    d: int
    depth: int
    offsets: tuple = field(init=False)

    def __post_init__(self):
        if self.d < 1 or self.depth < 1:
            raise InvalidArgument(
                f"dimension and depth must be >= 1, got d={self.d}, depth={self.depth}")
        offs, size = [0], 1
        for _ in range(self.depth):
            size *= self.d
            offs.append(offs[-1] + size)
        object.__setattr__(self, "offsets", tuple(offs))

    @property
    def total(self) -> int:
        return self.offsets[-1]

    def level_slice(self, k: int) -> slice:
        if not 1 <= k <= self.depth:
            raise InvalidArgument(f"level {k} outside 1..{self.depth}")
        return slice(self.offsets[k - 1], self.offsets[k])


def tensor_shape(d: int, depth: int) -> TensorShape:
    return TensorShape(d, depth)


def effective_dim(d: int, kind) -> int:
    if kind is None or kind == "none":
        return d
    if kind not in KINDS:
        raise InvalidArgument(f"unknown transform {kind!r}")
    return d + 1 if kind == "time_augment" else 2 * d


# -------------------------------------------------------------------- kernels
def _tf(transform) -> int:
    if transform == "none":
        transform = None
    return ops.transform_code(transform)


def _times(times, L, dev):
    if times is None:
        return None
    t = torch.as_tensor(times, dtype=torch.float64, device=dev).contiguous()
    if t.shape != (L,):
        raise InvalidArgument(f"time grid has shape {tuple(t.shape)}, expected ({L},)")
    return t


def signature_forward(x, depth: int, transform=None, times=None) -> torch.Tensor:
    """(B, L, d) CUDA float64 -> (B, total) signatures (C ABI sk_signature)."""
    lib = _lib.load()
    x = ops._paths(x, "x")
    B, L, d = x.shape
    tf = _tf(transform)
    total = lib.sk_signature_length(effective_dim(d, transform if transform != "none" else None),
                                    depth)
    if total <= 0:
        raise InvalidArgument("signature too large")
    t = _times(times, L, x.device)
    out = torch.empty((B, total), dtype=torch.float64, device=x.device)
    with ops._on(x.device):
        nb = lib.sk_signature_workspace_bytes(B, L, d, depth, tf)
        if B and nb == 0:
            _lib.check(lib.sk_signature(None, None, B, L, d, depth, tf, None, None, 0, None))
        ws = ops._workspace(nb, x.device)
        _lib.check(lib.sk_signature(ops._ptr(x), ops._ptr(t), B, L, d, depth, tf, ops._ptr(out),
                                    ops._ptr(ws), ws.numel(), ops._stream(x.device)))
    return out


def signature_backward_t(x, depth: int, cot, transform=None, times=None) -> torch.Tensor:
    """dF/dx (B, L, d) for cot = dF/d(signature) (B, total) (C ABI sk_signature_backward)."""
    lib = _lib.load()
    x = ops._paths(x, "x")
    B, L, d = x.shape
    tf = _tf(transform)
    total = lib.sk_signature_length(effective_dim(d, transform if transform != "none" else None),
                                    depth)
    cot = ops._cotangent(cot, (B, total), x)
    t = _times(times, L, x.device)
    grad = torch.empty_like(x)
    if B == 0:
        return grad
    with ops._on(x.device):
        nb = lib.sk_signature_backward_workspace_bytes(B, L, d, depth, tf)
        if nb == 0:
            _lib.check(lib.sk_signature_backward(None, None, B, L, d, depth, tf, None, None, None,
                                                 0, None))
        ws = ops._workspace(nb, x.device)
        _lib.check(lib.sk_signature_backward(ops._ptr(x), ops._ptr(t), B, L, d, depth, tf,
                                             ops._ptr(cot), ops._ptr(grad), ops._ptr(ws),
                                             ws.numel(), ops._stream(x.device)))
    return grad


class _SignatureFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, depth, transform, times):
        ctx.save_for_backward(x)
        ctx.cfg = (depth, transform, times)
        return signature_forward(x, depth, transform, times)

    @staticmethod
    def backward(ctx, cot):
        (x,) = ctx.saved_tensors
        depth, transform, times = ctx.cfg
        return signature_backward_t(x, depth, cot, transform, times), None, None, None


def signature(x, depth: int, transform=None, times=None) -> torch.Tensor:
    """Truncated signatures (levels 1..depth, reference layout) of a (B, L, d)
    batch -> (B, total), or of one (L, d) path -> (total,).  Differentiable.
    transform: None, "time_augment" (times: optional (L,) grid) or "lead_lag",
    applied inside the kernel (reference fused_increments, transforms.py:91-120).
    Float32 inputs are computed in float64 and returned as float32."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise InvalidArgument("x must be a CUDA tensor (no CPU fallback)")
    if depth < 1:
        raise InvalidArgument(f"depth must be >= 1, got {depth}")
    sq = x.dim() == 2
    xb = x.unsqueeze(0) if sq else x
    out_dtype = x.dtype if x.is_floating_point() else torch.float64
    s = _SignatureFn.apply(xb.to(torch.float64), int(depth), transform, times)
    s = s.to(out_dtype)
    return s[0] if sq else s


# ---------------------------------------------------------------- numpy facade
@dataclass
class PathBatch:
    """B x L x d path points, optional shared strictly increasing time grid
    (reference signature.py:23-55)."""

    data: np.ndarray
    times: np.ndarray | None = None

    def __post_init__(self):
        self.data = np.ascontiguousarray(self.data)
        if self.data.ndim == 2:
            self.data = self.data[None]
        if self.data.ndim != 3:
            raise InvalidArgument(f"path batch must be (B, L, d) or (L, d), "
                                  f"got shape {self.data.shape}")
        if self.times is not None:
            self.times = np.asarray(self.times, dtype=self.data.dtype)
            if self.times.shape != (self.L,):
                raise InvalidArgument(
                    f"time grid has shape {self.times.shape}, expected ({self.L},)")
            if np.any(np.diff(self.times) <= 0):
                raise InvalidArgument("time grid must be strictly increasing")

    @property
    def B(self) -> int:
        return self.data.shape[0]

    @property
    def L(self) -> int:
        return self.data.shape[1]

    @property
    def d(self) -> int:
        return self.data.shape[2]


@dataclass(frozen=True)
class SigOptions:
    """Truncation depth, update rule, fused transform, scalar width (signature.py:58-80)."""

    depth: int
    method: str = "horner"
    transform: str | None = None
    scalar_width: int = 64

    def __post_init__(self):
        if self.depth < 1:
            raise InvalidArgument(f"depth must be >= 1, got {self.depth}")
        if self.method not in METHODS:
            raise InvalidArgument(f"method must be one of {METHODS}, got {self.method!r}")
        if self.transform not in (None, "none") + KINDS:
            raise InvalidArgument(f"unknown transform {self.transform!r}")
        if self.scalar_width not in WIDTHS:
            raise InvalidArgument(f"scalar width must be 32 or 64, got {self.scalar_width}")

    @property
    def dtype(self):
        return np.float32 if self.scalar_width == 32 else np.float64


def sig_tensor_shape(path_dim: int, opts: SigOptions) -> TensorShape:
    return tensor_shape(effective_dim(path_dim, opts.transform), opts.depth)


def _as_batch(batch) -> PathBatch:
    return batch if isinstance(batch, PathBatch) else PathBatch(np.asarray(batch))


def _validated(pb: PathBatch, opts: SigOptions):
    if pb.L < 2:
        raise InvalidArgument(f"signature needs at least 2 points, got L={pb.L}")
    data = pb.data
    if not np.isfinite(data).all():
        raise InvalidArgument("path batch contains non-finite values")
    if data.dtype != opts.dtype:
        data = data.astype(opts.dtype)
    x = torch.as_tensor(np.ascontiguousarray(data, dtype=np.float64),
                        device=torch.device("cuda", torch.cuda.current_device()))
    return x


def signature_np(batch, opts: SigOptions, threads: int | None = None) -> np.ndarray:
    """sigcore.signature: (B, total) (or (total,) for one unbatched path);
    `threads` accepted and ignored (results never depend on it)."""
    pb = _as_batch(batch)
    squeeze = not isinstance(batch, PathBatch) and np.asarray(batch).ndim == 2
    x = _validated(pb, opts)
    out = signature_forward(x, opts.depth, opts.transform, pb.times).cpu().numpy()
    out = out.astype(opts.dtype, copy=False)
    return out[0] if squeeze else out


def signature_backward_np(batch, opts: SigOptions, cot, threads: int | None = None) -> np.ndarray:
    """sigcore.signature_backward: gradient shaped like the input batch."""
    pb = _as_batch(batch)
    squeeze = not isinstance(batch, PathBatch) and np.asarray(batch).ndim == 2
    shape = sig_tensor_shape(pb.d, opts)
    cot = np.ascontiguousarray(np.asarray(cot, dtype=opts.dtype))
    if cot.ndim == 1:
        cot = cot[None]
    if cot.shape != (pb.B, shape.total):
        raise InvalidArgument(
            f"cotangent has shape {cot.shape}, expected ({pb.B}, {shape.total})")
    x = _validated(pb, opts)
    c = torch.as_tensor(cot.astype(np.float64), device=x.device)
    g = signature_backward_t(x, opts.depth, c, opts.transform, pb.times).cpu().numpy()
    g = g.astype(opts.dtype, copy=False)
    return g[0] if squeeze else g
