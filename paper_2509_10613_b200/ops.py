"""Tensor-level calls into libsigkernel (device memory, current torch stream).

These are the thin shims the autograd Functions (api.py) and the numpy facade
(sigcore_compat.py) sit on.  Inputs must be CUDA float64 tensors; outputs and
workspaces are torch allocations handed to the C ABI as borrowed pointers.
"""

from __future__ import annotations

import os

import torch

from . import _lib
from .errors import InvalidArgument


def _ptr(t):
    return t.data_ptr() if t is not None else None


def _dev_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    return device.index if device.index is not None else torch.cuda.current_device()


def _stream(device=None):
    """Raw handle of torch's current stream on `device` (no Stream object)."""
    return torch._C._cuda_getCurrentRawStream(_dev_index(device))


class _NoDevSwitch:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_NO_SWITCH = _NoDevSwitch()


def _on(device):
    """Make `device` current for the enclosed launches; free when it already is
    (the common case: small calls pay no device switch)."""
    if device.index is None or device.index == torch.cuda.current_device():
        return _NO_SWITCH
    return torch.cuda.device(device)


def _same_device(t, ref, name):
    if t is not None and t.device != ref.device:
        raise InvalidArgument(f"{name} is on {t.device}, expected {ref.device}")


def _cotangent(cot, shape, ref, name="cotangent"):
    """Validated float64 contiguous cotangent of exactly `shape` on ref's device
    (the kernels index it as a dense array of that shape)."""
    if not isinstance(cot, torch.Tensor):
        raise InvalidArgument(f"{name} must be a torch tensor")
    if tuple(cot.shape) != tuple(shape):
        raise InvalidArgument(f"{name} must have shape {tuple(shape)}, got {tuple(cot.shape)}")
    _same_device(cot, ref, name)
    return cot.to(torch.float64).contiguous()


_WSQ_CACHE: dict = {}


def _wsq(fn, *args) -> int:
    """Workspace-size query of the C ABI, memoised per (entry point, current
    device, arguments): the answer depends only on those (plans are cached per
    device on the C side too)."""
    # SK_NO_MMA (read per plan on the C side) selects other instances
    key = (fn.__name__, torch.cuda.current_device(), os.environ.get("SK_NO_MMA"),
           os.environ.get("SK_MMA_DY"), args)
    nb = _WSQ_CACHE.get(key)
    if nb is None:
        nb = fn(*args)
        _WSQ_CACHE[key] = nb
    return nb


_WS_CACHE: dict = {}
_WS_CACHE_MAX = 64 << 20  # small workspaces are kept per (device, stream)


def _workspace(nbytes: int, device) -> torch.Tensor:
    """Scratch for one C-ABI call.  Workspaces up to 64 MiB are cached per
    (device, current stream) and reused: calls on one stream run in order, so
    a later call never overwrites scratch a queued kernel still reads.  Larger
    ones come from the caching allocator per call."""
    nbytes = max(int(nbytes), 1)
    # (no caching under CUDA-graph capture: that memory belongs to the graph's pool)
    if nbytes > _WS_CACHE_MAX or torch.cuda.is_current_stream_capturing():
        return torch.empty(nbytes, dtype=torch.uint8, device=device)
    idx = _dev_index(device)
    key = (idx, torch._C._cuda_getCurrentRawStream(idx))
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf[:nbytes]


def _paths(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        raise InvalidArgument(f"{name} must be a torch tensor")
    if t.dim() != 3:
        raise InvalidArgument(f"{name} must be (B, L, d), got shape {tuple(t.shape)}")
    if t.shape[1] < 2:
        raise InvalidArgument(f"{name} needs at least 2 points per path")
    if not t.is_cuda:
        raise InvalidArgument(f"{name} must live on a CUDA device")
    if t.dtype is torch.float64 and t.is_contiguous():
        return t
    return t.to(torch.float64).contiguous()


def _grad_buffer(g, ref, name):
    if g.shape != ref.shape or g.dtype != torch.float64 or not g.is_contiguous():
        raise InvalidArgument(f"{name} must be a contiguous float64 tensor of shape "
                              f"{tuple(ref.shape)}")
    _same_device(g, ref, name)


def static_kind(static_kernel):
    """(kind, sigma) for a static kernel spec: None/'linear'/LinearKernel or RBFKernel."""
    if static_kernel is None or static_kernel == "linear":
        return _lib.STATIC_LINEAR, 1.0
    kind = getattr(static_kernel, "kind", None)
    if kind == "linear":
        return _lib.STATIC_LINEAR, 1.0
    if kind == "rbf":
        return _lib.STATIC_RBF, float(static_kernel.sigma)
    raise InvalidArgument(f"unknown static kernel {static_kernel!r}")


def transform_code(transform) -> int:
    """C-ABI code of a path transform: None, "time_augment" or "lead_lag"."""
    if isinstance(transform, int) and transform in (0, 1, 2):
        return transform
    if transform not in _lib.TRANSFORMS:
        raise InvalidArgument(f"unknown transform {transform!r}, expected one of "
                              f"(None, 'time_augment', 'lead_lag')")
    return _lib.TRANSFORMS[transform]


def effective_shape(L: int, d: int, tf: int):
    """(points, dimension) of the transformed path (reference transforms.py:123-135)."""
    return (2 * L - 1 if tf == 2 else L), (d + 1 if tf == 1 else 2 * d if tf == 2 else d)


def forward_batch(x, y, lam1: int, lam2: int, kind: int, sigma: float,
                  transform=None) -> torch.Tensor:
    lib = _lib.load()
    tf = transform_code(transform)
    x = _paths(x, "x")
    y = _paths(y, "y")
    B, L1, d = x.shape
    if y.shape[0] != B:
        raise InvalidArgument(f"batch sizes differ: {B} vs {y.shape[0]}")
    if y.shape[2] != d:
        raise InvalidArgument(f"path dimensions differ: {d} vs {y.shape[2]}")
    _same_device(y, x, "y")
    L2 = y.shape[1]
    out = torch.empty(B, dtype=torch.float64, device=x.device)
    if B == 0:
        return out
    dev = x.device
    with _on(dev):
        nb = _wsq(lib.sk_forward_batch_tf_workspace_bytes, B, L1, L2, d, lam1, lam2, kind, tf)
        # (few short pairs need no workspace: BASELINE config 1's small-pair kernel)
        ws = _workspace(nb, dev) if nb else None
        _lib.check(lib.sk_forward_batch_tf(x.data_ptr(), y.data_ptr(), B, L1, L2, d, lam1, lam2,
                                           kind, sigma, tf, out.data_ptr(), _ptr(ws),
                                           ws.numel() if nb else 0, _stream(dev)))
    return out


def _transpose_cross(y, rows, kind, L1, L2, lam1, lam2, tf) -> bool:
    """Whole linear cross Grams whose y paths have the longer fine axis: the
    kernels put the longer axis on the grid rows (kernel.py:137-140), and only
    the un-swapped orientation shares one column path across a Gram tile (the
    DMMA kernels), so the forward solves G^T = Gram(y, x) instead.
    k(x, y) == k(y, x) bitwise and the DMMA forward is bitwise the FMA-pipe
    forward, so the values equal the swapped-orientation (row-range) call's.
    (The backward keeps the swapped orientation: its tile sums would differ in
    the last bits from row-split calls, which must stay bitwise equal.)"""
    if y is None or rows is not None or kind != 0:
        return False
    L1e, _ = effective_shape(L1, 1, tf)
    L2e, _ = effective_shape(L2, 1, tf)
    return ((L2e - 1) << lam2) > ((L1e - 1) << lam1)


def forward_gram(x, y, lam1: int, lam2: int, kind: int, sigma: float,
                 rows: tuple[int, int] | None = None, out: torch.Tensor | None = None,
                 transform=None):
    """G[a - r0, b] = k(x_a, y_b) for a in rows; y None -> symmetric (y is x)."""
    lib = _lib.load()
    tf = transform_code(transform)
    x, yy, sym, n1, n2, L1, L2, d = _gram_args(x, y)
    if not sym and _transpose_cross(y, rows, kind, L1, L2, lam1, lam2, tf):
        gt = forward_gram(yy, x, lam2, lam1, kind, sigma, transform=transform)
        if out is None:
            return gt.t().contiguous()
        if tuple(out.shape) != (n1, n2):
            raise InvalidArgument(f"out must have shape {(n1, n2)}")
        out.copy_(gt.t())
        return out
    r0, r1 = _rows(rows, n1)
    if out is None:
        out = torch.empty((r1 - r0, n2), dtype=torch.float64, device=x.device)
    if n1 == 0 or n2 == 0 or r1 <= r0:
        return out
    with _on(x.device):
        nb = _wsq(lib.sk_forward_gram_tf_workspace_bytes, n1, n2, L1, L2, d, lam1, lam2, kind, int(sym),
                                                    tf)
        ws = _workspace(nb, x.device)
        _lib.check(lib.sk_forward_gram_tf(_ptr(x), None if sym else _ptr(yy), n1, n2, L1, L2, d,
                                          lam1, lam2, kind, sigma, tf, r0, r1, _ptr(out),
                                          _ptr(ws), ws.numel(), _stream(x.device)))
    return out


def _paths32(t, name):
    t = _paths(t, name) if t.dtype != torch.float32 else t
    if t.dim() != 3 or t.shape[1] < 2:
        raise InvalidArgument(f"{name} must be (B, L, d) with L >= 2")
    if not t.is_cuda:
        raise InvalidArgument(f"{name} must live on a CUDA device")
    return t.to(torch.float32).contiguous()


def forward_batch_f32(x, y, lam1: int, lam2: int, transform=None) -> torch.Tensor:
    """FP32-arithmetic forward (linear static kernel): float32 in, float32 out.
    The cell uses the small-correction form (sk_cell.cuh Coef32)."""
    lib = _lib.load()
    tf = transform_code(transform)
    x = _paths32(x, "x")
    y = _paths32(y, "y")
    B, L1, d = x.shape
    if y.shape[0] != B or y.shape[2] != d:
        raise InvalidArgument(f"shapes differ: {tuple(x.shape)} vs {tuple(y.shape)}")
    _same_device(y, x, "y")
    out = torch.empty(B, dtype=torch.float32, device=x.device)
    if B == 0:
        return out
    with _on(x.device):
        nb = _wsq(lib.sk_forward_batch_f32_workspace_bytes, B, L1, y.shape[1], d, lam1, lam2, tf)
        ws = _workspace(nb, x.device)
        _lib.check(lib.sk_forward_batch_f32(_ptr(x), _ptr(y), B, L1, y.shape[1], d, lam1, lam2,
                                            tf, _ptr(out), _ptr(ws), ws.numel(),
                                            _stream(x.device)))
    return out


def forward_gram_f32(x, y, lam1: int, lam2: int, rows=None, transform=None) -> torch.Tensor:
    """FP32-arithmetic Gram forward (linear static kernel); y None = symmetric."""
    lib = _lib.load()
    tf = transform_code(transform)
    x = _paths32(x, "x")
    sym = y is None
    yy = x if sym else _paths32(y, "y")
    n1, L1, d = x.shape
    n2, L2 = yy.shape[0], yy.shape[1]
    if yy.shape[2] != d:
        raise InvalidArgument(f"path dimensions differ: {d} vs {yy.shape[2]}")
    _same_device(yy, x, "y")
    r0, r1 = _rows(rows, n1)
    out = torch.empty((r1 - r0, n2), dtype=torch.float32, device=x.device)
    if n1 == 0 or n2 == 0 or r1 <= r0:
        return out
    with _on(x.device):
        nb = _wsq(lib.sk_forward_gram_f32_workspace_bytes, n1, n2, L1, L2, d, lam1, lam2, int(sym), tf)
        ws = _workspace(nb, x.device)
        _lib.check(lib.sk_forward_gram_f32(_ptr(x), None if sym else _ptr(yy), n1, n2, L1, L2, d,
                                           lam1, lam2, tf, r0, r1, _ptr(out), _ptr(ws),
                                           ws.numel(), _stream(x.device)))
    return out


def solve_delta(delta: torch.Tensor, lam1: int, lam2: int) -> torch.Tensor:
    """Kernel values for given increment matrices delta (B, r1, r2)."""
    lib = _lib.load()
    delta = delta.to(torch.float64).contiguous()
    B, r1, r2 = delta.shape
    out = torch.empty(B, dtype=torch.float64, device=delta.device)
    with _on(delta.device):
        nb = _wsq(lib.sk_solve_delta_workspace_bytes, B, r1, r2, lam1, lam2)
        ws = _workspace(nb, delta.device)
        _lib.check(lib.sk_solve_delta(_ptr(delta), B, r1, r2, lam1, lam2, _ptr(out), _ptr(ws),
                                      ws.numel(), _stream(delta.device)))
    return out


def solve_delta_grid(delta: torch.Tensor, lam1: int, lam2: int) -> torch.Tensor:
    lib = _lib.load()
    delta = delta.to(torch.float64).contiguous()
    r1, r2 = delta.shape
    grid = torch.empty(((r1 << lam1) + 1, (r2 << lam2) + 1), dtype=torch.float64,
                       device=delta.device)
    with _on(delta.device):
        _lib.check(lib.sk_solve_delta_grid(_ptr(delta), r1, r2, lam1, lam2, _ptr(grid),
                                           _stream(delta.device)))
    return grid


def backward_batch(x, y, lam1, lam2, kind, sigma, cot, want_values=False, transform=None):
    """(values or None, grad_x, grad_y) of sum_b cot[b] k(x_b, y_b)."""
    lib = _lib.load()
    tf = transform_code(transform)
    x = _paths(x, "x")
    y = _paths(y, "y")
    B, L1, d = x.shape
    L2 = y.shape[1]
    if y.shape[0] != B:
        raise InvalidArgument(f"batch sizes differ: {B} vs {y.shape[0]}")
    if y.shape[2] != d:
        raise InvalidArgument(f"path dimensions differ: {d} vs {y.shape[2]}")
    _same_device(y, x, "y")
    cot = _cotangent(cot, (B,), x) if cot is not None else None
    gx = torch.empty_like(x)
    gy = torch.empty_like(y)
    vals = torch.empty(B, dtype=torch.float64, device=x.device) if want_values else None
    if B == 0:
        return vals, gx, gy
    with _on(x.device):
        nb = _wsq(lib.sk_backward_batch_tf_workspace_bytes, B, L1, L2, d, lam1, lam2, kind, tf)
        ws = _workspace(nb, x.device)
        _lib.check(lib.sk_backward_batch_tf(_ptr(x), _ptr(y), B, L1, L2, d, lam1, lam2, kind,
                                            sigma, tf, _ptr(cot), _ptr(vals), _ptr(gx), _ptr(gy),
                                            _ptr(ws), ws.numel(), _stream(x.device)))
    return vals, gx, gy


class GradAcc:
    """Exact (order-independent) accumulator of a Gram gradient for n paths of
    shape (L, d): int64 fixed-point limbs (include/sigkernel.h, sk_grad_acc_*).

    Sums into it are bitwise independent of tile order, of how the Gram rows
    are split across calls, and of how many GPUs contributed (gram_dist sums
    the limbs of all ranks as integers).  `limbs` and `meta` are int64 views
    for collectives: limbs add (SUM), meta combines with MAX.  With a path
    transform the limbs hold the transformed-path gradient; finalize() maps it
    back to the raw paths."""

    META = 8

    def __init__(self, n, L, d, device, transform=None):
        lib = _lib.load()
        self.shape = (int(n), int(L), int(d))
        self.tf = transform_code(transform)
        Le, de = effective_shape(int(L), int(d), self.tf)
        self.tshape = (int(n), Le, de)
        nbytes = lib.sk_grad_acc_bytes(*self.tshape)
        self.blob = torch.empty(nbytes // 8, dtype=torch.int64, device=device)
        self.meta = self.blob[: self.META]
        self.limbs = self.blob[self.META:]

    def init(self, cot, n1, n2, symmetric):
        """Zero the limbs and fix the anchor from the FULL (n1, n2) cotangent
        (every call and rank sharing this gradient must pass the same one)."""
        lib = _lib.load()
        cot = _cotangent(cot, (n1, n2), self.blob)
        with _on(self.blob.device):
            _lib.check(lib.sk_grad_acc_init(_ptr(self.blob), *self.tshape, _ptr(cot), n1, n2,
                                            int(bool(symmetric)), _stream(self.blob.device)))
        return self

    def finalize(self, out=None, accumulate=False):
        """fp64 gradient (n, L, d) of the raw paths: out = value, or out += value."""
        lib = _lib.load()
        if out is None:
            out = torch.empty(self.shape, dtype=torch.float64, device=self.blob.device)
            accumulate = False
        if (tuple(out.shape) != self.shape or out.dtype != torch.float64
                or not out.is_contiguous()):
            raise InvalidArgument(f"out must be a contiguous float64 tensor of shape {self.shape}")
        _same_device(out, self.blob, "out")
        dev = self.blob.device
        with _on(dev):
            if self.tf == 0:
                _lib.check(lib.sk_grad_acc_finalize(_ptr(self.blob), *self.tshape, _ptr(out),
                                                    int(bool(accumulate)), _stream(dev)))
            else:
                gt = torch.empty(self.tshape, dtype=torch.float64, device=dev)
                _lib.check(lib.sk_grad_acc_finalize(_ptr(self.blob), *self.tshape, _ptr(gt), 0,
                                                    _stream(dev)))
                _lib.check(lib.sk_transform_adjoint(_ptr(gt), *self.shape, self.tf, _ptr(out),
                                                    int(bool(accumulate)), _stream(dev)))
        return out


def transform_adjoint(gt: torch.Tensor, L: int, d: int, transform) -> torch.Tensor:
    """Point gradients of the transformed paths gt (n, L', d') -> the raw paths'
    (n, L, d) (reference transform_adjoint, transforms.py:66-88, same addition
    order) by the C-ABI kernel sk_transform_adjoint."""
    lib = _lib.load()
    tf = transform_code(transform)
    if not isinstance(gt, torch.Tensor) or not gt.is_cuda or gt.dim() != 3:
        raise InvalidArgument("gt must be a (n, L', d') CUDA tensor")
    gt = gt.to(torch.float64).contiguous()
    n = gt.shape[0]
    Le, de = effective_shape(L, d, tf)
    if tuple(gt.shape[1:]) != (Le, de):
        raise InvalidArgument(f"gradient of the transformed paths must be ({n}, {Le}, {de}), "
                              f"got {tuple(gt.shape)}")
    out = torch.empty((n, L, d), dtype=torch.float64, device=gt.device)
    if n == 0:
        return out
    with _on(gt.device):
        _lib.check(lib.sk_transform_adjoint(gt.data_ptr(), n, L, d, tf, out.data_ptr(), 0,
                                            _stream(gt.device)))
    return out


def _gram_args(x, y):
    x = _paths(x, "x")
    sym = y is None
    yy = x if sym else _paths(y, "y")
    n1, L1, d = x.shape
    n2, L2 = yy.shape[0], yy.shape[1]
    if yy.shape[2] != d:
        raise InvalidArgument(f"path dimensions differ: {d} vs {yy.shape[2]}")
    _same_device(yy, x, "y")
    return x, yy, sym, n1, n2, L1, L2, d


def _rows(rows, n1):
    r0, r1 = (0, n1) if rows is None else (int(rows[0]), int(rows[1]))
    if r0 < 0 or r1 > n1 or r0 > r1:
        raise InvalidArgument(f"row range {(r0, r1)} out of bounds for {n1} rows")
    return r0, r1


def _check_acc(acc, n, L, d, tf, x, name):
    if not isinstance(acc, GradAcc) or acc.shape != (n, L, d) or acc.tf != tf:
        raise InvalidArgument(f"{name} must be a GradAcc of shape {(n, L, d)} and the call's "
                              f"transform")
    _same_device(acc.blob, x, name)


def _transpose_cross_bwd(kind, L1, L2, lam1, lam2, d, tf) -> bool:
    """Cross-Gram backwards whose y paths are longer run as G^T on the DMMA
    backward (sk_backward_gram_acc_cols: the row range of G is the column range
    of G^T, so row splits stay bitwise the whole call): linear kernel, dyadic
    order 0, transformed dimension <= 16."""
    if kind != 0 or lam1 or lam2 or os.environ.get("SK_NO_MMA") == "1":
        return False
    L1e, de = effective_shape(L1, d, tf)
    L2e, _ = effective_shape(L2, d, tf)
    return de <= 16 and L2e > L1e


def _gram_backward_t(x, yy, n1, n2, L1, L2, d, lam1, lam2, kind, cot, r0, r1, out, grad_x,
                     grad_y, acc_x, acc_y, transform, tf):
    """The transposed cross-Gram backward (see _transpose_cross_bwd)."""
    lib = _lib.load()
    dev = x.device
    own = acc_x is None
    if own:  # anchors from the original (n1, n2) cotangent, as the C path would
        ax = GradAcc(n1, L1, d, dev, transform).init(cot, n1, n2, False)
        ay = GradAcc(n2, L2, d, dev, transform).init(cot, n1, n2, False)
    else:
        _check_acc(acc_x, n1, L1, d, tf, x, "acc_x")
        _check_acc(acc_y, n2, L2, d, tf, x, "acc_y")
        ax, ay = acc_x, acc_y
    out_t = None if out is None else torch.empty((n2, r1 - r0), dtype=torch.float64, device=dev)
    if n1 and n2 and r1 > r0:
        cot_t = cot.t().contiguous()
        with _on(dev):
            nb = _wsq(lib.sk_backward_gram_acc_tf_workspace_bytes, n2, n1, L2, L1, d, lam2, lam1,
                      kind, 0, tf)
            ws = _workspace(nb, dev)
            _lib.check(lib.sk_backward_gram_acc_cols(
                _ptr(yy), _ptr(x), n2, n1, L2, L1, d, lam2, lam1, tf, 0, n2, r0, r1, _ptr(cot_t),
                _ptr(out_t), _ptr(ay.blob), _ptr(ax.blob), _ptr(ws), ws.numel(), _stream(dev)))
    if out is not None and out_t is not None:
        out.copy_(out_t.t())
    if not own:
        return acc_x, acc_y
    gx = ax.finalize() if grad_x is None else ax.finalize(out=grad_x, accumulate=True)
    gy = ay.finalize() if grad_y is None else ay.finalize(out=grad_y, accumulate=True)
    return gx, gy


def _gram_backward(x, y, lam1, lam2, kind, sigma, cot, rows, out, grad_x, grad_y, acc_x, acc_y,
                   transform):
    """Shared body of backward_gram (out None) and value_and_grad_gram."""
    lib = _lib.load()
    tf = transform_code(transform)
    x, yy, sym, n1, n2, L1, L2, d = _gram_args(x, y)
    r0, r1 = _rows(rows, n1)
    if not sym and _transpose_cross_bwd(kind, L1, L2, lam1, lam2, d, tf):
        if grad_x is not None:
            _grad_buffer(grad_x, x, "grad_x")
        if grad_y is not None:
            _grad_buffer(grad_y, yy, "grad_y")
        return _gram_backward_t(x, yy, n1, n2, L1, L2, d, lam1, lam2, kind,
                                _cotangent(cot, (n1, n2), x), r0, r1, out, grad_x, grad_y,
                                acc_x, acc_y, transform, tf)
    cot = _cotangent(cot, (n1, n2), x)
    dev = x.device
    if acc_x is not None:
        _check_acc(acc_x, n1, L1, d, tf, x, "acc_x")
        if not sym:
            _check_acc(acc_y, n2, L2, d, tf, x, "acc_y")
        if n1 == 0 or n2 == 0 or r1 <= r0:
            return acc_x, acc_y
        with _on(dev):
            nb = _wsq(lib.sk_backward_gram_acc_tf_workspace_bytes, n1, n2, L1, L2, d, lam1, lam2, kind,
                                                             int(sym), tf)
            ws = _workspace(nb, dev)
            _lib.check(lib.sk_backward_gram_acc_tf(
                _ptr(x), None if sym else _ptr(yy), n1, n2, L1, L2, d, lam1, lam2, kind, sigma,
                tf, r0, r1, _ptr(cot), _ptr(out), _ptr(acc_x.blob),
                None if sym else _ptr(acc_y.blob), _ptr(ws), ws.numel(), _stream(dev)))
        return acc_x, acc_y
    if grad_x is None:
        grad_x = torch.zeros_like(x)
    if grad_y is None and not sym:
        grad_y = torch.zeros_like(yy)
    _grad_buffer(grad_x, x, "grad_x")
    if not sym:
        _grad_buffer(grad_y, yy, "grad_y")
    if n1 == 0 or n2 == 0 or r1 <= r0:
        return grad_x, grad_y
    with _on(dev):
        nb = _wsq(lib.sk_backward_gram_tf_workspace_bytes, n1, n2, L1, L2, d, lam1, lam2, kind,
                                                     int(sym), tf)
        ws = _workspace(nb, dev)
        _lib.check(lib.sk_backward_gram_tf(_ptr(x), None if sym else _ptr(yy), n1, n2, L1, L2, d,
                                           lam1, lam2, kind, sigma, tf, r0, r1, _ptr(cot),
                                           _ptr(out), _ptr(grad_x),
                                           _ptr(grad_y) if not sym else None, _ptr(ws),
                                           ws.numel(), _stream(dev)))
    return grad_x, grad_y


def backward_gram(x, y, lam1, lam2, kind, sigma, cot, rows=None, grad_x=None, grad_y=None,
                  acc_x=None, acc_y=None, transform=None):
    """dF/dx (and dF/dy) of F = sum cot[a, b] G[a, b] over the pairs with a in
    rows; cot is the full (n1, n2) cotangent.

    Default: grad_x (grad_y) += this call's gradient (new zero buffers if None);
    the sum inside the call is exact, so one call is bitwise reproducible.
    With acc_x (acc_y) GradAcc accumulators, the call adds into them instead and
    returns them (finalize() at the end): any tile-aligned split of the rows into
    calls then gives bitwise the same gradient."""
    return _gram_backward(x, y, lam1, lam2, kind, sigma, cot, rows, None, grad_x, grad_y, acc_x,
                          acc_y, transform)


def value_and_grad_gram(x, y, lam1, lam2, kind, sigma, cot, rows=None, out=None, grad_x=None,
                        grad_y=None, acc_x=None, acc_y=None, transform=None):
    """One fused pass: G rows [r0, r1) (as forward_gram) and dF/dx (dF/dy) of
    F = sum cot[a, b] G[a, b] (as backward_gram, including its accumulator
    mode), from the backward's own forward solve."""
    xx = _paths(x, "x")
    n1 = xx.shape[0]
    n2 = n1 if y is None else y.shape[0]
    r0, r1 = _rows(rows, n1)
    if out is None:
        out = torch.empty((r1 - r0, n2), dtype=torch.float64, device=xx.device)
    if tuple(out.shape) != (r1 - r0, n2) or out.dtype != torch.float64 or not out.is_contiguous():
        raise InvalidArgument(f"out must be a contiguous float64 ({r1 - r0}, {n2}) tensor")
    _same_device(out, xx, "out")
    g1, g2 = _gram_backward(xx, y, lam1, lam2, kind, sigma, cot, rows, out, grad_x, grad_y, acc_x,
                            acc_y, transform)
    return out, g1, g2


def f32_backward_supported(lam1: int, lam2: int, d: int, transform=None, L1=None,
                           L2=None) -> bool:
    """Shapes the FP32-arithmetic Gram backward covers (sk_backward_gram_acc_f32):
    linear, order 0, d <= 16, no transform, and (cross Grams) y no longer than
    x -- a longer y puts the y paths on the grid rows (kernel.py:137-140), which
    the DMMA Gram tiles (shared column path) do not cover."""
    return (lam1 == 0 and lam2 == 0 and 1 <= d <= 16 and transform_code(transform) == 0
            and (L1 is None or L2 is None or L2 <= L1))


def value_and_grad_gram_f32(x, y, cot, rows=None, out=None, acc_x=None, acc_y=None):
    """FP32-arithmetic fused Gram value + gradient (linear kernel, dyadic order
    0, d <= 16): the forward, recompute and adjoint recurrences in float
    (small-correction forms), p = <dx, dy>, gx, gy on the FP64 tensor cores.
    x, y: float32 or float64 points (float64 copies are made; exact for float32
    inputs).  Returns (G rows [r0, r1) as float64 of the float results, gx, gy)
    with float64 gradients (exact fixed-point sums of the float adjoints)."""
    lib = _lib.load()
    x, yy, sym, n1, n2, L1, L2, d = _gram_args(x.to(torch.float64), None if y is None else y.to(torch.float64))
    if not f32_backward_supported(0, 0, d, None, L1, L2):
        raise InvalidArgument("FP32 backward supports d <= 16 and (cross Grams) y no longer "
                              "than x")
    r0, r1 = _rows(rows, n1)
    cot = _cotangent(cot, (n1, n2), x)
    dev = x.device
    if out is None:
        out = torch.empty((r1 - r0, n2), dtype=torch.float64, device=dev)
    own = acc_x is None
    if own:
        acc_x = GradAcc(n1, L1, d, dev).init(cot, n1, n2, sym)
        if not sym:
            acc_y = GradAcc(n2, L2, d, dev).init(cot, n1, n2, False)
    else:
        _check_acc(acc_x, n1, L1, d, 0, x, "acc_x")
        if not sym:
            _check_acc(acc_y, n2, L2, d, 0, x, "acc_y")
    if n1 and n2 and r1 > r0:
        with _on(dev):
            nb = _wsq(lib.sk_backward_gram_acc_f32_workspace_bytes, n1, n2, L1, L2, d, 0, 0,
                      int(sym))
            ws = _workspace(nb, dev)
            _lib.check(lib.sk_backward_gram_acc_f32(
                _ptr(x), None if sym else _ptr(yy), n1, n2, L1, L2, d, 0, 0, r0, r1, _ptr(cot),
                _ptr(out), _ptr(acc_x.blob), None if sym else _ptr(acc_y.blob), _ptr(ws),
                ws.numel(), _stream(dev)))
    if not own:
        return out, acc_x, acc_y
    return out, acc_x.finalize(), (None if sym else acc_y.finalize())


def mirror_upper(G: torch.Tensor) -> torch.Tensor:
    """In place: lower triangle := upper triangle (kernel.py:177-179)."""
    lib = _lib.load()
    n = G.shape[0]
    with _on(G.device):
        _lib.check(lib.sk_mirror_upper(_ptr(G), n, G.stride(0), _stream(G.device)))
    return G


def dfma_peak(iters: int = 4096, reps: int = 3) -> float:
    """Measured FP64 FMA rate (FMA/s) of this device: the roofline denominator."""
    lib = _lib.load()
    import ctypes
    dev = torch.device("cuda", torch.cuda.current_device())
    scratch = torch.empty(lib.sk_dfma_probe_scratch_bytes() // 8 + 1, dtype=torch.float64,
                          device=dev)
    cnt = ctypes.c_double(0.0)
    _lib.check(lib.sk_dfma_probe(_ptr(scratch), 64, ctypes.byref(cnt), _stream()))  # warm
    best = 0.0
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.sk_dfma_probe(_ptr(scratch), iters, ctypes.byref(cnt), _stream()))
        e1.record()
        e1.synchronize()
        best = max(best, cnt.value / (e0.elapsed_time(e1) * 1e-3))
    return best
