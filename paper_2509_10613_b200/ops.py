"""Tensor-level calls into libsigkernel (device memory, current torch stream).

These are the thin shims the autograd Functions (api.py) and the numpy facade
(sigcore_compat.py) sit on.  Inputs must be CUDA float64 tensors; outputs and
workspaces are torch allocations handed to the C ABI as borrowed pointers.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import InvalidArgument


def _ptr(t):
    return t.data_ptr() if t is not None else None


def _stream(device=None):
    return torch.cuda.current_stream(device).cuda_stream


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


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _paths(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        raise InvalidArgument(f"{name} must be a torch tensor")
    if t.dim() != 3:
        raise InvalidArgument(f"{name} must be (B, L, d), got shape {tuple(t.shape)}")
    if t.shape[1] < 2:
        raise InvalidArgument(f"{name} needs at least 2 points per path")
    if not t.is_cuda:
        raise InvalidArgument(f"{name} must live on a CUDA device")
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


def forward_batch(x, y, lam1: int, lam2: int, kind: int, sigma: float) -> torch.Tensor:
    lib = _lib.load()
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
    with torch.cuda.device(x.device):
        nb = lib.sk_forward_batch_workspace_bytes(B, L1, L2, d, lam1, lam2, kind)
        ws = _workspace(nb, x.device)
        _lib.check(lib.sk_forward_batch(_ptr(x), _ptr(y), B, L1, L2, d, lam1, lam2, kind, sigma,
                                        _ptr(out), _ptr(ws), ws.numel(), _stream(x.device)))
    return out


def forward_gram(x, y, lam1: int, lam2: int, kind: int, sigma: float,
                 rows: tuple[int, int] | None = None, out: torch.Tensor | None = None):
    """G[a - r0, b] = k(x_a, y_b) for a in rows; y None -> symmetric (y is x)."""
    lib = _lib.load()
    x = _paths(x, "x")
    sym = y is None
    yy = x if sym else _paths(y, "y")
    n1, L1, d = x.shape
    n2, L2 = yy.shape[0], yy.shape[1]
    if yy.shape[2] != d:
        raise InvalidArgument(f"path dimensions differ: {d} vs {yy.shape[2]}")
    _same_device(yy, x, "y")
    r0, r1 = (0, n1) if rows is None else (int(rows[0]), int(rows[1]))
    if out is None:
        out = torch.empty((r1 - r0, n2), dtype=torch.float64, device=x.device)
    if n1 == 0 or n2 == 0 or r1 <= r0:
        return out
    with torch.cuda.device(x.device):
        nb = lib.sk_forward_gram_workspace_bytes(n1, n2, L1, L2, d, lam1, lam2, kind, int(sym))
        ws = _workspace(nb, x.device)
        _lib.check(lib.sk_forward_gram(_ptr(x), None if sym else _ptr(yy), n1, n2, L1, L2, d,
                                       lam1, lam2, kind, sigma, r0, r1, _ptr(out), _ptr(ws),
                                       ws.numel(), _stream(x.device)))
    return out


def solve_delta(delta: torch.Tensor, lam1: int, lam2: int) -> torch.Tensor:
    """Kernel values for given increment matrices delta (B, r1, r2)."""
    lib = _lib.load()
    delta = delta.to(torch.float64).contiguous()
    B, r1, r2 = delta.shape
    out = torch.empty(B, dtype=torch.float64, device=delta.device)
    with torch.cuda.device(delta.device):
        nb = lib.sk_solve_delta_workspace_bytes(B, r1, r2, lam1, lam2)
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
    with torch.cuda.device(delta.device):
        _lib.check(lib.sk_solve_delta_grid(_ptr(delta), r1, r2, lam1, lam2, _ptr(grid),
                                           _stream(delta.device)))
    return grid


def backward_batch(x, y, lam1, lam2, kind, sigma, cot, want_values=False):
    """(values or None, grad_x, grad_y) of sum_b cot[b] k(x_b, y_b)."""
    lib = _lib.load()
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
    with torch.cuda.device(x.device):
        nb = lib.sk_backward_batch_workspace_bytes(B, L1, L2, d, lam1, lam2, kind)
        ws = _workspace(nb, x.device)
        _lib.check(lib.sk_backward_batch(_ptr(x), _ptr(y), B, L1, L2, d, lam1, lam2, kind, sigma,
                                         _ptr(cot), _ptr(vals), _ptr(gx), _ptr(gy), _ptr(ws),
                                         ws.numel(), _stream(x.device)))
    return vals, gx, gy


def backward_gram(x, y, lam1, lam2, kind, sigma, cot, rows=None, grad_x=None, grad_y=None):
    """Accumulate dF/dx (and dF/dy) of F = sum cot[a, b] G[a, b] into grad buffers.

    cot is the full (n1, n2) cotangent; rows restricts the solved X rows."""
    lib = _lib.load()
    x = _paths(x, "x")
    sym = y is None
    yy = x if sym else _paths(y, "y")
    n1, L1, d = x.shape
    n2, L2 = yy.shape[0], yy.shape[1]
    if yy.shape[2] != d:
        raise InvalidArgument(f"path dimensions differ: {d} vs {yy.shape[2]}")
    _same_device(yy, x, "y")
    r0, r1 = (0, n1) if rows is None else (int(rows[0]), int(rows[1]))
    cot = _cotangent(cot, (n1, n2), x)
    if grad_x is None:
        grad_x = torch.zeros_like(x)
    if grad_y is None and not sym:
        grad_y = torch.zeros_like(yy)
    _grad_buffer(grad_x, x, "grad_x")
    if not sym:
        _grad_buffer(grad_y, yy, "grad_y")
    if n1 == 0 or n2 == 0 or r1 <= r0:
        return grad_x, grad_y
    with torch.cuda.device(x.device):
        nb = lib.sk_backward_gram_workspace_bytes(n1, n2, L1, L2, d, lam1, lam2, kind, int(sym))
        ws = _workspace(nb, x.device)
        _lib.check(lib.sk_backward_gram(_ptr(x), None if sym else _ptr(yy), n1, n2, L1, L2, d,
                                        lam1, lam2, kind, sigma, r0, r1, _ptr(cot), _ptr(grad_x),
                                        _ptr(grad_y) if not sym else None, _ptr(ws), ws.numel(),
                                        _stream(x.device)))
    return grad_x, grad_y


def value_and_grad_gram(x, y, lam1, lam2, kind, sigma, cot, rows=None, out=None, grad_x=None,
                        grad_y=None):
    """One fused pass: G rows [r0, r1) (as forward_gram) and dF/dx (dF/dy) of
    F = sum cot[a, b] G[a, b] (accumulated as backward_gram), from the
    backward's own forward solve (sk_value_and_grad_gram)."""
    lib = _lib.load()
    x = _paths(x, "x")
    sym = y is None
    yy = x if sym else _paths(y, "y")
    n1, L1, d = x.shape
    n2, L2 = yy.shape[0], yy.shape[1]
    if yy.shape[2] != d:
        raise InvalidArgument(f"path dimensions differ: {d} vs {yy.shape[2]}")
    _same_device(yy, x, "y")
    r0, r1 = (0, n1) if rows is None else (int(rows[0]), int(rows[1]))
    cot = _cotangent(cot, (n1, n2), x)
    if out is None:
        out = torch.empty((r1 - r0, n2), dtype=torch.float64, device=x.device)
    if grad_x is None:
        grad_x = torch.zeros_like(x)
    if grad_y is None and not sym:
        grad_y = torch.zeros_like(yy)
    _grad_buffer(grad_x, x, "grad_x")
    if not sym:
        _grad_buffer(grad_y, yy, "grad_y")
    if n1 == 0 or n2 == 0 or r1 <= r0:
        return out, grad_x, grad_y
    with torch.cuda.device(x.device):
        nb = lib.sk_backward_gram_workspace_bytes(n1, n2, L1, L2, d, lam1, lam2, kind, int(sym))
        ws = _workspace(nb, x.device)
        _lib.check(lib.sk_value_and_grad_gram(_ptr(x), None if sym else _ptr(yy), n1, n2, L1, L2,
                                              d, lam1, lam2, kind, sigma, r0, r1, _ptr(cot),
                                              _ptr(out), _ptr(grad_x),
                                              _ptr(grad_y) if not sym else None, _ptr(ws),
                                              ws.numel(), _stream(x.device)))
    return out, grad_x, grad_y


def mirror_upper(G: torch.Tensor) -> torch.Tensor:
    """In place: lower triangle := upper triangle (kernel.py:177-179)."""
    lib = _lib.load()
    n = G.shape[0]
    with torch.cuda.device(G.device):
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
