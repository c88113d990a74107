"""ctypes wrapper for the CPU oracle (oracle/sk_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker and CPU baseline.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  The product package
(paper_2509_10613_b200) never imports it.

Function names mirror the reference API they restate
(/root/reference/pkg/src/sigcore/kernel.py and kernel_grad.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libsk_oracle.so")

LINEAR = 0
RBF = 1

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc -fopenmp)."""
    if force or not os.path.exists(_SO) or (
            os.path.getmtime(_SO) < os.path.getmtime(os.path.join(_HERE, "sk_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        i64, ci, cd = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.sko_kernel_batch.argtypes = [dp, dp, i64, i64, i64, i64, ci, ci, ci, cd, dp, ci]
        L.sko_kernel_gram.argtypes = [dp, dp, i64, i64, i64, i64, i64, ci, ci, ci, cd, ci,
                                      i64, i64, dp, ci]
        L.sko_kernel_batch_backward.argtypes = [dp, dp, i64, i64, i64, i64, ci, ci, ci, cd, dp,
                                                dp, dp, dp, ci]
        L.sko_gram_backward.argtypes = [dp, dp, i64, i64, i64, i64, i64, ci, ci, ci, cd, ci,
                                        i64, i64, dp, dp, dp, ci]
        L.sko_solve_goursat.argtypes = [dp, i64, i64, ci, ci, dp]
        L.sko_solve_goursat.restype = cd
        L.sko_increment_gram.argtypes = [dp, dp, i64, i64, i64, dp]
        L.sko_rbf_increment_gram.argtypes = [dp, dp, i64, i64, i64, cd, dp]
        L.sko_max_threads.restype = ci
        L.sko_signature.argtypes = [dp, i64, i64, i64, ci, dp, ci]
        L.sko_signature_backward.argtypes = [dp, i64, i64, i64, ci, dp, dp, ci]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _kind(static_kernel):
    if static_kernel in (None, "linear", LINEAR):
        return LINEAR, 1.0
    if isinstance(static_kernel, tuple) and static_kernel[0] == "rbf":
        return RBF, float(static_kernel[1])
    raise ValueError(f"unknown static kernel {static_kernel!r}")


def max_threads() -> int:
    return int(lib().sko_max_threads())


def increment_gram(x, y, static_kernel=None):
    """kernel.py:60-77 for one (L,d) pair; RBF -> second difference of K."""
    x, y = _f64(x), _f64(y)
    kind, sigma = _kind(static_kernel)
    out = np.empty((x.shape[0] - 1, y.shape[0] - 1))
    if kind == RBF:
        lib().sko_rbf_increment_gram(_p(x), _p(y), x.shape[0], y.shape[0], x.shape[1], sigma,
                                     _p(out))
    else:
        lib().sko_increment_gram(_p(x), _p(y), x.shape[0], y.shape[0], x.shape[1], _p(out))
    return out


def solve_goursat(delta, lam1=0, lam2=0, store_grid=False):
    """kernel.py:94-122: value (and the full grid when store_grid)."""
    delta = _f64(delta)
    r1, r2 = delta.shape
    grid = np.empty(((r1 << lam1) + 1, (r2 << lam2) + 1)) if store_grid else None
    v = lib().sko_solve_goursat(_p(delta), r1, r2, lam1, lam2,
                                _p(grid) if grid is not None else None)
    return float(v), grid


def kernel_batch(x, y, lam1=0, lam2=0, static_kernel=None, threads=0):
    """kernel.py:125-148."""
    x, y = _f64(x), _f64(y)
    B, L1, d = x.shape
    L2 = y.shape[1]
    kind, sigma = _kind(static_kernel)
    out = np.empty(B)
    rc = lib().sko_kernel_batch(_p(x), _p(y), B, L1, L2, d, lam1, lam2, kind, sigma, _p(out),
                                threads)
    if rc:
        raise MemoryError("oracle allocation failed")
    return out


def kernel_gram(x, y=None, lam1=0, lam2=0, static_kernel=None, threads=0, rows=None):
    """kernel.py:151-180 (symmetric when y is None)."""
    symmetric = y is None
    x = _f64(x)
    y = x if symmetric else _f64(y)
    n1, L1, d = x.shape
    n2, L2 = y.shape[0], y.shape[1]
    r0, r1 = (0, n1) if rows is None else rows
    kind, sigma = _kind(static_kernel)
    out = np.zeros((r1 - r0, n2))
    rc = lib().sko_kernel_gram(_p(x), _p(y), n1, n2, L1, L2, d, lam1, lam2, kind, sigma,
                               int(symmetric), r0, r1, _p(out), threads)
    if rc:
        raise MemoryError("oracle allocation failed")
    return out


def kernel_batch_backward(x, y, lam1=0, lam2=0, cot=None, static_kernel=None, threads=0):
    """kernel_grad.py:64-98: (values, grad_x, grad_y)."""
    x, y = _f64(x), _f64(y)
    B, L1, d = x.shape
    L2 = y.shape[1]
    kind, sigma = _kind(static_kernel)
    cot = np.ones(B) if cot is None else _f64(cot)
    vals = np.empty(B)
    gx = np.empty_like(x)
    gy = np.empty_like(y)
    rc = lib().sko_kernel_batch_backward(_p(x), _p(y), B, L1, L2, d, lam1, lam2, kind, sigma,
                                         _p(cot), _p(vals), _p(gx), _p(gy), threads)
    if rc:
        raise MemoryError("oracle allocation failed")
    return vals, gx, gy


def gram_backward(x, y=None, cot=None, lam1=0, lam2=0, static_kernel=None, threads=0):
    """Gram backward composed from kernel_backward per pair.

    Returns grad_x (and grad_y when y is given)."""
    symmetric = y is None
    x = _f64(x)
    y = x if symmetric else _f64(y)
    n1, L1, d = x.shape
    n2, L2 = y.shape[0], y.shape[1]
    kind, sigma = _kind(static_kernel)
    cot = np.ones((n1, n2)) if cot is None else _f64(cot)
    gx = np.zeros_like(x)
    gy = np.zeros_like(y) if not symmetric else np.zeros((1,))
    rc = lib().sko_gram_backward(_p(x), _p(y), n1, n2, L1, L2, d, lam1, lam2, kind, sigma,
                                 int(symmetric), 0, n1, _p(cot), _p(gx), _p(gy), threads)
    if rc:
        raise MemoryError("oracle allocation failed")
    return gx if symmetric else (gx, gy)


# ------------------------------------------------------------ truncated signatures
def _linspace_times(L):
    """transforms.py:30-34 default_times (numpy.linspace)."""
    return np.zeros(1) if L == 1 else np.linspace(0.0, 1.0, L)


def fused_increments(x, kind=None, times=None):
    """transforms.py:91-120: increments of the transformed path, (B, M', d')."""
    x = _f64(x)
    B, L, d = x.shape
    dx = np.diff(x, axis=1)
    if kind is None:
        return np.ascontiguousarray(dx)
    if kind == "time_augment":
        t = _linspace_times(L) if times is None else np.asarray(times, dtype=np.float64)
        out = np.empty((B, L - 1, d + 1))
        out[:, :, :d] = dx
        out[:, :, d] = np.diff(t)
        return out
    out = np.zeros((B, 2 * L - 2, 2 * d))
    out[:, 0::2, :d] = dx
    out[:, 1::2, d:] = dx
    return out


def transform_adjoint(g, kind):
    """transforms.py:69-90."""
    if kind is None:
        return g
    if kind == "time_augment":
        return g[:, :, :-1].copy()
    d = g.shape[2] // 2
    lead, lag = g[:, :, :d], g[:, :, d:]
    out = lead[:, 0::2] + lag[:, 0::2]
    out[:, :-1] += lag[:, 1::2]
    out[:, 1:] += lead[:, 1::2]
    return out


def signature_length(d, depth):
    return sum(d ** k for k in range(1, depth + 1))


def signature(x, depth, kind=None, times=None, threads=0):
    """signature.py:104-121 (Horner; the C restatement of _kernels.py:115-172)."""
    inc = fused_increments(x, kind, times)
    B, M, d = inc.shape
    out = np.empty((B, signature_length(d, depth)))
    if lib().sko_signature(_p(inc), B, M, d, depth, _p(out), threads):
        raise MemoryError("oracle allocation failed")
    return out


def signature_backward(x, depth, cot, kind=None, times=None, threads=0):
    """signature_grad.py:20-53: the C restatement of sig_backward_path
    (_kernels.py:182-266), then the telescoping and the transform adjoint."""
    x = _f64(x)
    inc = fused_increments(x, kind, times)
    B, M, d = inc.shape
    cot = _f64(cot).reshape(B, -1)
    g = np.empty((B, M, d))
    if lib().sko_signature_backward(_p(inc), B, M, d, depth, _p(cot), _p(g), threads):
        raise MemoryError("oracle allocation failed")
    grad_eff = np.zeros((B, M + 1, d))
    grad_eff[:, :-1] -= g
    grad_eff[:, 1:] += g
    return transform_adjoint(grad_eff, kind)
