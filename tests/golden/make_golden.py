"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (it imports sigcore from /root/reference,
which does not exist on the GPU box):

    cd /tmp && NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_golden.py

The reference tree is read-only; numba's cache goes to /tmp.  Outputs are
small .npz files next to this script; tests/test_oracle.py pins the C
oracle against them and the GPU parity tests use them as fixed vectors.

Inputs follow the reference bench generator (sigcore/bench.py:53-56) and the
test helpers (tests/conftest.py:24-27).
"""

import os
import sys

import numpy as np

import sigcore as sc  # the reference, via PYTHONPATH

OUT = os.path.dirname(os.path.abspath(__file__))


def make_paths(rng, batch, length, dim):
    """sigcore/bench.py:53-56 (fp64 branch)."""
    steps = rng.standard_normal((batch, length, dim)) / np.sqrt(max(length, 1))
    return np.cumsum(steps, axis=1, dtype=np.float64)


def random_paths(rng, b, length, d, scale=1.0):
    """tests/conftest.py:24-27."""
    steps = rng.standard_normal((b, length, d)) / np.sqrt(max(length - 1, 1))
    return np.cumsum(steps, axis=1) * scale


def rbf_delta(x, y, sigma):
    """RBF second difference; no reference exists."""
    d2 = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    K = np.exp(-d2 / (2.0 * sigma * sigma))
    return (K[1:, 1:] - K[1:, :-1]) - (K[:-1, 1:] - K[:-1, :-1])


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def main():
    # C1: the reference's own CPU-runnable config (BASELINE.json configs[0])
    rng = np.random.default_rng(0)
    x = make_paths(rng, 32, 64, 4)
    y = make_paths(rng, 32, 64, 4)
    save("c1_kernel_batch", x=x, y=y, lam=np.array([0, 0]),
         out=sc.kernel_batch(x, y, sc.KernelConfig(0, 0)))

    # mixed lengths and dyadic orders (both swap branches of kernel.py:137-140)
    rng = np.random.default_rng(1)
    x = random_paths(rng, 4, 9, 3)
    y = random_paths(rng, 4, 13, 3)
    save("batch_mixed", x=x, y=y,
         out_12=sc.kernel_batch(x, y, sc.KernelConfig(1, 2)),
         out_21=sc.kernel_batch(x, y, sc.KernelConfig(2, 1)),
         out_30=sc.kernel_batch(x, y, sc.KernelConfig(3, 0)),
         out_03=sc.kernel_batch(x, y, sc.KernelConfig(0, 3)))

    # Gram: symmetric and cross
    rng = np.random.default_rng(2)
    xs = random_paths(rng, 6, 10, 2)
    xc = random_paths(rng, 3, 7, 2)
    yc = random_paths(rng, 5, 11, 2)
    save("gram_small", xs=xs, xc=xc, yc=yc,
         g_sym_11=sc.kernel_gram(xs, cfg=sc.KernelConfig(1, 1)),
         g_cross_01=sc.kernel_gram(xc, yc, sc.KernelConfig(0, 1)),
         g_cross_20=sc.kernel_gram(xc, yc, sc.KernelConfig(2, 0)))

    # batch backward (kernel_grad.py:64-98) with a random cotangent
    rng = np.random.default_rng(3)
    x = rng.standard_normal((3, 5, 2)) * 0.5
    y = rng.standard_normal((3, 7, 2)) * 0.5
    cot = rng.standard_normal(3)
    arrs = {"x": x, "y": y, "cot": cot}
    for l1, l2 in ((0, 0), (1, 2), (2, 1), (0, 3)):
        v, gx, gy = sc.kernel_batch_backward(x, y, sc.KernelConfig(l1, l2), cot)
        arrs[f"v_{l1}{l2}"], arrs[f"gx_{l1}{l2}"], arrs[f"gy_{l1}{l2}"] = v, gx, gy
    save("batch_backward_small", **arrs)

    # full grid + adjoint for a small delta (goursat_grid / goursat_backward)
    rng = np.random.default_rng(4)
    delta = rng.standard_normal((3, 2)) * 0.4
    cfg = sc.KernelConfig(1, 1, store_grid=True)
    res = sc.solve_goursat(delta, cfg)
    save("solve_grid", delta=delta, value=np.array(res.value), grid=res.grid)

    # C2-shaped pairs (L=256, d=8, lambda=2), linear kernel, fwd+bwd on 2 pairs
    rng = np.random.default_rng(5)
    x = make_paths(rng, 2, 256, 8)
    y = make_paths(rng, 2, 256, 8)
    v, gx, gy = sc.kernel_batch_backward(x, y, sc.KernelConfig(2, 2))
    save("c2_linear_pairs", x=x, y=y, v=v, gx=gx, gy=gy)

    # RBF: our delta restatement fed to the REFERENCE solver + adjoint, so the
    # solver part of the RBF path is pinned (SURVEY.md 8c "parity unpinned")
    rng = np.random.default_rng(6)
    x = make_paths(rng, 1, 24, 3)[0]
    y = make_paths(rng, 1, 17, 3)[0]
    sigma = 1.0
    drbf = rbf_delta(x, y, sigma)
    cfgr = sc.KernelConfig(2, 2, store_grid=True)
    res = sc.solve_goursat(drbf, cfgr)
    from sigcore import _kernels  # reference adjoint on an arbitrary delta
    d1 = np.empty_like(res.grid)
    d2 = np.zeros_like(drbf)
    _kernels.goursat_backward(drbf, 2, 2, cfgr.scale, res.grid, 1.0, d1, d2)
    save("rbf_pinned_solver", x=x, y=y, sigma=np.array(sigma), delta=drbf,
         value=np.array(res.value), d2=d2)

    # C3-shaped symmetric sub-Gram (L=512, d=16)
    rng = np.random.default_rng(7)
    X = make_paths(rng, 4, 512, 16)
    save("c3_subgram", x=X, g=sc.kernel_gram(X, cfg=sc.KernelConfig(0, 0)))

    # C4-shaped long pair (d=4, lambda=1), shortened to L=4096 to keep the fixture small
    rng = np.random.default_rng(8)
    x = make_paths(rng, 1, 4096, 4)
    y = make_paths(rng, 1, 4096, 4)
    save("c4_long_pair", x=x, y=y, out=sc.kernel_batch(x, y, sc.KernelConfig(1, 1)))

    # C5-shaped pair gradient (L=1024, d=8) via kernel_backward
    rng = np.random.default_rng(9)
    x = make_paths(rng, 1, 1024, 8)[0]
    y = make_paths(rng, 1, 1024, 8)[0]
    cfg = sc.KernelConfig(0, 0, store_grid=True)
    res = sc.solve_goursat(sc.increment_gram(x, y), cfg)
    gx, gy = sc.kernel_backward(x, y, cfg, res, 1.0)
    save("c5_pair_grad", x=x, y=y, value=np.array(res.value), gx=gx, gy=gy)

    # dyadic-convergence oracle: depth-12 truncated signature inner products of
    # low-variation paths (reference tests/conftest.py:40-52, 93-100)
    rng = np.random.default_rng(4)
    xs, ys, oracles = [], [], []
    for _ in range(5):
        steps = rng.uniform(0.2, 1.0, size=(4, 2))
        steps *= 1.0 / steps.sum()
        x = np.zeros((5, 2)); x[1:] = np.cumsum(steps, axis=0)
        steps = rng.uniform(0.2, 1.0, size=(5, 2))
        steps *= 1.0 / steps.sum()
        y = np.zeros((6, 2)); y[1:] = np.cumsum(steps, axis=0)
        shape = sc.tensor_shape(2, 12)
        opts = sc.SigOptions(12)
        sx = sc.TruncatedSig(shape, sc.signature(x, opts))
        sy = sc.TruncatedSig(shape, sc.signature(y, opts))
        xs.append(x); ys.append(y); oracles.append(sc.dot(sx, sy))
    save("dyadic_convergence", x=np.array(xs), y=np.array(ys), oracle=np.array(oracles))

    # SGT1 files written by the reference's io.write_array (io.py:27-39)
    rng = np.random.default_rng(12)
    a3 = rng.standard_normal((2, 5, 3))
    a2 = rng.standard_normal((4, 2)).astype(np.float32)
    a1 = np.arange(7, dtype=np.int64)  # integers are widened to float64
    sc.write_array(a3, os.path.join(OUT, "ref_f64_3d.sgt"))
    sc.write_array(a2, os.path.join(OUT, "ref_f32_2d.sgt"))
    sc.write_array(a1, os.path.join(OUT, "ref_int_1d.sgt"))
    save("sgt_contents", a3=a3, a2=a2, a1=a1)

    # path transforms (transforms.py:37-66) and their adjoints (69-90)
    rng = np.random.default_rng(13)
    xt = rng.standard_normal((3, 6, 2))
    gt_ta = rng.standard_normal((3, 6, 3))
    gt_ll = rng.standard_normal((3, 11, 4))
    save("transforms", x=xt, time_augment=sc.transform(xt, "time_augment"),
         lead_lag=sc.transform(xt, "lead_lag"), g_ta=gt_ta, g_ll=gt_ll,
         adj_ta=sc.transform_adjoint(gt_ta, "time_augment"),
         adj_ll=sc.transform_adjoint(gt_ll, "lead_lag"))

    print("reference:", sc.__file__, "numba", __import__("numba").__version__,
          "numpy", np.__version__, file=sys.stderr)


if __name__ == "__main__":
    main()
