"""Pin the C oracle (oracle/sk_oracle.c) against vectors produced by the
reference implementation itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import golden, rel_err

TOL = 1e-12  # oracle vs reference: only BLAS summation order differs in delta


def test_known_answers(oracle):
    # test_kernel.py:40-46 of the reference: zero delta -> 1, one cell delta=1 -> 2.25
    v, _ = oracle.solve_goursat(np.zeros((3, 4)), 1, 2)
    assert v == 1.0
    v, _ = oracle.solve_goursat(np.array([[1.0]]))
    assert v == 2.25
    x = np.array([[0.0], [1.0]])
    vals, gx, gy = oracle.kernel_batch_backward(x[None], x[None])
    # test_kernel_grad.py:19-26: grads [[-1.5],[1.5]]
    np.testing.assert_allclose(gx[0], [[-1.5], [1.5]], rtol=1e-15)
    np.testing.assert_allclose(gy[0], [[-1.5], [1.5]], rtol=1e-15)
    assert vals[0] == 2.25


def test_overflow_is_inf(oracle):
    v, _ = oracle.solve_goursat(np.full((40, 40), 1e300))
    assert np.isinf(v)


def test_solve_grid(oracle):
    g = golden("solve_grid")
    v, grid = oracle.solve_goursat(g["delta"], 1, 1, store_grid=True)
    assert rel_err(grid, g["grid"]) < 1e-15
    assert v == float(g["value"])
    v2, _ = oracle.solve_goursat(g["delta"], 1, 1)
    assert v2 == v  # strip march == grid march bitwise (test_kernel.py:65-71)


def test_c1(oracle):
    g = golden("c1_kernel_batch")
    got = oracle.kernel_batch(g["x"], g["y"])
    assert rel_err(got, g["out"]) < TOL


def test_batch_mixed(oracle):
    g = golden("batch_mixed")
    for l1, l2 in ((1, 2), (2, 1), (3, 0), (0, 3)):
        got = oracle.kernel_batch(g["x"], g["y"], l1, l2)
        assert rel_err(got, g[f"out_{l1}{l2}"]) < TOL


def test_gram(oracle):
    g = golden("gram_small")
    got = oracle.kernel_gram(g["xs"], None, 1, 1)
    assert rel_err(got, g["g_sym_11"]) < TOL
    np.testing.assert_array_equal(got, got.T)
    assert rel_err(oracle.kernel_gram(g["xc"], g["yc"], 0, 1), g["g_cross_01"]) < TOL
    assert rel_err(oracle.kernel_gram(g["xc"], g["yc"], 2, 0), g["g_cross_20"]) < TOL


def test_batch_backward(oracle):
    g = golden("batch_backward_small")
    for l1, l2 in ((0, 0), (1, 2), (2, 1), (0, 3)):
        v, gx, gy = oracle.kernel_batch_backward(g["x"], g["y"], l1, l2, g["cot"])
        assert rel_err(v, g[f"v_{l1}{l2}"]) < TOL
        assert rel_err(gx, g[f"gx_{l1}{l2}"]) < 1e-11
        assert rel_err(gy, g[f"gy_{l1}{l2}"]) < 1e-11


def test_c2_linear_pairs(oracle):
    g = golden("c2_linear_pairs")
    v, gx, gy = oracle.kernel_batch_backward(g["x"], g["y"], 2, 2)
    assert rel_err(v, g["v"]) < TOL
    assert rel_err(gx, g["gx"]) < 1e-11
    assert rel_err(gy, g["gy"]) < 1e-11


def test_rbf_solver_part_pinned(oracle):
    g = golden("rbf_pinned_solver")
    sig = float(g["sigma"])
    delta = oracle.increment_gram(g["x"], g["y"], ("rbf", sig))
    assert rel_err(delta, g["delta"]) < 1e-13
    v = oracle.kernel_batch(g["x"][None], g["y"][None], 2, 2, ("rbf", sig))
    assert rel_err(v, [float(g["value"])]) < TOL


def test_rbf_gradient_matches_fd(oracle):
    """RBF adjoint has no reference: check it against central differences."""
    rng = np.random.default_rng(11)
    x = rng.standard_normal((1, 5, 2)) * 0.5
    y = rng.standard_normal((1, 4, 2)) * 0.5
    sk = ("rbf", 0.7)
    _, gx, gy = oracle.kernel_batch_backward(x, y, 1, 1, static_kernel=sk)
    h = 1e-6
    for arr, g in ((x, gx), (y, gy)):
        fd = np.zeros_like(arr)
        for idx in np.ndindex(arr.shape):
            ap = arr.copy(); ap[idx] += h
            am = arr.copy(); am[idx] -= h
            xa, ya = (ap, y) if arr is x else (x, ap)
            xb, yb = (am, y) if arr is x else (x, am)
            fd[idx] = (oracle.kernel_batch(xa, ya, 1, 1, sk)[0] -
                       oracle.kernel_batch(xb, yb, 1, 1, sk)[0]) / (2 * h)
        assert rel_err(g, fd, floor=1e-9) < 1e-6


def test_c3_subgram(oracle):
    g = golden("c3_subgram")
    assert rel_err(oracle.kernel_gram(g["x"]), g["g"]) < TOL


def test_c4_long_pair(oracle):
    g = golden("c4_long_pair")
    assert rel_err(oracle.kernel_batch(g["x"], g["y"], 1, 1), g["out"]) < TOL


def test_c5_pair_grad(oracle):
    g = golden("c5_pair_grad")
    v, gx, gy = oracle.kernel_batch_backward(g["x"][None], g["y"][None])
    assert rel_err(v, [float(g["value"])]) < TOL
    assert rel_err(gx[0], g["gx"]) < 1e-11
    assert rel_err(gy[0], g["gy"]) < 1e-11


def test_gram_backward_composition(oracle):
    """Gram backward == sum over pairs of kernel_batch_backward (cot-weighted)."""
    rng = np.random.default_rng(12)
    X = rng.standard_normal((4, 6, 2)) * 0.4
    C = rng.standard_normal((4, 4))
    # symmetric Gram mirrors the upper triangle (kernel.py:177-179); with
    # lam1 == lam2 that equals the full square of pairwise kernels
    gx = oracle.gram_backward(X, None, C, 1, 1)
    want = np.zeros_like(X)
    for a in range(4):
        for b in range(4):
            _, ga, gb = oracle.kernel_batch_backward(X[a:a + 1], X[b:b + 1], 1, 1,
                                                     np.array([C[a, b]]))
            want[a] += ga[0]
            want[b] += gb[0]
    assert rel_err(gx, want) < 1e-12
    Y = rng.standard_normal((3, 5, 2)) * 0.4
    C2 = rng.standard_normal((4, 3))
    gx2, gy2 = oracle.gram_backward(X, Y, C2, 0, 1)
    wx, wy = np.zeros_like(X), np.zeros_like(Y)
    for a in range(4):
        for b in range(3):
            _, ga, gb = oracle.kernel_batch_backward(X[a:a + 1], Y[b:b + 1], 0, 1,
                                                     np.array([C2[a, b]]))
            wx[a] += ga[0]
            wy[b] += gb[0]
    assert rel_err(gx2, wx) < 1e-12 and rel_err(gy2, wy) < 1e-12


def test_signature_oracle_pinned_to_reference(oracle):
    """The C restatement of the reference's signature kernels against vectors
    the reference itself produced (tests/golden/make_golden_signature.py):
    forward and backward bitwise (same operations in the same order)."""
    g = golden("signature")
    kinds = {0: None, 1: "time_augment", 2: "lead_lag"}
    for i in range(int(g["n"])):
        depth, tf, custom = (int(v) for v in g[f"s{i}_meta"])
        times = g[f"s{i}_times"] if custom else None
        x = g[f"s{i}_x"]
        sig = oracle.signature(x, depth, kinds[tf], times)
        np.testing.assert_array_equal(sig, g[f"s{i}_sig"])
        grad = oracle.signature_backward(x, depth, g[f"s{i}_cot"], kinds[tf], times)
        np.testing.assert_array_equal(grad, g[f"s{i}_grad"])


def _rbf_sigkernel_torch(x, y, lam1, lam2, sigma):
    """Independent differentiable restatement (torch fp64, autograd) of the RBF
    signature kernel: node kernel K, coarse second difference, the reference's
    cell recurrence (_kernels.py:286-290, dyadic refinement as in
    goursat_strip, _kernels.py:293-338) -- reverse-mode of the same
    discretisation, no hand-written adjoint."""
    import torch
    K = torch.exp(-((x[:, None, :] - y[None, :, :]) ** 2).sum(-1) / (2.0 * sigma * sigma))
    delta = (K[1:, 1:] - K[1:, :-1]) - (K[:-1, 1:] - K[:-1, :-1])
    scale = 2.0 ** -(lam1 + lam2)
    M1, M2 = (x.shape[0] - 1) << lam1, (y.shape[0] - 1) << lam2
    one = torch.ones((), dtype=torch.float64)
    prev = [one] * (M2 + 1)
    for s in range(1, M1 + 1):
        cur = [one]
        for t in range(1, M2 + 1):
            p = delta[(s - 1) >> lam1, (t - 1) >> lam2] * scale
            a = 1.0 + p * 0.5 + p * p * (1.0 / 12.0)
            b = 1.0 - p * p * (1.0 / 12.0)
            cur.append((prev[t] + cur[t - 1]) * a - prev[t - 1] * b)
        prev = cur
    return prev[M2]


@pytest.mark.parametrize("L1,L2,d,lam1,lam2,sigma", [(5, 4, 2, 1, 1, 0.7), (4, 6, 3, 2, 0, 1.3),
                                                      (6, 5, 1, 0, 2, 0.5)])
def test_rbf_adjoint_pinned_by_autograd(oracle, L1, L2, d, lam1, lam2, sigma):
    """The RBF kappa adjoint (no reference counterpart) against torch autograd of
    an independent restatement: values and both gradients to 1e-12 -- pins the
    oracle the GPU RBF backward tests compare with."""
    import torch
    rng = np.random.default_rng(L1 * 10 + L2 + d)
    x = rng.standard_normal((L1, d)) * 0.5
    y = rng.standard_normal((L2, d)) * 0.5
    xt = torch.tensor(x, requires_grad=True)
    yt = torch.tensor(y, requires_grad=True)
    k = _rbf_sigkernel_torch(xt, yt, lam1, lam2, sigma)
    k.backward()
    v, gx, gy = oracle.kernel_batch_backward(x[None], y[None], lam1, lam2,
                                             static_kernel=("rbf", sigma))
    assert abs(v[0] - k.item()) <= 1e-12 * abs(k.item())
    assert rel_err(gx[0], xt.grad.numpy()) < 1e-12
    assert rel_err(gy[0], yt.grad.numpy()) < 1e-12
