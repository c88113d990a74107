"""GPU parity of the forward wavefront kernels against the reference-pinned
golden vectors and the C oracle (fp64 tolerance 1e-10)."""

import numpy as np
import pytest
import torch

from conftest import golden, make_paths, random_paths, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def sk():
    import paper_2509_10613_b200 as sk
    from paper_2509_10613_b200 import ops
    return sk, ops


def cu(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")


def test_known_answers(sk):
    _, ops = sk
    assert ops.solve_delta(cu([[[1.0]]]), 0, 0).item() == 2.25
    assert ops.solve_delta(cu(np.zeros((1, 3, 4))), 1, 2).item() == 1.0
    s, _ = sk
    x = cu([[0.0], [1.0]])
    assert s.sig_kernel(x, x).item() == 2.25


def test_c1_golden(sk):
    s, _ = sk
    g = golden("c1_kernel_batch")
    got = s.sig_kernel(cu(g["x"]), cu(g["y"])).cpu().numpy()
    assert rel_err(got, g["out"]) < TOL


def test_batch_mixed_golden(sk):
    s, _ = sk
    g = golden("batch_mixed")
    for l1, l2 in ((1, 2), (2, 1), (3, 0), (0, 3)):
        got = s.sig_kernel(cu(g["x"]), cu(g["y"]), (l1, l2)).cpu().numpy()
        assert rel_err(got, g[f"out_{l1}{l2}"]) < TOL, (l1, l2)


def test_swap_symmetry_bitwise(sk):
    s, _ = sk
    rng = np.random.default_rng(6)
    x = cu(random_paths(rng, 4, 6, 3))
    y = cu(random_paths(rng, 4, 9, 3))
    k1 = s.sig_kernel(x, y, (1, 2)).cpu().numpy()
    k2 = s.sig_kernel(y, x, (2, 1)).cpu().numpy()
    np.testing.assert_array_equal(k1, k2)


def test_gram_golden(sk):
    s, _ = sk
    g = golden("gram_small")
    G = s.sig_kernel_gram(cu(g["xs"]), dyadic_order=1).cpu().numpy()
    assert rel_err(G, g["g_sym_11"]) < TOL
    np.testing.assert_array_equal(G, G.T)
    assert rel_err(s.sig_kernel_gram(cu(g["xc"]), cu(g["yc"]), (0, 1)).cpu().numpy(),
                   g["g_cross_01"]) < TOL
    assert rel_err(s.sig_kernel_gram(cu(g["xc"]), cu(g["yc"]), (2, 0)).cpu().numpy(),
                   g["g_cross_20"]) < TOL


def test_gram_equals_batch_bitwise(sk):
    s, _ = sk
    rng = np.random.default_rng(9)
    x = random_paths(rng, 5, 7, 2)
    y = random_paths(rng, 6, 11, 2)
    G = s.sig_kernel_gram(cu(x), cu(y), (0, 1)).cpu().numpy()
    xa = np.repeat(x, 6, axis=0)
    yb = np.tile(y, (5, 1, 1))
    kb = s.sig_kernel(cu(xa), cu(yb), (0, 1)).cpu().numpy().reshape(5, 6)
    np.testing.assert_array_equal(G, kb)


def test_c3_subgram(sk):
    s, _ = sk
    g = golden("c3_subgram")
    assert rel_err(s.sig_kernel_gram(cu(g["x"])).cpu().numpy(), g["g"]) < TOL


def test_c4_long_pair(sk):
    s, _ = sk
    g = golden("c4_long_pair")
    got = s.sig_kernel(cu(g["x"]), cu(g["y"]), 1).cpu().numpy()
    assert rel_err(got, g["out"]) < TOL


def test_rbf_pinned_solver(sk):
    s, ops = sk
    g = golden("rbf_pinned_solver")
    v = s.sig_kernel(cu(g["x"]), cu(g["y"]), 2, s.RBFKernel(float(g["sigma"]))).item()
    assert rel_err([v], [float(g["value"])]) < TOL
    # the pinned solver on the (numpy) RBF delta: bitwise-independent of our delta
    v2 = ops.solve_delta(cu(g["delta"])[None], 2, 2).item()
    assert rel_err([v2], [float(g["value"])]) < 1e-12


def test_solve_grid(sk):
    _, ops = sk
    g = golden("solve_grid")
    grid = ops.solve_delta_grid(cu(g["delta"]), 1, 1).cpu().numpy()
    assert rel_err(grid, g["grid"]) < 1e-14
    v = ops.solve_delta(cu(g["delta"])[None], 1, 1).item()
    assert v == grid[-1, -1]  # strip == grid bitwise (test_kernel.py:65-71)


@pytest.mark.parametrize("L1,L2,d,l1,l2,B", [
    (2, 2, 1, 0, 0, 3), (3, 40, 2, 0, 0, 5), (70, 33, 5, 1, 0, 7), (17, 17, 9, 2, 3, 4),
    (129, 100, 16, 0, 1, 3), (64, 64, 20, 0, 0, 2), (300, 5, 3, 0, 4, 2),
    (1030, 260, 4, 1, 0, 2)])
def test_random_shapes_vs_oracle(sk, oracle, L1, L2, d, l1, l2, B):
    s, _ = sk
    rng = np.random.default_rng(L1 * 7 + L2)
    x = make_paths(rng, B, L1, d)
    y = make_paths(rng, B, L2, d)
    want = oracle.kernel_batch(x, y, l1, l2)
    got = s.sig_kernel(cu(x), cu(y), (l1, l2)).cpu().numpy()
    assert rel_err(got, want) < TOL


@pytest.mark.parametrize("n,L,d,l", [(9, 12, 3, 0), (33, 20, 8, 1), (40, 65, 16, 0)])
def test_sym_gram_vs_oracle(sk, oracle, n, L, d, l):
    s, _ = sk
    rng = np.random.default_rng(n)
    X = make_paths(rng, n, L, d)
    G = s.sig_kernel_gram(cu(X), dyadic_order=l).cpu().numpy()
    assert rel_err(G, oracle.kernel_gram(X, None, l, l)) < TOL
    np.testing.assert_array_equal(G, G.T)


def test_rbf_batch_vs_oracle(sk, oracle):
    s, _ = sk
    rng = np.random.default_rng(3)
    x = make_paths(rng, 6, 40, 5)
    y = make_paths(rng, 6, 31, 5)
    for lam in ((0, 0), (2, 2), (1, 3)):
        want = oracle.kernel_batch(x, y, *lam, ("rbf", 0.8))
        got = s.sig_kernel(cu(x), cu(y), lam, s.RBFKernel(0.8)).cpu().numpy()
        assert rel_err(got, want) < TOL


def test_empty_and_errors(sk):
    s, _ = sk
    e = s.sig_kernel(cu(np.zeros((0, 5, 2))), cu(np.zeros((0, 5, 2))))
    assert e.shape == (0,)
    with pytest.raises(s.InvalidArgument):
        s.sig_kernel(cu(np.zeros((2, 1, 2))), cu(np.zeros((2, 5, 2))))
    with pytest.raises(s.InvalidArgument):
        s.sig_kernel(cu(np.zeros((2, 3, 2))), cu(np.zeros((3, 5, 2))))
    with pytest.raises(ValueError):
        s.sig_kernel(cu(np.zeros((2, 3, 2))), cu(np.zeros((2, 5, 3))))


def test_overflow_inf(sk):
    _, ops = sk
    v = ops.solve_delta(cu(np.full((1, 40, 40), 1e300)), 0, 0).item()
    assert np.isinf(v)


def test_fp32_storage_fp64_math(sk, oracle):
    s, _ = sk
    rng = np.random.default_rng(4)
    x = make_paths(rng, 3, 50, 3).astype(np.float32)
    y = make_paths(rng, 3, 60, 3).astype(np.float32)
    got = s.sig_kernel(torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda"), 1)
    assert got.dtype == torch.float32
    want = oracle.kernel_batch(x.astype(np.float64), y.astype(np.float64), 1, 1)
    assert rel_err(got.cpu().numpy(), want) < 1e-6
