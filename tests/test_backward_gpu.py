"""GPU parity of the reverse-wavefront backward against the reference-pinned
golden vectors, the C oracle (fp64, 1e-10) and torch.autograd.gradcheck."""

import numpy as np
import pytest
import torch

from conftest import golden, make_paths, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def sk():
    import paper_2509_10613_b200 as sk
    from paper_2509_10613_b200 import ops
    return sk, ops


def cu(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")


def bwd(ops, x, y, l1, l2, cot=None, static=(0, 1.0)):
    v, gx, gy = ops.backward_batch(cu(x), cu(y), l1, l2, static[0], static[1],
                                   None if cot is None else cu(cot), want_values=True)
    return v.cpu().numpy(), gx.cpu().numpy(), gy.cpu().numpy()


def test_single_cell_hand_value(sk):
    _, ops = sk
    x = np.array([[[0.0], [1.0]]])
    v, gx, gy = bwd(ops, x, x, 0, 0)
    assert v[0] == 2.25
    np.testing.assert_allclose(gx[0], [[-1.5], [1.5]], rtol=1e-15)
    np.testing.assert_allclose(gy[0], [[-1.5], [1.5]], rtol=1e-15)


def test_batch_backward_golden(sk):
    _, ops = sk
    g = golden("batch_backward_small")
    for l1, l2 in ((0, 0), (1, 2), (2, 1), (0, 3)):
        v, gx, gy = bwd(ops, g["x"], g["y"], l1, l2, g["cot"])
        assert rel_err(v, g[f"v_{l1}{l2}"]) < TOL
        assert rel_err(gx, g[f"gx_{l1}{l2}"]) < TOL, (l1, l2)
        assert rel_err(gy, g[f"gy_{l1}{l2}"]) < TOL, (l1, l2)


def test_c2_linear_golden(sk):
    _, ops = sk
    g = golden("c2_linear_pairs")
    v, gx, gy = bwd(ops, g["x"], g["y"], 2, 2)
    assert rel_err(v, g["v"]) < TOL
    assert rel_err(gx, g["gx"]) < TOL
    assert rel_err(gy, g["gy"]) < TOL


def test_c5_pair_golden(sk):
    _, ops = sk
    g = golden("c5_pair_grad")
    v, gx, gy = bwd(ops, g["x"][None], g["y"][None], 0, 0)
    assert rel_err(v, [float(g["value"])]) < TOL
    assert rel_err(gx[0], g["gx"]) < TOL
    assert rel_err(gy[0], g["gy"]) < TOL


@pytest.mark.parametrize("B,L1,L2,d,l1,l2", [
    (3, 2, 2, 1, 0, 0), (4, 5, 40, 2, 0, 0), (3, 70, 33, 5, 1, 0), (2, 17, 17, 9, 2, 3),
    (3, 129, 100, 16, 0, 1), (2, 300, 5, 3, 0, 4), (2, 40, 37, 4, 3, 1), (2, 65, 66, 8, 0, 0),
    (1, 520, 200, 6, 0, 0), (2, 33, 35, 12, 1, 1)])
def test_random_vs_oracle(sk, oracle, B, L1, L2, d, l1, l2):
    _, ops = sk
    rng = np.random.default_rng(B * 1000 + L1 + L2)
    x = make_paths(rng, B, L1, d)
    y = make_paths(rng, B, L2, d)
    cot = rng.standard_normal(B)
    wv, wx, wy = oracle.kernel_batch_backward(x, y, l1, l2, cot)
    v, gx, gy = bwd(ops, x, y, l1, l2, cot)
    assert rel_err(v, wv) < TOL
    assert rel_err(gx, wx) < TOL
    assert rel_err(gy, wy) < TOL


@pytest.mark.parametrize("lam", [(0, 0), (2, 2), (1, 3)])
def test_rbf_vs_oracle(sk, oracle, lam):
    _, ops = sk
    rng = np.random.default_rng(77)
    x = make_paths(rng, 3, 30, 4)
    y = make_paths(rng, 3, 23, 4)
    cot = rng.standard_normal(3)
    wv, wx, wy = oracle.kernel_batch_backward(x, y, *lam, cot, ("rbf", 0.9))
    v, gx, gy = bwd(ops, x, y, *lam, cot, static=(1, 0.9))
    assert rel_err(v, wv) < TOL
    assert rel_err(gx, wx) < TOL
    assert rel_err(gy, wy) < TOL


def test_batch_equals_single_bitwise(sk):
    _, ops = sk
    rng = np.random.default_rng(4)
    x = rng.standard_normal((3, 40, 2)) * 0.5
    y = rng.standard_normal((3, 60, 2)) * 0.5
    v, gx, gy = bwd(ops, x, y, 1, 0)
    for b in range(3):
        vb, gxb, gyb = bwd(ops, x[b:b + 1], y[b:b + 1], 1, 0)
        assert v[b] == vb[0]
        np.testing.assert_array_equal(gx[b], gxb[0])
        np.testing.assert_array_equal(gy[b], gyb[0])


def test_linear_in_cotangent(sk):
    _, ops = sk
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, 30, 3)) * 0.5
    y = rng.standard_normal((2, 50, 3)) * 0.5
    _, g1x, g1y = bwd(ops, x, y, 1, 1, np.ones(2))
    _, g2x, g2y = bwd(ops, x, y, 1, 1, -2.5 * np.ones(2))
    assert rel_err(g2x, -2.5 * g1x) < 1e-13
    assert rel_err(g2y, -2.5 * g1y) < 1e-13


@pytest.mark.parametrize("n,L,d,lam", [(5, 9, 2, (1, 1)), (13, 40, 8, (0, 0)),
                                       (6, 70, 16, (0, 0)), (4, 20, 3, (2, 1))])
def test_gram_sym_vs_oracle(sk, oracle, n, L, d, lam):
    _, ops = sk
    rng = np.random.default_rng(n + L)
    X = make_paths(rng, n, L, d)
    C = rng.standard_normal((n, n))
    want = oracle.gram_backward(X, None, C, *lam)
    gx, _ = ops.backward_gram(cu(X), None, *lam, 0, 1.0, cu(C))
    assert rel_err(gx.cpu().numpy(), want) < TOL


def test_gram_cross_vs_oracle(sk, oracle):
    _, ops = sk
    rng = np.random.default_rng(5)
    X = make_paths(rng, 5, 20, 3)
    Y = make_paths(rng, 7, 31, 3)
    C = rng.standard_normal((5, 7))
    for lam in ((0, 0), (0, 1), (2, 0)):
        wx, wy = oracle.gram_backward(X, Y, C, *lam)
        gx, gy = ops.backward_gram(cu(X), cu(Y), *lam, 0, 1.0, cu(C))
        assert rel_err(gx.cpu().numpy(), wx) < TOL
        assert rel_err(gy.cpu().numpy(), wy) < TOL


def test_gram_rbf_vs_oracle(sk, oracle):
    _, ops = sk
    rng = np.random.default_rng(8)
    X = make_paths(rng, 6, 15, 3)
    C = rng.standard_normal((6, 6))
    want = oracle.gram_backward(X, None, C, 1, 1, ("rbf", 0.7))
    gx, _ = ops.backward_gram(cu(X), None, 1, 1, 1, 0.7, cu(C))
    assert rel_err(gx.cpu().numpy(), want) < TOL


def test_autograd_gradcheck(sk):
    s, _ = sk
    torch.manual_seed(0)
    x = (torch.randn(2, 6, 2, dtype=torch.float64, device="cuda") * 0.4).requires_grad_()
    y = (torch.randn(2, 5, 2, dtype=torch.float64, device="cuda") * 0.4).requires_grad_()
    assert torch.autograd.gradcheck(lambda a, b: s.sig_kernel(a, b, (1, 0)), (x, y))
    assert torch.autograd.gradcheck(
        lambda a, b: s.sig_kernel(a, b, 1, s.RBFKernel(0.8)), (x, y))
    X = (torch.randn(3, 5, 2, dtype=torch.float64, device="cuda") * 0.4).requires_grad_()
    assert torch.autograd.gradcheck(lambda a: s.sig_kernel_gram(a, dyadic_order=1), (X,))
    assert torch.autograd.gradcheck(lambda a, b: s.sig_kernel_gram(a, b, (0, 1)), (X, y))


def test_autograd_loss_backward(sk, oracle):
    s, _ = sk
    rng = np.random.default_rng(3)
    X = make_paths(rng, 8, 30, 4)
    C = rng.standard_normal((8, 8))
    Xt = cu(X).requires_grad_()
    G = s.sig_kernel_gram(Xt, dyadic_order=0)
    (G * cu(C)).sum().backward()
    assert rel_err(Xt.grad.cpu().numpy(), oracle.gram_backward(X, None, C)) < TOL


@pytest.mark.parametrize("B,L1,L2,d,l1,l2", [
    (3, 20, 17, 33, 0, 0), (2, 40, 31, 64, 0, 0), (2, 25, 30, 50, 1, 2), (2, 12, 70, 100, 2, 0)])
def test_wide_paths_vs_oracle(sk, oracle, B, L1, L2, d, l1, l2):
    """d > 32: DP-chunked dot products, coarse adjoint mapped chunk by chunk
    after the sweep (the reference handles any d, kernel_grad.py:27-61)."""
    _, ops = sk
    rng = np.random.default_rng(d + L1)
    x = make_paths(rng, B, L1, d)
    y = make_paths(rng, B, L2, d)
    cot = rng.standard_normal(B)
    wv, wx, wy = oracle.kernel_batch_backward(x, y, l1, l2, cot)
    v, gx, gy = bwd(ops, x, y, l1, l2, cot)
    assert rel_err(v, wv) < TOL
    assert rel_err(gx, wx) < TOL
    assert rel_err(gy, wy) < TOL


@pytest.mark.parametrize("n1,n2,L,d,lam", [(7, None, 21, 33, 0), (5, 6, 18, 64, 1), (9, None, 15, 40, 1)])
def test_wide_gram_vs_oracle(sk, oracle, n1, n2, L, d, lam):
    """Gram backward and the fused value + gradient at d > 32."""
    s, ops = sk
    rng = np.random.default_rng(n1 * d + L)
    X = make_paths(rng, n1, L, d)
    Y = None if n2 is None else make_paths(rng, n2, L + 2, d)
    C = rng.standard_normal((n1, n1 if n2 is None else n2))
    G, gx, gy = s.sig_kernel_gram_value_and_grad(cu(X), None if Y is None else cu(Y), cu(C),
                                                 dyadic_order=lam)
    assert rel_err(G.cpu().numpy(), oracle.kernel_gram(X, Y, lam, lam)) < TOL
    want = oracle.gram_backward(X, Y, C, lam, lam)
    if Y is None:
        assert rel_err(gx.cpu().numpy(), want) < TOL
    else:
        assert rel_err(gx.cpu().numpy(), want[0]) < TOL
        assert rel_err(gy.cpu().numpy(), want[1]) < TOL
    # autograd through sig_kernel_gram
    xt = cu(X).requires_grad_(True)
    Gt = s.sig_kernel_gram(xt, None if Y is None else cu(Y), dyadic_order=lam)
    (Gt * cu(C)).sum().backward()
    assert rel_err(xt.grad.cpu().numpy(), want if Y is None else want[0]) < TOL


@pytest.mark.parametrize("B,L1,L2,d,l1,l2,static", [
    (6, 130, 120, 8, 2, 2, (1, 0.8)),   # 516 fine rows: 8 rows per lane, one 4-warp strip
    (5, 700, 650, 7, 0, 0, (0, 1.0)),   # cross-warp, lambda 0, d padded to 8
    (4, 400, 390, 5, 1, 2, (1, 1.3)),   # RBF, mixed orders
    (3, 300, 310, 8, 2, 1, (0, 1.0)),   # 1196 fine rows: taller than one 4-row strip of 128 lanes
    (4, 65, 80, 3, 3, 3, (0, 1.0)),     # short axis at order 3
])
def test_cross_warp_pairs_vs_oracle(sk, oracle, B, L1, L2, d, l1, l2, static):
    """Few long pairs take the cross-warp kernels (one pair per CTA: 8 rows per
    lane past 512 fine rows, LAG-chunked forward hops); values and both
    gradients vs the oracle at shapes around the instance boundaries."""
    rng = np.random.default_rng(B * 1000 + L1 + d)
    x = make_paths(rng, B, L1, d)
    y = make_paths(rng, B, L2, d)
    cot = rng.standard_normal(B)
    kind, sigma = static
    st = ("rbf", sigma) if kind == 1 else None
    _, ops = sk
    wv, wx, wy = oracle.kernel_batch_backward(x, y, l1, l2, cot, st)
    v, gx, gy = ops.backward_batch(cu(x), cu(y), l1, l2, kind, sigma, cu(cot), want_values=True)
    assert rel_err(v.cpu().numpy(), wv) < TOL
    assert rel_err(gx.cpu().numpy(), wx) < TOL
    assert rel_err(gy.cpu().numpy(), wy) < TOL
    f = ops.forward_batch(cu(x), cu(y), l1, l2, kind, sigma).cpu().numpy()
    np.testing.assert_array_equal(f, v.cpu().numpy())


@pytest.mark.parametrize("B,L1,L2,d,lam,sk_kind", [(6, 40, 33, 3, 0, None),
                                                   (5, 50, 50, 8, (1, 2), None),
                                                   (4, 30, 41, 5, 1, ("rbf", 0.8)),
                                                   (256, 256, 256, 8, 2, ("rbf", 1.0))])  # C2
def test_sig_kernel_value_and_grad_matches_oracle(B, L1, L2, d, lam, sk_kind):
    """The torch form of kernel_batch_backward (kernel_grad.py:64-98): values
    and both gradients from one pass, against the oracle's batch backward."""
    import paper_2509_10613_b200 as sk
    from oracle import oracle as orc
    rng = np.random.default_rng(21)
    x = np.cumsum(rng.standard_normal((B, L1, d)) / np.sqrt(L1), axis=1)
    y = np.cumsum(rng.standard_normal((B, L2, d)) / np.sqrt(L2), axis=1)
    cot = rng.standard_normal(B)
    l1, l2 = (lam, lam) if isinstance(lam, int) else lam
    static = None if sk_kind is None else sk.RBFKernel(sk_kind[1])
    k, gx, gy = sk.sig_kernel_value_and_grad(torch.as_tensor(x, device="cuda"),
                                             torch.as_tensor(y, device="cuda"),
                                             torch.as_tensor(cot, device="cuda"),
                                             dyadic_order=(l1, l2), static_kernel=static)
    wv, wx, wy = orc.kernel_batch_backward(x, y, l1, l2, cot, sk_kind)
    for got, want in ((k, wv), (gx, wx), (gy, wy)):
        assert np.abs(got.cpu().numpy() - want).max() / np.abs(want).max() < 1e-10
    k2 = sk.sig_kernel(torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda"),
                       dyadic_order=(l1, l2), static_kernel=static)
    assert np.abs(k.cpu().numpy() - k2.cpu().numpy()).max() / np.abs(wv).max() < 1e-13


def test_sig_kernel_value_and_grad_single_pair_and_transform():
    """(L, d) inputs give a 0-d k; a transform runs inside the kernels and the
    result equals sig_kernel + autograd on the same call (values and gradients)."""
    import paper_2509_10613_b200 as sk
    rng = np.random.default_rng(22)
    x = torch.as_tensor(np.cumsum(rng.standard_normal((30, 3)) / 6, axis=0), device="cuda")
    y = torch.as_tensor(np.cumsum(rng.standard_normal((25, 3)) / 5, axis=0), device="cuda")
    k, gx, gy = sk.sig_kernel_value_and_grad(x, y, dyadic_order=1, transform="lead_lag")
    assert k.dim() == 0 and gx.shape == x.shape and gy.shape == y.shape
    xr, yr = x.clone().requires_grad_(True), y.clone().requires_grad_(True)
    k2 = sk.sig_kernel(xr, yr, dyadic_order=1, transform="lead_lag")
    k2.backward()
    assert abs(k.item() - k2.item()) <= 1e-13 * abs(k2.item())
    assert torch.allclose(gx, xr.grad, rtol=0, atol=1e-13 * xr.grad.abs().max().item())
    assert torch.allclose(gy, yr.grad, rtol=0, atol=1e-13 * yr.grad.abs().max().item())
