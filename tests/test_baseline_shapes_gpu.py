"""GPU parity at BASELINE.json's own shapes (configs C1-C5), against the C
oracle (the pinned restatement of the reference, tests/test_oracle.py).

Each config runs exactly the kernel instance the bench / a user hits at that
shape; where the full config is too large for the CPU oracle (C3, C5 Gram,
C4's 128 pairs) a sub-block of the same shape is compared and the sub-block is
stated.  Tolerance: rel_err (reference tests/conftest.py:16-21) <= 1e-10 fp64.
Data: the reference bench generator (bench.py:53-56), seed 0, x then y.
"""

import numpy as np
import pytest
import torch

from conftest import make_paths, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


def cu(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")


@pytest.fixture(scope="module")
def sk():
    import paper_2509_10613_b200 as sk
    from paper_2509_10613_b200 import ops
    return sk, ops


def test_c1_full(sk, oracle):
    """C1: sig_kernel forward, 32 pairs, L=64, d=4, lambda=0 (whole config)."""
    s, _ = sk
    rng = np.random.default_rng(0)
    x = make_paths(rng, 32, 64, 4)
    y = make_paths(rng, 32, 64, 4)
    got = s.sig_kernel(cu(x), cu(y), dyadic_order=0).cpu().numpy()
    assert rel_err(got, oracle.kernel_batch(x, y, 0, 0)) < TOL


def test_c2_full_rbf_fwd_bwd(sk, oracle):
    """C2 exactly as configured: 256 pairs, L=256, d=8, lambda=2, RBF sigma=1,
    forward + backward (cotangent ones), values and both gradients."""
    s, ops = sk
    rng = np.random.default_rng(0)
    x = make_paths(rng, 256, 256, 8)
    y = make_paths(rng, 256, 256, 8)
    wv, wx, wy = oracle.kernel_batch_backward(x, y, 2, 2, None, ("rbf", 1.0))
    v, gx, gy = ops.backward_batch(cu(x), cu(y), 2, 2, 1, 1.0, None, want_values=True)
    assert rel_err(v.cpu().numpy(), wv) < TOL
    assert rel_err(gx.cpu().numpy(), wx) < TOL
    assert rel_err(gy.cpu().numpy(), wy) < TOL
    # the public autograd path gives the same values and gradients
    xt = cu(x).requires_grad_(True)
    yt = cu(y).requires_grad_(True)
    k = s.sig_kernel(xt, yt, dyadic_order=2, static_kernel=s.RBFKernel(1.0))
    k.sum().backward()
    assert rel_err(k.detach().cpu().numpy(), wv) < TOL
    assert rel_err(xt.grad.cpu().numpy(), wx) < TOL
    assert rel_err(yt.grad.cpu().numpy(), wy) < TOL


def test_c3_subgram_value_and_grad(sk, oracle):
    """C3 shape (L=512, d=16, lambda=0, symmetric, DMMA kernels): a 20-path
    sub-Gram of the config's own paths, random cotangent (seed 1)."""
    s, _ = sk
    rng = np.random.default_rng(0)
    X = make_paths(rng, 20, 512, 16)
    C = np.random.default_rng(1).standard_normal((20, 20))
    G, gx, gy = s.sig_kernel_gram_value_and_grad(cu(X), None, cu(C))
    assert gy is None
    assert rel_err(G.cpu().numpy(), oracle.kernel_gram(X, None, 0, 0)) < TOL
    assert rel_err(gx.cpu().numpy(), oracle.gram_backward(X, None, C, 0, 0)) < TOL


def test_c4_long_pairs(sk, oracle):
    """C4 shape: L=8192, d=4, lambda=1 (cross-warp strip pipeline, one pair per
    CTA); 3 pairs of the config (the full 128 take the oracle minutes)."""
    s, _ = sk
    rng = np.random.default_rng(0)
    x = make_paths(rng, 3, 8192, 4)
    y = make_paths(rng, 3, 8192, 4)
    got = s.sig_kernel(cu(x), cu(y), dyadic_order=1).cpu().numpy()
    assert rel_err(got, oracle.kernel_batch(x, y, 1, 1)) < TOL


def test_c5_subgram_value_and_grad(sk, oracle):
    """C5 shape: L=1024, d=8, lambda=0 -> the DP = 8 DMMA backward
    (gram_bwd_mma<8, 2>), the north-star kernel.  A 16-path symmetric sub-Gram
    with a random cotangent (seed 1): G and dF/dX."""
    s, _ = sk
    rng = np.random.default_rng(0)
    X = make_paths(rng, 16, 1024, 8)
    C = np.random.default_rng(1).standard_normal((16, 16))
    G, gx, _ = s.sig_kernel_gram_value_and_grad(cu(X), None, cu(C))
    assert rel_err(G.cpu().numpy(), oracle.kernel_gram(X, None, 0, 0)) < TOL
    assert rel_err(gx.cpu().numpy(), oracle.gram_backward(X, None, C, 0, 0)) < TOL
    # the autograd split (forward Gram kernel, then the backward kernel)
    Xt = cu(X).requires_grad_(True)
    Gt = s.sig_kernel_gram(Xt)
    (Gt * cu(C)).sum().backward()
    assert rel_err(Gt.detach().cpu().numpy(), oracle.kernel_gram(X, None, 0, 0)) < TOL
    assert rel_err(Xt.grad.cpu().numpy(), oracle.gram_backward(X, None, C, 0, 0)) < TOL


def test_c5_cross_block(sk, oracle):
    """C5 shape, cross Gram block (the off-diagonal tiles a sharded run solves):
    9 x 7 paths, random cotangent, both gradients."""
    s, _ = sk
    rng = np.random.default_rng(0)
    X = make_paths(rng, 9, 1024, 8)
    Y = make_paths(rng, 7, 1024, 8)
    C = np.random.default_rng(1).standard_normal((9, 7))
    G, gx, gy = s.sig_kernel_gram_value_and_grad(cu(X), cu(Y), cu(C))
    assert rel_err(G.cpu().numpy(), oracle.kernel_gram(X, Y, 0, 0)) < TOL
    wx, wy = oracle.gram_backward(X, Y, C, 0, 0)
    assert rel_err(gx.cpu().numpy(), wx) < TOL
    assert rel_err(gy.cpu().numpy(), wy) < TOL


@pytest.mark.parametrize("L1,L2,d,lam", [(64, 64, 4, 0), (40, 64, 3, 0), (17, 9, 8, 1),
                                         (33, 33, 20, 0), (2, 65, 1, 0), (9, 5, 4, 3)])
def test_small_pairs_path(sk, oracle, L1, L2, d, lam):
    """Few short pairs run the small-pair kernel (sk_small.cu: one warp per pair
    from a shared coefficient tile); the same pairs inside a large batch run the
    general batch kernel -- values are bitwise equal, and match the oracle."""
    s, ops = sk
    rng = np.random.default_rng(L1 * 31 + L2 + d)
    n_big = 4 * torch.cuda.get_device_properties(0).multi_processor_count + 8
    x = make_paths(rng, n_big, L1, d)
    y = make_paths(rng, n_big, L2, d)
    small = ops.forward_batch(cu(x[:32]), cu(y[:32]), lam, lam, 0, 1.0).cpu().numpy()
    big = ops.forward_batch(cu(x), cu(y), lam, lam, 0, 1.0).cpu().numpy()
    np.testing.assert_array_equal(small, big[:32])
    assert rel_err(small, oracle.kernel_batch(x[:32], y[:32], lam, lam)) < TOL
