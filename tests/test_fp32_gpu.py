"""FP32-arithmetic kernels (precision="fp32", linear static kernel) against the
fp64 oracle: north_star's "<= 1e-4 relative in fp32" (rel_err, reference
tests/conftest.py:16-21), at every BASELINE config shape the bound holds for,
and the measured error at config 4's long paths, where fp32 cannot hold it
(error grows ~linearly with the fine-axis length; 16382 fine
cells per axis there) -- that config is an fp64 config."""

import numpy as np
import pytest
import torch

from conftest import make_paths, rel_err

pytestmark = pytest.mark.gpu
TOL32 = 1e-4


@pytest.fixture(scope="module")
def sk():
    import paper_2509_10613_b200 as sk
    return sk


def f32(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float32), device="cuda")


@pytest.mark.parametrize("B,L,d,lam", [(32, 64, 4, 0),      # C1
                                       (64, 256, 8, 2),     # C2 shape (linear)
                                       (16, 512, 16, 0),    # C3 shape
                                       (8, 1024, 8, 0),     # C5 shape
                                       (5, 300, 40, 1)])    # d > 32
def test_batch_fp32_within_1e4(sk, oracle, B, L, d, lam):
    rng = np.random.default_rng(0)
    x = make_paths(rng, B, L, d).astype(np.float32)
    y = make_paths(rng, B, L, d).astype(np.float32)
    k = sk.sig_kernel(f32(x), f32(y), dyadic_order=lam, precision="fp32")
    assert k.dtype == torch.float32
    want = oracle.kernel_batch(x.astype(np.float64), y.astype(np.float64), lam, lam)
    assert rel_err(k.cpu().numpy(), want) < TOL32


@pytest.mark.parametrize("n,L,d,lam", [(24, 512, 16, 0), (20, 1024, 8, 0), (12, 100, 3, 2),
                                       (10, 300, 32, 0), (16, 130, 20, 1)])  # DMMA + float recurrence
def test_gram_fp32_within_1e4(sk, oracle, n, L, d, lam):
    rng = np.random.default_rng(1)
    X = make_paths(rng, n, L, d).astype(np.float32)
    G = sk.sig_kernel_gram(f32(X), dyadic_order=lam, precision="fp32").cpu().numpy()
    want = oracle.kernel_gram(X.astype(np.float64), None, lam, lam)
    assert rel_err(G, want) < TOL32
    np.testing.assert_array_equal(G, G.T)
    Y = make_paths(rng, 7, L // 2, d).astype(np.float32)
    Gc = sk.sig_kernel_gram(f32(X), f32(Y), dyadic_order=lam, precision="fp32").cpu().numpy()
    assert rel_err(Gc, oracle.kernel_gram(X.astype(np.float64), Y.astype(np.float64), lam, lam)) < TOL32


def test_c4_fp32_error_reported(sk, oracle):
    """Config 4 (L=8192, lambda=1): fp32 arithmetic is ~1e-3 off -- measured and
    bounded here, not claimed within 1e-4 (use the fp64 path there)."""
    rng = np.random.default_rng(0)
    x = make_paths(rng, 2, 8192, 4).astype(np.float32)
    y = make_paths(rng, 2, 8192, 4).astype(np.float32)
    k = sk.sig_kernel(f32(x), f32(y), dyadic_order=1, precision="fp32").cpu().numpy()
    err = rel_err(k, oracle.kernel_batch(x.astype(np.float64), y.astype(np.float64), 1, 1))
    print(f"C4 fp32 rel err {err:.2e}")
    assert err < 5e-3


def test_fp32_autograd_uses_fp64_backward(sk, oracle):
    rng = np.random.default_rng(3)
    x = make_paths(rng, 4, 40, 3).astype(np.float32)
    y = make_paths(rng, 4, 33, 3).astype(np.float32)
    xt = f32(x).requires_grad_(True)
    k = sk.sig_kernel(xt, f32(y), dyadic_order=1, precision="fp32")
    k.sum().backward()
    _, wx, _ = oracle.kernel_batch_backward(x.astype(np.float64), y.astype(np.float64), 1, 1)
    assert xt.grad.dtype == torch.float32
    assert rel_err(xt.grad.cpu().numpy(), wx) < 1e-6


def test_fp32_rejects_rbf(sk):
    from paper_2509_10613_b200 import InvalidArgument
    x = torch.zeros((1, 4, 2), device="cuda")
    with pytest.raises(InvalidArgument):
        sk.sig_kernel(x, x, static_kernel=sk.RBFKernel(1.0), precision="fp32")
