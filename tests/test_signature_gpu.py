"""Truncated signatures on the GPU against the reference:
golden vectors the reference produced (tests/golden/signature.npz, forward
BITWISE: same operations in the same order, no FMA contraction), the C
oracle (its restatement, itself pinned bitwise to the goldens) at random
shapes, and the reference's own known answers and invariants
(/root/reference/pkg/tests/test_signature.py, test_signature_grad.py)."""

import numpy as np
import pytest
import torch

from conftest import golden, random_paths, rel_err

pytestmark = pytest.mark.gpu
KINDS = {0: None, 1: "time_augment", 2: "lead_lag"}


@pytest.fixture(scope="module")
def sc():
    from paper_2509_10613_b200 import sigcore_compat as sc
    return sc


def cu(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")


def test_golden_forward_bitwise_backward_close(sc):
    g = golden("signature")
    for i in range(int(g["n"])):
        depth, tf, custom = (int(v) for v in g[f"s{i}_meta"])
        times = g[f"s{i}_times"] if custom else None
        opts = sc.SigOptions(depth, transform=KINDS[tf])
        pb = sc.PathBatch(g[f"s{i}_x"], times=times)
        np.testing.assert_array_equal(sc.signature(pb, opts), g[f"s{i}_sig"])
        grad = sc.signature_backward(pb, opts, g[f"s{i}_cot"])
        assert rel_err(grad, g[f"s{i}_grad"]) < 1e-12, i


@pytest.mark.parametrize("B,L,d,depth,kind", [
    (3, 30, 2, 12, None), (2, 17, 3, 7, "time_augment"), (4, 50, 4, 6, None),
    (2, 25, 5, 5, "lead_lag"), (3, 40, 8, 4, None), (2, 12, 12, 3, None), (2, 9, 16, 4, None),
    (1, 6, 30, 3, None), (2, 8, 16, 3, "lead_lag"), (5, 2, 3, 3, None), (2, 100, 1, 16, None)])
def test_random_vs_oracle(sc, oracle, B, L, d, depth, kind):
    rng = np.random.default_rng(B * 100 + L + d + depth)
    x = random_paths(rng, B, L, d)
    opts = sc.SigOptions(depth, transform=kind)
    want = oracle.signature(x, depth, kind)
    got = sc.signature(x, opts)
    np.testing.assert_array_equal(got, want)
    cot = rng.standard_normal(want.shape)
    gw = oracle.signature_backward(x, depth, cot, kind)
    gg = sc.signature_backward(x, opts, cot)
    assert rel_err(gg, gw) < 1e-11


def test_known_answers(sc):
    """reference tests/test_signature.py:11-23 and test_signature_grad.py:9-12."""
    s = sc.signature(np.array([[0.0], [1.0]]), sc.SigOptions(3))
    np.testing.assert_allclose(s, [1.0, 0.5, 1.0 / 6.0], rtol=1e-15)
    s = sc.signature(np.array([[0.0], [1.0], [2.0]]), sc.SigOptions(2))
    np.testing.assert_allclose(s, [2.0, 2.0], rtol=1e-15)
    s = sc.signature(np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]]), sc.SigOptions(2))
    np.testing.assert_allclose(s[:2], [1.0, 1.0], rtol=1e-15)
    np.testing.assert_allclose(s[2:], [0.5, 1.0, 0.0, 0.5], atol=1e-15)
    g = sc.signature_backward(np.array([[0.0], [1.0]]), sc.SigOptions(1), np.array([2.5]))
    np.testing.assert_array_equal(g, [[-2.5], [2.5]])


def test_invariants(sc):
    """Chen identity, midpoint insertion, repeated points bit-exact, level 1 =
    total increment (reference tests/test_signature.py:43-86)."""
    rng = np.random.default_rng(11)
    opts = sc.SigOptions(4)
    x = random_paths(rng, 1, 6, 2)[0]
    base = sc.signature(x, opts)
    for seg in range(5):
        mid = (x[seg] + x[seg + 1]) / 2
        assert rel_err(sc.signature(np.insert(x, seg + 1, mid, axis=0), opts), base) < 1e-12
    np.testing.assert_array_equal(sc.signature(np.concatenate([x, x[-1:]], 0), opts), base)
    np.testing.assert_array_equal(sc.signature(np.insert(x, 2, x[2], axis=0), opts), base)
    y = random_paths(rng, 2, 6, 3)
    s = sc.signature(y, sc.SigOptions(2))
    np.testing.assert_allclose(s[:, :3], y[:, -1] - y[:, 0], rtol=1e-14, atol=1e-15)


def test_backward_properties(sc):
    """Zero cotangent, level-1 cotangent hits the endpoints, linearity, batch ==
    per path bitwise, run-to-run bitwise (reference test_signature_grad.py)."""
    rng = np.random.default_rng(3)
    x = random_paths(rng, 3, 6, 2)
    opts = sc.SigOptions(3)
    total = sc.sig_tensor_shape(2, opts).total
    assert not sc.signature_backward(x, opts, np.zeros((3, total))).any()
    cot = np.zeros(total)
    cot[:2] = [1.0, -2.0]
    g = sc.signature_backward(x[0], opts, cot)
    np.testing.assert_array_equal(g[0], [-1.0, 2.0])
    np.testing.assert_array_equal(g[-1], [1.0, -2.0])
    np.testing.assert_array_equal(g[1:-1], np.zeros((4, 2)))
    c1, c2 = rng.standard_normal((3, total)), rng.standard_normal((3, total))
    comb = sc.signature_backward(x, opts, 0.7 * c1 - 1.3 * c2)
    split = 0.7 * sc.signature_backward(x, opts, c1) - 1.3 * sc.signature_backward(x, opts, c2)
    assert rel_err(comb, split) < 1e-13
    gb = sc.signature_backward(x, opts, c1)
    for b in range(3):
        np.testing.assert_array_equal(sc.signature_backward(x[b], opts, c1[b]), gb[b])
    np.testing.assert_array_equal(sc.signature_backward(x, opts, c1), gb)


def test_validation(sc):
    from paper_2509_10613_b200 import InvalidArgument
    with pytest.raises(InvalidArgument):
        sc.signature(np.zeros((1, 2)), sc.SigOptions(2))
    bad = np.zeros((3, 2))
    bad[1, 0] = np.nan
    with pytest.raises(InvalidArgument):
        sc.signature(bad, sc.SigOptions(2))
    with pytest.raises(InvalidArgument):
        sc.SigOptions(0)
    with pytest.raises(InvalidArgument):
        sc.signature_backward(random_paths(np.random.default_rng(6), 2, 4, 2), sc.SigOptions(2),
                              np.zeros((2, 5)))
    s = sc.signature(random_paths(np.random.default_rng(15), 2, 8, 2).astype(np.float32),
                     sc.SigOptions(3, scalar_width=32))
    assert s.dtype == np.float32


def test_torch_api_autograd(sc, oracle):
    import paper_2509_10613_b200 as sk
    rng = np.random.default_rng(21)
    x = random_paths(rng, 2, 7, 2)
    xt = cu(x).requires_grad_(True)
    s = sk.signature(xt, 4, transform="lead_lag")
    np.testing.assert_array_equal(s.detach().cpu().numpy(), oracle.signature(x, 4, "lead_lag"))
    w = torch.as_tensor(rng.standard_normal(s.shape), device="cuda")
    (s * w).sum().backward()
    want = oracle.signature_backward(x, 4, w.cpu().numpy(), "lead_lag")
    assert rel_err(xt.grad.cpu().numpy(), want) < 1e-12
    assert torch.autograd.gradcheck(lambda a: sk.signature(a, 3, "time_augment"),
                                    (cu(x[:1, :4]).requires_grad_(True),))
    one = sk.signature(cu(x[0]), 3)
    assert one.shape == (2 + 4 + 8,)
