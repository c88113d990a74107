"""Path transforms of the torch API against the reference (tests/golden/transforms.npz):
forward values and, through autograd, the reference's transform_adjoint."""

import numpy as np
import pytest
import torch

from conftest import golden, make_paths, rel_err
from paper_2509_10613_b200.api import path_transform


@pytest.mark.parametrize("kind,gkey,akey", [("time_augment", "g_ta", "adj_ta"),
                                            ("lead_lag", "g_ll", "adj_ll")])
def test_transform_and_adjoint_match_reference(kind, gkey, akey):
    g = golden("transforms")
    x = torch.as_tensor(g["x"]).requires_grad_(True)
    z = path_transform(x, kind)
    np.testing.assert_array_equal(z.detach().numpy(), g[kind])
    (z * torch.as_tensor(g[gkey])).sum().backward()
    np.testing.assert_allclose(x.grad.numpy(), g[akey], rtol=0, atol=1e-15)


@pytest.mark.gpu
def test_transformed_kernel_vs_oracle(oracle):
    import paper_2509_10613_b200 as sk
    g = golden("transforms")
    rng = np.random.default_rng(5)
    x = make_paths(rng, 3, 12, 2)
    y = make_paths(rng, 3, 9, 2)
    for kind in ("time_augment", "lead_lag"):
        xt = path_transform(torch.as_tensor(x), kind).numpy()
        yt = path_transform(torch.as_tensor(y), kind).numpy()
        want = oracle.kernel_batch(xt, yt, 1, 1)
        got = sk.sig_kernel(torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda"),
                            1, transform=kind).cpu().numpy()
        assert rel_err(got, want) < 1e-10
    X = torch.as_tensor(x, device="cuda").requires_grad_(True)
    assert torch.autograd.gradcheck(
        lambda a: sk.sig_kernel_gram(a, dyadic_order=0, transform="lead_lag"), (X,))
    del g


def _np_adjoint(g, kind):
    """The reference's transform_adjoint (transforms.py:69-90), numpy."""
    if kind == "time_augment":
        return g[:, :, :-1].copy()
    d = g.shape[2] // 2
    lead, lag = g[:, :, :d], g[:, :, d:]
    out = lead[:, 0::2] + lag[:, 0::2]
    out[:, :-1] += lag[:, 1::2]
    out[:, 1:] += lead[:, 1::2]
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("kind,gkey,akey", [("time_augment", "g_ta", "adj_ta"),
                                            ("lead_lag", "g_ll", "adj_ll")])
def test_adjoint_kernel_matches_reference_golden(kind, gkey, akey):
    """sk_transform_adjoint on the reference's golden gradient: same additions
    in the same order as transform_adjoint -> bitwise."""
    from paper_2509_10613_b200 import _lib, ops
    g = golden("transforms")
    lib = _lib.load()
    n, L, d = g["x"].shape
    gt = torch.as_tensor(g[gkey], device="cuda")
    out = torch.empty((n, L, d), dtype=torch.float64, device="cuda")
    _lib.check(lib.sk_transform_adjoint(gt.data_ptr(), n, L, d, ops.transform_code(kind),
                                        out.data_ptr(), 0, torch.cuda.current_stream().cuda_stream))
    np.testing.assert_array_equal(out.cpu().numpy(), g[akey])


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["time_augment", "lead_lag"])
@pytest.mark.parametrize("lam,static", [((0, 0), None), ((1, 2), None), ((1, 0), ("rbf", 0.8))])
def test_fused_transform_batch(oracle, kind, lam, static):
    """Transform inside the kernels' input preparation: values bitwise those of
    the materialised transform (same subtractions), gradients vs the oracle on
    the transformed paths mapped back by the reference's adjoint."""
    import paper_2509_10613_b200 as sk
    from paper_2509_10613_b200 import ops
    rng = np.random.default_rng(11)
    x = make_paths(rng, 4, 20, 3)
    y = make_paths(rng, 4, 15, 3)
    cot = rng.standard_normal(4)
    kind_c, sigma = (1, static[1]) if static else (0, 1.0)
    xt = path_transform(torch.as_tensor(x), kind).numpy()
    yt = path_transform(torch.as_tensor(y), kind).numpy()
    cu = lambda a: torch.as_tensor(a, device="cuda")
    v, gx, gy = ops.backward_batch(cu(x), cu(y), *lam, kind_c, sigma, cu(cot), want_values=True,
                                   transform=kind)
    k_mat = ops.forward_batch(cu(xt), cu(yt), *lam, kind_c, sigma).cpu().numpy()
    k_fused = ops.forward_batch(cu(x), cu(y), *lam, kind_c, sigma, transform=kind).cpu().numpy()
    np.testing.assert_array_equal(k_fused, k_mat)
    np.testing.assert_array_equal(v.cpu().numpy(), k_mat)
    wv, wxt, wyt = oracle.kernel_batch_backward(xt, yt, *lam, cot, static)
    assert rel_err(v.cpu().numpy(), wv) < 1e-10
    assert rel_err(gx.cpu().numpy(), _np_adjoint(wxt, kind)) < 1e-10
    assert rel_err(gy.cpu().numpy(), _np_adjoint(wyt, kind)) < 1e-10
    # public autograd API
    X = cu(x).requires_grad_(True)
    k = sk.sig_kernel(X, cu(y), dyadic_order=lam,
                      static_kernel=sk.RBFKernel(static[1]) if static else None, transform=kind)
    (k * cu(cot)).sum().backward()
    np.testing.assert_array_equal(k.detach().cpu().numpy(), k_mat)
    assert rel_err(X.grad.cpu().numpy(), _np_adjoint(wxt, kind)) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["time_augment", "lead_lag"])
def test_fused_transform_gram(oracle, kind):
    """Gram (symmetric DMMA path at lambda 0, and cross) with the transform
    inside the call: G, fused value + gradient, exact accumulators."""
    import paper_2509_10613_b200 as sk
    from paper_2509_10613_b200 import ops
    rng = np.random.default_rng(12)
    X = make_paths(rng, 10, 17, 3)
    Y = make_paths(rng, 6, 17, 3)
    C = rng.standard_normal((10, 10))
    cu = lambda a: torch.as_tensor(a, device="cuda")
    Xt = path_transform(torch.as_tensor(X), kind).numpy()
    Yt = path_transform(torch.as_tensor(Y), kind).numpy()
    G = sk.sig_kernel_gram(cu(X), transform=kind).cpu().numpy()
    np.testing.assert_array_equal(G, ops.forward_gram(cu(Xt), None, 0, 0, 0, 1.0).cpu().numpy())
    Gv, gx, _ = sk.sig_kernel_gram_value_and_grad(cu(X), None, cu(C), transform=kind)
    np.testing.assert_array_equal(Gv.cpu().numpy(), G)
    want = _np_adjoint(oracle.gram_backward(Xt, None, C, 0, 0), kind)
    assert rel_err(gx.cpu().numpy(), want) < 1e-10
    acc = ops.GradAcc(10, 17, 3, torch.device("cuda"), transform=kind).init(cu(C), 10, 10, True)
    for rg in ((0, 8), (8, 10)):
        ops.backward_gram(cu(X), None, 0, 0, 0, 1.0, cu(C), rows=rg, acc_x=acc, transform=kind)
    np.testing.assert_array_equal(acc.finalize().cpu().numpy(), gx.cpu().numpy())
    # cross Gram, dyadic order 1, autograd
    Cx = rng.standard_normal((10, 6))
    xt_ = cu(X).requires_grad_(True)
    yt_ = cu(Y).requires_grad_(True)
    Gc = sk.sig_kernel_gram(xt_, yt_, dyadic_order=1, transform=kind)
    (Gc * cu(Cx)).sum().backward()
    assert rel_err(Gc.detach().cpu().numpy(), oracle.kernel_gram(Xt, Yt, 1, 1)) < 1e-10
    wx, wy = oracle.gram_backward(Xt, Yt, Cx, 1, 1)
    assert rel_err(xt_.grad.cpu().numpy(), _np_adjoint(wx, kind)) < 1e-10
    assert rel_err(yt_.grad.cpu().numpy(), _np_adjoint(wy, kind)) < 1e-10


@pytest.mark.gpu
def test_fused_transform_fp32(oracle):
    import paper_2509_10613_b200 as sk
    rng = np.random.default_rng(13)
    x = make_paths(rng, 8, 100, 4).astype(np.float32)
    y = make_paths(rng, 8, 100, 4).astype(np.float32)
    for kind in ("time_augment", "lead_lag"):
        k = sk.sig_kernel(torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda"),
                          transform=kind, precision="fp32").cpu().numpy()
        xt = path_transform(torch.as_tensor(x.astype(np.float64)), kind).numpy()
        yt = path_transform(torch.as_tensor(y.astype(np.float64)), kind).numpy()
        assert rel_err(k, oracle.kernel_batch(xt, yt, 0, 0)) < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("kind,gkey,akey", [("time_augment", "g_ta", "adj_ta"),
                                            ("lead_lag", "g_ll", "adj_ll")])
def test_sigcore_facade_transforms_match_reference(kind, gkey, akey):
    """The facade's reference-named utilities (transforms.py:37-135) against
    the reference's own outputs (tests/golden/transforms.npz, bitwise), and
    fused_increments == np.diff of the transformed path."""
    from paper_2509_10613_b200 import sigcore_compat as sc
    g = golden("transforms")
    x = g["x"]
    np.testing.assert_array_equal(sc.transform(x, kind), g[kind])
    np.testing.assert_array_equal(sc.transform(x[0], kind), g[kind][0])
    np.testing.assert_array_equal(sc.transform_adjoint(g[gkey], kind), g[akey])
    inc = sc.fused_increments(x, kind)
    np.testing.assert_array_equal(inc, np.diff(g[kind], axis=1))
    assert sc.effective_dim(x.shape[2], kind) == g[kind].shape[2]
    assert sc.effective_length(x.shape[1], kind) == g[kind].shape[1]
    with pytest.raises(sc.InvalidArgument):
        sc.transform(x, "bogus")
