"""GPU parity of the DMMA (FP64 tensor-core) Gram kernels.

The DMMA kernels serve linear-kernel Gram tiles at dyadic order 0 (BASELINE
configs C3 / C5).  They must agree with the C oracle (rel 1e-10)
and bitwise with the r01 FMA-pipe kernels (SK_NO_MMA=1), which form <dx, dy>
in the same sequential FMA order (tools/dmma_probe.cu)."""

import os

import numpy as np
import pytest
import torch

from conftest import random_paths, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def mods():
    from oracle import oracle as orc
    from paper_2509_10613_b200 import ops
    return ops, orc


def cu(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")


class _NoMMA:
    def __enter__(self):
        os.environ["SK_NO_MMA"] = "1"

    def __exit__(self, *a):
        os.environ.pop("SK_NO_MMA", None)


SHAPES = [  # (n1, n2, L, d)
    (1, 1, 2, 1), (3, 3, 3, 2), (9, 9, 9, 4), (8, 8, 17, 5), (17, 17, 33, 8),
    (5, 12, 64, 3), (16, 16, 70, 16), (11, 11, 130, 13), (24, 24, 41, 7), (4, 4, 300, 16),
    (10, 10, 45, 17), (9, 13, 60, 32), (12, 12, 129, 24),  # DP = 32 instance
]


@pytest.mark.parametrize("n1,n2,L,d", SHAPES)
def test_gram_forward_mma(mods, n1, n2, L, d):
    ops, orc = mods
    rng = np.random.default_rng(n1 * 1000 + L * 10 + d)
    X = random_paths(rng, n1, L, d)
    Y = random_paths(rng, n2, L, d) if n1 != n2 else None
    want = orc.kernel_gram(X, Y, 0, 0)
    got = ops.forward_gram(cu(X), None if Y is None else cu(Y), 0, 0, 0, 1.0).cpu().numpy()
    assert rel_err(got, want) < TOL
    with _NoMMA():
        old = ops.forward_gram(cu(X), None if Y is None else cu(Y), 0, 0, 0, 1.0).cpu().numpy()
    np.testing.assert_array_equal(got, old)
    if Y is None:
        np.testing.assert_array_equal(got, got.T)


@pytest.mark.parametrize("n1,n2,L1,L2,d,l1,l2", [
    (9, 9, 20, 20, 4, 1, 1), (7, 7, 13, 13, 8, 2, 2), (6, 11, 17, 15, 5, 1, 2),
    (10, 10, 9, 9, 16, 3, 0), (5, 8, 30, 12, 3, 0, 2), (12, 12, 33, 33, 24, 1, 1),
    (4, 6, 25, 40, 8, 2, 1),  # longer columns' fine axis: the cross Gram swaps
])
def test_gram_forward_mma_dyadic(mods, n1, n2, L1, L2, d, l1, l2):
    """DMMA Gram forward at dyadic orders > 0 (coarse p tiles, duplicated
    coarse rows in the B operand, a tile spanning 8 << lam2 fine columns):
    vs the oracle, and bitwise the FMA-pipe kernels' values (same p chain)."""
    ops, orc = mods
    rng = np.random.default_rng(n1 * 100 + L1 + d + l1 + 7 * l2)
    X = random_paths(rng, n1, L1, d)
    Y = random_paths(rng, n2, L2, d) if (n1 != n2 or L1 != L2) else None
    want = orc.kernel_gram(X, Y, l1, l2)
    got = ops.forward_gram(cu(X), None if Y is None else cu(Y), l1, l2, 0, 1.0).cpu().numpy()
    assert rel_err(got, want) < TOL
    with _NoMMA():
        old = ops.forward_gram(cu(X), None if Y is None else cu(Y), l1, l2, 0, 1.0).cpu().numpy()
    np.testing.assert_array_equal(got, old)


@pytest.mark.parametrize("n1,n2,L1,L2,d,l1,l2", [
    (9, 9, 15, 15, 16, 1, 1), (7, 7, 11, 11, 12, 2, 1), (6, 9, 13, 10, 16, 0, 2),
    (10, 10, 9, 9, 10, 1, 0), (5, 7, 12, 17, 16, 1, 1),  # longer columns: swapped cross Gram
])
def test_gram_backward_mma_dyadic(mods, n1, n2, L1, L2, d, l1, l2):
    """DMMA Gram backward at dyadic orders > 0 (opt-in DY instance: coarse p
    tiles, fine -> coarse sums of the increment gradients, the dyadic factor
    on the dY side): G and both gradients vs the oracle and the FMA pipe."""
    ops, orc = mods
    rng = np.random.default_rng(n1 * 31 + L1 + d + 5 * l1 + l2)
    X = random_paths(rng, n1, L1, d)
    Y = random_paths(rng, n2, L2, d) if (n1 != n2 or L1 != L2) else None
    C = rng.standard_normal((n1, n2))
    os.environ["SK_MMA_DY"] = "1"  # the DY instance is opt-in (sk_capi.cu plan_backward)
    try:
        G, gx, gy = ops.value_and_grad_gram(cu(X), None if Y is None else cu(Y), l1, l2, 0,
                                            1.0, cu(C))
        bx, by = ops.backward_gram(cu(X), None if Y is None else cu(Y), l1, l2, 0, 1.0, cu(C))
    finally:
        os.environ.pop("SK_MMA_DY", None)
    assert rel_err(G.cpu().numpy(), orc.kernel_gram(X, Y, l1, l2)) < TOL
    want = orc.gram_backward(X, Y, C, l1, l2)
    if Y is None:
        assert rel_err(gx.cpu().numpy(), want) < TOL
    else:
        assert rel_err(gx.cpu().numpy(), want[0]) < TOL
        assert rel_err(gy.cpu().numpy(), want[1]) < TOL
    np.testing.assert_array_equal(bx.cpu().numpy(), gx.cpu().numpy())
    with _NoMMA():
        ox, oy = ops.backward_gram(cu(X), None if Y is None else cu(Y), l1, l2, 0, 1.0, cu(C))
    assert rel_err(gx.cpu().numpy(), ox.cpu().numpy()) < 1e-12


def test_gram_forward_mma_cross_lengths(mods):
    ops, orc = mods
    rng = np.random.default_rng(3)
    X = random_paths(rng, 6, 40, 6)
    Y = random_paths(rng, 5, 23, 6)  # shorter columns: no orientation swap
    got = ops.forward_gram(cu(X), cu(Y), 0, 0, 0, 1.0).cpu().numpy()
    assert rel_err(got, orc.kernel_gram(X, Y, 0, 0)) < TOL
    got2 = ops.forward_gram(cu(Y), cu(X), 0, 0, 0, 1.0).cpu().numpy()  # swapped orientation
    np.testing.assert_array_equal(got2, got.T)


def test_gram_forward_mma_row_range(mods):
    ops, orc = mods
    rng = np.random.default_rng(4)
    X = random_paths(rng, 20, 33, 8)
    full = orc.kernel_gram(X, None, 0, 0)
    got = ops.forward_gram(cu(X), None, 0, 0, 0, 1.0, rows=(5, 13)).cpu().numpy()
    # a symmetric row block holds the upper triangle (b >= a); the rest is the
    # all-gather's job (gram_dist.py)
    for i, a in enumerate(range(5, 13)):
        assert rel_err(got[i, a:], full[a, a:]) < TOL


BWD_SHAPES = [  # (n1, n2, L, d) -- DMMA backward serves d <= 16 (d <= 4 padded to 8)
    (1, 1, 2, 5), (3, 3, 3, 6), (6, 6, 19, 1), (7, 9, 25, 3), (9, 9, 40, 4), (9, 9, 9, 8), (8, 8, 17, 5), (17, 17, 33, 8),
    (5, 12, 64, 7), (16, 16, 70, 16), (11, 11, 130, 13), (10, 10, 41, 12),
]


@pytest.mark.parametrize("n1,n2,L,d", BWD_SHAPES)
def test_gram_backward_mma(mods, n1, n2, L, d):
    ops, orc = mods
    rng = np.random.default_rng(n1 * 7 + L * 3 + d)
    X = random_paths(rng, n1, L, d)
    Y = random_paths(rng, n2, L, d) if n1 != n2 else None
    C = rng.standard_normal((n1, n2))
    want = orc.gram_backward(X, Y, C, 0, 0)
    gx, gy = ops.backward_gram(cu(X), None if Y is None else cu(Y), 0, 0, 0, 1.0, cu(C))
    if Y is None:
        assert rel_err(gx.cpu().numpy(), want) < TOL
    else:
        assert rel_err(gx.cpu().numpy(), want[0]) < TOL
        assert rel_err(gy.cpu().numpy(), want[1]) < TOL
    with _NoMMA():
        ox, oy = ops.backward_gram(cu(X), None if Y is None else cu(Y), 0, 0, 0, 1.0, cu(C))
    assert rel_err(gx.cpu().numpy(), ox.cpu().numpy()) < 1e-13


def test_gram_backward_mma_row_blocks_sum(mods):
    """Row blocks (the multi-GPU split, gram_dist.py) add up to the full gradient:
    bitwise through the exact accumulators for tile-aligned blocks (the ones
    gram_dist makes), within rounding for arbitrary blocks summed in fp64."""
    ops, orc = mods
    rng = np.random.default_rng(11)
    X = random_paths(rng, 21, 37, 8)
    C = rng.standard_normal((21, 21))
    full, _ = ops.backward_gram(cu(X), None, 0, 0, 0, 1.0, cu(C))
    acc = ops.GradAcc(21, 37, 8, torch.device("cuda")).init(cu(C), 21, 21, True)
    for r in ((0, 8), (8, 16), (16, 21)):
        ops.backward_gram(cu(X), None, 0, 0, 0, 1.0, cu(C), rows=r, acc_x=acc)
    np.testing.assert_array_equal(acc.finalize().cpu().numpy(), full.cpu().numpy())
    g = torch.zeros_like(full)
    for r in ((0, 4), (4, 13), (13, 21)):
        ops.backward_gram(cu(X), None, 0, 0, 0, 1.0, cu(C), rows=r, grad_x=g)
    assert rel_err(g.cpu().numpy(), full.cpu().numpy()) < 1e-13
    assert rel_err(full.cpu().numpy(), orc.gram_backward(X, None, C, 0, 0)) < TOL


@pytest.mark.parametrize("n1,n2,L,d,lam", [(9, 9, 33, 8, 0), (6, 11, 40, 16, 0), (12, 12, 70, 5, 0),
                                           (5, 5, 17, 3, 1), (4, 7, 12, 6, 1)])
def test_value_and_grad_gram(mods, n1, n2, L, d, lam):
    """Fused G + gradient == separate forward Gram and backward (bitwise for the
    values: same forward arithmetic), vs the oracle within 1e-10."""
    import paper_2509_10613_b200 as sk
    ops, orc = mods
    rng = np.random.default_rng(n1 + 3 * L + d)
    X = random_paths(rng, n1, L, d)
    Y = None if n1 == n2 else random_paths(rng, n2, L, d)
    C = rng.standard_normal((n1, n2))
    G, gx, gy = sk.sig_kernel_gram_value_and_grad(cu(X), None if Y is None else cu(Y), cu(C),
                                                  dyadic_order=lam)
    Gf = ops.forward_gram(cu(X), None if Y is None else cu(Y), lam, lam, 0, 1.0)
    np.testing.assert_array_equal(G.cpu().numpy(), Gf.cpu().numpy())
    assert rel_err(G.cpu().numpy(), orc.kernel_gram(X, Y, lam, lam)) < TOL
    want = orc.gram_backward(X, Y, C, lam, lam)
    if Y is None:
        assert gy is None
        assert rel_err(gx.cpu().numpy(), want) < TOL
    else:
        assert rel_err(gx.cpu().numpy(), want[0]) < TOL
        assert rel_err(gy.cpu().numpy(), want[1]) < TOL


def test_value_and_grad_gram_long_and_ragged(mods):
    """Long paths (many 8-column tiles, several strips) and a tile count that is
    not a multiple of 8 pairs, symmetric, against the oracle on a sub-block."""
    import paper_2509_10613_b200 as sk
    ops, orc = mods
    rng = np.random.default_rng(21)
    X = random_paths(rng, 13, 1030, 9)
    C = rng.standard_normal((13, 13))
    G, gx, _ = sk.sig_kernel_gram_value_and_grad(cu(X), None, cu(C))
    assert rel_err(G.cpu().numpy(), orc.kernel_gram(X, None, 0, 0)) < TOL
    assert rel_err(gx.cpu().numpy(), orc.gram_backward(X, None, C, 0, 0)) < TOL


def test_value_and_grad_row_blocks_assemble(mods):
    """The multi-GPU split (gram_dist.row_blocks) run sequentially on one GPU:
    the row blocks' G rows and summed gradients equal the single call."""
    import paper_2509_10613_b200 as sk
    from paper_2509_10613_b200 import gram_dist
    ops, _ = mods
    rng = np.random.default_rng(22)
    X = random_paths(rng, 19, 45, 8)
    C = torch.ones((19, 19), dtype=torch.float64, device="cuda")
    G, gx, _ = sk.sig_kernel_gram_value_and_grad(cu(X), None, C)
    world = 3
    Gs = torch.zeros_like(G)
    gs = torch.zeros_like(gx)
    for r in range(world):
        for rg in gram_dist.row_blocks(19, world, r, True):
            out, _, _ = ops.value_and_grad_gram(cu(X), None, 0, 0, 0, 1.0, C, rows=rg, grad_x=gs)
            Gs[rg[0]:rg[1]] = out
    ops.mirror_upper(Gs)
    np.testing.assert_array_equal(Gs.cpu().numpy(), G.cpu().numpy())
    assert rel_err(gs.cpu().numpy(), gx.cpu().numpy()) < 1e-13


def test_value_and_grad_gram_swapped_orientation(mods):
    """Cross Gram whose column paths are longer (the orientation swap of
    kernel.py:164-170: r01 kernels) still returns G and both gradients."""
    import paper_2509_10613_b200 as sk
    ops, orc = mods
    rng = np.random.default_rng(31)
    X = random_paths(rng, 5, 14, 6)
    Y = random_paths(rng, 6, 29, 6)
    C = rng.standard_normal((5, 6))
    G, gx, gy = sk.sig_kernel_gram_value_and_grad(cu(X), cu(Y), cu(C))
    assert rel_err(G.cpu().numpy(), orc.kernel_gram(X, Y, 0, 0)) < TOL
    wx, wy = orc.gram_backward(X, Y, C, 0, 0)
    assert rel_err(gx.cpu().numpy(), wx) < TOL
    assert rel_err(gy.cpu().numpy(), wy) < TOL


@pytest.mark.parametrize("lam", [0, 1])
def test_sig_mmd(mods, lam):
    """MMD^2 from the Gram hot path: value vs the oracle Grams, gradients of the
    fused API vs autograd vs the oracle Gram backward."""
    import paper_2509_10613_b200 as sk
    ops, orc = mods
    rng = np.random.default_rng(41 + lam)
    X = random_paths(rng, 7, 30, 8)
    Y = random_paths(rng, 5, 30, 8)
    want = (orc.kernel_gram(X, None, lam, lam).mean() + orc.kernel_gram(Y, None, lam, lam).mean()
            - 2 * orc.kernel_gram(X, Y, lam, lam).mean())
    xt = cu(X).requires_grad_(True)
    yt = cu(Y).requires_grad_(True)
    v = sk.sig_mmd(xt, yt, lam)
    v.backward()
    v2, gx2, gy2 = sk.sig_mmd_value_and_grad(cu(X), cu(Y), lam)
    assert abs(v.item() - want) <= 1e-10 * abs(want) + 1e-14
    assert abs(v2.item() - want) <= 1e-10 * abs(want) + 1e-14
    gxw = (orc.gram_backward(X, None, np.full((7, 7), 1 / 49), lam, lam)
           + orc.gram_backward(X, Y, np.full((7, 5), -2 / 35), lam, lam)[0])
    gyw = (orc.gram_backward(Y, None, np.full((5, 5), 1 / 25), lam, lam)
           + orc.gram_backward(X, Y, np.full((7, 5), -2 / 35), lam, lam)[1])
    assert rel_err(xt.grad.cpu().numpy(), gxw) < TOL
    assert rel_err(yt.grad.cpu().numpy(), gyw) < TOL
    assert rel_err(gx2.cpu().numpy(), gxw) < TOL
    assert rel_err(gy2.cpu().numpy(), gyw) < TOL


def test_sig_mmd_same_sample(mods):
    """MMD^2(X, X) = 0 with zero gradients (a minimum), through the fused API
    with the same tensor twice (the cross term must stay a cross
    Gram); dtype follows the input."""
    import paper_2509_10613_b200 as sk
    rng = np.random.default_rng(5)
    X = random_paths(rng, 6, 25, 4)
    xt = cu(X)
    v, gx, gy = sk.sig_mmd_value_and_grad(xt, xt)
    assert abs(v.item()) < 1e-13
    assert gx.abs().max().item() < 1e-12 and gy.abs().max().item() < 1e-12
    v32, _, _ = sk.sig_mmd_value_and_grad(xt.float(), xt.float())
    assert v32.dtype == torch.float32


@pytest.mark.parametrize("no_mma", [False, True])
def test_backward_workspace_budget_caps_slots(mods, no_mma):
    """With a tiny workspace budget the backward runs on fewer resident slots
    (each warp loops over more tiles) and returns the same gradient."""
    ops, orc = mods
    rng = np.random.default_rng(51)
    X = random_paths(rng, 20, 37, 8)
    C = rng.standard_normal((20, 20))
    if no_mma:
        os.environ["SK_NO_MMA"] = "1"
    try:
        full, _ = ops.backward_gram(cu(X), None, 0, 0, 0, 1.0, cu(C))
        os.environ["SK_WS_BUDGET_GB"] = "0.000001"
        capped, _ = ops.backward_gram(cu(X), None, 0, 0, 0, 1.0, cu(C))
    finally:
        os.environ.pop("SK_WS_BUDGET_GB", None)
        os.environ.pop("SK_NO_MMA", None)
    assert rel_err(capped.cpu().numpy(), full.cpu().numpy()) < 1e-13
    assert rel_err(full.cpu().numpy(), orc.gram_backward(X, None, C, 0, 0)) < TOL


def test_cross_gram_forward_longer_y_bitwise_row_range():
    """A whole cross Gram whose y paths are longer is solved as G^T on the DMMA
    tiles (ops._transpose_cross): bitwise equal to the swapped-orientation
    row-range call and to the oracle within 1e-10."""
    from paper_2509_10613_b200 import ops
    from oracle import oracle as orc
    rng = np.random.default_rng(31)
    X = np.cumsum(rng.standard_normal((13, 40, 16)) / 7, axis=1)
    Y = np.cumsum(rng.standard_normal((9, 57, 16)) / 7, axis=1)
    xt, yt = torch.as_tensor(X, device="cuda"), torch.as_tensor(Y, device="cuda")
    for lam in ((0, 0), (1, 0)):
        G = ops.forward_gram(xt, yt, lam[0], lam[1], 0, 1.0)
        Gr = ops.forward_gram(xt, yt, lam[0], lam[1], 0, 1.0, rows=(0, 13))
        assert torch.equal(G, Gr)
        want = orc.kernel_gram(X, Y, lam[0], lam[1])
        assert np.abs(G.cpu().numpy() - want).max() / np.abs(want).max() < 1e-10


@pytest.mark.parametrize("tf", [None, "lead_lag"])
def test_cross_gram_backward_longer_y_transposed(tf):
    """Cross Grams whose y paths are longer: the backward runs as G^T on the
    DMMA kernels with the row range of G as the column range of G^T
    (sk_backward_gram_acc_cols).  Whole call vs the oracle, row splits with
    accumulators bitwise the whole call, values bitwise the forward."""
    from paper_2509_10613_b200 import ops
    from oracle import oracle as orc
    rng = np.random.default_rng(32)
    d = 3 if tf else 8
    X = np.cumsum(rng.standard_normal((21, 30, d)) / 6, axis=1)
    Y = np.cumsum(rng.standard_normal((11, 45, d)) / 6, axis=1)
    C = rng.standard_normal((21, 11))
    xt, yt = torch.as_tensor(X, device="cuda"), torch.as_tensor(Y, device="cuda")
    Ct = torch.as_tensor(C, device="cuda")
    G, gx, gy = ops.value_and_grad_gram(xt, yt, 0, 0, 0, 1.0, Ct, transform=tf)
    assert torch.equal(G, ops.forward_gram(xt, yt, 0, 0, 0, 1.0, transform=tf))
    if tf is None:
        wx, wy = orc.gram_backward(X, Y, C, 0, 0)
        assert rel_err(gx.cpu().numpy(), wx) < 1e-10
        assert rel_err(gy.cpu().numpy(), wy) < 1e-10
        assert rel_err(G.cpu().numpy(), orc.kernel_gram(X, Y, 0, 0)) < 1e-10
    ax = ops.GradAcc(21, 30, d, xt.device, tf).init(Ct, 21, 11, False)
    ay = ops.GradAcc(11, 45, d, xt.device, tf).init(Ct, 21, 11, False)
    for rg in ((0, 8), (8, 16), (16, 21)):
        ops.backward_gram(xt, yt, 0, 0, 0, 1.0, Ct, rows=rg, acc_x=ax, acc_y=ay, transform=tf)
    assert torch.equal(ax.finalize(), gx) and torch.equal(ay.finalize(), gy)
