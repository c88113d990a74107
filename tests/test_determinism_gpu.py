"""Bitwise determinism of the Gram gradients (exact fixed-point accumulation,
sk_common.cuh FixAcc): run to run, across row-block splits of the Gram and
across emulated GPU counts (per-rank accumulators summed as integers, as
gram_dist's all-reduce does).  The reference contract: results may not depend
on thread count / reduction order (/root/reference/SPEC.md:261,
pkg/tests/test_kernel.py:156-171)."""

import numpy as np
import pytest
import torch

from conftest import make_paths, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from oracle import oracle as orc
    from paper_2509_10613_b200 import gram_dist, ops
    return ops, gram_dist, orc


def cu(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")


# (n1, n2 or None, L, d, lam, kind): DMMA tiles (lam 0, d <= 16, sym and cross),
# FMA-pipe kernels (lam 1; d 20; a cross Gram with longer y paths, which swaps
# the grid orientation), RBF
CASES = [(21, None, 37, 8, 0, 0), (19, 13, 41, 16, 0, 0), (17, None, 25, 5, 1, 0),
         (12, 9, 30, 20, 0, 0), (10, 7, -25, 4, 0, 0), (11, None, 20, 3, 1, 1)]


def _inputs(n1, n2, L, d, seed):
    """L < 0: y paths 5 points longer than x's (|L|)."""
    rng = np.random.default_rng(seed)
    X = make_paths(rng, n1, abs(L), d)
    Y = None if n2 is None else make_paths(rng, n2, abs(L) + (5 if L < 0 else 0), d)
    C = rng.standard_normal((n1, n1 if n2 is None else n2))
    return X, Y, C


@pytest.mark.parametrize("n1,n2,L,d,lam,kind", CASES)
def test_run_to_run_bitwise(mods, n1, n2, L, d, lam, kind):
    ops, _, orc = mods
    X, Y, C = _inputs(n1, n2, L, d, n1 + abs(L))
    outs = []
    for _ in range(3):
        gx, gy = ops.backward_gram(cu(X), None if Y is None else cu(Y), lam, lam, kind, 0.8, cu(C))
        outs.append((gx.cpu().numpy(), None if gy is None else gy.cpu().numpy()))
    for o in outs[1:]:
        np.testing.assert_array_equal(o[0], outs[0][0])
        if Y is not None:
            np.testing.assert_array_equal(o[1], outs[0][1])
    static = None if kind == 0 else ("rbf", 0.8)
    want = orc.gram_backward(X, Y, C, lam, lam, static)
    if Y is None:
        assert rel_err(outs[0][0], want) < 1e-10
    else:
        assert rel_err(outs[0][0], want[0]) < 1e-10
        assert rel_err(outs[0][1], want[1]) < 1e-10


@pytest.mark.parametrize("n1,n2,L,d,lam,kind", CASES)
def test_row_splits_and_gpu_counts_bitwise(mods, n1, n2, L, d, lam, kind):
    """Full Gram in one call == any tile-aligned split into calls == per-rank
    accumulators (gram_dist.row_blocks for 2, 4 and 8 'GPUs') summed as integers."""
    ops, gram_dist, _ = mods
    X, Y, C = _inputs(n1, n2, L, d, 7 * n1 + abs(L))
    L = abs(L)
    x, y, c = cu(X), (None if Y is None else cu(Y)), cu(C)
    sym = Y is None
    nn2 = n1 if sym else n2

    def accs():
        ax = ops.GradAcc(n1, L, d, x.device).init(c, n1, nn2, sym)
        ay = None if sym else ops.GradAcc(n2, Y.shape[1], d, x.device).init(c, n1, nn2, False)
        return ax, ay

    full_x, full_y = ops.backward_gram(x, y, lam, lam, kind, 0.8, c)
    for cuts in ([], [8], [8, 16]):
        bounds = [0] + [c for c in cuts if c < n1] + [n1]
        split = list(zip(bounds[:-1], bounds[1:]))
        ax, ay = accs()
        for rg in split:
            ops.backward_gram(x, y, lam, lam, kind, 0.8, c, rows=rg, acc_x=ax, acc_y=ay)
        np.testing.assert_array_equal(ax.finalize().cpu().numpy(), full_x.cpu().numpy())
        if not sym:
            np.testing.assert_array_equal(ay.finalize().cpu().numpy(), full_y.cpu().numpy())
    for world in (2, 4, 8):
        ranks = []
        for r in range(world):
            ax, ay = accs()
            for rg in gram_dist.row_blocks(n1, world, r, sym):
                ops.backward_gram(x, y, lam, lam, kind, 0.8, c, rows=rg, acc_x=ax, acc_y=ay)
            ranks.append((ax, ay))
        ax0, ay0 = ranks[0]
        for ax, ay in ranks[1:]:  # what the NCCL all-reduce (SUM limbs, MAX meta) does
            ax0.limbs += ax.limbs
            ax0.meta.copy_(torch.maximum(ax0.meta, ax.meta))
            if not sym:
                ay0.limbs += ay.limbs
        np.testing.assert_array_equal(ax0.finalize().cpu().numpy(), full_x.cpu().numpy())
        if not sym:
            np.testing.assert_array_equal(ay0.finalize().cpu().numpy(), full_y.cpu().numpy())


def test_value_and_grad_acc_matches_plain(mods):
    import paper_2509_10613_b200 as sk
    ops, _, _ = mods
    X, _, C = _inputs(18, None, 45, 8, 3)
    x, c = cu(X), cu(C)
    G, gx, _ = sk.sig_kernel_gram_value_and_grad(x, None, c)
    acc = ops.GradAcc(18, 45, 8, x.device).init(c, 18, 18, True)
    blocks = [ops.value_and_grad_gram(x, None, 0, 0, 0, 1.0, c, rows=rg, acc_x=acc)[0]
              for rg in ((0, 8), (8, 18))]
    np.testing.assert_array_equal(acc.finalize().cpu().numpy(), gx.cpu().numpy())
    np.testing.assert_array_equal(blocks[0].cpu().numpy()[:, 0:], G.cpu().numpy()[0:8, :])


def test_autograd_gram_backward_bitwise(mods):
    import paper_2509_10613_b200 as sk
    X, _, C = _inputs(14, None, 33, 6, 9)
    grads = []
    for _ in range(2):
        xt = cu(X).requires_grad_(True)
        (sk.sig_kernel_gram(xt) * cu(C)).sum().backward()
        grads.append(xt.grad.cpu().numpy())
    np.testing.assert_array_equal(grads[0], grads[1])


def test_nonfinite_contributions_fail_loudly(mods):
    """A kernel value that overflows (reference: inf, kernel.py:97-99) makes its
    gradient contributions non-finite: the accumulator flags it and the Gram
    gradient comes back NaN instead of a silently wrong number."""
    ops, _, _ = mods
    rng = np.random.default_rng(0)
    X = np.cumsum(rng.standard_normal((4, 64, 2)) * 40.0, axis=1)
    C = np.ones((4, 4))
    G = ops.forward_gram(cu(X), None, 0, 0, 0, 1.0).cpu().numpy()
    assert not np.isfinite(G).all()
    gx, _ = ops.backward_gram(cu(X), None, 0, 0, 0, 1.0, cu(C))
    assert np.isnan(gx.cpu().numpy()).all()


@pytest.mark.parametrize("n,L,d,lam", [(19, 45, 8, 0), (7, 30, 16, 0), (9, 25, 5, 1), (6, 20, 40, 0)])
def test_uninitialised_workspace_is_never_read(mods, n, L, d, lam):
    """Workspaces come from torch's caching allocator uninitialised: poison
    the cache with NaN first; the gradients must be unaffected (bitwise)."""
    ops, _, orc = mods
    X, _, C = _inputs(n, None, L, d, n + L)
    ref, _ = ops.backward_gram(cu(X), None, lam, lam, 0, 1.0, cu(C))
    for _ in range(3):
        junk = torch.full((64 << 20,), float("nan"), dtype=torch.float64, device="cuda")
        del junk
        got, _ = ops.backward_gram(cu(X), None, lam, lam, 0, 1.0, cu(C))
        np.testing.assert_array_equal(got.cpu().numpy(), ref.cpu().numpy())
    assert rel_err(ref.cpu().numpy(), orc.gram_backward(X, None, C, lam, lam)) < 1e-10
