"""Host logic of the sharded Gram (gram_dist.py) on CPU: row-block balance and
the all-gather assembly / fixed-order gradient sum with gloo, world size 2."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_10613_b200 import gram_dist


@pytest.mark.parametrize("n,world", [(1024, 2), (1024, 8), (8192, 8), (37, 4), (5, 8)])
def test_row_blocks_cover_and_balance(n, world):
    seen = []
    counts = []
    for r in range(world):
        rg = gram_dist.row_blocks(n, world, r, True)
        for lo, hi in rg:
            seen.extend(range(lo, hi))
        counts.append(gram_dist.pair_count(rg, n, True))
    assert sorted(seen) == list(range(n))
    assert sum(counts) == n * (n + 1) // 2
    # one contiguous range per rank (one kernel launch), balanced in the fused
    # kernel's work units (super-items) to within one 8-row block of them
    items = [gram_dist.super_item_count(gram_dist.row_blocks(n, world, r, True), n)
             for r in range(world)]
    assert sum(items) == gram_dist.super_item_count([(0, n)], n)
    gran = max(gram_dist._super_items_per_block(n))
    assert max(items) - sum(items) / world <= gran
    assert all(len(gram_dist.row_blocks(n, world, r, True)) <= 1 for r in range(world))


def test_row_blocks_c3_one_wave_per_rank_at_8():
    """C3 (n = 1024) on 8 GPUs: every rank's items fit one wave of the fused
    kernel's 1184 resident warps (148 SMs x 8), against 7 waves on one GPU."""
    items = [gram_dist.super_item_count(gram_dist.row_blocks(1024, 8, r, True), 1024)
             for r in range(8)]
    assert max(items) <= 148 * 8 < gram_dist.super_item_count([(0, 1024)], 1024)


def test_row_blocks_cross():
    rg = [gram_dist.row_blocks(10, 3, r, False) for r in range(3)]
    assert rg == [[(0, 8)], [(8, 10)], []]
    rg = [gram_dist.row_blocks(100, 3, r, False) for r in range(3)]
    assert rg == [[(0, 40)], [(40, 80)], [(80, 100)]]


@pytest.mark.parametrize("n,world", [(1024, 8), (37, 4), (1000, 3)])
def test_row_blocks_tile_aligned(n, world):
    """Every boundary is a multiple of the 8-path Gram tile (or n): each rank
    sees the same tiles as a one-GPU run (bitwise-equal exact gradients)."""
    for sym in (True, False):
        for r in range(world):
            for lo, hi in gram_dist.row_blocks(n, world, r, sym):
                assert lo % gram_dist.TILE == 0
                assert hi % gram_dist.TILE == 0 or hi == n


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, m = 19, 23
    full = torch.arange(n * m, dtype=torch.float64).reshape(n, m)
    ok = True
    for sym in (False, True):
        nn = n if sym else m
        ref = full[:, :nn].clone()
        ranges_all = [gram_dist.row_blocks(n, world, r, sym) for r in range(world)]
        mine = torch.cat([ref[lo:hi] for lo, hi in ranges_all[rank]], 0)
        G = gram_dist._gather_rows(mine, ranges_all, n, nn, None, symmetric=sym)
        if sym:  # only the upper triangle travels
            iu = torch.triu_indices(n, n)
            ok = ok and torch.equal(G[iu[0], iu[1]], ref[iu[0], iu[1]])
        else:
            ok = ok and torch.equal(G, ref)
    # exact accumulators: limbs add as integers, metadata by MAX
    acc = _CpuAcc(2, 3, 1)
    acc.limbs.fill_(rank + 1)
    acc.meta[1] = rank
    gram_dist._allreduce_acc(acc, None)
    ok = ok and bool((acc.limbs == 3).all()) and int(acc.meta[1]) == 1
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


def test_gather_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok in res:
        assert ok


class _CpuAcc:
    """CPU stand-in for ops.GradAcc with the same limb format (tests/fixpt_ref.py)."""

    def __init__(self, n, L, d, device=None):
        self.shape = (n, L, d)
        self.blob = torch.zeros(8 + n * L * d * 4, dtype=torch.int64)
        self.meta = self.blob[:8]
        self.limbs = self.blob[8:]

    def init(self, cot, n1, n2, symmetric):
        import fixpt_ref as fx
        self.E = fx.anchor(float(cot.abs().max()), max(n1, n2) * (2.0 if symmetric else 1.0))
        self.blob.zero_()
        return self

    def add(self, g):
        import fixpt_ref as fx
        acc = self.limbs.view(-1, 4).numpy()
        fx.accumulate(acc, g.ravel(), self.E)

    def finalize(self):
        import fixpt_ref as fx
        return torch.from_numpy(fx.finalize(self.limbs.view(-1, 4).numpy(), self.E)
                                .reshape(self.shape))


def _fused_worker(rank, world, port, q):
    """gram_dist.value_and_grad_sharded with the per-block GPU call replaced by
    the C oracle on the same row block (test infrastructure only), its gradient
    added into the CPU accumulator stand-in."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_2509_10613_b200 import ops

    def block_grad(X, cot, l1, l2, r0, r1):
        n = X.shape[0]
        gx = np.zeros_like(X)
        rc = orc.lib().sko_gram_backward(orc._p(X), orc._p(X), n, n, X.shape[1], X.shape[1],
                                         X.shape[2], l1, l2, 0, 1.0, 1, r0, r1,
                                         orc._p(np.ascontiguousarray(cot.numpy())), orc._p(gx),
                                         orc._p(np.zeros(1)), 1)
        assert rc == 0
        return gx

    def fake_value_and_grad(x, y, l1, l2, kind, sigma, cot, rows=None, out=None, grad_x=None,
                            grad_y=None, acc_x=None, acc_y=None):
        X = x.numpy()
        r0, r1 = rows
        G = orc.kernel_gram(X, None, l1, l2)
        acc_x.add(block_grad(X, cot, l1, l2, r0, r1))
        blk = torch.from_numpy(G[r0:r1].copy())
        blk[:, :r0] = float("nan")  # rows of a symmetric block hold b >= r0 only
        return blk, acc_x, acc_y

    def fake_mirror(G):
        iu = torch.triu_indices(G.shape[0], G.shape[0], 1)
        G[iu[1], iu[0]] = G[iu[0], iu[1]]
        return G

    ops.value_and_grad_gram = fake_value_and_grad
    ops.mirror_upper = fake_mirror
    ops.GradAcc = _CpuAcc
    rng = np.random.default_rng(5)
    X = torch.from_numpy(np.cumsum(rng.standard_normal((19, 7, 2)) / 3.0, axis=1))
    C = torch.from_numpy(rng.standard_normal((19, 19)))
    G, gx, gy = gram_dist.value_and_grad_sharded(X, None, C)
    Gw = orc.kernel_gram(X.numpy(), None, 0, 0)
    gw = orc.gram_backward(X.numpy(), None, C.numpy(), 0, 0)
    # the one-GPU accumulation over the same row blocks, in one accumulator
    one = _CpuAcc(*X.shape).init(C, 19, 19, True)
    for r in range(world):
        for lo, hi in gram_dist.row_blocks(19, world, r, True):
            one.add(block_grad(X.numpy(), C, 0, 0, lo, hi))
    ok = (gy is None and np.allclose(G.numpy(), Gw, rtol=0, atol=1e-13)
          and np.abs(gx.numpy() - gw).max() <= 1e-12 * np.abs(gw).max()
          and np.array_equal(gx.numpy(), one.finalize().numpy()))
    q.put((rank, bool(ok), gx.numpy().tobytes()))
    dist.destroy_process_group()


def test_value_and_grad_sharded_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_fused_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), [r[:2] for r in res]
    assert res[0][2] == res[1][2]  # every rank holds the same bits
