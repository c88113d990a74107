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
    if n >= 64 * world:
        assert max(counts) / (sum(counts) / world) < 1.01  # balanced to 1%


def test_row_blocks_cross():
    rg = [gram_dist.row_blocks(10, 3, r, False) for r in range(3)]
    assert rg == [[(0, 4)], [(4, 8)], [(8, 10)]]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, m = 9, 4
    full = torch.arange(n * m, dtype=torch.float64).reshape(n, m)
    ranges_all = [gram_dist.row_blocks(n, world, r, True) for r in range(world)]
    mine = torch.cat([full[lo:hi] for lo, hi in ranges_all[rank]], 0)
    G = gram_dist._gather_rows(mine, ranges_all, n, m, None)
    part = torch.full((3, 2), float(rank + 1), dtype=torch.float64)
    s = gram_dist._gather_sum(part, None)
    q.put((rank, bool(torch.equal(G, full)), s.tolist()))
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
    for rank, ok, s in res:
        assert ok
        assert np.allclose(s, 3.0)


def _fused_worker(rank, world, port, q):
    """gram_dist.value_and_grad_sharded with the per-block GPU call replaced by
    the C oracle on the same row block (test infrastructure only)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_2509_10613_b200 import ops

    def fake_value_and_grad(x, y, l1, l2, kind, sigma, cot, rows=None, out=None, grad_x=None,
                            grad_y=None):
        X = x.numpy()
        n = X.shape[0]
        r0, r1 = rows
        G = orc.kernel_gram(X, None, l1, l2)
        gx = np.zeros_like(X)
        rc = orc.lib().sko_gram_backward(orc._p(X), orc._p(X), n, n, X.shape[1], X.shape[1],
                                         X.shape[2], l1, l2, 0, 1.0, 1, r0, r1,
                                         orc._p(np.ascontiguousarray(cot.numpy())), orc._p(gx),
                                         orc._p(np.zeros(1)), 1)
        assert rc == 0
        grad_x += torch.from_numpy(gx)
        blk = torch.from_numpy(G[r0:r1].copy())
        blk[:, :r0] = float("nan")  # rows of a symmetric block hold b >= r0 only
        return blk, grad_x, grad_y

    def fake_mirror(G):
        iu = torch.triu_indices(G.shape[0], G.shape[0], 1)
        G[iu[1], iu[0]] = G[iu[0], iu[1]]
        return G

    ops.value_and_grad_gram = fake_value_and_grad
    ops.mirror_upper = fake_mirror
    rng = np.random.default_rng(5)
    X = torch.from_numpy(np.cumsum(rng.standard_normal((11, 7, 2)) / 3.0, axis=1))
    C = torch.from_numpy(rng.standard_normal((11, 11)))
    G, gx, gy = gram_dist.value_and_grad_sharded(X, None, C)
    Gw = orc.kernel_gram(X.numpy(), None, 0, 0)
    gw = orc.gram_backward(X.numpy(), None, C.numpy(), 0, 0)
    ok = (gy is None and np.allclose(G.numpy(), Gw, rtol=0, atol=1e-13)
          and np.abs(gx.numpy() - gw).max() <= 1e-12 * np.abs(gw).max())
    q.put((rank, bool(ok)))
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
    assert all(ok for _, ok in res), res
