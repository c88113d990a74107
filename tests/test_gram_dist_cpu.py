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
