"""Gram matrices sharded across the GPUs of one box.

One process per GPU (torch.distributed, NCCL over NVLink).  Each rank solves
one contiguous range of Gram rows, cut so every rank holds the same number of
the fused kernel's work units (the upper triangle of a symmetric Gram: row a
holds n-a pairs, so the top ranges are short), in one kernel launch.
The only data-path collectives are all-gathers: one for the assembled Gram
matrix, one for the gradients (each rank's partial gradient is gathered and
summed in fixed rank order, so every rank holds bit-identical results and
the result does not depend on NCCL's reduction order).

The reference has no distributed code; this is the north
star's "Gram tiling sharded across the 8 GPUs of one box".
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import ops
from .api import _orders
from .errors import InvalidArgument


TILE = 8  # Gram tile height of the DMMA kernels (pairs (a0 + g, b), g < 8)


SUPER_B = 8  # column chunk of the DMMA kernels' super-items (SK_SUPER_B, sk_common.cuh)


def _super_items_per_block(n: int) -> list[int]:
    """Super-items (8 rows x SUPER_B column paths, the fused kernel's work unit,
    sk_common.cuh super_chunks) of each 8-row block of a symmetric (n, n) Gram."""
    return [(n - 1) // SUPER_B - (TILE * ab) // SUPER_B + 1 for ab in range(-(-n // TILE))]


def row_blocks(n: int, world: int, rank: int, symmetric: bool = True) -> list[tuple[int, int]]:
    """Row ranges owned by `rank`.

    symmetric: ONE contiguous range per rank, its boundaries chosen so every
    rank holds the same number of the kernel's work units (super-items; row a
    of the upper triangle holds n - a pairs, so the top ranges are short) --
    one kernel launch per rank.  (Round 1/2 gave each rank two equal row
    blocks, r and 2P-1-r: two launches, the second a nearly empty wave -- C3 on
    8 GPUs would have taken 2 waves per rank against 7 on one GPU.)
    Otherwise one contiguous block of equal rows.  Boundaries are multiples of
    TILE (the kernels' 8-path Gram tile height), so every rank sees the same
    tiles as a one-GPU run and the exact gradient accumulators sum to bitwise
    the one-GPU gradient."""
    if world <= 1:
        return [(0, n)]
    if not symmetric:
        step = -(-n // world)
        step = -(-step // TILE) * TILE
        lo, hi = min(n, rank * step), min(n, (rank + 1) * step)
        return [(lo, hi)] if hi > lo else []
    w = _super_items_per_block(n)
    cum = [0]
    for v in w:
        cum.append(cum[-1] + v)
    total = cum[-1]

    def cut(r):  # 8-row block index of boundary r (nearest to r / world of the items)
        if r <= 0:
            return 0
        if r >= world:
            return len(w)
        t = total * r / world
        return min(range(len(cum)), key=lambda k: (abs(cum[k] - t), k))

    lo, hi = min(n, TILE * cut(rank)), min(n, TILE * cut(rank + 1))
    return [(lo, hi)] if hi > lo else []


def super_item_count(ranges, n: int) -> int:
    """Super-items (kernel work units) of the given row ranges of a symmetric Gram."""
    w = _super_items_per_block(n)
    return sum(sum(w[lo // TILE: -(-hi // TILE)]) for lo, hi in ranges)


def pair_count(ranges, n: int, symmetric: bool, n2: int | None = None) -> int:
    """Number of solved pairs for the given row ranges."""
    if not symmetric:
        return sum((hi - lo) for lo, hi in ranges) * (n2 if n2 is not None else n)
    return sum(sum(n - a for a in range(lo, hi)) for lo, hi in ranges)


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def _upper_mask(ranges, n, device):
    """Boolean mask of the solved (b >= a) entries of the concatenated row
    blocks `ranges` of a symmetric (n, n) Gram."""
    rows = torch.cat([torch.arange(lo, hi, device=device) for lo, hi in ranges]) if ranges \
        else torch.zeros(0, dtype=torch.long, device=device)
    return torch.arange(n, device=device).view(1, n) >= rows.view(-1, 1)


def _gather_rows(local_rows: torch.Tensor, ranges_all, n1: int, n2: int, group,
                 symmetric: bool = False) -> torch.Tensor:
    """All-gather per-rank row blocks into a full (n1, n2).  Symmetric: only the
    solved upper-triangle entries travel (packed, padded to the largest rank),
    about half the bytes of full rows; the caller mirrors."""
    world = len(ranges_all)
    dev = local_rows.device
    if symmetric:
        counts = [int(sum((n2 - a) for lo, hi in r for a in range(lo, hi))) for r in ranges_all]
        rank = dist.get_rank(group)
        mine = local_rows[_upper_mask(ranges_all[rank], n2, dev)]
        pad = torch.zeros(max(counts), dtype=local_rows.dtype, device=dev)
        pad[: mine.numel()] = mine
        gathered = torch.empty(world * max(counts), dtype=pad.dtype, device=dev)
        dist.all_gather_into_tensor(gathered, pad, group=group)
        G = torch.zeros((n1, n2), dtype=pad.dtype, device=dev)
        for r, ranges in enumerate(ranges_all):
            if not ranges:
                continue
            idx = torch.cat([torch.arange(lo, hi, device=dev) for lo, hi in ranges])
            blk = G[idx]
            blk[_upper_mask(ranges, n2, dev)] = gathered[r * max(counts): r * max(counts) + counts[r]]
            G[idx] = blk
        return G
    maxrows = max(sum(hi - lo for lo, hi in r) for r in ranges_all)
    pad = torch.zeros((maxrows, n2), dtype=local_rows.dtype, device=dev)
    pad[: local_rows.shape[0]] = local_rows
    gathered = torch.empty((world * maxrows, n2), dtype=pad.dtype, device=dev)
    dist.all_gather_into_tensor(gathered, pad, group=group)
    G = torch.empty((n1, n2), dtype=pad.dtype, device=dev)
    for r, ranges in enumerate(ranges_all):
        off = r * maxrows
        for lo, hi in ranges:
            G[lo:hi] = gathered[off: off + hi - lo]
            off += hi - lo
    return G


def _allreduce_acc(acc, group):
    """Combine the exact gradient accumulators of all ranks: the limbs add as
    integers (exact, order-free), the metadata (identical anchor, OR of the
    overflow flags) by MAX."""
    dist.all_reduce(acc.limbs, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(acc.meta, op=dist.ReduceOp.MAX, group=group)
    return acc


def gram_forward_sharded(x, y, l1, l2, kind, sigma, group=None) -> torch.Tensor:
    world, rank = _world(group)
    sym = y is None
    n1, n2 = x.shape[0], (x.shape[0] if sym else y.shape[0])
    if world == 1:
        return ops.forward_gram(x, y, l1, l2, kind, sigma)
    ranges_all = [row_blocks(n1, world, r, sym) for r in range(world)]
    mine = ranges_all[rank]
    parts = [ops.forward_gram(x, y, l1, l2, kind, sigma, rows=rg) for rg in mine]
    local = torch.cat(parts, 0) if parts else torch.zeros((0, n2), dtype=torch.float64,
                                                         device=x.device)
    G = _gather_rows(local, ranges_all, n1, n2, group, symmetric=sym)
    if sym:
        ops.mirror_upper(G)
    return G


def _accumulators(x, y, cot, sym):
    n1, L1, d = x.shape
    acc_x = ops.GradAcc(n1, L1, d, x.device).init(cot, n1, y.shape[0] if y is not None else n1,
                                                   sym)
    acc_y = None
    if not sym:
        acc_y = ops.GradAcc(y.shape[0], y.shape[1], d, x.device).init(cot, n1, y.shape[0], False)
    return acc_x, acc_y


def gram_backward_sharded(x, y, l1, l2, kind, sigma, cot, group=None):
    world, rank = _world(group)
    sym = y is None
    n1 = x.shape[0]
    acc_x, acc_y = _accumulators(x, y, cot, sym)
    ranges = row_blocks(n1, world, rank, sym) if world > 1 else [(0, n1)]
    for rg in ranges:
        ops.backward_gram(x, y, l1, l2, kind, sigma, cot, rows=rg, acc_x=acc_x, acc_y=acc_y)
    if world > 1:
        _allreduce_acc(acc_x, group)
        if acc_y is not None:
            _allreduce_acc(acc_y, group)
    return acc_x.finalize(), (None if acc_y is None else acc_y.finalize())


class _ShardedGramFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, y, l1, l2, kind, sigma, group):
        ctx.sym = y is None
        ctx.cfg = (l1, l2, kind, sigma, group)
        ctx.save_for_backward(x) if ctx.sym else ctx.save_for_backward(x, y)
        return gram_forward_sharded(x, y, l1, l2, kind, sigma, group)

    @staticmethod
    def backward(ctx, cot):
        l1, l2, kind, sigma, group = ctx.cfg
        if ctx.sym:
            (x,) = ctx.saved_tensors
            gx, _ = gram_backward_sharded(x, None, l1, l2, kind, sigma, cot, group)
            return gx, None, None, None, None, None, None
        x, y = ctx.saved_tensors
        gx, gy = gram_backward_sharded(x, y, l1, l2, kind, sigma, cot, group)
        return gx, gy, None, None, None, None, None


def sig_kernel_gram_sharded(x, y=None, dyadic_order=0, static_kernel=None, group=None):
    """sig_kernel_gram across all ranks of `group`; every rank gets the full G.

    The upstream gradient (cotangent) must be identical on all ranks, as it is
    for a loss computed redundantly from the replicated G."""
    if x.dim() != 3:
        raise InvalidArgument("x must be (n, L, d)")
    sym = y is None or y is x
    l1, l2 = _orders(dyadic_order)
    kind, sigma = ops.static_kind(static_kernel)
    xx = x.to(torch.float64)
    yy = None if sym else y.to(torch.float64)
    return _ShardedGramFn.apply(xx, yy, l1, l2, kind, sigma, group)


def value_and_grad_sharded(x, y=None, cotangent=None, dyadic_order=0, static_kernel=None,
                           group=None):
    """Fused G + gradient across all ranks of `group` (sig_kernel_gram_value_and_grad
    sharded by balanced row blocks): every rank gets the full G (all-gather of
    its rows, then the mirror) and the full dF/dx (dF/dy) (all-gather of the
    partials, summed in rank order).  cotangent must be identical on all ranks."""
    if x.dim() != 3:
        raise InvalidArgument("x must be (n, L, d)")
    sym = y is None or y is x
    l1, l2 = _orders(dyadic_order)
    kind, sigma = ops.static_kind(static_kernel)
    xx = x.detach().to(torch.float64)
    yy = None if sym else y.detach().to(torch.float64)
    world, rank = _world(group)
    n1, n2 = xx.shape[0], (xx.shape[0] if sym else yy.shape[0])
    if cotangent is None:
        cotangent = torch.ones((n1, n2), dtype=torch.float64, device=xx.device)
    if world == 1:
        return ops.value_and_grad_gram(xx, yy, l1, l2, kind, sigma, cotangent)
    ranges_all = [row_blocks(n1, world, r, sym) for r in range(world)]
    acc_x, acc_y = _accumulators(xx, yy, cotangent, sym)
    parts = []
    for rg in ranges_all[rank]:
        out, _, _ = ops.value_and_grad_gram(xx, yy, l1, l2, kind, sigma, cotangent, rows=rg,
                                            acc_x=acc_x, acc_y=acc_y)
        parts.append(out)
    local = torch.cat(parts, 0) if parts else torch.zeros((0, n2), dtype=torch.float64,
                                                         device=xx.device)
    G = _gather_rows(local, ranges_all, n1, n2, group, symmetric=sym)
    if sym:
        ops.mirror_upper(G)
    _allreduce_acc(acc_x, group)
    if acc_y is not None:
        _allreduce_acc(acc_y, group)
    return G, acc_x.finalize(), (None if acc_y is None else acc_y.finalize())
