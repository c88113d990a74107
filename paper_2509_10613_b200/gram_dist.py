"""Gram matrices sharded across the GPUs of one box.

One process per GPU (torch.distributed, NCCL over NVLink).  Rows of the Gram
are split into 2P equal blocks and rank r solves blocks r and 2P-1-r, which
balances the upper-triangle work of a symmetric Gram (row a holds n-a pairs).
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


def row_blocks(n: int, world: int, rank: int, symmetric: bool = True) -> list[tuple[int, int]]:
    """Row ranges owned by `rank`.

    symmetric: 2*world equal blocks, rank gets blocks rank and 2*world-1-rank
    (balanced upper-triangle pair counts); otherwise one contiguous block."""
    if world <= 1:
        return [(0, n)]
    if not symmetric:
        step = -(-n // world)
        lo, hi = min(n, rank * step), min(n, (rank + 1) * step)
        return [(lo, hi)] if hi > lo else []
    nb = 2 * world
    bounds = [round(k * n / nb) for k in range(nb + 1)]
    out = []
    for k in (rank, nb - 1 - rank):
        lo, hi = bounds[k], bounds[k + 1]
        if hi > lo:
            out.append((lo, hi))
    return sorted(out)


def pair_count(ranges, n: int, symmetric: bool, n2: int | None = None) -> int:
    """Number of solved pairs for the given row ranges."""
    if not symmetric:
        return sum((hi - lo) for lo, hi in ranges) * (n2 if n2 is not None else n)
    return sum(sum(n - a for a in range(lo, hi)) for lo, hi in ranges)


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def _gather_rows(local_rows: torch.Tensor, ranges_all, n1: int, n2: int, group) -> torch.Tensor:
    """All-gather per-rank row blocks (padded to equal size) into a full (n1, n2)."""
    world = len(ranges_all)
    maxrows = max(sum(hi - lo for lo, hi in r) for r in ranges_all)
    pad = torch.zeros((maxrows, n2), dtype=local_rows.dtype, device=local_rows.device)
    pad[: local_rows.shape[0]] = local_rows
    gathered = torch.empty((world * maxrows, n2), dtype=pad.dtype, device=pad.device)
    dist.all_gather_into_tensor(gathered, pad, group=group)
    G = torch.empty((n1, n2), dtype=pad.dtype, device=pad.device)
    for r, ranges in enumerate(ranges_all):
        off = r * maxrows
        for lo, hi in ranges:
            G[lo:hi] = gathered[off: off + hi - lo]
            off += hi - lo
    return G


def _gather_sum(t: torch.Tensor, group) -> torch.Tensor:
    """All-gather equal-shape partials and sum them in fixed rank order."""
    world, _ = _world(group)
    t = t.contiguous()
    flat = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                       device=t.device)
    dist.all_gather_into_tensor(flat, t, group=group)
    buf = flat.view((world,) + tuple(t.shape))
    out = buf[0].clone()
    for r in range(1, world):
        out += buf[r]
    return out


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
    G = _gather_rows(local, ranges_all, n1, n2, group)
    if sym:
        ops.mirror_upper(G)
    return G


def gram_backward_sharded(x, y, l1, l2, kind, sigma, cot, group=None):
    world, rank = _world(group)
    sym = y is None
    n1 = x.shape[0]
    gx = torch.zeros_like(x, dtype=torch.float64)
    gy = None if sym else torch.zeros_like(y, dtype=torch.float64)
    ranges = row_blocks(n1, world, rank, sym) if world > 1 else [(0, n1)]
    for rg in ranges:
        ops.backward_gram(x, y, l1, l2, kind, sigma, cot, rows=rg, grad_x=gx, grad_y=gy)
    if world > 1:
        gx = _gather_sum(gx, group)
        if gy is not None:
            gy = _gather_sum(gy, group)
    return gx, gy


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
    gx = torch.zeros_like(xx)
    gy = None if sym else torch.zeros_like(yy)
    parts = []
    for rg in ranges_all[rank]:
        out, _, _ = ops.value_and_grad_gram(xx, yy, l1, l2, kind, sigma, cotangent, rows=rg,
                                            grad_x=gx, grad_y=gy)
        parts.append(out)
    local = torch.cat(parts, 0) if parts else torch.zeros((0, n2), dtype=torch.float64,
                                                         device=xx.device)
    G = _gather_rows(local, ranges_all, n1, n2, group)
    if sym:
        ops.mirror_upper(G)
    gx = _gather_sum(gx, group)
    if gy is not None:
        gy = _gather_sum(gy, group)
    return G, gx, gy
