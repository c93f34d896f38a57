"""Row-sharded msGeMM over several GPUs (one process per GPU).

The path shards naturally by rows: every output row is an independent
consumer of the read-only tables (gemm.py:136-152 splits work
the same way across threads).  Rank r of G owns rows
[r*m/G, (r+1)*m/G) of W, builds the tables for the (replicated) X itself
and computes its Y slice; the only exchange is one all-gather of the
row-major Y slices (contiguous in Y), done with torch.distributed (NCCL over
NVLink/NVSwitch on the GPU box, gloo in the CPU tests).

Row-chunking is bitwise safe: each row's result depends only on that row's
weights and X, so the gathered Y equals the single-GPU Y of the same kernel
configuration row by row (the k-split, and hence the fp32 summation order,
depends on the shard height; results are within the stated tolerance and
bit-exact for integer-valued X).
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from .packing import PackedWeightMatrix, PerGroup, PerRow


def shard_bounds(m: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [lo, hi) of rank `rank`; the first m % world ranks get one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_rows(pwm: PackedWeightMatrix, world: int, rank: int) -> PackedWeightMatrix:
    """This rank's row block as a PackedWeightMatrix (data and scales sliced)."""
    lo, hi = shard_bounds(pwm.m, world, rank)
    scales = pwm.scales
    if isinstance(scales, PerRow):
        scales = PerRow(q=scales.q[lo:hi])
    elif isinstance(scales, PerGroup):
        scales = PerGroup(group_size=scales.group_size, q=scales.q[lo:hi])
    return PackedWeightMatrix(m=hi - lo, k=pwm.k, width=pwm.width, data=pwm.data[lo:hi],
                              codebook=pwm.codebook, scales=scales)


def gather_rows(y_local, m: int, group=None):
    """All-gather row slices (possibly unequal heights) into the full (m, ...) Y.

    Uses all_gather_into_tensor when the slices are equal (the common case:
    m divisible by the world size), else pads to the largest slice.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_bounds(m, world, r) for r in range(world)]
    heights = [hi - lo for lo, hi in sizes]
    tail = tuple(y_local.shape[1:])
    hmax = max(heights)
    if all(h == hmax for h in heights):
        out = torch.empty((m,) + tail, dtype=y_local.dtype, device=y_local.device)
        dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
        return out
    pad = torch.zeros((hmax,) + tail, dtype=y_local.dtype, device=y_local.device)
    pad[: heights[rank]] = y_local
    buf = torch.empty((hmax * world,) + tail, dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(buf, pad, group=group)
    return torch.cat([buf[r * hmax: r * hmax + heights[r]] for r in range(world)])


def msgemm_sharded(pwm_local: PackedWeightMatrix, X, d: int, m_total: int, group=None,
                   local_fn: Callable | None = None, **kw):
    """Y = W @ X for row-sharded W: local msGeMM on this rank's rows, then one
    all-gather.  X (replicated) and the result are torch tensors on this
    rank's device.  `local_fn(pwm, X, d, **kw)` defaults to msgemm (tests
    substitute the CPU oracle to exercise the gloo path without a GPU).
    """
    import torch

    if local_fn is None:
        from .gemm import msgemm as local_fn
    y = local_fn(pwm_local, X, d, **kw)
    if not isinstance(y, torch.Tensor):
        y = torch.from_numpy(np.ascontiguousarray(y))
    return gather_rows(y, m_total, group)
