"""Row-sharded msGeMM over several GPUs (one process per GPU).

The path shards naturally by rows: every output row is an independent
consumer of the read-only tables (gemm.py:136-152 splits work
the same way across threads).  Rank r of G owns rows
[r*m/G, (r+1)*m/G) of W, builds the tables for the (replicated) X itself
and computes its Y slice; the only exchange is one all-gather of the
row-major Y slices (contiguous in Y), done with torch.distributed (NCCL over
NVLink/NVSwitch on the GPU box, gloo in the CPU tests) -- or, opt-in, fused
into the finishing kernels as peer stores over symmetric memory (PeerY,
msgemm_sharded_fused below).

Row-chunking is bitwise safe: each row's result depends only on that row's
weights and X, so the gathered Y equals the single-GPU Y of the same kernel
configuration row by row (the k-split, and hence the fp32 summation order,
depends on the shard height; results are within the stated tolerance and
bit-exact for integer-valued X).
"""

from __future__ import annotations

import math
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


# ----------------------------------------------------------------------------
# All-gather fused into the epilogue: Y lives in
# symmetric memory (every rank maps every rank's buffer over NVLink), and the
# finishing kernels of rank r store its rows straight into all G copies
# (msg_gemm_fanout) -- no NCCL call, no extra pass over Y; one barrier on the
# symmetric-memory signal pads before any rank reads.
# ----------------------------------------------------------------------------
def peer_targets(buffer_ptrs, rank: int, row_lo: int, row_bytes: int) -> list[int]:
    """Addresses of row `row_lo` in every OTHER rank's Y buffer (the fan-out
    destinations of this rank's slice)."""
    if not 0 <= rank < len(buffer_ptrs):
        raise ValueError(f"bad rank {rank} of {len(buffer_ptrs)}")
    if len(buffer_ptrs) > 8:
        raise ValueError("the fused all-gather fans out to at most 7 peers")
    return [int(p) + row_lo * row_bytes for r, p in enumerate(buffer_ptrs) if r != rank]


class PeerY:
    """The full Y (m, b) of a row-sharded msGeMM in symmetric memory.

    Needs the NCCL/CUDA symmetric-memory allocator of torch.distributed (one
    process per GPU, peers on NVLink); raises RuntimeError where that is not
    available so callers can fall back to `gather_rows`.
    """

    def __init__(self, m: int, b: int, dtype, device, group=None):
        import torch.distributed as dist
        try:
            import torch.distributed._symmetric_memory as symm
        except ImportError as e:  # pragma: no cover
            raise RuntimeError(f"symmetric memory unavailable: {e}") from e
        self.m, self.b = m, b
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        gname = (group or dist.group.WORLD).group_name
        try:
            self.buf = symm.empty((m, b), dtype=dtype, device=device)
            self.handle = symm.rendezvous(self.buf, gname)
        except Exception as e:
            raise RuntimeError(f"symmetric memory rendezvous failed: {e}") from e
        self.row_bytes = b * self.buf.element_size()
        self.ptrs = [int(p) for p in self.handle.buffer_ptrs]
        self.lo, self.hi = shard_bounds(m, self.world, self.rank)

    def local(self):
        """This rank's rows of its own copy (the `out` of the local msGeMM)."""
        return self.buf[self.lo:self.hi]

    def targets(self) -> list[int]:
        return peer_targets(self.ptrs, self.rank, self.lo, self.row_bytes)

    def barrier(self):
        """Every rank's stores have landed everywhere (on the current stream)."""
        self.handle.barrier()


def msgemm_sharded_fused(pwm_local: PackedWeightMatrix, X, d: int, peer_y: PeerY, **kw):
    """Y = W @ X for row-sharded W with the all-gather fused into the finishing
    kernels: returns this rank's full (m, b) Y (a view of symmetric memory,
    valid until the next call).  X: CUDA tensor (replicated)."""
    from .gemm import msgemm

    peer_y.barrier()          # nobody still reads the previous call's Y
    if peer_y.hi > peer_y.lo:
        msgemm(pwm_local, X, d, out=peer_y.local(), _fan=peer_y.targets(), **kw)
    peer_y.barrier()
    return peer_y.buf


# ----------------------------------------------------------------------------
# k-split: every rank owns a slice of the inner
# dimension for ALL rows, so the table build is split too (the replicated
# build is the Amdahl term of row sharding, §8(e)); the exchange is an fp32
# sum of the partial Y (all-reduce, or reduce-scatter when the consumer wants
# row shards).
# ----------------------------------------------------------------------------
def k_split_bounds(k: int, d: int, world: int, rank: int, group_size: int = 0) -> tuple[int, int]:
    """Columns [lo, hi) of rank `rank`'s k-slice.

    Boundaries fall on multiples of lcm(2, d, group_size): whole bytes of the
    packed rows (packing.py:99-114), whole d-groups (so the slices' lookup
    blocks are exactly the global blocks, gemm.py:116-133) and whole scale
    groups.  The last rank also takes the remainder, which holds the global
    k % d tail (gemm.py:81-83), so the slices' results sum to the full Y.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if d < 1:
        raise ValueError("depth d must be >= 1")
    a = math.lcm(2, d, group_size or 1)
    base, extra = divmod(k // a, world)
    lo = (rank * base + min(rank, extra)) * a
    hi = lo + (base + (1 if rank < extra else 0)) * a
    return lo, (k if rank == world - 1 else hi)


def shard_cols(pwm: PackedWeightMatrix, d: int, world: int, rank: int) -> tuple[PackedWeightMatrix, int, int]:
    """This rank's k-slice of W as a PackedWeightMatrix, with its bounds.

    The packed payload is sliced on byte boundaries (lo is even); per-row
    scales are kept (scaling is linear, so each slice may apply them), per-group
    scales are sliced by column group.
    """
    gs = pwm.scales.group_size if isinstance(pwm.scales, PerGroup) else 0
    lo, hi = k_split_bounds(pwm.k, d, world, rank, gs)
    data = pwm.data[:, lo // 2:(hi + 1) // 2]
    scales = pwm.scales
    if isinstance(scales, PerGroup):
        scales = PerGroup(group_size=gs, q=scales.q[:, lo // gs:hi // gs])
    return (PackedWeightMatrix(m=pwm.m, k=hi - lo, width=pwm.width, data=data,
                               codebook=pwm.codebook, scales=scales), lo, hi)


def msgemm_ksplit(pwm_slice: PackedWeightMatrix, X, d: int, lo: int, hi: int, group=None,
                  local_fn: Callable | None = None, reduce: str = "all"):
    """Y = W @ X for a k-split W: this rank's partial product over columns
    [lo, hi) in fp32 (int64 for integer X), then one sum across ranks.

    reduce="all": every rank gets the full (m, b) Y (all-reduce).
    reduce="scatter": rank r gets rows shard_bounds(m, world, r) (reduce-scatter).
    The result has X's dtype (reference semantics, gemm.py:113, 153).  X is the
    full (k, b) activation matrix (replicated); `local_fn(pwm, Xs, d)` must
    return the partial in its accumulation dtype (default: msgemm with fp32
    output; the CPU tests substitute the oracle).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    Xt = X if isinstance(X, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(X))
    vec = Xt.dim() == 1
    X2 = Xt[:, None] if vec else Xt
    out_dtype = X2.dtype
    exact = not X2.is_floating_point()
    acc_dtype = torch.int64 if exact else torch.float32
    m, b = pwm_slice.m, X2.shape[1]
    if hi > lo:
        if local_fn is None:
            from .gemm import msgemm

            y = msgemm(pwm_slice, X2[lo:hi], d, out_dtype=None if exact else np.float32)
        else:
            y = local_fn(pwm_slice, X2[lo:hi], d)
        y = y if isinstance(y, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(y))
        y = y.to(acc_dtype).reshape(m, b)
    else:
        y = torch.zeros((m, b), dtype=acc_dtype, device=X2.device)
    if reduce == "all":
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
        out = y.to(out_dtype)
        return out[:, 0] if vec else out
    if reduce != "scatter":
        raise ValueError(f"reduce must be 'all' or 'scatter', got {reduce!r}")
    spans = [shard_bounds(m, world, r) for r in range(world)]
    hmax = max(h - l for l, h in spans)
    if dist.get_backend(group) == "gloo":  # gloo has no reduce-scatter: sum, then slice
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
        part = y[spans[rank][0]:spans[rank][1]]
    elif all(h - l == hmax for l, h in spans):
        part = torch.empty((hmax, b), dtype=acc_dtype, device=y.device)
        dist.reduce_scatter_tensor(part, y.contiguous(), op=dist.ReduceOp.SUM, group=group)
    else:  # unequal row shards: pad every shard to hmax rows
        pad = torch.zeros((hmax * world, b), dtype=acc_dtype, device=y.device)
        for r, (l, h) in enumerate(spans):
            pad[r * hmax: r * hmax + (h - l)] = y[l:h]
        part = torch.empty((hmax, b), dtype=acc_dtype, device=y.device)
        dist.reduce_scatter_tensor(part, pad, op=dist.ReduceOp.SUM, group=group)
        part = part[: spans[rank][1] - spans[rank][0]]
    out = part.to(out_dtype)
    return out[:, 0] if vec else out
