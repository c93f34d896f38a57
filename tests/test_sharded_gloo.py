"""Multi-process (world_size 2, gloo, CPU) tests of the row-sharded path.

The GPU compute is replaced by the CPU oracle as the local function (tests may
use the oracle), so what is exercised here is exactly the host-side logic the
B200 run uses: row shard bounds, weight/scale slicing and the all-gather that
reassembles Y.  Row-chunking is bitwise safe for the oracle, so the gathered
result must equal the unsharded oracle bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc
from paper_2310_06178_b200.sharded import gather_rows, msgemm_sharded, shard_bounds, shard_rows

VALS = orc.int4_values()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_local(pwm, X, d, **kw):
    mode, gs, q = None, 0, None
    if isinstance(pwm.scales, mg.PerRow):
        mode, q = "per_row", pwm.scales.q
    return orc.msgemm(np.asarray(pwm.data), pwm.m, pwm.k, 4, VALS, X, d, mode, gs, q)


def _case(m, k, b, dtype, seed, scaled):
    rng = np.random.default_rng(seed)
    data = rng.integers(0, 256, size=(m, (k + 1) // 2), dtype=np.uint8)
    if k % 2:
        data[:, -1] &= 0xF
    scales = mg.PerRow(q=rng.integers(1, 5, size=m).astype(np.int64)) if scaled else None
    pwm = mg.PackedWeightMatrix(m=m, k=k, width=4, data=data, codebook=mg.int4_codebook(),
                                scales=scales)
    if np.issubdtype(dtype, np.integer):
        X = rng.integers(-100, 100, size=(k, b)).astype(dtype)
    else:
        X = rng.standard_normal((k, b)).astype(dtype)
    return pwm, X


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for m, k, b, dtype, seed, scaled, d in cases:
            pwm, X = _case(m, k, b, dtype, seed, scaled)
            local = shard_rows(pwm, world, rank)
            lo, hi = shard_bounds(m, world, rank)
            assert local.m == hi - lo
            y = msgemm_sharded(local, X, d, m, local_fn=_oracle_local)
            full = _oracle_local(pwm, X, d)
            assert y.shape == full.shape
            assert np.array_equal(y.numpy().view(np.uint8), full.view(np.uint8)), (m, k, b, dtype)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


CASES = [
    (64, 48, 3, np.int64, 1, False, 3),     # equal shards, tail, exact
    (11, 30, 2, np.int64, 2, True, 2),      # unequal shards (6/5), per-row scales
    (40, 64, 8, np.float16, 3, False, 3),   # fp16 X
    (33, 17, 1, np.float32, 4, False, 1),   # f32, vector-like b=1, unequal
]


@pytest.mark.timeout(180)
def test_row_sharded_allgather_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=170) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert res == {0: "ok", 1: "ok"}, res


def test_shard_bounds_cover_rows():
    for m in (0, 1, 7, 64, 65536, 65537):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_shard_rows_slices_scales():
    pwm, _ = _case(10, 8, 1, np.int64, 5, True)
    s = shard_rows(pwm, 3, 1)
    lo, hi = shard_bounds(10, 3, 1)
    assert np.array_equal(s.data, pwm.data[lo:hi])
    assert np.array_equal(s.scales.q, pwm.scales.q[lo:hi])


# ---------------------------------------------------------------------------
# k-split (row f4): slices of the inner dimension, fp32/int64 partial sums
# ---------------------------------------------------------------------------
from paper_2310_06178_b200.sharded import k_split_bounds, msgemm_ksplit, shard_cols  # noqa: E402


def _oracle_partial(pwm, X, d):
    """The slice's partial product, accumulated wide (int64 / float64) like the
    kernels' fp32 partials, so the cross-rank sum adds no fp16 rounding."""
    X = np.asarray(X)
    Xw = X.astype(np.int64) if np.issubdtype(X.dtype, np.integer) else X.astype(np.float64)
    mode, gs, q = None, 0, None
    if isinstance(pwm.scales, mg.PerRow):
        mode, q = "per_row", pwm.scales.q
    elif isinstance(pwm.scales, mg.PerGroup):
        mode, gs, q = "per_group", pwm.scales.group_size, pwm.scales.q
    return orc.msgemm(np.asarray(pwm.data), pwm.m, pwm.k, 4, VALS, Xw, d, mode, gs, q)


def _kcase(m, k, b, dtype, seed, scale, d):
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 16, size=(m, k), dtype=np.uint8)
    data = orc.pack_rows(codes, 4)
    scales = None
    if scale == "row":
        scales = mg.PerRow(q=rng.integers(1, 5, size=m).astype(np.int64))
    elif scale == "group":
        gs = 2 * d
        scales = mg.PerGroup(group_size=gs, q=rng.integers(1, 4, size=(m, k // gs)).astype(np.int64))
    pwm = mg.PackedWeightMatrix(m=m, k=k, width=4, data=data, codebook=mg.int4_codebook(),
                                scales=scales)
    if np.issubdtype(dtype, np.integer):
        X = rng.integers(-100, 100, size=(k, b)).astype(dtype)
    else:
        X = rng.standard_normal((k, b)).astype(dtype)
    return pwm, X


def _kworker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for m, k, b, dtype, seed, scale, d, red in cases:
            pwm, X = _kcase(m, k, b, dtype, seed, scale, d)
            local, lo, hi = shard_cols(pwm, d, world, rank)
            y = msgemm_ksplit(local, X, d, lo, hi, local_fn=_oracle_partial, reduce=red)
            full = _oracle_partial(pwm, X, d)
            if red == "scatter":
                r0, r1 = shard_bounds(m, world, rank)
                full = full[r0:r1]
            assert y.dtype == torch.from_numpy(X).dtype and tuple(y.shape) == full.shape
            if np.issubdtype(X.dtype, np.integer):
                assert np.array_equal(y.numpy(), full), (m, k, b, d, scale)  # exact
            else:
                W = orc.dense(np.asarray(pwm.data), k, 4, VALS,
                              None if scale is None else ("per_row" if scale == "row" else "per_group"),
                              0 if scale != "group" else pwm.scales.group_size,
                              None if scale is None else pwm.scales.q, apply_scales=True)
                tol = 1e-5 if X.dtype == np.float32 else 2e-3
                ref = np.abs(W) @ np.abs(X.astype(np.float64))
                if red == "scatter":
                    ref = ref[r0:r1]
                assert np.all(np.abs(y.numpy().astype(np.float64) - full) <= tol * ref + 1e-30)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


KCASES = [
    (24, 50, 3, np.int64, 7, None, 3, "all"),       # tail (50 % 3 = 2) on the last rank
    (17, 36, 2, np.int64, 8, "row", 2, "all"),      # per-row scales
    (16, 48, 4, np.int64, 9, "group", 3, "all"),    # per-group scales, slices on group bounds
    (40, 66, 8, np.float32, 10, None, 3, "all"),    # f32: fp32 partials, tolerance
    (21, 30, 5, np.int64, 11, None, 3, "scatter"),  # reduce-scatter, unequal row shards
    (8, 6, 1, np.int64, 12, None, 3, "all"),        # one aligned unit: rank 1 gets an empty slice
]


@pytest.mark.timeout(180)
def test_k_split_allreduce_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_kworker, args=(r, world, port, KCASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=170) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert res == {0: "ok", 1: "ok"}, res


def test_k_split_bounds_align_and_cover():
    for k in (0, 1, 5, 6, 7, 48, 8192, 8193):
        for d in (1, 2, 3, 4):
            for gs in (0, 12):
                if gs and (k % gs or gs % d):
                    continue
                for world in (1, 2, 3, 8):
                    spans = [k_split_bounds(k, d, world, r, gs) for r in range(world)]
                    assert spans[0][0] == 0 and spans[-1][1] == k
                    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
                    a = np.lcm.reduce([2, d, gs or 1])
                    assert all(lo % a == 0 for lo, _ in spans)
    with pytest.raises(ValueError):
        k_split_bounds(10, 3, 2, 2)


def test_peer_targets_offsets():
    """Fan-out destinations of the fused all-gather: every other rank's buffer
    at this rank's first row (pure address arithmetic, sharded.peer_targets)."""
    from paper_2310_06178_b200.sharded import peer_targets, shard_bounds
    ptrs = [0x1000_0000, 0x2000_0000, 0x3000_0000, 0x4000_0000]
    m, b, item = 1030, 8, 2
    for r in range(4):
        lo, _ = shard_bounds(m, 4, r)
        t = peer_targets(ptrs, r, lo, b * item)
        assert len(t) == 3 and ptrs[r] + lo * b * item not in t
        assert t == [p + lo * b * item for i, p in enumerate(ptrs) if i != r]
    with pytest.raises(ValueError):
        peer_targets(ptrs, 4, 0, 16)
    with pytest.raises(ValueError):
        peer_targets(list(range(9)), 0, 0, 16)
