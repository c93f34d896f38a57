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
