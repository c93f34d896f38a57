"""k-split slices on the GPU (row f4): the per-rank partial products of
shard_cols(...) slices, computed by the B200 kernels with fp32 output, sum to
the full product.  One process plays every rank (no collective: the sum is
done here), so the kernels never wait on one another; the collective itself
is covered by the gloo world-2 test."""

import numpy as np
import pytest
import torch

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc
from paper_2310_06178_b200.sharded import shard_cols

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,b,d,world,scale", [
    (4096, 4096, 1, 3, 2, None), (4096, 4096, 1, 3, 8, None), (1000, 8192, 8, 3, 4, None),
    (513, 1027, 3, 2, 3, "row"), (256, 768, 4, 3, 2, "group"), (300, 50, 2, 3, 4, None)])
def test_ksplit_partials_sum_to_full(m, k, b, d, world, scale):
    rng = np.random.default_rng(m + k + world)
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    scales = None
    if scale == "row":
        scales = mg.PerRow(q=rng.uniform(0.5, 2, m).astype(np.float32))
    elif scale == "group":
        scales = mg.PerGroup(group_size=96, q=rng.uniform(0.5, 2, (m, k // 96)).astype(np.float32))
    pwm = mg.from_codes(codes, mg.int4_codebook(), scales=scales)
    X = rng.standard_normal((k, b)).astype(np.float16)
    acc = np.zeros((m, b), np.float64)
    for r in range(world):
        part, lo, hi = shard_cols(pwm, d, world, r)
        if hi > lo:
            y = mg.msgemm(part, torch.from_numpy(X[lo:hi]).cuda(), d, out_dtype=np.float32)
            acc += y.cpu().numpy().astype(np.float64)
    W = orc.dense(np.asarray(pwm.data), k, 4, orc.int4_values(),
                  None if scale is None else ("per_row" if scale == "row" else "per_group"),
                  96 if scale == "group" else 0, None if scale is None else pwm.scales.q,
                  apply_scales=True)
    assert orc.rel_error(acc.astype(np.float16), W, X) <= 2e-3


def test_ksplit_integer_exact():
    rng = np.random.default_rng(3)
    m, k, d = 2048, 4096, 3
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, mg.int4_codebook())
    X = rng.integers(-127, 128, (k, 2)).astype(np.float16)
    acc = np.zeros((m, 2), np.float64)
    for r in range(4):
        part, lo, hi = shard_cols(pwm, d, 4, r)
        acc += mg.msgemm(part, X[lo:hi], d, out_dtype=np.float32,
                          table_dtype=np.float32).astype(np.float64)
    ref = orc.naive_gemm(orc.dense(np.asarray(pwm.data), k, 4, orc.int4_values()), X.astype(np.int64))
    assert np.array_equal(acc.astype(np.int64), ref)
