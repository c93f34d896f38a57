"""Small calls through every kernel family (odd shapes, tails, scales, sparse
rows, every table/layout variant), each checked against the CPU oracle -- the
program compute-sanitizer runs (tools/sanitize.sh) and a quick all-paths probe.

    python tools/sanitize_probe.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402
from oracle import msgemm_oracle as orc  # noqa: E402

rng = np.random.default_rng(3)
cb = mg.int4_codebook()
TOL = {np.float16: 2e-3, np.float32: 1e-5, np.float64: 1e-12}


def check(m, k, b, d, dt, scales=None, codebook=cb, sparse=False, **kw):
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    if sparse:
        codes[::7] = 0                            # all-zero rows
        codes[3::7, 1:] = 0                       # single-nonzero rows
    pwm = mg.from_codes(codes, codebook, scales)
    X = rng.standard_normal((k, b)).astype(dt)
    Xa = X[:, 0].copy() if b == 1 else X
    Y = mg.msgemm(pwm, Xa, d, **kw)
    W = orc.dense(pwm.data, k, 4, np.asarray(codebook.values))
    if isinstance(scales, mg.PerRow):
        W = W * np.asarray(scales.q)[:, None]
    elif isinstance(scales, mg.PerGroup):
        W = W * np.repeat(np.asarray(scales.q), scales.group_size, axis=1)
    err = orc.rel_error(np.asarray(Y, dtype=np.float64).reshape(m, b), W, X)
    assert err <= TOL[dt], (m, k, b, d, dt, err)
    if sparse:
        assert (np.asarray(Y).reshape(m, b)[::7] == 0).all()


# lane GEMV (b=1): tail, several chunks, per-row scale, sparse rows (fix-up path)
check(97, 301, 1, 3, np.float16)
check(700, 1000, 1, 3, np.float16, scales=mg.PerRow(q=rng.random(700).astype(np.float32) + 0.5))
check(200, 400, 1, 3, np.float16, sparse=True)
# row-block kernels: BC=8 in TMEM (b=8, 16), BC=4 (b=4), BC=2 (b=2), tails
check(300, 200, 8, 3, np.float16)
check(130, 301, 16, 3, np.float16)
check(300, 200, 4, 3, np.float16)
check(257, 98, 2, 3, np.float16, sparse=True)
# fused quad kernel: fp32 X, fp32 tables, full tables, per-group scales, uint4
check(64, 50, 3, 2, np.float32)
check(90, 300, 8, 3, np.float16, table_dtype=np.float32)
check(90, 300, 8, 3, np.float16, symmetric=False)
check(64, 96, 4, 3, np.float16, scales=mg.PerGroup(group_size=24, q=rng.random((64, 4)).astype(np.float32)))
check(70, 99, 5, 3, np.float32, codebook=mg.uint4_codebook())
# generic global-table kernels: f64, d=4
check(40, 30, 2, 4, np.float64)
# phase-1 / packing kernels
x = rng.standard_normal(31).astype(np.float32)
assert np.array_equal(np.asarray(mg.build_lut(x, cb, 3).entries), orc.lut_full(x, orc.int4_values(), 3))
pwm = mg.pack(rng.integers(-8, 8, (9, 13)), cb)
assert np.array_equal(mg.group_indices(pwm, 3), orc.group_indices(np.asarray(pwm.data), 13, 4, 3))
# dense product and the K4 comparison kernel
W = rng.integers(-8, 8, (33, 70))
Xi = rng.integers(-99, 99, (70, 3))
assert np.array_equal(mg.naive_gemm(W, Xi), orc.naive_gemm(W, Xi))
Xh = rng.standard_normal((200, 16)).astype(np.float16)
pwm = mg.from_codes(rng.integers(0, 16, (256, 200), dtype=np.uint8), cb)
Yk = mg.dequant_gemm(pwm, torch.from_numpy(Xh).cuda()).cpu().numpy()
assert orc.rel_error(Yk, orc.dense(pwm.data, 200, 4, orc.int4_values()), Xh) <= 2e-3
# the weight-streaming dense kernel (mma.sync, cluster split-k over DSMEM): b = 1, 8, 13
Xh2 = rng.standard_normal((2080, 13)).astype(np.float16)
pwm2 = mg.from_codes(rng.integers(0, 16, (300, 2080), dtype=np.uint8), cb)
W2 = orc.dense(pwm2.data, 2080, 4, orc.int4_values())
for nb in (1, 8, 13):
    Yh = mg.dequant_gemm(pwm2, torch.from_numpy(np.ascontiguousarray(Xh2[:, :nb])).cuda(), kernel="hmma").cpu().numpy()
    assert orc.rel_error(Yh, W2, Xh2[:, :nb]) <= 2e-3
# Y fan-out of the finishing kernels (same-device stand-in peers)
Xf = torch.from_numpy(rng.standard_normal((700, 8)).astype(np.float16)).cuda()
pwm3 = mg.from_codes(rng.integers(0, 16, (2100, 700), dtype=np.uint8), cb)
own = torch.empty((2100, 8), dtype=torch.float16, device="cuda")
peers = [torch.empty_like(own) for _ in range(2)]
mg.msgemm(pwm3, Xf, 3, out=own, _fan=[p.data_ptr() for p in peers])
assert all(torch.equal(p, own) for p in peers)
torch.cuda.synchronize()
print("sanitize probe ok")
