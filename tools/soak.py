"""Randomised parity soak of the round-2 additions (run under gpurun; not part
of pytest): dense HMMA kernel on random shapes / splits, b = 1 finishing
kernel with ragged rows and misaligned outputs, Y fan-out on random routes.
    python tools/soak.py [seconds]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402
from oracle import msgemm_oracle as orc  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(os.environ.get("SOAK_SEED", "7")))
t0 = time.time()
n = {"hmma": 0, "lane": 0, "fan": 0, "host": 0}
while time.time() - t0 < budget:
    # ---- dense HMMA kernel: integer X bit-exact against numpy
    m = int(rng.integers(1, 3000)); k = 32 * int(rng.integers(1, 200)); b = int(rng.integers(1, 17))
    os.environ["MSG_DH_SPLIT"] = str(int(rng.choice([0, 1, 2, 3, 4, 5, 6, 7, 8])))
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    book, vals = ((mg.int4_codebook(), orc.int4_values()) if rng.random() < 0.5
                  else (mg.uint4_codebook(), orc.uint4_values()))
    pwm = mg.from_codes(codes, book)
    Xi = rng.integers(-20, 21, (k, b))
    xd = torch.from_numpy(Xi.astype(np.float16)).cuda()
    if rng.random() < 0.3:      # a misaligned activation view
        buf = torch.empty(k * b + 1, dtype=torch.float16, device="cuda")
        buf[1:] = xd.reshape(-1)
        xd = buf[1:].reshape(k, b)
    y = mg.dequant_gemm(pwm, xd, kernel="hmma").cpu().numpy()
    ref = vals[codes].astype(np.int64) @ Xi.astype(np.int64)
    assert np.array_equal(y.astype(np.int64), ref), ("hmma", m, k, b, os.environ["MSG_DH_SPLIT"])
    n["hmma"] += 1
    # ---- b = 1 lane path: ragged m, fp16 / fp32 Y, aligned and misaligned out
    m = int(rng.integers(1, 2500)); k = int(rng.integers(3, 1500))
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, mg.int4_codebook())
    x = rng.standard_normal(k).astype(np.float16)
    xt = torch.from_numpy(x).cuda()
    odt = np.float32 if rng.random() < 0.5 else None
    ref = mg.msgemm(pwm, xt, 3, out_dtype=odt)
    W = orc.int4_values()[codes]
    assert orc.rel_error(ref.cpu().numpy(), W, x) <= 2e-3
    off = int(rng.integers(0, 9))
    big = torch.full((m + 16,), 3, dtype=ref.dtype, device="cuda")
    out = big[off:off + m]
    peers = [torch.full((m + 16,), 3, dtype=ref.dtype, device="cuda") for _ in range(int(rng.integers(0, 3)))]
    mg.msgemm(pwm, xt, 3, out_dtype=odt, out=out,
              _fan=[p.data_ptr() + off * ref.element_size() for p in peers] or None)
    torch.cuda.synchronize()
    for bufr in [big] + peers:
        assert torch.equal(bufr[off:off + m], ref), ("lane", m, k, off, odt)
        assert bool((bufr[:off] == 3).all()) and bool((bufr[off + m:] == 3).all()), ("lane guard", m, k, off)
    n["lane"] += 1
    # ---- fan-out on a random batched route
    m = int(rng.integers(1, 3000)); k = int(rng.integers(3, 900)); b = int(rng.integers(2, 17))
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    if rng.random() < 0.3:
        codes[::13] = 0
    pwm = mg.from_codes(codes, mg.int4_codebook())
    X = torch.from_numpy(rng.standard_normal((k, b)).astype(np.float16)).cuda()
    ref = mg.msgemm(pwm, X, 3)
    assert orc.rel_error(ref.cpu().numpy(), orc.int4_values()[codes], X.cpu().numpy()) <= 2e-3
    own = torch.full((m + 2, b), 5, dtype=ref.dtype, device="cuda")
    peers = [torch.full((m + 2, b), 5, dtype=ref.dtype, device="cuda") for _ in range(int(rng.integers(1, 4)))]
    ob = b * ref.element_size()
    mg.msgemm(pwm, X, 3, out=own[1:1 + m], _fan=[p.data_ptr() + ob for p in peers])
    torch.cuda.synchronize()
    # (an out at another alignment may take the other finishing kernel, whose
    # slice-group count and hence fp32 summation order differ: compare the
    # copies of ONE call bitwise, and that call with the oracle)
    assert orc.rel_error(own[1:1 + m].cpu().numpy(), orc.int4_values()[codes], X.cpu().numpy()) <= 2e-3
    for bufr in peers:
        assert torch.equal(bufr, own), ("fan", m, k, b)
    assert bool((own[0] == 5).all()) and bool((own[m + 1] == 5).all())
    n["fan"] += 1
    # ---- host path (numpy in / numpy out, graph replays from the 2nd call) vs the device path
    os.environ.pop("MSG_DH_SPLIT", None)
    m = int(rng.integers(1, 2000)); k = int(rng.integers(3, 1200)); b = int(rng.choice([1, 1, 2, 3, 4, 8, 13]))
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    if rng.random() < 0.3:
        codes[::7] = 0
    pwm = mg.from_codes(codes, mg.int4_codebook())
    for _ in range(3):
        Xn = rng.standard_normal((k, b)).astype(np.float16)
        yh = mg.msgemm(pwm, Xn, 3)
        yd = mg.msgemm(pwm, torch.from_numpy(Xn).cuda(), 3).cpu().numpy()
        assert yh.shape == (m, b) and np.array_equal(yh.view(np.uint16), yd.view(np.uint16)), ("host", m, k, b)
    n["host"] += 1
print("soak ok", n, f"{time.time() - t0:.0f}s")
