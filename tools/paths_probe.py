"""Small msgemm calls through every kernel family (odd shapes, tails), each
checked against the oracle -- a quick all-paths probe.

    python tools/paths_probe.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402
from oracle import msgemm_oracle as orc  # noqa: E402

rng = np.random.default_rng(3)
cb = mg.int4_codebook()
for (m, k, b, d, dt) in [(97, 301, 1, 3, np.float16),    # lane GEMV (+ tail)
                         (700, 1000, 1, 3, np.float16),   # lane, several chunks
                         (300, 200, 8, 3, np.float16),    # row-block BC=8
                         (300, 200, 4, 3, np.float16),    # row-block BC=4 (512 threads)
                         (64, 50, 3, 2, np.float32),      # row-block f32
                         (40, 30, 2, 4, np.float64)]:     # generic
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, cb)
    X = rng.standard_normal((k, b)).astype(dt)
    Y = mg.msgemm(pwm, X, d)
    W = orc.dense(pwm.data, k, 4, orc.int4_values())
    tol = {np.float16: 2e-3, np.float32: 1e-5, np.float64: 1e-12}[dt]
    assert orc.rel_error(Y, W, X) <= tol, (m, k, b, d)
Xh = rng.standard_normal((200, 16)).astype(np.float16)
pwm = mg.from_codes(rng.integers(0, 16, (256, 200), dtype=np.uint8), cb)
mg.dequant_gemm(pwm, torch.from_numpy(Xh).cuda())           # K4
torch.cuda.synchronize()
print("sanitize probe ok")
