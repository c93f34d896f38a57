"""Break down the end-to-end msgemm call (host X in, host Y out) on the GPU.

    python tools/e2e_probe.py [cfg4b1]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402
from paper_2310_06178_b200.workloads import CONFIGS, activations, weights  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4b1"]
dev = torch.device("cuda", 0)
pwm = mg.PackedWeightMatrix(m=cfg.m, k=cfg.k, width=4, data=torch.from_numpy(weights(cfg)).to(dev),
                            codebook=mg.int4_codebook())
X = activations(cfg)
Xpin = torch.from_numpy(X).pin_memory()
xd = Xpin.to(dev)
Ypin = torch.empty((cfg.m, cfg.b), dtype=xd.dtype, pin_memory=True)
Yd = torch.empty((cfg.m, cfg.b), dtype=xd.dtype, device=dev)


def bench(name, fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {1e6 * (time.perf_counter() - t0) / n:8.1f} us")


bench("e2e: pinned X -> pinned Y", lambda: mg.msgemm(pwm, Xpin, cfg.d, out=Ypin))
bench("device X -> device Y (async)", lambda: mg.msgemm(pwm, xd, cfg.d, out=Yd))
bench("device X -> device Y + sync", lambda: (mg.msgemm(pwm, xd, cfg.d, out=Yd), torch.cuda.synchronize()))
bench("H2D X + D2H Y copies only", lambda: (xd.copy_(Xpin, non_blocking=True), Ypin.copy_(Yd)))
bench("numpy X -> numpy Y", lambda: mg.msgemm(pwm, X, cfg.d))
