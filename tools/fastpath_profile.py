"""cProfile of the drop-in host path (pinned tensors vs numpy arrays) at a GEMV shape.
    python tools/fastpath_profile.py [cfg4b1]"""
import cProfile
import pstats
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
Ypin = torch.empty((cfg.m, cfg.b) if X.ndim == 2 else (cfg.m,), dtype=Xpin.dtype, pin_memory=True)
print("X", X.shape, "Ypin", tuple(Ypin.shape))
Xnp_view = Xpin.numpy()
X2 = X + 1


def pinned_rewritten():
    np.copyto(Xnp_view, X2)     # a serving loop writes fresh activations into its pinned buffer
    return mg.msgemm(pwm, Xpin, cfg.d, out=Ypin)


for name, fn in (("pinned", lambda: mg.msgemm(pwm, Xpin, cfg.d, out=Ypin)), ("pinned, X rewritten", pinned_rewritten),
                 ("numpy", lambda: mg.msgemm(pwm, X, cfg.d))):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(500):
        fn()
    print(name, f"{1e6 * (time.perf_counter() - t0) / 500:.1f} us per call")
    if "-p" not in sys.argv:
        continue
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(500):
        fn()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
