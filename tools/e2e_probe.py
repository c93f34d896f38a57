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

# a CUDA graph holding H2D (pinned staging) -> msGeMM kernels -> D2H (pinned staging)
from paper_2310_06178_b200 import _lib, gemm  # noqa: E402
xs_h = torch.empty_like(Xpin).pin_memory()
ys_h = torch.empty_like(Ypin).pin_memory()
xs_d = torch.empty_like(xd)
ys_d = torch.empty_like(Yd)
for _ in range(3):
    mg.msgemm(pwm, xs_d, cfg.d, out=ys_d)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(2):
        mg.msgemm(pwm, xs_d, cfg.d, out=ys_d)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        xs_d.copy_(xs_h, non_blocking=True)
        mg.msgemm(pwm, xs_d, cfg.d, out=ys_d)
        ys_h.copy_(ys_d, non_blocking=True)
torch.cuda.synchronize()
cur = torch.cuda.current_stream()
Xn = np.ascontiguousarray(X)
xs_np = xs_h.numpy()


def graph_call():
    np.copyto(xs_np, Xn)
    g.replay()
    cur.synchronize()
    return ys_h.numpy().copy()


bench("graph: numpy X -> numpy Y", graph_call)
bench("graph replay + sync only", lambda: (g.replay(), cur.synchronize()))
y1 = graph_call()
y2 = mg.msgemm(pwm, X, cfg.d)
print("graph result matches:", np.array_equal(y1.view(np.uint16), y2.view(np.uint16)))
