"""msGeMM vs the dense baseline across batch sizes on one weight matrix
(8192 x 8192 int4, fp16 X, d = 3): device time per call, CUDA-graph replay,
weights rotated over >= 3x L2.

    python tools/batch_sweep.py [m] [k]
"""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
L2 = 126 * 2 ** 20
rng = np.random.default_rng(0)
data = rng.integers(0, 256, (m, k // 2), dtype=np.uint8)
nc = max(2, math.ceil(3 * L2 / data.nbytes))
base = torch.from_numpy(data).cuda()
pwms = [mg.PackedWeightMatrix(m=m, k=k, width=4, data=base if c == 0 else base.clone(),
                              codebook=mg.int4_codebook()) for c in range(nc)]


def timed(fn):
    for i in range(nc):
        fn(i)
    torch.cuda.synchronize()
    n = nc * max(1, 24 // nc)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(n):
                fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (4 * n)


print(f"{'b':>4s} {'msGeMM us':>10s} {'dense us':>9s} {'ratio':>6s}")
for b in [int(v) for v in __import__("os").environ.get("BS", "1,2,3,4,6,8,12,16,32").split(",")]:
    x = torch.from_numpy(rng.standard_normal((k, b)).astype(np.float16)).cuda()
    Y = torch.empty((m, b), dtype=torch.float16, device="cuda")
    Yd = torch.empty((m, b), dtype=torch.float32, device="cuda")
    t_ms = timed(lambda i: mg.msgemm(pwms[i % nc], x, 3, out=Y))
    t_d = timed(lambda i: mg.dequant_gemm(pwms[i % nc], x, out=Yd))
    print(f"{b:4d} {t_ms:10.1f} {t_d:9.1f} {t_d / t_ms:6.2f}", flush=True)
