"""Dense baseline (K4) kernels timed per config: weight-streaming mma.sync vs CUDA-core GEMV vs tcgen05,
weights rotated over >= 3x L2, CUDA-graph replay, CUDA events.

    python tools/dense_probe.py
"""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402

L2 = 126 * 2 ** 20
PEAK = 6549.1
rng = np.random.default_rng(0)
for (m, k, bs) in ((8192, 8192, (1, 8)), (4096, 4096, (1,))):
    data = rng.integers(0, 256, (m, k // 2), dtype=np.uint8)
    nc = max(2, math.ceil(3 * L2 / data.nbytes))
    base = torch.from_numpy(data).cuda()
    pwms = [mg.PackedWeightMatrix(m=m, k=k, width=4, data=base if c == 0 else base.clone(),
                                  codebook=mg.int4_codebook()) for c in range(nc)]
    for b in bs:
        x = torch.from_numpy(rng.standard_normal((k, b)).astype(np.float16)).cuda()
        for kern in ("hmma",):
            if (kern == "gemv" and b > 8) or (kern == "hmma" and b > 16):
                continue
            Y = torch.empty((m, b), dtype=torch.float32, device="cuda")
            for p in pwms:
                mg.dequant_gemm(p, x, out=Y, kernel=kern)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    for p in pwms * max(1, 16 // nc):
                        mg.dequant_gemm(p, x, out=Y, kernel=kern)
            torch.cuda.synchronize()
            n = nc * max(1, 16 // nc)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * n)
            byts = m * k / 2 + k * b * 2 + m * b * 4
            print(f"{m}x{k} b={b:3d} {kern:4s} {us:8.1f} us  {byts / us / 1e3:7.0f} GB/s  "
                  f"({byts / us / 1e3 / PEAK:.1%} HBM)  {2 * m * k * b / us / 1e6:8.1f} TOP/s", flush=True)
