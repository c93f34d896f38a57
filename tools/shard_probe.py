"""Per-rank step time of config 5 at N = 1, 2, 4, 8 for both multi-GPU splits,
emulated on one GPU (the shard each rank would run; collectives excluded).

    python tools/shard_probe.py [cfg5]
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402
from paper_2310_06178_b200.sharded import k_split_bounds  # noqa: E402
from paper_2310_06178_b200.workloads import CONFIGS, activations, weights  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
dev = torch.device("cuda", 0)
W = weights(cfg)
X = activations(cfg)
L2 = 126 * 2 ** 20
FLAGS = int(os.environ.get("MSG_BENCH_FLAGS", "0"))  # e.g. 128: 4096-row CTAs


def time_shard(data, kr, xs, yd):
    ncopies = max(2, math.ceil(3 * L2 / data.nbytes))
    base = torch.from_numpy(np.ascontiguousarray(data)).to(dev)
    pwms = [mg.PackedWeightMatrix(m=data.shape[0], k=kr, width=4, data=base if c == 0 else base.clone(),
                                  codebook=mg.int4_codebook()) for c in range(ncopies)]
    xd = torch.from_numpy(np.ascontiguousarray(xs)).to(dev)
    Y = torch.empty((data.shape[0], cfg.b), dtype=yd, device=dev)
    for i in range(ncopies):
        mg.msgemm(pwms[i], xd, cfg.d, out=Y, out_dtype=None if yd == xd.dtype else np.float32,
                  _flags=FLAGS)
    torch.cuda.synchronize()
    n = ncopies * max(1, math.ceil(20 / ncopies))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n):
            mg.msgemm(pwms[i % ncopies], xd, cfg.d, out=Y,
                      out_dtype=None if yd == xd.dtype else np.float32, _flags=FLAGS)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * n)


for N in (1, 2, 4, 8):
    mr = cfg.m // N
    t_rows = time_shard(W[:mr], cfg.k, X, torch.float16)
    k0, k1 = k_split_bounds(cfg.k, cfg.d, N, 0)
    t_k = time_shard(W[:, k0 // 2:(k1 + 1) // 2], k1 - k0, X[k0:k1], torch.float32)
    print(f"N={N}: row shard {mr}x{cfg.k}: {t_rows:8.1f} us/step   "
          f"k shard {cfg.m}x{k1 - k0}: {t_k:8.1f} us/step   (N=1 x 1/N: {t_rows if N == 1 else 0:.0f})",
          flush=True)
