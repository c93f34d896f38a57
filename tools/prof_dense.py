"""A few dense-baseline calls on one shape (a short program for ncu).
    python tools/prof_dense.py [m] [k] [b] [gemv|mma]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402

m, k, b = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 8192, 1)))
kern = sys.argv[4] if len(sys.argv) > 4 else "gemv"
rng = np.random.default_rng(0)
pwm = mg.PackedWeightMatrix(m=m, k=k, width=4, codebook=mg.int4_codebook(),
                            data=torch.from_numpy(rng.integers(0, 256, (m, k // 2), dtype=np.uint8)).cuda())
x = torch.from_numpy(rng.standard_normal((k, b)).astype(np.float16)).cuda()
for _ in range(4):
    y = mg.dequant_gemm(pwm, x, kernel=kern)
torch.cuda.synchronize()
print("ok", float(y.abs().mean()))
