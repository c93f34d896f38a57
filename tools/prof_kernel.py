"""Run msgemm a few times on one shape (a short program for ncu captures).

    python tools/prof_kernel.py [m] [k] [b] [flags] [dtype]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
b = int(sys.argv[3]) if len(sys.argv) > 3 else 8
flags = int(sys.argv[4]) if len(sys.argv) > 4 else 0
dt = np.float32 if (len(sys.argv) > 5 and sys.argv[5] == "f32") else np.float16
rng = np.random.default_rng(7)
data = rng.integers(0, 256, size=(m, (k + 1) // 2), dtype=np.uint8)
pwm = mg.PackedWeightMatrix(m=m, k=k, width=4, data=torch.from_numpy(data).cuda(),
                            codebook=mg.int4_codebook())
x = torch.from_numpy(rng.standard_normal((k, b)).astype(dt)).cuda()
for _ in range(4):
    y = mg.msgemm(pwm, x, 3, _flags=flags)
torch.cuda.synchronize()
print("ok", float(y.float().abs().mean()))
