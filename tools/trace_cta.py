"""Per-CTA timeline of one msgemm launch (diagnostics; uses msg_set_tracing)."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg
from paper_2310_06178_b200 import _lib
from paper_2310_06178_b200.workloads import CONFIGS, activations, weights

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4b1"
cfg = CONFIGS[name]
pwm = mg.PackedWeightMatrix(m=cfg.m, k=cfg.k, width=4, data=torch.from_numpy(weights(cfg)).cuda(),
                            codebook=mg.int4_codebook())
xd = torch.from_numpy(activations(cfg)).cuda()
for _ in range(3):
    mg.msgemm(pwm, xd, cfg.d)
torch.cuda.synchronize()
_lib.lib().msg_set_tracing(1)
mg.msgemm(pwm, xd, cfg.d)
torch.cuda.synchronize()
tr = _lib.read_trace()
_lib.lib().msg_set_tracing(0)
t0 = tr[:, 1].min()
start = (tr[:, 1] - t0) / 1e3
end = (tr[:, 2] - t0) / 1e3
dur = end - start
print(f"{name}: {len(tr)} CTAs; start us min/max {start.min():.2f}/{start.max():.2f}; "
      f"end min/med/max {end.min():.2f}/{np.median(end):.2f}/{end.max():.2f}; "
      f"dur min/med/max {dur.min():.2f}/{np.median(dur):.2f}/{dur.max():.2f}")
order = np.argsort(dur)
for i in list(order[:5]) + list(order[-8:]):
    print(f"  cta {i:4d} sm {int(tr[i,0]):3d} start {start[i]:6.2f} dur {dur[i]:6.2f} units {int(tr[i,3])}")
