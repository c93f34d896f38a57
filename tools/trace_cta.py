"""Per-CTA timeline of one msgemm launch (diagnostics; uses msg_set_tracing).

    python tools/trace_cta.py [cfg4b1] [flags]

Lane kernel phase columns: build = summed table-build time (thread 0),
wait = warp 0's summed mbarrier waits, loop = end of the main loop,
count = after the tile-arrival counters (before the finishing writes).
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402
from paper_2310_06178_b200 import _lib  # noqa: E402
from paper_2310_06178_b200.workloads import CONFIGS, activations, weights  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4b1"
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = CONFIGS[name]
pwm = mg.PackedWeightMatrix(m=cfg.m, k=cfg.k, width=4, data=torch.from_numpy(weights(cfg)).cuda(),
                            codebook=mg.int4_codebook())
xd = torch.from_numpy(activations(cfg)).cuda()
for _ in range(3):
    mg.msgemm(pwm, xd, cfg.d, _flags=flags)
torch.cuda.synchronize()
_lib.lib().msg_set_tracing(1)
mg.msgemm(pwm, xd, cfg.d, _flags=flags)
torch.cuda.synchronize()
tr = _lib.read_trace().astype(np.float64)
_lib.lib().msg_set_tracing(0)
t0 = tr[:, 1].min()
start = (tr[:, 1] - t0) / 1e3
end = (tr[:, 2] - t0) / 1e3
dur = end - start
build = tr[:, 4] / 1e3
wait = np.where(tr[:, 5] > 0, (tr[:, 5] - t0) / 1e3, np.nan)  # lane: thread 0 at the 2nd build
loop = np.where(tr[:, 6] > 0, (tr[:, 6] - t0) / 1e3, np.nan)
count = np.where(tr[:, 7] > 0, (tr[:, 7] - t0) / 1e3, np.nan)
print(f"{name}: {len(tr)} CTAs; start us min/max {start.min():.2f}/{start.max():.2f}; "
      f"end min/med/max {end.min():.2f}/{np.median(end):.2f}/{end.max():.2f}; "
      f"dur min/med/max {dur.min():.2f}/{np.median(dur):.2f}/{dur.max():.2f}")
print(f"  build med {np.median(build):.2f}  wait(w0) med {np.median(wait):.2f}  "
      f"loop-end med/max {np.nanmedian(loop):.2f}/{np.nanmax(loop):.2f}  "
      f"count-end med/max {np.nanmedian(count):.2f}/{np.nanmax(count):.2f}")
order = np.argsort(dur)
for i in list(order[:5]) + list(order[-8:]):
    print(f"  cta {i:4d} sm {int(tr[i,0]):3d} start {start[i]:6.2f} dur {dur[i]:6.2f} "
          f"tiles {int(tr[i,3]) & 0xffffffff} fin {int(tr[i,3]) >> 32} build {build[i]:5.2f} wait {wait[i]:5.2f} "
          f"loop {loop[i]:6.2f} count {count[i]:6.2f} end {end[i]:6.2f}")
