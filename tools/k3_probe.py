"""K3 repack throughput per layout (one-time weight re-layout), CUDA events.

    python tools/k3_probe.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_06178_b200 import _lib  # noqa: E402

lib = _lib.lib()
peak = 6549.1
for (m, k) in ((65536, 8192), (8192, 8192), (4096, 4096)):
    rng = np.random.default_rng(0)
    data = torch.from_numpy(rng.integers(0, 256, (m, (k + 1) // 2), dtype=np.uint8)).cuda()
    for name, layout in (("lane", _lib.LAYOUT_LANE), ("rb4", _lib.LAYOUT_RB4), ("rb4s", _lib.LAYOUT_RB4S), ("rb8", _lib.LAYOUT_RB8),
                         ("rb16", _lib.LAYOUT_RB16), ("quad", _lib.LAYOUT_QUAD)):
        nbytes = int(lib.msg_repacked_bytes(m, k, 3, layout))
        out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream

        def run():
            _lib.check(lib.msg_repack(_lib.ptr(data), m, k, 3, layout, 1, _lib.ptr(out), st))
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        tot = data.numel() + nbytes
        print(f"{m}x{k} {name:5s} {ms * 1e3:9.1f} us  {tot / ms / 1e6:8.1f} GB/s  ({tot / ms / 1e6 / peak:.1%} of HBM)")
