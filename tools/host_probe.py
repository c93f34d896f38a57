"""Host-side cost of the msgemm call pieces (device-resident X and Y).

    python tools/host_probe.py
"""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2310_06178_b200 as mg
from paper_2310_06178_b200 import _lib, gemm
from paper_2310_06178_b200.workloads import CONFIGS, activations, weights
cfg = CONFIGS["cfg4b1"]
dev = torch.device("cuda", 0)
pwm = mg.PackedWeightMatrix(m=cfg.m, k=cfg.k, width=4, data=torch.from_numpy(weights(cfg)).to(dev), codebook=mg.int4_codebook())
xd = torch.from_numpy(activations(cfg)).to(dev)
Y = torch.empty((cfg.m, 1), dtype=torch.float16, device=dev)
for _ in range(5): mg.msgemm(pwm, xd, 3, out=Y)
torch.cuda.synchronize()
def T(name, fn, n=2000):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(n): fn()
    t1=time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:30s} {1e6*(t1-t0)/n:7.2f} us (host, before sync)")
stream = _lib.current_stream_handle(dev)
call = gemm._call_plan(pwm, dev, stream, 1, _lib.F16, xd.dtype, 3, None, True, None, 0)
T("msgemm device", lambda: mg.msgemm(pwm, xd, 3, out=Y), 500)
T("call.launch only", lambda: call.launch(xd, Y), 500)
T("require_device", lambda: _lib.require_device())
T("current_stream", lambda: torch.cuda.current_stream(dev))
T("_call_plan lookup", lambda: gemm._call_plan(pwm, dev, stream, 1, _lib.F16, xd.dtype, 3, None, True, None, 0))
T("_as_matrix", lambda: gemm._as_matrix(xd))
T("dtype_code", lambda: _lib.dtype_code(xd.dtype))
T("np_dtype", lambda: gemm._np_dtype(xd))
