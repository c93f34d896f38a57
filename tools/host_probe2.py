import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2310_06178_b200 as mg
from paper_2310_06178_b200 import _lib, gemm
from paper_2310_06178_b200.workloads import CONFIGS, activations, weights
cfg = CONFIGS["cfg4b1"]
dev = torch.device("cuda", 0)
pwm = mg.PackedWeightMatrix(m=cfg.m, k=cfg.k, width=4, data=torch.from_numpy(weights(cfg)).to(dev), codebook=mg.int4_codebook())
X = activations(cfg)
Xpin = torch.from_numpy(X).pin_memory(); Ypin = torch.empty((cfg.m,1), dtype=torch.float16).pin_memory()
for _ in range(5): mg.msgemm(pwm, Xpin, 3, out=Ypin)
torch.cuda.synchronize()
def T(name, fn, n=300):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(n): fn()
    t1=time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:30s} {1e6*(t1-t0)/n:7.2f} us")
stream = _lib.current_stream_handle(dev)
call = gemm._call_plan(pwm, dev, stream, 1, _lib.F16, torch.float16, 3, None, True, None, 0)
T("msgemm pinned->pinned", lambda: mg.msgemm(pwm, Xpin, 3, out=Ypin))
T("run_host", lambda: call.run_host(Xpin, Ypin, stream))
print("graphs", len(call._graphs), "seen", len(call._seen))
Xn = X.copy()
T("msgemm numpy->numpy", lambda: mg.msgemm(pwm, Xn, 3))
T("run_host numpy", lambda: call.run_host(Xn, None, stream))
print("graphs", len(call._graphs), "seen", len(call._seen))
g = next(iter(call._graphs.values()))[0]
cur = torch.cuda.current_stream(dev)
T("replay+sync", lambda: (g.replay(), cur.synchronize()))
T("replay only", lambda: g.replay(), 100)
T("is_pinned", lambda: Xpin.is_pinned())
T("current_stream", lambda: torch.cuda.current_stream(dev))
T("is_capturing", lambda: torch.cuda.is_current_stream_capturing())
T("require_device", lambda: _lib.require_device())
T("current_stream_handle", lambda: _lib.current_stream_handle(dev))
T("ensure_device_pwm", lambda: gemm._ensure_device_pwm(pwm))
T("data_ptr", lambda: Xpin.data_ptr())
T("empty sync", lambda: cur.synchronize())
