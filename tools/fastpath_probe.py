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
keys=[k for k in pwm._device_cache if k[0]=="fast"]
print("fast keys", len(keys))
ent = pwm._device_cache[keys[0]]
print("ent returns", type(ent(Xpin, Ypin)))
def T(name, fn, n=300):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(n): fn()
    t1=time.perf_counter()
    print(f"{name:30s} {1e6*(t1-t0)/n:7.2f} us")
T("msgemm", lambda: mg.msgemm(pwm, Xpin, 3, out=Ypin))
T("ent", lambda: ent(Xpin, Ypin))
stream = _lib.current_stream_handle(dev)
call = gemm._call_plan(pwm, dev, stream, 1, _lib.F16, torch.float16, 3, None, True, None, 0)
T("run_host", lambda: call.run_host(Xpin, Ypin, stream))
T("host_call", lambda: gemm._host_call(call, Xpin, Ypin, stream, True, False))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(200): mg.msgemm(pwm, Xpin, 3, out=Ypin)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)
