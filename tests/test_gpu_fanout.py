"""Y fan-out of the finishing kernels (msg_gemm_fanout, include/msgemm_b200.h):
the row-sharded all-gather fused into the epilogue.  One
GPU stands in for the peers with extra buffers on the same device -- the
kernels only see addresses -- and a world-size-1 symmetric-memory run covers
the torch plumbing; the reference has no distributed path,
so the check is bitwise equality with the plain call."""

import os

import numpy as np
import pytest

import paper_2310_06178_b200 as mg
from paper_2310_06178_b200 import sharded

pytestmark = pytest.mark.gpu

CASES = [  # (m, k, b, d, x dtype, kwargs): one per finishing kernel / route
    (1003, 600, 1, 3, np.float16, {}),                          # lane finish, ragged rows
    (4096, 512, 1, 3, np.float16, {"out_dtype": np.float32}),   # lane finish, fp32 Y
    (2100, 700, 8, 3, np.float16, {}),                          # rb_tmem + vec4 finish
    (515, 300, 4, 3, np.float16, {}),                           # rb_lut<4>
    (333, 301, 3, 3, np.float16, {}),                           # rb_lut, scalar finish
    (640, 256, 2, 2, np.float32, {}),                           # fused quad, fp32 X
    (700, 300, 8, 3, np.float16, {"symmetric": False}),         # full tables
]


@pytest.mark.parametrize("m,k,b,d,dt,kw", CASES)
@pytest.mark.parametrize("sparse", [False, True])
def test_fanout_matches_plain_call(m, k, b, d, dt, kw, sparse):
    import torch
    rng = np.random.default_rng(m + k + b)
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    if sparse:
        codes[3::17] = 0       # all-zero rows: the full-table fix-up scatters into every copy
    pwm = mg.from_codes(codes, mg.int4_codebook())
    X = torch.from_numpy(rng.standard_normal((k, b)).astype(dt)).cuda()
    ref = mg.msgemm(pwm, X, d, **kw)
    lo, hi = 0, m              # "this rank's rows" inside three full-height copies of Y
    own = torch.full((m + 8, b), 7, dtype=ref.dtype, device="cuda")
    peers = [torch.full((m + 8, b), 7, dtype=ref.dtype, device="cuda") for _ in range(2)]
    off = 8 * b * ref.element_size()   # the slice starts 8 rows down: offsets travel with the pointers
    mg.msgemm(pwm, X, d, out=own[8:8 + m], _fan=[p.data_ptr() + off for p in peers], **kw)
    torch.cuda.synchronize()
    for buf in [own] + peers:
        assert torch.equal(buf[8:8 + m].view(torch.uint8), ref.reshape(m, b).view(torch.uint8))
        assert bool((buf[:8] == 7).all())          # nothing before the slice is touched


def test_fanout_rejects_what_it_cannot_do():
    import torch
    rng = np.random.default_rng(1)
    pwm = mg.from_codes(rng.integers(0, 16, (64, 40), dtype=np.uint8), mg.int4_codebook())
    X = torch.from_numpy(rng.standard_normal((40, 2))).cuda()            # f64: generic path
    out = torch.empty((64, 2), dtype=torch.float64, device="cuda")
    peer = torch.empty_like(out)
    with pytest.raises(NotImplementedError):
        mg.msgemm(pwm, X, 4, out=out, _fan=[peer.data_ptr()])
    with pytest.raises(ValueError):
        mg.msgemm(pwm, X.cpu().numpy(), 4, _fan=[peer.data_ptr()])       # host path: no fan-out
    with pytest.raises(ValueError):
        mg.msgemm(pwm, X, 4, out=out, _fan=[peer.data_ptr()] * 8)


_WORLD1 = r"""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg
from paper_2310_06178_b200 import sharded
os.environ["MASTER_ADDR"] = "127.0.0.1"
os.environ["MASTER_PORT"] = sys.argv[1]
try:
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
except Exception as e:
    print("SKIP: process group:", e); sys.exit(0)
rng = np.random.default_rng(5)
m, k, b = 1024, 768, 8
pwm = mg.from_codes(rng.integers(0, 16, (m, k), dtype=np.uint8), mg.int4_codebook())
X = torch.from_numpy(rng.standard_normal((k, b)).astype(np.float16)).cuda()
try:
    py = sharded.PeerY(m, b, torch.float16, torch.device("cuda", 0))
except RuntimeError as e:
    print("SKIP: symmetric memory:", e); sys.exit(0)
assert py.targets() == [] and (py.lo, py.hi) == (0, m)
y = sharded.msgemm_sharded_fused(sharded.shard_rows(pwm, 1, 0), X, 3, py)
y2 = sharded.msgemm_sharded_fused(sharded.shard_rows(pwm, 1, 0), X, 3, py)   # reuse of the buffer
torch.cuda.synchronize()
assert torch.equal(y, mg.msgemm(pwm, X, 3)) and y2.data_ptr() == y.data_ptr()
print("OK")
dist.destroy_process_group()
"""


def test_symmetric_memory_world1(tmp_path):
    """PeerY + msgemm_sharded_fused with one rank: rendezvous, barrier, view.
    In a subprocess with a time limit: a process group must not leak into (or
    hang) the test session."""
    import socket
    import subprocess
    import sys
    from pathlib import Path
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    script = tmp_path / "world1.py"
    script.write_text(_WORLD1)
    try:
        r = subprocess.run([sys.executable, str(script), str(port)], cwd=Path(__file__).resolve().parents[1],
                           capture_output=True, text=True, timeout=240)
    except subprocess.TimeoutExpired:
        pytest.skip("symmetric-memory rendezvous did not finish in time on this box")
    out = r.stdout + r.stderr
    if "SKIP:" in r.stdout:
        pytest.skip(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0 and "OK" in r.stdout, out[-3000:]
