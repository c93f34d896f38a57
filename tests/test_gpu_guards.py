"""Guard bands around every device buffer a kernel writes (Y, workspace) and
reads (X): out-of-bounds writes of any kernel family show up as changed
canary bytes (compute-sanitizer's memcheck is not available on this pool).

Buffers are carved out of one allocation as [canary | buffer | canary], with
the buffer at an odd 256-byte offset so a write past either end cannot land in
padding that the allocator would hide.  Results are also checked against the
oracle so a read of a canary shows up as a wrong value.
"""

import numpy as np
import pytest

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc
from paper_2310_06178_b200 import _lib

pytestmark = pytest.mark.gpu
GUARD = 4096
CANARY = 0xA5


class Guarded:
    def __init__(self, nbytes, dev, fill=CANARY):
        import torch
        self.n = int(nbytes)
        self.raw = torch.full((GUARD + 256 + self.n + GUARD,), fill, dtype=torch.uint8, device=dev)
        self.lo = GUARD + 256
        self.view = self.raw[self.lo:self.lo + self.n]

    def intact(self):
        raw = self.raw.cpu().numpy()
        return bool((raw[:self.lo] == CANARY).all() and (raw[self.lo + self.n:] == CANARY).all())


@pytest.fixture
def guarded_workspaces(monkeypatch):
    made = []

    def workspace(nbytes, dev, kind="scratch"):
        g = Guarded(max(int(nbytes), 256), dev)
        g.view.zero_()                      # the lane workspace must start zero
        made.append(g)
        return g.view

    monkeypatch.setattr(_lib, "workspace", workspace)
    return made


CASES = [  # (m, k, b, d, x dtype, kwargs) -- one per kernel family
    (97, 301, 1, 3, np.float16, {}),                       # lane GEMV + finish
    (700, 1000, 1, 3, np.float16, {}),
    (300, 200, 8, 3, np.float16, {}),                      # rb_tmem
    (130, 301, 16, 3, np.float16, {}),
    (300, 200, 4, 3, np.float16, {}),                      # rb_lut<4>
    (257, 98, 2, 3, np.float16, {}),                       # rb_lut<2>
    (64, 50, 3, 2, np.float32, {}),                        # fused quad, fp32
    (90, 300, 8, 3, np.float16, {"table_dtype": np.float32}),
    (90, 300, 8, 3, np.float16, {"symmetric": False}),
    (40, 30, 2, 4, np.float64, {}),                        # generic
]


@pytest.mark.parametrize("m,k,b,d,dt,kw", CASES)
def test_no_out_of_bounds_writes(guarded_workspaces, m, k, b, d, dt, kw):
    import torch
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(m * 7 + k + b)
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    codes[::9] = 0                                          # zero rows: the fix-up path too
    pwm = mg.from_codes(codes, mg.int4_codebook())
    X = rng.standard_normal((k, b)).astype(dt)
    xt = torch.from_numpy(X[:, 0].copy() if b == 1 else X)
    xg = Guarded(xt.numel() * xt.element_size(), dev)
    xd = xg.view.view(xt.dtype).reshape(xt.shape)
    xd.copy_(xt.cuda())
    y_dt = xt.dtype if "table_dtype" not in kw else torch.float32
    kw = dict(kw, out_dtype=np.float32) if "table_dtype" in kw else kw
    yg = Guarded(m * b * torch.empty((), dtype=y_dt).element_size(), dev)
    yd = yg.view.view(y_dt).reshape((m,) if b == 1 else (m, b))
    for _ in range(2):
        out = mg.msgemm(pwm, xd, d, out=yd, **kw)
    torch.cuda.synchronize()
    assert out.data_ptr() == yd.data_ptr()
    assert yg.intact() and xg.intact()
    assert guarded_workspaces and all(g.intact() for g in guarded_workspaces)
    W = orc.dense(np.asarray(pwm.data), k, 4, orc.int4_values())
    tol = {np.float16: 2e-3, np.float32: 1e-5, np.float64: 1e-12}[dt]
    assert orc.rel_error(yd.cpu().numpy().astype(np.float64).reshape(m, b), W, X) <= tol
    assert (yd.cpu().numpy().reshape(m, b)[::9] == 0).all()


def test_dequant_mma_no_out_of_bounds_writes(guarded_workspaces):
    import torch
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    for m, k, b in ((256, 200, 16), (128, 64, 1), (384, 320, 200)):
        pwm = mg.from_codes(rng.integers(0, 16, (m, k), dtype=np.uint8), mg.int4_codebook())
        X = rng.standard_normal((k, b)).astype(np.float16)
        yg = Guarded(m * b * 4, dev)
        yd = yg.view.view(torch.float32).reshape(m, b)
        mg.dequant_gemm(pwm, torch.from_numpy(X).cuda(), out=yd)
        torch.cuda.synchronize()
        assert yg.intact() and all(g.intact() for g in guarded_workspaces)
        W = orc.dense(np.asarray(pwm.data), k, 4, orc.int4_values())
        assert orc.rel_error(yd.cpu().numpy(), W, X) <= 2e-3
