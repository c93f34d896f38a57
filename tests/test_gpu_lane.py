"""The b=1 lane kernel (msg_lane.cu) and the cached host path.

The lane kernel sums chunk partials in int64 fixed point across CTAs, so its
Y must be bitwise independent of how rows are split over launches, and its
workspace must come back to zero after every call.  Tolerance bar as in
test_gpu_parity (fp16 X: 2e-3 * sum_j |W_ij||x_j|, suites.py:106-124);
integer-valued X whose tables fit fp16 exactly: bit-exact.
"""

import ctypes

import numpy as np
import pytest

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc
from paper_2310_06178_b200 import _lib

pytestmark = pytest.mark.gpu


def _plan_layout(m, k, b, d, x_code=_lib.F16, flags=0):
    vals = _lib.host_doubles(mg.int4_codebook().values)
    lay, sym, ws = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    _lib.check(_lib.lib().msg_gemm_plan(m, k, 4, vals, x_code, b, d, 0, 0, flags,
                                        ctypes.byref(lay), ctypes.byref(sym), ctypes.byref(ws)))
    return lay.value


def _case(m, k, seed, scales=None):
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, mg.int4_codebook(), scales=scales)
    x = rng.standard_normal(k).astype(np.float16)
    return pwm, x, rng


def _lane_workspaces_zero():
    import torch
    torch.cuda.synchronize()
    # a 1-row matrix runs on full tables (its row is ill-conditioned for the
    # half tables), so no lane workspace may exist yet when it runs first
    bufs = [buf for key, buf in _lib._ws.items() if key[2] == "lane"]
    return all(int(torch.count_nonzero(b)) == 0 for b in bufs)


def test_lane_layout_selected_for_b1_fp16_d3():
    assert _plan_layout(4096, 4096, 1, 3) == _lib.LAYOUT_LANE
    assert _plan_layout(4096, 4096, 2, 3) != _lib.LAYOUT_LANE     # b > 1: row-block kernel
    assert _plan_layout(4096, 4096, 1, 2) != _lib.LAYOUT_LANE     # d != 3
    assert _plan_layout(4096, 4096, 1, 3, _lib.F32) != _lib.LAYOUT_LANE  # f32 X: f32 tables
    assert _plan_layout(4096, 4096, 1, 3, flags=_lib.FLAG_NO_LANE) != _lib.LAYOUT_LANE


@pytest.mark.parametrize("m,k", [(1, 3), (31, 95), (33, 97), (257, 98), (1000, 3001),
                                 (4096, 4096)])
def test_lane_matches_oracle(m, k):
    pwm, x, _ = _case(m, k, m + k)
    y = mg.msgemm(pwm, x, 3)
    W = orc.dense(pwm.data, k, 4, orc.int4_values())
    assert y.dtype == np.float16 and y.shape == (m,)
    assert orc.rel_error(y, W, x) <= 2e-3
    assert _lane_workspaces_zero()


def test_lane_integer_x_bitexact():
    m, k = 777, 2050                     # k % 3 == 1: one tail column
    pwm, _, rng = _case(m, k, 11)
    xi = rng.integers(-8, 9, k)          # |table entries| <= 180: exact in fp16
    y = mg.msgemm(pwm, xi.astype(np.float16), 3, out_dtype=np.float32)
    ref = orc.msgemm(pwm.data, m, k, 4, orc.int4_values(), xi.astype(np.int64), 3)
    assert np.array_equal(y.astype(np.int64), ref)


def test_lane_rows_split_bitwise_invariant():
    """Fixed-point sums: a row's Y does not depend on the launch's CTA split."""
    m, k = 3000, 4099
    pwm, x, _ = _case(m, k, 12)
    full = mg.msgemm(pwm, x, 3)
    for r0, r1 in [(0, 1), (5, 700), (1111, 3000), (2999, 3000)]:
        part = mg.from_codes(orc.unpack_rows(pwm.data[r0:r1], k, 4), mg.int4_codebook())
        y = mg.msgemm(part, x, 3)
        assert np.array_equal(y.view(np.uint16), full[r0:r1].view(np.uint16)), (r0, r1)


def test_lane_per_row_scales():
    m, k = 500, 1201
    rng = np.random.default_rng(13)
    q = rng.uniform(0.5, 2.0, m).astype(np.float32)
    pwm, x, _ = _case(m, k, 13, scales=mg.PerRow(q=q))
    y = mg.msgemm(pwm, x, 3)
    W = orc.dense(pwm.data, k, 4, orc.int4_values()) * q[:, None].astype(np.float64)
    assert orc.rel_error(y, W, x) <= 2e-3


def test_lane_interleaved_with_other_paths_and_repeat():
    """Lane calls keep their own self-cleaning workspace: row-block and generic
    calls on the same stream between them do not disturb it."""
    pwm, x, rng = _case(2048, 3072, 14)
    X8 = rng.standard_normal((3072, 8)).astype(np.float16)
    a = mg.msgemm(pwm, x, 3)
    mg.msgemm(pwm, X8, 3)                                  # row-block kernel (scratch)
    mg.msgemm(pwm, x.astype(np.float64), 3)                # generic kernel (scratch)
    b = mg.msgemm(pwm, x, 3)
    assert np.array_equal(a.view(np.uint16), b.view(np.uint16))
    assert _lane_workspaces_zero()


def test_lut_phase_only_then_reset():
    import torch
    pwm, x, _ = _case(1024, 2048, 15)
    ref = mg.msgemm(pwm, x, 3)
    xd = torch.from_numpy(x).cuda()
    mg.msgemm(pwm, xd, 3, _flags=_lib.FLAG_LUT_PHASE_ONLY)   # leaves its sums behind
    torch.cuda.synchronize()
    _lib.reset_workspaces()
    assert np.array_equal(mg.msgemm(pwm, x, 3).view(np.uint16), ref.view(np.uint16))


def test_host_staging_paths_agree():
    import torch
    pwm, x, rng = _case(1500, 2500, 16)
    X = rng.standard_normal((2500, 4)).astype(np.float16)
    for Xin in (x, X):
        ref = mg.msgemm(pwm, torch.from_numpy(Xin).cuda(), 3).cpu().numpy()
        assert np.array_equal(mg.msgemm(pwm, Xin, 3), ref)                       # numpy
        assert np.array_equal(mg.msgemm(pwm, torch.from_numpy(Xin), 3).numpy(), ref)  # CPU torch
        pin = torch.from_numpy(Xin).pin_memory()
        out = torch.empty((1500, Xin.reshape(2500, -1).shape[1]), dtype=torch.float16,
                          pin_memory=True)
        mg.msgemm(pwm, pin, 3, out=out)
        assert np.array_equal(out.numpy().reshape(ref.shape), ref)               # pinned in/out
        # the returned numpy array is private: a later call must not change it
        first = mg.msgemm(pwm, Xin, 3)
        mg.msgemm(pwm, np.zeros_like(Xin), 3)
        assert np.array_equal(first, ref)


def test_side_stream():
    import torch
    pwm, x, _ = _case(999, 1999, 17)
    ref = mg.msgemm(pwm, x, 3)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y = mg.msgemm(pwm, torch.from_numpy(x).cuda(), 3)
    s.synchronize()
    assert np.array_equal(y.cpu().numpy().view(np.uint16), ref.view(np.uint16))


@pytest.mark.parametrize("cbname", ["uint4", "custom_antisym"])
def test_lane_other_antisymmetric_codebooks(cbname):
    """uint4 (beta = 7.5) and a custom antisymmetric codebook take the lane path
    with their own symmetry shift and fixed-point grid."""
    if cbname == "uint4":
        cb = mg.uint4_codebook()
        vals = np.arange(16, dtype=np.float64)
    else:
        vals = np.array([-7.5, -6.0, -4.25, -3.0, -2.0, -1.5, -0.75, -0.25,
                         0.25, 0.75, 1.5, 2.0, 3.0, 4.25, 6.0, 7.5])
        # antisymmetric: v[c] + v[~c] == 0
        assert np.allclose(vals + vals[::-1], 0)
        cb = mg.custom_codebook(list(vals))
    rng = np.random.default_rng(21)
    m, k = 640, 3001
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, cb)
    x = rng.standard_normal(k).astype(np.float16)
    vals_c = _lib.host_doubles(cb.values)
    lay, sym, ws = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    _lib.check(_lib.lib().msg_gemm_plan(m, k, 4, vals_c, _lib.F16, 1, 3, 0, 0, 0,
                                        ctypes.byref(lay), ctypes.byref(sym), ctypes.byref(ws)))
    assert lay.value == _lib.LAYOUT_LANE
    y = mg.msgemm(pwm, x, 3)
    W = vals[codes.astype(np.int64)]
    assert orc.rel_error(y, W, x) <= 2e-3


def test_lane_long_k():
    """Many chunks (k = 60000: 625 chunks) keep the fixed-point grid inside int64."""
    rng = np.random.default_rng(22)
    m, k = 96, 60000
    pwm = mg.from_codes(rng.integers(0, 16, (m, k), dtype=np.uint8), mg.int4_codebook())
    x = rng.standard_normal(k).astype(np.float16)
    y = mg.msgemm(pwm, x, 3)
    W = orc.dense(pwm.data, k, 4, orc.int4_values())
    assert orc.rel_error(y, W, x) <= 2e-3


def test_concurrent_host_calls_share_staging_safely():
    """Host-staged calls from several Python threads on one plan serialise on
    its staging buffers (results match the single-threaded ones)."""
    import threading
    pwm, x, rng = _case(1024, 2048, 23)
    xs = [rng.standard_normal(2048).astype(np.float16) for _ in range(8)]
    refs = [mg.msgemm(pwm, v, 3) for v in xs]
    outs = [None] * len(xs)

    def work(i):
        for _ in range(5):
            outs[i] = mg.msgemm(pwm, xs[i], 3)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(xs))]
    for t_ in th:
        t_.start()
    for t_ in th:
        t_.join()
    for o, r in zip(outs, refs):
        assert np.array_equal(o.view(np.uint16), r.view(np.uint16))


def test_device_out_vector():
    import torch
    pwm, x, _ = _case(300, 600, 24)
    ref = mg.msgemm(pwm, x, 3)
    out = torch.empty(300, dtype=torch.float16, device="cuda")
    y = mg.msgemm(pwm, torch.from_numpy(x).cuda(), 3, out=out)
    assert y.data_ptr() == out.data_ptr()
    assert np.array_equal(out.cpu().numpy().view(np.uint16), ref.view(np.uint16))
