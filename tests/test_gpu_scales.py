"""Per-group / per-row scales on the fused row-block kernels.

The reference applies per-group scales after summing each group's block
entries (gemm.py:75-79) and per-row scales after the row sum (gemm.py:84-85).
On the GPU a per-group scale group that is a whole number of quads (4 groups
of d) becomes one k-slice of the fused kernel and the finish kernel weights
slice s of row i by q[i, s].  Checked against the oracle (and exact fp64)
with the north_star tolerances; uint4 / custom codebooks too.
"""

import numpy as np
import pytest

import paper_2310_06178_b200 as mg
from paper_2310_06178_b200 import _lib
from oracle import msgemm_oracle as orc

pytestmark = pytest.mark.gpu
FUSED = (_lib.LAYOUT_QUAD, _lib.LAYOUT_RB4, _lib.LAYOUT_RB4S, _lib.LAYOUT_RB8, _lib.LAYOUT_RB16)

RTOL = {np.float32: 1e-5, np.float16: 2e-3}


def _plan_layout(pwm, d, b, xdt):
    import ctypes
    lay, sym, ws = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    mode, gs = (_lib.SCALE_PER_GROUP, pwm.scales.group_size) if isinstance(
        pwm.scales, mg.PerGroup) else ((_lib.SCALE_PER_ROW, 0) if pwm.scales is not None else (0, 0))
    _lib.check(_lib.lib().msg_gemm_plan(pwm.m, pwm.k, 4, _lib.host_doubles(pwm.codebook.values),
                                        xdt, b, d, mode, gs, 0, ctypes.byref(lay),
                                        ctypes.byref(sym), ctypes.byref(ws)))
    return lay.value


def _case(m, k, b, d, gs, xdtype, cb, seed, per_row=False):
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    if per_row:
        q = rng.uniform(-2, 2, m).astype(np.float32)
        scales = mg.PerRow(q=q)
        Wd = np.asarray(cb.values, np.float64)[codes] * q[:, None]
        mode = "per_row"
    else:
        q = rng.uniform(-2, 2, (m, k // gs)).astype(np.float32)
        scales = mg.PerGroup(group_size=gs, q=q)
        Wd = np.asarray(cb.values, np.float64)[codes] * np.repeat(q, gs, axis=1)
        mode = "per_group"
    pwm = mg.from_codes(codes, cb, scales=scales)
    X = rng.standard_normal((k, b)).astype(xdtype)
    return pwm, X, Wd, q, mode


@pytest.mark.parametrize("m,k,b,d,gs", [
    (300, 384, 1, 3, 96), (257, 384, 5, 3, 48), (128, 256, 8, 2, 64), (200, 128, 3, 1, 16),
    (64, 1536, 16, 3, 192), (1000, 768, 2, 2, 32), (96, 96, 9, 3, 12), (33, 64, 4, 1, 4)])
@pytest.mark.parametrize("xdtype", [np.float16, np.float32])
def test_per_group_fused_matches_oracle(m, k, b, d, gs, xdtype):
    cb = mg.int4_codebook()
    pwm, X, Wd, q, mode = _case(m, k, b, d, gs, xdtype, cb, seed=m * 7 + k + b + d)
    xcode = _lib.F16 if xdtype == np.float16 else _lib.F32
    assert _plan_layout(pwm, d, b, xcode) in FUSED                  # not the generic path
    y = mg.msgemm(pwm, X, d)
    assert y.dtype == X.dtype and y.shape == (m, b)
    assert orc.rel_error(y, Wd, X) <= RTOL[xdtype]
    ref = orc.msgemm(np.asarray(pwm.data), m, k, 4, cb.values, X, d, scale_mode=mode,
                     group_size=gs, q=q)
    scale = np.abs(Wd) @ np.abs(X.astype(np.float64))
    diff = np.abs(y.astype(np.float64) - ref.astype(np.float64))
    assert np.all(diff <= 2 * RTOL[xdtype] * np.maximum(scale, 1e-30) + 1e-30)


@pytest.mark.parametrize("cbname", ["uint4", "custom"])
@pytest.mark.parametrize("per_row", [False, True])
def test_scales_with_other_codebooks(cbname, per_row):
    cb = mg.uint4_codebook() if cbname == "uint4" else mg.custom_codebook(
        [-8, -6, -5, -4, -3, -2, -1, 0, 1, 2, 3, 4, 5, 6, 7, 9])  # not antisymmetric
    m, k, b, d, gs = 500, 768, 4, 3, 96
    pwm, X, Wd, q, mode = _case(m, k, b, d, gs, np.float16, cb, seed=11, per_row=per_row)
    assert _plan_layout(pwm, d, b, _lib.F16) in FUSED
    y = mg.msgemm(pwm, X, d)
    assert orc.rel_error(y, Wd, X) <= 2e-3


def test_per_group_unaligned_falls_back_and_matches():
    # per = group_size / d = 2 groups: not a whole quad -> generic kernels, same answer
    cb = mg.int4_codebook()
    m, k, b, d, gs = 200, 96, 3, 3, 6
    pwm, X, Wd, q, mode = _case(m, k, b, d, gs, np.float32, cb, seed=5)
    assert _plan_layout(pwm, d, b, _lib.F32) == _lib.LAYOUT_NONE
    y = mg.msgemm(pwm, X, d)
    assert orc.rel_error(y, Wd, X) <= 1e-5


@pytest.mark.parametrize("m,k,b", [(256, 8192 + 2, 4), (256, 8192 + 2, 8), (300, 4097, 12),
                                   (100, 3000, 6), (4096, 2048, 16)])
@pytest.mark.parametrize("per_row", [False, True])
def test_row_block_finish_paths(m, k, b, per_row):
    """Small m over long k gives many k-slices: the float4 finish with slice
    groups (b % 4 == 0), the plain float4 finish and the scalar slice-group
    finish (b % 4 != 0) -- each against the oracle, tails and per-row scales
    included, and bitwise repeatable."""
    rng = np.random.default_rng(m + k + b)
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    q = rng.uniform(0.5, 2.0, m).astype(np.float32) if per_row else None
    pwm = mg.from_codes(codes, mg.int4_codebook(), scales=mg.PerRow(q=q) if per_row else None)
    X = rng.standard_normal((k, b)).astype(np.float16)
    y1 = mg.msgemm(pwm, X, 3)
    y2 = mg.msgemm(pwm, X, 3)
    assert np.array_equal(y1.view(np.uint16), y2.view(np.uint16))
    W = orc.dense(pwm.data, k, 4, orc.int4_values()).astype(np.float64)
    if per_row:
        W = W * q[:, None].astype(np.float64)
    assert orc.rel_error(y1, W, X) <= 2e-3
