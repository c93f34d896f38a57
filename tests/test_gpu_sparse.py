"""Sparse and all-zero weight rows on every kernel route (round-2 parity gap).

The reference's tolerance is per element, |y - y_exact| <= rtol *
sum_j |W_ij||x_j| (suites.py:104-124), so a row without a nonzero weight must
come out exactly 0 -- the reference's all-zero table index is exactly 0
(lut.py:59-72, pinned by test_lut.py:22-27).  Sign-symmetric half tables
cannot promise that (their rounding error follows sum |v - beta||x|), so
msgemm routes ill-conditioned rows to full tables (gemm.py _CallPlan).  The
fixtures come from the reference itself (tests/golden/make_golden.py,
sparse_cases): a mostly dense matrix with a few special rows (the fix-up
path), a matrix of special rows only (the full-table fallback) and a
config-1-like d=2 matrix.
"""

import numpy as np
import pytest
import torch

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc
from paper_2310_06178_b200 import _lib
from paper_2310_06178_b200.gemm import _call_plan, _symmetric_threshold
from paper_2310_06178_b200.sharded import shard_cols
from tests.golden_io import load

pytestmark = pytest.mark.gpu

SPARSE = {meta["name"]: (meta, a) for meta, a in load("sparse_cases.npz")}
RTOL = {"float16": 2e-3, "float32": 1e-5}
ROUTES = ["default", "nolane", "f32tab", "nosym", "generic", "device", "ksplit"]


def _case(name, dt, b):
    meta, a = SPARSE[name]
    X = a[f"X_{dt}"]
    Xb = X[:, 0].copy() if b == 1 else np.ascontiguousarray(X[:, :b])
    return meta, a, Xb, a[f"Y_{dt}_b{b}"]


def _pwm(meta, a):
    return mg.PackedWeightMatrix(m=meta["m"], k=meta["k"], width=4, data=a["data"],
                                 codebook=mg.int4_codebook())


def _run(route, pwm, X, d):
    if route == "default":
        return mg.msgemm(pwm, X, d)
    if route == "nolane":
        return mg.msgemm(pwm, X, d, _flags=_lib.FLAG_NO_LANE)
    if route == "f32tab":
        return mg.msgemm(pwm, X, d, table_dtype=np.float32)
    if route == "nosym":
        return mg.msgemm(pwm, X, d, symmetric=False)
    if route == "generic":
        return mg.msgemm(pwm, X, d, _flags=_lib.FLAG_FORCE_GENERIC)
    if route == "device":
        return mg.msgemm(pwm, torch.from_numpy(X).cuda(), d).cpu().numpy()
    assert route == "ksplit"    # 4 column slices, fp32 partial Y summed in order
    acc = None
    for r in range(4):
        part, lo, hi = shard_cols(pwm, d, 4, r)
        if hi > lo:
            y = mg.msgemm(part, X[lo:hi], d, out_dtype=np.float32).astype(np.float32)
            acc = y if acc is None else acc + y
    return acc.astype(X.dtype)


def _zero_rows(W):
    return np.flatnonzero(~W.any(axis=1))


@pytest.mark.parametrize("route", ROUTES)
@pytest.mark.parametrize("b", [1, 4, 8, 16])
@pytest.mark.parametrize("name,dt", [("mixed", "float16"), ("mixed", "float32"),
                                     ("special", "float16"), ("special", "float32"),
                                     ("cfg1like", "float32")])
def test_sparse_rows_within_reference_bound(name, dt, b, route):
    meta, a, X, Yref = _case(name, dt, b)
    pwm = _pwm(meta, a)
    W = orc.dense(a["data"], meta["k"], 4, orc.int4_values())
    y = _run(route, pwm, X, meta["d"])
    assert y.dtype == Yref.dtype and y.shape == Yref.shape
    tol = RTOL[dt]
    err = orc.rel_error(y, W, X)
    assert err <= tol, (route, err)
    zr = _zero_rows(W)
    assert len(zr) > 0
    assert np.all(y.reshape(meta["m"], -1)[zr] == 0), route            # exactly 0
    # and against the reference's own rounded output
    scale = np.abs(W.astype(np.float64)) @ np.abs(X.astype(np.float64))
    diff = np.abs(y.astype(np.float64) - Yref.astype(np.float64))
    assert np.all(diff <= 2 * tol * scale), route


@pytest.mark.parametrize("route", ["default", "nolane", "ksplit"])
@pytest.mark.parametrize("b", [1, 8])
@pytest.mark.parametrize("name", ["mixed", "special", "cfg1like"])
def test_sparse_rows_integer_exact(name, b, route):
    meta, a = SPARSE[name]
    Xi = a["X_int"][:, 0].copy() if b == 1 else a["X_int"]
    Yref = a[f"Y_int_b{b}"]
    pwm = _pwm(meta, a)
    X16 = Xi.astype(np.float16)
    d = meta["d"]
    if route == "ksplit":
        y = sum(mg.msgemm(part, X16[lo:hi], d, out_dtype=np.float32, table_dtype=np.float32)
                .astype(np.float64) for part, lo, hi in
                (shard_cols(pwm, d, 4, r) for r in range(4)) if hi > lo)
    else:
        y = mg.msgemm(pwm, X16, d, out_dtype=np.float32, table_dtype=np.float32,
                      _flags=_lib.FLAG_NO_LANE if route == "nolane" else 0)
    assert np.array_equal(np.asarray(y).astype(np.int64), Yref)


def _ratio_numpy(codes, d, beta):
    v = orc.int4_values().astype(np.float64)[codes]
    k = codes.shape[1]
    nb = k // d
    sj = np.abs(v[:, :nb * d] - beta).reshape(codes.shape[0], nb, d).sum(axis=2)
    wabs = np.abs(v).sum(axis=1)
    nnz = (v != 0).sum(axis=1)
    ok = (wabs > 0) & (nnz >= min(8, (k + 1) // 2))
    return np.where(ok, np.sqrt((sj ** 2).sum(axis=1)) / np.where(ok, wabs, 1), np.inf)


@pytest.mark.parametrize("name", ["mixed", "special", "cfg1like"])
def test_conditioning_ratio_and_routing(name):
    meta, a = SPARSE[name]
    pwm = _pwm(meta, a)
    dev = _lib.require_device()
    d = meta["d"]
    codes = orc.unpack_rows(a["data"], meta["k"], 4)
    want = _ratio_numpy(codes, d, -0.5)
    got = pwm.symmetric_conditioning(dev, d, -0.5).cpu().numpy().astype(np.float64)
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin)
    np.testing.assert_allclose(got[fin], want[fin], rtol=1e-5)
    # the plan: a few ill rows -> fix-up on full tables; mostly ill -> full tables
    thr = _symmetric_threshold(_lib.F16, 2)
    n_ill = int((want > thr).sum())
    stream = _lib.current_stream_handle(dev)
    call = _call_plan(pwm, dev, stream, 8, _lib.F16, np.dtype(np.float16), d, None, True,
                      None, 0)
    if name == "mixed":
        assert 0 < n_ill * 8 <= meta["m"] and call.fix is not None and call.fix[2] == n_ill
    if name == "special":
        assert n_ill * 8 > meta["m"] and call.fix is None
        assert call._flags & _lib.FLAG_NO_SYMMETRY


def test_nonfinite_activations_propagate():
    """NaN in X poisons every row (every table entry that touches it is NaN
    in the reference); inf gives a non-finite row wherever the reference's
    row is non-finite -- on the b=1 lane kernel (fixed-point reduction) and
    the row-block kernel alike."""
    rng = np.random.default_rng(77)
    m, k, d = 96, 3 * 400 + 2, 3
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, mg.int4_codebook())
    for b in (1, 8):
        for bad in (np.nan, np.inf):
            X = rng.standard_normal((k, b)).astype(np.float16)
            X[17, 0] = bad
            Xb = X[:, 0].copy() if b == 1 else X
            ref = orc.msgemm(np.asarray(pwm.data), m, k, 4, orc.int4_values(), Xb, d)
            y = mg.msgemm(pwm, Xb, d)
            ref = ref.reshape(m, -1)
            y = y.reshape(m, -1)
            assert np.array_equal(np.isfinite(y), np.isfinite(ref)), (b, bad)
            if np.isnan(bad):
                assert np.isnan(y[:, 0]).all()
    # the self-cleaning lane workspace is clean again: a finite call is exact
    Xi = rng.integers(-127, 128, (k,)).astype(np.float16)
    yi = mg.msgemm(pwm, Xi, d, table_dtype=np.float32, out_dtype=np.float32)
    ref = orc.naive_gemm(orc.dense(np.asarray(pwm.data), k, 4, orc.int4_values()),
                         Xi.astype(np.int64))
    assert np.array_equal(yi.astype(np.int64), ref)
    y1 = mg.msgemm(pwm, rng.standard_normal(k).astype(np.float16), d)
    assert np.isfinite(y1).all()


def test_out_argument_contract():
    rng = np.random.default_rng(5)
    m, k, d = 64, 96, 3
    pwm = mg.from_codes(rng.integers(0, 16, (m, k), dtype=np.uint8), mg.int4_codebook())
    X = torch.from_numpy(rng.standard_normal((k, 4)).astype(np.float16)).cuda()
    with pytest.raises(ValueError):      # (m,) is only for a vector X
        mg.msgemm(pwm, X, d, out=torch.empty(m, dtype=torch.float16, device="cuda"))
    out = torch.empty((m, 4), dtype=torch.float16, device="cuda")
    Xh = X.cpu().numpy()
    r = mg.msgemm(pwm, Xh, d, out=out)   # host X, device out: written in place
    assert r is out
    np.testing.assert_array_equal(out.cpu().numpy(), mg.msgemm(pwm, Xh, d))
    x1 = torch.from_numpy(rng.standard_normal(k).astype(np.float16)).cuda()
    o1 = torch.empty(m, dtype=torch.float16, device="cuda")
    mg.msgemm(pwm, x1, d, out=o1)
    np.testing.assert_array_equal(o1.cpu().numpy(), mg.msgemm(pwm, x1.cpu().numpy(), d))


def test_misaligned_activation_view():
    """A 1-D fp16 view at an odd element offset (row i of an (n, k) tensor
    with odd k) must not fault the b=1 kernel's 4-byte activation copies."""
    rng = np.random.default_rng(6)
    m, k, d = 128, 3 * 101, 3                         # k odd
    pwm = mg.from_codes(rng.integers(0, 16, (m, k), dtype=np.uint8), mg.int4_codebook())
    Xs = torch.from_numpy(rng.standard_normal((3, k)).astype(np.float16)).cuda()
    x = Xs[1]                                         # byte offset 2*k: not 4-aligned
    assert x.data_ptr() % 4 != 0
    y = mg.msgemm(pwm, x, d).cpu().numpy()
    np.testing.assert_array_equal(y, mg.msgemm(pwm, x.cpu().numpy(), d))
    out = torch.empty((m, 4), dtype=torch.float32, device="cuda")
    X4 = torch.from_numpy(rng.standard_normal((k, 4)).astype(np.float16)).cuda()
    ob = torch.empty(m * 4 + 1, dtype=torch.float32, device="cuda")[1:].view(m, 4)  # 4-B aligned
    mg.msgemm(pwm, X4, d, out_dtype=np.float32, out=ob)
    mg.msgemm(pwm, X4, d, out_dtype=np.float32, out=out)
    torch.testing.assert_close(ob, out, rtol=0, atol=0)
