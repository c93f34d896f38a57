"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz).

Bit-exact for every dtype: the oracle restates the reference's numpy
algorithm with the same primitives and association order.  Also checks the
reference's hand-derived known answers (test_gemm.py:26-34, test_lut.py:16-69,
test_packing.py:9-41).
"""

import numpy as np
import pytest

from oracle import msgemm_oracle as orc
from tests.golden_io import load

PACK = load("packing_lut.npz")
GEMM = load("gemm_cases.npz")


def _values(meta):
    vals = meta["values"]
    if all(float(v).is_integer() for v in vals):
        return np.asarray([int(v) for v in vals])
    return np.asarray(vals)


def test_running_example_known_answers():
    meta, a = next(c for c in PACK if c[0]["kind"] == "running_example")
    vals = orc.int4_values()
    data = orc.pack_rows(orc.nearest_codes(a["W"], vals) & 0xF, 4)
    assert np.array_equal(data, a["data"])
    assert list(data[0]) == [0x42, 0x53]                      # test_packing.py:9-11
    gi = orc.group_indices(data, 4, 4, 2)
    assert np.array_equal(gi, a["gidx"])
    assert gi[0, 0] == 66 and gi[0, 1] == 83                   # test_packing.py:38-41
    lut = orc.lut_full(a["x"], vals, 2)
    assert np.array_equal(lut, a["lut"])
    assert lut[0, 66] == 42 and lut[1, 83] == 5300             # test_lut.py:16-19, 66-69
    y = orc.msgemm(data, 12, 4, 4, vals, a["x"], 2)
    assert np.array_equal(y, a["y"]) and y[0] == 5342          # test_gemm.py:26-34
    assert np.array_equal(a["trace_idx"], gi)
    assert np.array_equal(a["trace_val"], lut[np.arange(2)[None, :], gi])


@pytest.mark.parametrize("i", [i for i, c in enumerate(PACK) if c[0]["kind"] == "packing"])
def test_packing_golden(i):
    meta, a = PACK[i]
    w, k = meta["width"], meta["k"]
    assert np.array_equal(orc.pack_rows(a["codes"], w), a["data"])
    assert np.array_equal(orc.unpack_rows(a["data"], k, w), a["unpacked"])
    for d in (1, 2, 3, 4):
        key = f"gidx_d{d}"
        if key in a:
            assert np.array_equal(orc.group_indices(a["data"], k, w, d), a[key])


def test_pack_scaled_golden():
    vals = orc.int4_values()
    for meta, a in (c for c in PACK if c[0]["kind"] == "pack_scaled"):
        m, k = a["Wscaled"].shape
        if meta["mode"] == "per_row":
            grid = np.broadcast_to(a["q"][:, None], (m, k))
        else:
            grid = np.repeat(a["q"], meta["group_size"], axis=1)
        codes = orc.nearest_codes(a["Wscaled"], vals, grid)
        assert np.array_equal(orc.pack_rows(codes, 4), a["data"])


@pytest.mark.parametrize("i", [i for i, c in enumerate(PACK) if c[0]["kind"] == "lut"])
def test_lut_golden_bitexact(i):
    meta, a = PACK[i]
    vals = orc.int4_values()
    tab = orc.lut_full(a["x"], vals, meta["d"])
    assert tab.dtype == a["entries"].dtype
    assert np.array_equal(tab.view(np.uint8), a["entries"].view(np.uint8))
    assert np.array_equal(orc.lut_block(a["x"], vals, meta["d"], 1), a["block1"])


@pytest.mark.parametrize("i", range(len(GEMM)))
def test_msgemm_golden_bitexact(i):
    meta, a = GEMM[i]
    y = orc.msgemm(a["data"], meta["m"], meta["k"], meta["width"], _values(meta), a["X"],
                   meta["d"], None if meta["scale_mode"] == "none" else meta["scale_mode"],
                   meta["group_size"], a["q"])
    assert y.dtype == a["Y"].dtype and y.shape == a["Y"].shape
    assert np.array_equal(y.view(np.uint8), a["Y"].view(np.uint8)), meta["tag"]


def test_oracle_matches_naive_within_reference_tolerance():
    # suites.py:106-124 convention, exact int and f32 rtol 1e-5
    for meta, a in GEMM:
        X = a["X"]
        if np.issubdtype(X.dtype, np.integer):
            assert np.array_equal(a["Y"], orc.naive_gemm(a["W"], X)), meta["tag"]
        elif X.dtype == np.float32:
            assert orc.rel_error(a["Y"], a["W"], X) <= 1e-5, meta["tag"]
        elif X.dtype == np.float16:
            assert orc.rel_error(a["Y"], a["W"], X) <= 2e-3, meta["tag"]


def test_error_order():
    vals = orc.int4_values()
    data = orc.pack_rows(np.zeros((4, 8), dtype=np.uint8), 4)
    with pytest.raises(ValueError):
        orc.msgemm(data, 4, 8, 4, vals, np.zeros((8, 1, 1)), 2)
    with pytest.raises(ValueError):
        orc.msgemm(data, 4, 8, 4, vals, np.zeros(7), 2)
    with pytest.raises(ValueError):
        orc.msgemm(data, 4, 8, 4, vals, np.zeros(8), 0)
    with pytest.raises(ValueError):
        orc.msgemm(data, 4, 8, 4, vals, np.zeros(8), 9)          # d*width > 32
    with pytest.raises(orc.OracleBudgetError):
        orc.msgemm(data, 4, 8, 4, vals, np.zeros(8, dtype=np.int64), 4, budget=1024)
    with pytest.raises(IndexError):
        orc.lut_block(np.zeros(4), vals, 2, 2)


def test_workers_invariant():
    rng = np.random.default_rng(0)
    vals = orc.int4_values()
    data = orc.pack_rows(rng.integers(0, 16, (20, 30), dtype=np.uint8), 4)
    X = rng.standard_normal((30, 6)).astype(np.float16)
    a = orc.msgemm(data, 20, 30, 4, vals, X, 3)
    b = orc.msgemm(data, 20, 30, 4, vals, X, 3, workers=4)
    assert np.array_equal(a.view(np.uint16), b.view(np.uint16))


# ---------------------------------------------------------------- CaseGen suites

def _casegen_digests():
    import json
    from pathlib import Path
    return json.loads((Path(__file__).parent / "golden" / "casegen_digests.json").read_text())["suites"]


@pytest.mark.parametrize("name", ["crit1_d1", "crit1_d2", "crit1_d3", "crit1_d4", "crit1_f32",
                                  "suite_exact_small", "suite_f32_small", "formula"])
def test_casegen_reproduces_reference_cases(name):
    """oracle/casegen.py draws the reference's own cases (suites.py:27-85),
    and on the exact suites the oracle's msgemm returns the reference's bytes."""
    import hashlib
    from oracle.casegen import CaseGen
    ent = _casegen_digests()[name]
    kw = {k: tuple(v) if isinstance(v, list) else v for k, v in ent["kwargs"].items()}
    gen = CaseGen(**kw)
    hc, hy = hashlib.sha256(), hashlib.sha256()
    for _ in range(ent["cases"]):
        c = gen.draw(**ent["draw"])
        c.digest_update(hc)
        if ent["Y_sha256"] is not None:
            y = orc.msgemm(orc.pack_rows(c.codes.astype(np.uint8), 4), c.m, c.k, 4, orc.int4_values(),
                           c.X, c.d, None if c.scale_mode == "none" else c.scale_mode,
                           c.group_size, c.q)
            hy.update(np.ascontiguousarray(y).tobytes())
    assert hc.hexdigest() == ent["cases_sha256"]
    if ent["Y_sha256"] is not None:
        assert hy.hexdigest() == ent["Y_sha256"]
