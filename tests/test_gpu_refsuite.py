"""The reference's own hot-path test suites, replayed through the GPU package.

Each test restates one reference test (cited per test) against
``paper_2310_06178_b200`` -- the drop-in -- on the B200:

* acceptance criteria 1-3 (``pkg/tests/test_acceptance.py:50-95``): the 5,000
  randomized oracle cases of ``run_oracle_suite`` (the reference's CaseGen
  draws, reproduced by ``oracle/casegen.py`` and pinned by
  ``tests/golden/casegen_digests.json``), the traced running example and the
  closed-form operation counts;
* ``pkg/tests/test_suites.py``, ``test_gemm.py``, ``test_lut.py`` and
  ``test_packing.py``.

Expected values come from the CPU oracle (``oracle/``), never from the
package under test.  Integer cases are bit-exact; f32 cases use the
reference's rule |dy| <= 1e-5 * sum_j |W_ij||x_j| (``suites.py:104-124``).
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc
from oracle.casegen import CRITERION1_SUITES, F32_RTOL, CaseGen

pytestmark = pytest.mark.gpu

CB = mg.int4_codebook()
DIGESTS = json.loads((Path(__file__).parent / "golden" / "casegen_digests.json").read_text())["suites"]
RUNNING_EXAMPLE = [  # test_acceptance.py:33-37
    [2, 4, 3, 5], [-1, 0, 1, -8], [7, -3, 2, 6], [0, 0, 0, 0],
    [1, 2, 3, 4], [-4, 5, -6, 7], [3, 3, 3, 3], [-8, -8, -8, -8],
    [6, 1, -2, 0], [5, -5, 5, -5], [0, 7, -1, 2], [-2, 4, 0, -7],
]


def _pwm(case):
    scales = None
    if case.scale_mode == "per_row":
        scales = mg.PerRow(q=case.q)
    elif case.scale_mode == "per_group":
        scales = mg.PerGroup(group_size=case.group_size, q=case.q)
    return mg.from_codes(case.codes, CB, scales)


def _expected(case):
    """naive_gemm(dense(pwm, apply_scales=True), X) on the CPU oracle (suites.py:113-115)."""
    W = orc.int4_values()[case.codes]
    if case.scale_mode == "per_row":
        W = W * case.q[:, None]
    elif case.scale_mode == "per_group":
        W = W * np.repeat(case.q, case.group_size, axis=1)
    return W, orc.naive_gemm(W, case.X)


def _case_ok(case, actual):
    """suites.py:104-124 (case_matches), the oracle on the expected side."""
    W, expected = _expected(case)
    if np.issubdtype(case.X.dtype, np.integer):
        return actual.dtype == expected.dtype and np.array_equal(actual, expected), 0.0
    scale = np.abs(W).astype(np.float64) @ np.abs(case.X.astype(np.float64))
    diff = np.abs(actual.astype(np.float64) - expected.astype(np.float64))
    rel = float(np.max(diff / np.maximum(scale, 1e-30))) if expected.size else 0.0
    return rel <= F32_RTOL and actual.dtype == case.X.dtype, rel


def _run_suite(gen, n, **draw_kw):
    failures, ys = [], hashlib.sha256()
    hc = hashlib.sha256()
    for _ in range(n):
        case = gen.draw(**draw_kw)
        case.digest_update(hc)
        y = mg.msgemm(_pwm(case), case.X, case.d)
        ys.update(np.ascontiguousarray(y).tobytes())
        ok, rel = _case_ok(case, y)
        if not ok:
            failures.append(f"case_seed={case.case_seed} m={case.m} k={case.k} b={case.b} "
                            f"d={case.d} scales={case.scale_mode} rel={rel:.3g}")
    return failures, hc.hexdigest(), ys.hexdigest()


# ---------------------------------------------------------------- acceptance

@pytest.mark.parametrize("name,kw", [(f"crit1_d{d}", CRITERION1_SUITES[d - 1]) for d in (1, 2, 3, 4)]
                         + [("crit1_f32", CRITERION1_SUITES[4])])
def test_criterion_1_oracle_equivalence(name, kw):
    """test_acceptance.py:50-61: 4 x 1000 exact + 1000 f32 CaseGen cases."""
    failures, cases_sha, y_sha = _run_suite(CaseGen(**kw), 1000)
    assert cases_sha == DIGESTS[name]["cases_sha256"], "not the reference's cases"
    assert not failures, failures[:5]
    if DIGESTS[name]["Y_sha256"] is not None:       # exact suites: the reference's own bytes
        assert y_sha == DIGESTS[name]["Y_sha256"]


def test_criterion_2_running_example_trace():
    """test_acceptance.py:64-74."""
    pwm = mg.pack(RUNNING_EXAMPLE, CB)
    x = np.array([1, 10, 100, 1000], dtype=np.int64)
    y, trace = mg.msgemm_traced(pwm, x, 2)
    assert [(j, idx) for j, idx, _ in trace[0]] == [(0, 0b0100_0010), (1, 0b0101_0011)]
    assert [v for _, _, v in trace[0]] == [42, 5300]
    assert y[0] == 5342
    assert np.array_equal(y, orc.naive_gemm(np.asarray(RUNNING_EXAMPLE), x))


def test_criterion_3_formula_agreement():
    """test_acceptance.py:77-95: counted ops equal the closed forms, 100 shapes."""
    rng = np.random.default_rng(77)
    shapes = [(12, 4, 1, 2)]
    while len(shapes) < 100:
        d = int(rng.integers(1, 5))
        k = d * int(rng.integers(1, 48 // d + 1))
        shapes.append((int(rng.integers(1, 65)), k, int(rng.integers(1, 9)), d))
    for m, k, b, d in shapes:
        codes = rng.integers(0, 16, size=(m, k))
        X = rng.integers(-9, 9, size=(k, b)).astype(np.int64)
        Y, c = mg.msgemm_counted(mg.from_codes(codes, CB), X, d)
        assert (c.fma, c.add, c.mem_weights, c.mem_activations) == \
            (2 ** (4 * d) * k * b, (k // d - 1) * m * b, m * k * b, k * b)
        assert np.array_equal(Y, orc.naive_gemm(orc.int4_values()[codes], X))
    _, c = mg.msgemm_counted(mg.from_codes(rng.integers(0, 16, size=(12, 4)), CB),
                             np.ones((4, 1), dtype=np.int64), 2)
    assert (c.fma, c.add) == (1024, 12)


# ---------------------------------------------------------------- test_suites.py

@pytest.mark.parametrize("name,kw", [("suite_exact_small", dict(seed=1)),
                                     ("suite_f32_small", dict(seed=2, mode="f32"))])
def test_small_oracle_suites(name, kw):
    """test_suites.py:6-14."""
    failures, cases_sha, y_sha = _run_suite(CaseGen(**kw), 100)
    assert cases_sha == DIGESTS[name]["cases_sha256"]
    assert not failures, failures[:3]
    if DIGESTS[name]["Y_sha256"] is not None:
        assert y_sha == DIGESTS[name]["Y_sha256"]


def test_formula_suite():
    """test_suites.py:35-37 (run_formula_suite, suites.py:142-156)."""
    gen = CaseGen(seed=5)
    hc = hashlib.sha256()
    for _ in range(50):
        case = gen.draw(divisible_only=True, scale_mode="none")
        case.digest_update(hc)
        Y, c = mg.msgemm_counted(_pwm(case), case.X, case.d)
        m, k, b, d = case.m, case.k, case.b, case.d
        assert (c.fma, c.add, c.mem_weights, c.mem_activations) == \
            (2 ** (4 * d) * k * b, (k // d - 1) * m * b, m * k * b, k * b)
        assert np.array_equal(Y, _expected(case)[1])
    assert hc.hexdigest() == DIGESTS["formula"]["cases_sha256"]


# ---------------------------------------------------------------- test_gemm.py

def _random_pwm(rng, m, k, scales=None):
    codes = rng.integers(0, 16, size=(m, k))
    return mg.from_codes(codes, CB, scales), orc.int4_values()[codes]


def test_naive_known_answers():
    """test_gemm.py:37-51: hand example, one-hot selection, empty output."""
    assert mg.naive_gemm(np.array([[2, 4, 3, 5]]), np.array([1, 10, 100, 1000]))[0] == 5342
    W = np.eye(4, dtype=np.int64)[[2, 0, 3]]
    x = np.array([5, -7, 11, 13], dtype=np.int64)
    assert np.array_equal(mg.naive_gemm(W, x), x[[2, 0, 3]])
    assert mg.naive_gemm(np.zeros((0, 4), dtype=np.int64), np.ones(4, dtype=np.int64)).shape == (0,)


def test_d1_equals_naive_bitwise():
    """test_gemm.py:53-57."""
    rng = np.random.default_rng(10)
    pwm, W = _random_pwm(rng, 12, 7)
    X = rng.integers(-100, 100, size=(7, 3)).astype(np.int64)
    assert np.array_equal(mg.msgemm(pwm, X, 1), mg.naive_gemm(mg.dense(pwm), X))
    assert np.array_equal(mg.msgemm(pwm, X, 1), orc.naive_gemm(W, X))


@pytest.mark.parametrize("d", [1, 2, 3, 4])
def test_exact_oracle_equivalence(d):
    """test_gemm.py:60-69."""
    rng = np.random.default_rng(20 + d)
    for _ in range(25):
        m, k, b = int(rng.integers(1, 65)), int(rng.integers(d, 49)), int(rng.integers(1, 9))
        pwm, W = _random_pwm(rng, m, k)
        X = rng.integers(-1000, 1001, size=(k, b)).astype(np.int64)
        assert np.array_equal(mg.msgemm(pwm, X, d), orc.naive_gemm(W, X))


def test_exact_with_tail_and_scales():
    """test_gemm.py:72-107: k % d tail, per-row and per-group scales."""
    rng = np.random.default_rng(30)
    pwm, W = _random_pwm(rng, 9, 11)
    x = rng.integers(-50, 50, size=11).astype(np.int64)
    assert np.array_equal(mg.msgemm(pwm, x, 3), orc.naive_gemm(W, x))
    rng = np.random.default_rng(31)
    q = rng.integers(1, 5, size=8).astype(np.int64)
    pwm, W = _random_pwm(rng, 8, 10, mg.PerRow(q=q))
    x = rng.integers(-30, 30, size=10).astype(np.int64)
    assert np.array_equal(mg.msgemm(pwm, x, 2), orc.naive_gemm(W * q[:, None], x))
    rng = np.random.default_rng(32)
    for r in (2, 4):
        q = rng.integers(1, 5, size=(6, 8 // r)).astype(np.int64)
        pwm, W = _random_pwm(rng, 6, 8, mg.PerGroup(group_size=r, q=q))
        x = rng.integers(-30, 30, size=8).astype(np.int64)
        assert np.array_equal(mg.msgemm(pwm, x, 2), orc.naive_gemm(W * np.repeat(q, r, axis=1), x))


def test_per_row_scale_linearity():
    """test_gemm.py:110-117."""
    rng = np.random.default_rng(33)
    q = rng.integers(1, 7, size=5).astype(np.int64)
    codes = rng.integers(0, 16, size=(5, 6))
    x = rng.integers(-20, 20, size=6).astype(np.int64)
    unscaled = mg.msgemm(mg.from_codes(codes, CB), x, 2)
    assert np.array_equal(mg.msgemm(mg.from_codes(codes, CB, mg.PerRow(q=q)), x, 2), q * unscaled)


def test_f32_oracle_equivalence():
    """test_gemm.py:120-131."""
    rng = np.random.default_rng(40)
    for d in (1, 2, 3):
        pwm, W = _random_pwm(rng, 32, 24)
        X = rng.standard_normal((24, 4)).astype(np.float32)
        actual = mg.msgemm(pwm, X, d)
        assert actual.dtype == np.float32
        assert orc.rel_error(actual, W, X) <= 1e-5


def test_batch_decomposition_bitwise():
    """test_gemm.py:134-140."""
    rng = np.random.default_rng(41)
    pwm, _ = _random_pwm(rng, 10, 12)
    X = rng.integers(-99, 99, size=(12, 5)).astype(np.int64)
    full = mg.msgemm(pwm, X, 3)
    for c in range(5):
        assert np.array_equal(full[:, c], mg.msgemm(pwm, X[:, c], 3))


def test_validation_errors():
    """test_gemm.py:143-161, 174-178: group size vs depth, k mismatch, budget."""
    rng = np.random.default_rng(42)
    pwm, _ = _random_pwm(rng, 4, 8, mg.PerGroup(group_size=4, q=np.ones((4, 2), dtype=np.int64)))
    with pytest.raises(ValueError):
        mg.msgemm(pwm, np.zeros(8, dtype=np.int64), 3)
    pwm2, _ = _random_pwm(rng, 4, 8, mg.PerGroup(group_size=2, q=np.ones((4, 4), dtype=np.int64)))
    with pytest.raises(ValueError):
        mg.msgemm(pwm2, np.zeros(8, dtype=np.int64), 4)
    pwm3, _ = _random_pwm(np.random.default_rng(43), 4, 8)
    with pytest.raises(ValueError):
        mg.msgemm(pwm3, np.zeros(7, dtype=np.int64), 2)
    pwm4, _ = _random_pwm(np.random.default_rng(45), 4, 8)
    with pytest.raises(mg.TableBudgetError):
        mg.msgemm(pwm4, np.zeros(8, dtype=np.int64), 4, budget=1024)


def test_streaming_and_workers_match_full_table():
    """test_gemm.py:164-171, 181-187."""
    rng = np.random.default_rng(44)
    pwm, W = _random_pwm(rng, 16, 12)
    X = rng.integers(-50, 50, size=(12, 2)).astype(np.int64)
    full = mg.msgemm(pwm, X, 2)
    assert np.array_equal(full, orc.naive_gemm(W, X))
    assert np.array_equal(mg.msgemm(pwm, X, 2, budget=256 * 8 * 3), full)
    rng = np.random.default_rng(46)
    pwm, W = _random_pwm(rng, 20, 16)
    X = rng.integers(-99, 99, size=(16, 6)).astype(np.int64)
    ref = mg.msgemm(pwm, X, 2)
    for workers in (2, 4):
        assert np.array_equal(mg.msgemm(pwm, X, 2, workers=workers), ref)


def test_counted_wrappers():
    """test_gemm.py:190-227."""
    rng = np.random.default_rng(50)
    pwm, _ = _random_pwm(rng, 12, 4)
    X = rng.integers(-10, 10, size=(4, 1)).astype(np.int64)
    Y, c = mg.msgemm_counted(pwm, X, 2)
    assert (c.fma, c.add, c.mem_weights, c.mem_activations) == (1024, 12, 48, 4)
    assert np.array_equal(Y, mg.msgemm(pwm, X, 2))
    rng = np.random.default_rng(51)
    codes = rng.integers(0, 16, size=(6, 8))
    X1 = rng.integers(-10, 10, size=(8, 1)).astype(np.int64)
    _, c1 = mg.msgemm_counted(mg.from_codes(codes, CB), X1, 2)
    _, c3 = mg.msgemm_counted(mg.from_codes(codes, CB), np.hstack([X1, X1, X1]), 2)
    for name in ("fma", "add", "mem_weights", "mem_activations"):
        assert getattr(c3, name) == 3 * getattr(c1, name)
    _, c = mg.msgemm_counted(mg.from_codes([[3, 5]], CB), np.ones((2, 1), dtype=np.int64), 2)
    assert c.add == 0
    with pytest.raises(ValueError):
        mg.msgemm_counted(_random_pwm(np.random.default_rng(52), 4, 7)[0],
                          np.zeros(7, dtype=np.int64), 2)
    pwm, _ = _random_pwm(np.random.default_rng(53), 4, 8,
                         mg.PerGroup(group_size=4, q=np.ones((4, 2), dtype=np.int64)))
    _, c = mg.msgemm_counted(pwm, np.zeros((8, 3), dtype=np.int64), 2)
    assert c.mul == 4 * 2 * 3 and c.add == (8 // 2 - 1) * 4 * 3
    _, c = mg.naive_gemm_counted(np.ones((3, 5), dtype=np.int64), np.ones((5, 2), dtype=np.int64))
    assert (c.fma, c.mem_weights, c.mem_activations) == (30, 15, 10)


# ---------------------------------------------------------------- test_lut.py

def _brute_entry(idx, xs):
    """test_lut.py:7-13: decode each nibble, dot with the x slice."""
    return sum(orc.int4_values()[(idx >> (4 * r)) & 0xF] * xs[r] for r in range(len(xs)))


def test_lut_known_answers():
    """test_lut.py:16-44, 66-75: worked entries, zero index, size, exhaustive d=2."""
    x = np.array([1, 10, 100, 1000], dtype=np.int64)
    t = mg.build_lut(x, CB, 2)
    ent = np.asarray(t.entries)
    assert ent[0, 0b0100_0010] == 42
    assert (t.num_blocks, ent.shape) == (2, (2, 256))
    for j in range(2):
        assert [int(v) for v in ent[j]] == [_brute_entry(i, x[2 * j:2 * j + 2]) for i in range(256)]
    assert mg.build_lut_block(x, CB, 2, 1)[0b0101_0011] == 5300
    with pytest.raises(IndexError):
        mg.build_lut_block(x, CB, 2, 2)
    xf = np.random.default_rng(0).standard_normal(12).astype(np.float32)
    for d in (1, 2, 3):
        assert (np.asarray(mg.build_lut(xf, CB, d).entries)[:, 0] == 0).all()


@pytest.mark.parametrize("d,k", [(1, 5), (2, 6), (3, 6), (4, 8)])
def test_lut_brute_force_small_shapes(d, k):
    """test_lut.py:47-54."""
    rng = np.random.default_rng(d * 100 + k)
    x = rng.integers(-50, 50, size=k).astype(np.int64)
    ent = np.asarray(mg.build_lut(x, CB, d).entries)
    for j in range(k // d):
        for idx in rng.integers(0, 2 ** (4 * d), size=200):
            assert ent[j, idx] == _brute_entry(int(idx), x[j * d:(j + 1) * d])


def test_lut_blocks_linearity_budget_workers_dtype():
    """test_lut.py:57-63, 78-113."""
    rng = np.random.default_rng(1)
    x = rng.integers(-9, 9, size=9).astype(np.int64)
    full = np.asarray(mg.build_lut(x, CB, 3).entries)
    for j in range(3):
        assert np.array_equal(mg.build_lut_block(x, CB, 3, j), full[j])
    x = np.random.default_rng(2).integers(-20, 20, size=8).astype(np.int64)
    assert np.array_equal(np.asarray(mg.build_lut(7 * x, CB, 2).entries),
                          7 * np.asarray(mg.build_lut(x, CB, 2).entries))
    with pytest.raises(mg.TableBudgetError):
        mg.build_lut(np.zeros(8, dtype=np.float32), CB, 4, budget=1024)
    for bad in (0, 5):
        with pytest.raises(ValueError):
            mg.build_lut(np.zeros(8, dtype=np.float32), CB, bad)
    xf = np.random.default_rng(3).standard_normal(24).astype(np.float32)
    ref = np.asarray(mg.build_lut(xf, CB, 2).entries)
    assert np.array_equal(ref, orc.lut_full(xf, orc.int4_values(), 2))
    for workers in (2, 3, 8):
        assert np.array_equal(np.asarray(mg.build_lut(xf, CB, 2, workers=workers).entries), ref)
    assert np.asarray(mg.build_lut(np.zeros(4, dtype=np.float32), CB, 2).entries).dtype == np.float32
    assert np.asarray(mg.build_lut(np.zeros(4, dtype=np.int64), CB, 2).entries).dtype == np.int64


# ---------------------------------------------------------------- test_packing.py

def test_packing_known_answers():
    """test_packing.py:9-54."""
    pwm = mg.pack([[2, 4, 3, 5]], CB)
    assert list(np.asarray(pwm.data)[0]) == [0x42, 0x53]
    assert not np.asarray(mg.pack(np.zeros((3, 6)), CB).data).any()
    with pytest.raises(ValueError):
        mg.pack([[8]], CB)
    assert mg.unpack(pwm, 0, 1) == 4 and mg.unpack(mg.pack([[-1]], CB), 0, 0) == -1
    for i, j in ((0, 4), (1, 0)):
        with pytest.raises(IndexError):
            mg.unpack(pwm, i, j)
    assert (mg.group_index(pwm, 0, 0, 2), mg.group_index(pwm, 0, 1, 2)) == (66, 83)
    with pytest.raises(IndexError):
        mg.group_index(pwm, 0, 2, 2)
    z = mg.pack(np.zeros((1, 8)), CB)
    assert all(mg.group_index(z, 0, j, d) == 0 for d in (1, 2, 4) for j in range(8 // d))


def test_pack_unpack_identity_and_shift_oracle():
    """test_packing.py:57-82."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        m, k = int(rng.integers(1, 9)), int(rng.integers(1, 17))
        w = rng.integers(-8, 8, size=(m, k))
        pwm = mg.pack(w, CB)
        assert np.array_equal(mg.dense(pwm), w)
        assert np.array_equal(np.asarray(pwm.data), orc.pack_rows(np.where(w < 0, w + 16, w), 4))
        i, j = int(rng.integers(m)), int(rng.integers(k))
        assert mg.unpack(pwm, i, j) == w[i, j]
    w = np.random.default_rng(4).integers(-8, 8, size=(5, 12))
    pwm = mg.pack(w, CB)
    enc = np.where(w < 0, w + 16, w)
    for d in (1, 2, 3, 4):
        idx = mg.group_indices(pwm, d)
        for i in range(5):
            for j in range(12 // d):
                want = sum(int(enc[i, j * d + r]) << (4 * r) for r in range(d))
                assert mg.group_index(pwm, i, j, d) == want and idx[i, j] == want


def test_pack_scales_and_range_checks():
    """test_packing.py:85-119."""
    w = np.array([[2.0, 4.0], [3.0, -6.0]])
    assert np.array_equal(mg.dense(mg.pack(w * np.array([[0.5], [2.0]]), CB,
                                           mg.PerRow(q=np.array([0.5, 2.0])))), w)
    q = np.array([[2.0, 3.0]])
    w = np.array([[1.0, -2.0, 4.0, 5.0]])
    scaled = w * np.repeat(q, 2, axis=1)
    pwm = mg.pack(scaled, CB, mg.PerGroup(group_size=2, q=q))
    assert np.array_equal(mg.dense(pwm), w)
    assert np.allclose(mg.dense(pwm, apply_scales=True), scaled)
    with pytest.raises(ValueError):
        mg.pack(np.zeros((2, 4)), CB, mg.PerRow(q=np.zeros(3)))
    with pytest.raises(ValueError):
        mg.pack(np.zeros((2, 4)), CB, mg.PerGroup(group_size=3, q=np.zeros((2, 1))))
    with pytest.raises(ValueError):
        mg.from_codes([[16]], CB)
    pwm = mg.from_codes(np.random.default_rng(5).integers(0, 16, size=(7, 11)), CB)
    assert mg.codes(pwm).max() < 16 and np.asarray(pwm.data).shape == (7, 6)
