"""naive_gemm (gemm.py:206-216) on the GPU against the CPU oracle's numpy product.

Integer operands: bit-exact int64, including products and sums past 2^53
(numpy wraps int64; so does msg_naive_gemm).  float16: bit-exact (numpy's
half matmul sums exact fp32 products in k order).  float32 / float64 and
mixed operands: numpy's BLAS order is unspecified, so the rule is the
reference's |dy| <= rtol * sum_j |W_ij||x_j| (suites.py:104-124) with rtol
1e-5 (f32) / 1e-12 (f64).
"""

import numpy as np
import pytest

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc

pytestmark = pytest.mark.gpu


def _bound_ok(actual, W, X, rtol):
    ref = orc.naive_gemm(W, X)
    assert actual.dtype == ref.dtype and actual.shape == ref.shape
    W64, X64 = np.asarray(W, dtype=np.float64), np.asarray(X, dtype=np.float64)
    scale = np.abs(W64) @ np.abs(X64)
    diff = np.abs(actual.astype(np.float64) - ref.astype(np.float64))
    assert (diff <= rtol * scale + 1e-300).all(), float(np.max(diff / np.maximum(scale, 1e-30)))


@pytest.mark.parametrize("m,k,b", [(1, 1, 1), (7, 33, 3), (65, 100, 17), (130, 1027, 9), (64, 4096, 1)])
@pytest.mark.parametrize("wdt,xdt", [(np.int64, np.int64), (np.int8, np.int32), (np.uint8, np.int16),
                                     (np.int32, np.int64)])
def test_integer_bit_exact(m, k, b, wdt, xdt):
    rng = np.random.default_rng(m * 1000 + k + b)
    info_w, info_x = np.iinfo(wdt), np.iinfo(xdt)
    W = rng.integers(max(info_w.min, -2 ** 20), min(info_w.max, 2 ** 20), size=(m, k)).astype(wdt)
    X = rng.integers(max(info_x.min, -2 ** 20), min(info_x.max, 2 ** 20), size=(k, b)).astype(xdt)
    y = mg.naive_gemm(W, X)
    ref = orc.naive_gemm(W, X)
    assert y.dtype == ref.dtype == np.int64 and np.array_equal(y, ref)


def test_integer_past_2_53_wraps_like_numpy():
    rng = np.random.default_rng(5)
    W = rng.integers(-2 ** 40, 2 ** 40, size=(33, 300), dtype=np.int64)
    X = rng.integers(-2 ** 40, 2 ** 40, size=(300, 4), dtype=np.int64)
    with np.errstate(over="ignore"):
        ref = orc.naive_gemm(W, X)
    assert np.array_equal(mg.naive_gemm(W, X), ref)


@pytest.mark.parametrize("m,k,b", [(3, 5, 1), (64, 333, 4), (200, 4096, 16), (17, 8192, 8)])
def test_float16_bit_exact(m, k, b):
    rng = np.random.default_rng(k + b)
    W = orc.int4_values()[rng.integers(0, 16, size=(m, k))].astype(np.float16)
    X = rng.standard_normal((k, b)).astype(np.float16)
    y = mg.naive_gemm(W, X)
    ref = orc.naive_gemm(W, X)
    assert y.dtype == np.float16 and np.array_equal(y.view(np.uint16), ref.view(np.uint16))
    # int4 weights as int8 with fp16 X: numpy promotes to float16 (same loop)
    Wi = orc.int4_values()[rng.integers(0, 16, size=(m, k))].astype(np.int8)
    assert np.array_equal(mg.naive_gemm(Wi, X).view(np.uint16), orc.naive_gemm(Wi, X).view(np.uint16))


@pytest.mark.parametrize("wdt,xdt,rtol", [(np.float32, np.float32, 1e-5), (np.int64, np.float32, 1e-12),
                                          (np.float64, np.float64, 1e-12), (np.float32, np.float16, 1e-5),
                                          (np.int8, np.float64, 1e-12)])
def test_float_within_reference_rule(wdt, xdt, rtol):
    rng = np.random.default_rng(11)
    for m, k, b in ((1, 1, 1), (31, 257, 5), (100, 8192, 3)):
        W = orc.int4_values()[rng.integers(0, 16, size=(m, k))].astype(wdt)
        X = rng.standard_normal((k, b)).astype(xdt)
        _bound_ok(mg.naive_gemm(W, X), W, X, rtol)


def test_vector_empty_and_device_inputs():
    import torch
    rng = np.random.default_rng(3)
    W = rng.integers(-8, 8, size=(9, 14))
    x = rng.integers(-50, 50, size=14)
    y = mg.naive_gemm(W, x)
    assert y.shape == (9,) and np.array_equal(y, orc.naive_gemm(W, x))
    assert mg.naive_gemm(np.zeros((0, 4), dtype=np.int64), np.ones(4, dtype=np.int64)).shape == (0,)
    assert mg.naive_gemm(np.zeros((3, 0), dtype=np.float32), np.ones((0, 2), dtype=np.float32)).tolist() == \
        [[0.0, 0.0]] * 3
    Wt = torch.as_tensor(W.astype(np.float16), device="cuda")
    Xt = torch.as_tensor(rng.standard_normal((14, 2)).astype(np.float16), device="cuda")
    yt = mg.naive_gemm(Wt, Xt)
    assert yt.is_cuda and yt.dtype == torch.float16
    assert np.array_equal(yt.cpu().numpy(), orc.naive_gemm(Wt.cpu().numpy(), Xt.cpu().numpy()))
    with pytest.raises(ValueError):
        mg.naive_gemm(W, np.ones(13))


def test_dense_of_packed_weights_matches_msgemm_exact():
    """naive_gemm(dense(pwm), X) is the spec msgemm is held to (suites.py:113-115)."""
    rng = np.random.default_rng(8)
    codes = rng.integers(0, 16, size=(300, 4096), dtype=np.uint8)
    pwm = mg.from_codes(codes, mg.int4_codebook())
    X = rng.integers(-127, 128, size=(4096, 4)).astype(np.int64)
    ref = orc.naive_gemm(orc.int4_values()[codes], X)
    assert np.array_equal(mg.naive_gemm(mg.dense(pwm), X), ref)
    assert np.array_equal(mg.msgemm(pwm, X, 3), ref)
