"""The dense comparison baseline (K4) on its three kernels -- the
weight-streaming mma.sync kernel for b <= 16 (csrc/msg_dense_hmma.cu), the
CUDA-core GEMV (csrc/msg_dense.cu) and the tcgen05 kernel (csrc/msg_mma.cu) -- against the oracle's naive_gemm(dense(pwm), X)
(gemm.py:206-216).  Integer-valued X: every product and partial sum is an
integer below 2^24, so every kernel must be bit-exact; fp16 X: the
reference's rule with rtol 2e-3 (suites.py:104-124)."""

import numpy as np
import pytest

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kernel", ["hmma", "gemv", "mma"])
@pytest.mark.parametrize("m,k,b", [(1, 32, 1), (37, 96, 2), (300, 1056, 3), (129, 4096, 4),
                                   (1000, 2048, 8), (64, 8192, 1), (8192, 1024, 5)])
@pytest.mark.parametrize("cb", ["int4", "uint4"])
def test_dense_baseline_matches_oracle(kernel, m, k, b, cb):
    import torch
    rng = np.random.default_rng(m + k + b)
    book = mg.int4_codebook() if cb == "int4" else mg.uint4_codebook()
    vals = orc.int4_values() if cb == "int4" else orc.uint4_values()
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, book)
    W = vals[codes]
    Xi = rng.integers(-60, 61, (k, b))
    yi = mg.dequant_gemm(pwm, torch.from_numpy(Xi.astype(np.float16)).cuda(), kernel=kernel).cpu().numpy()
    assert np.array_equal(yi.astype(np.int64), orc.naive_gemm(W, Xi.astype(np.int64)))
    X = rng.standard_normal((k, b)).astype(np.float16)
    y = mg.dequant_gemm(pwm, torch.from_numpy(X).cuda(), kernel=kernel).cpu().numpy()
    assert orc.rel_error(y, W, X) <= 2e-3
    y16 = mg.dequant_gemm(pwm, torch.from_numpy(X).cuda(), out_dtype=np.float16, kernel=kernel)
    assert y16.dtype == torch.float16 and orc.rel_error(y16.cpu().numpy(), W, X) <= 2e-3


def test_dense_baseline_vector_and_auto_dispatch():
    import torch
    rng = np.random.default_rng(3)
    codes = rng.integers(0, 16, (513, 2048), dtype=np.uint8)
    pwm = mg.from_codes(codes, mg.int4_codebook())
    x = rng.standard_normal(2048).astype(np.float16)
    y = mg.dequant_gemm(pwm, torch.from_numpy(x).cuda()).cpu().numpy()
    assert y.shape == (513,)
    assert orc.rel_error(y, orc.int4_values()[codes], x) <= 2e-3
    with pytest.raises(NotImplementedError):
        mg.dequant_gemm(mg.from_codes(codes[:, :100], mg.int4_codebook()),
                        torch.from_numpy(x[:100]).cuda(), kernel="gemv")      # k % 32 != 0


@pytest.mark.parametrize("m,k,b", [(130, 128, 9), (777, 4096, 16), (1, 8192, 13), (4096, 4096, 1),
                                   (2049, 2080, 11), (256, 32, 16), (8192, 8192, 8)])
@pytest.mark.parametrize("split", [None, "1", "2", "8"])
def test_dense_hmma_wide_batches_and_splits(m, k, b, split, monkeypatch):
    """b = 9..16 (second n-tile), every cluster size of the k split, ragged
    rows and k tails -- bit-exact against numpy for integer X, repeatable."""
    import torch
    if split is None:
        monkeypatch.delenv("MSG_DH_SPLIT", raising=False)
    else:
        monkeypatch.setenv("MSG_DH_SPLIT", split)
    rng = np.random.default_rng(m * 7 + k + b)
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, mg.int4_codebook())
    W = orc.int4_values()[codes]
    Xi = rng.integers(-30, 31, (k, b))
    xd = torch.from_numpy(Xi.astype(np.float16)).cuda()
    y1 = mg.dequant_gemm(pwm, xd, kernel="hmma")
    y2 = mg.dequant_gemm(pwm, xd, kernel="hmma")
    assert torch.equal(y1, y2)
    assert np.array_equal(y1.cpu().numpy().astype(np.int64), W.astype(np.int64) @ Xi.astype(np.int64))
    X = rng.standard_normal((k, b)).astype(np.float16)
    y = mg.dequant_gemm(pwm, torch.from_numpy(X).cuda(), kernel="hmma").cpu().numpy()
    assert orc.rel_error(y, W, X) <= 2e-3
