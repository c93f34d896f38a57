"""Full-size BASELINE configurations on the GPU.

At full size the CPU oracle would take minutes, so parity is shown three
ways (size-independent, as the task asks):
  1. a sample of rows is checked against the oracle run on those rows only
     (row-chunking the oracle is bitwise safe);
  2. the whole Y is checked against a dense float64/float32 torch product of
     the same inputs, with the reference's tolerance convention;
  3. algebraic properties: linearity (msgemm(2X) == 2*msgemm(X) bitwise),
     symmetric-vs-full-table agreement, determinism.
"""

import numpy as np
import pytest
import torch

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc
from paper_2310_06178_b200.workloads import CONFIGS, activations, weights

pytestmark = pytest.mark.gpu

INT4 = orc.int4_values()


def _dense_check(data, m, k, X, Y, tol, exact):
    """Whole-output check against a dense GPU product (W dequantised exactly)."""
    dev = torch.device("cuda")
    pwm = mg.PackedWeightMatrix(m=m, k=k, width=4, data=data, codebook=mg.int4_codebook())
    codes = mg.codes(mg.PackedWeightMatrix(m=m, k=k, width=4, data=torch.from_numpy(data).to(dev),
                                           codebook=mg.int4_codebook()))
    W = torch.where(codes < 8, codes.to(torch.int32), codes.to(torch.int32) - 16).to(torch.float64)
    Xd = torch.from_numpy(np.asarray(X, dtype=np.float64)).to(dev)
    exact_y = W @ Xd
    Yd = torch.from_numpy(np.asarray(Y, dtype=np.float64)).to(dev)
    if exact:
        assert torch.equal(Yd, exact_y)
        return 0.0
    scale = W.abs() @ Xd.abs()
    rel = ((Yd - exact_y).abs() / scale.clamp_min(1e-30)).max().item()
    assert rel <= tol, rel
    return rel


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg2int", "cfg3", "cfg4b1", "cfg4b4",
                                  "cfg4b16", "cfg4b64", "cfg4b256", "cfg5", "cfg5b1"])
def test_config_parity(name):
    cfg = CONFIGS[name]
    data = weights(cfg)
    X = activations(cfg)
    pwm = mg.PackedWeightMatrix(m=cfg.m, k=cfg.k, width=4, data=data, codebook=mg.int4_codebook())
    exact = cfg.x_dtype == "int"
    if exact:
        # integer-valued X as fp16 on the device, fp32 tables and fp32 Y: bit-exact
        Y = mg.msgemm(pwm, X.astype(np.float16), cfg.d, table_dtype=np.float32,
                      out_dtype=np.float32)
        assert Y.dtype == np.float32
    else:
        Y = mg.msgemm(pwm, X, cfg.d)
        assert Y.dtype == X.dtype
    assert Y.shape == (cfg.m, cfg.b)
    tol = 1e-5 if cfg.x_dtype == "float32" else 2e-3
    # 1. oracle on a row sample
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([[0, cfg.m - 1], rng.choice(cfg.m, 62, replace=False)]))
    if exact:
        ref = orc.msgemm(data[rows], len(rows), cfg.k, 4, INT4, X, cfg.d)
        assert np.array_equal(Y[rows].astype(np.int64), ref)
    else:
        ref = orc.msgemm(data[rows], len(rows), cfg.k, 4, INT4, X, cfg.d)
        W = orc.dense(data[rows], cfg.k, 4, INT4)
        assert orc.rel_error(Y[rows], W, X) <= tol
        assert orc.rel_error(ref, W, X) <= tol
    # 2. whole output vs dense product
    _dense_check(data, cfg.m, cfg.k, X, Y, tol, exact)


def test_cfg2_int_fp16_device_bitexact():
    """The north_star's bit-exact check: integer X in [-127,127] as fp16 on the
    device, fp32 tables (fp16 cannot hold entries up to 3*8*127), fp32 Y."""
    cfg = CONFIGS["cfg2int"]
    data = weights(cfg)
    X = activations(cfg)
    pwm = mg.PackedWeightMatrix(m=cfg.m, k=cfg.k, width=4, data=data, codebook=mg.int4_codebook())
    xd = torch.from_numpy(X.astype(np.float16)).cuda()
    Yh = mg.msgemm(pwm, xd, cfg.d, table_dtype=np.float32)          # fp16 out (rounded)
    Yf = mg.msgemm(pwm, xd, cfg.d, table_dtype=np.float32, out_dtype=np.float32)
    ref = orc.msgemm(data, cfg.m, cfg.k, 4, INT4, X, cfg.d)          # int64 oracle, full size
    assert np.array_equal(Yf.cpu().numpy().astype(np.int64), ref)
    assert np.array_equal(Yf.cpu().numpy(), ref.astype(np.float32))
    for sym in (True, False):
        Ys = mg.msgemm(pwm, xd.float(), cfg.d, symmetric=sym)      # fp32 X path too
        assert np.array_equal(Ys.cpu().numpy().astype(np.int64), ref)
    # fp16 output is the fp16 rounding of the exact value
    assert np.array_equal(Yh.cpu().numpy(), ref.astype(np.float16))


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg5"])
def test_properties(name):
    cfg = CONFIGS[name]
    data = weights(cfg)
    X = activations(cfg)
    pwm = mg.PackedWeightMatrix(m=cfg.m, k=cfg.k, width=4, data=data, codebook=mg.int4_codebook())
    xd = torch.from_numpy(X).cuda()
    xf = xd.float()   # fp32 tables: no subnormal rounding, so scaling by 2 is exact
    y1f = mg.msgemm(pwm, xf, cfg.d)
    assert torch.equal(mg.msgemm(pwm, 2 * xf, cfg.d), 2 * y1f)     # linearity, bitwise
    y1 = mg.msgemm(pwm, xd, cfg.d)
    assert torch.equal(mg.msgemm(pwm, xd, cfg.d), y1)               # determinism
    yn = mg.msgemm(pwm, xd, cfg.d, symmetric=False)
    W = orc.dense(data[:256], cfg.k, 4, INT4)
    assert orc.rel_error(yn[:256].cpu().numpy(), W, X) <= 2e-3
    # column decomposition (within tolerance: the column tile changes the k-split)
    for c in (0, cfg.b - 1):
        yc = mg.msgemm(pwm, xd[:, c].contiguous(), cfg.d)
        assert orc.rel_error(yc[:256].cpu().numpy(), W, X[:, c]) <= 2e-3


@pytest.mark.parametrize("m,k,b", [(128, 64, 1), (300, 200, 3), (1024, 1024, 16), (8192, 8192, 1),
                                   (8192, 8192, 16), (8192, 8192, 64), (8192, 8192, 256),
                                   (11008, 4096, 16), (4096, 4096, 1)])
def test_dequant_mma_matches_dense(m, k, b):
    """K4 (tcgen05 kind::f16, fp32 TMEM accumulation) against the exact dense
    product: bit-exact for integer-valued X (partials < 2^24), 2e-3 rule for
    N(0,1) fp16 X."""
    rng = np.random.default_rng(m + k + b)
    data = rng.integers(0, 256, size=(m, (k + 1) // 2), dtype=np.uint8)
    pwm = mg.PackedWeightMatrix(m=m, k=k, width=4, data=data, codebook=mg.int4_codebook())
    W = orc.dense(data, k, 4, INT4)
    Xi = rng.integers(-127, 128, size=(k, b))
    yi = mg.dequant_gemm(pwm, Xi.astype(np.float16))
    assert yi.dtype == np.float32 and yi.shape == (m, b)
    assert np.array_equal(yi.astype(np.int64), W.astype(np.int64) @ Xi)
    X = rng.standard_normal((k, b)).astype(np.float16)
    y = mg.dequant_gemm(pwm, X)
    assert orc.rel_error(y, W, X) <= 2e-3
    y16 = mg.dequant_gemm(pwm, torch.from_numpy(X).cuda(), out_dtype=np.float16)
    assert y16.dtype == torch.float16


def test_dequant_mma_uint4_and_vector():
    rng = np.random.default_rng(9)
    codes = rng.integers(0, 16, size=(200, 96))
    pwm = mg.from_codes(codes, mg.uint4_codebook())
    x = rng.integers(-50, 50, size=96).astype(np.float16)
    y = mg.dequant_gemm(pwm, x)
    assert y.shape == (200,)
    assert np.array_equal(y.astype(np.int64), codes.astype(np.int64) @ x.astype(np.int64))
