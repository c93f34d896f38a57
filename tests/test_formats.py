"""MSGW/MSGA/MSGY files (row f1): byte-identical to the reference's, pinned by the
reference's golden 12x4 hex (test_acceptance.py:39-43), plus the device loader."""

import numpy as np
import pytest

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc
from paper_2310_06178_b200 import formats as F

RUNNING = [
    [2, 4, 3, 5], [-1, 0, 1, -8], [7, -3, 2, 6], [0, 0, 0, 0],
    [1, 2, 3, 4], [-4, 5, -6, 7], [3, 3, 3, 3], [-8, -8, -8, -8],
    [6, 1, -2, 0], [5, -5, 5, -5], [0, 7, -1, 2], [-2, 4, 0, -7],
]
GOLDEN_MSGW_HEX = (
    "4d534757010000000c000000000000000400000000000000040000000000"
    "42530f81d762000021435c7a33338888160eb5b5702f4e90"
)


def _pwm(data, m, k, scales=None):
    return mg.PackedWeightMatrix(m=m, k=k, width=4, data=data, codebook=mg.int4_codebook(),
                                 scales=scales)


def test_golden_msgw_bytes(tmp_path):
    data = orc.pack_rows(orc.nearest_codes(RUNNING, orc.int4_values()) & 0xF, 4)
    p = tmp_path / "g.msgw"
    F.write_weights(p, _pwm(data, 12, 4))
    assert p.read_bytes().hex() == GOLDEN_MSGW_HEX
    back = F.read_weights(p)
    assert np.array_equal(back.data, data) and back.m == 12 and back.k == 4


def test_roundtrip_scales_and_matrices(tmp_path):
    rng = np.random.default_rng(70)
    for i in range(30):
        m, k = int(rng.integers(1, 33)), 2 * int(rng.integers(1, 17))
        data = orc.pack_rows(rng.integers(0, 16, (m, k), dtype=np.uint8), 4)
        scales = None
        if i % 3 == 1:
            scales = mg.PerRow(q=rng.random(m).astype(np.float32))
        elif i % 3 == 2:
            scales = mg.PerGroup(group_size=2, q=rng.random((m, k // 2)).astype(np.float32))
        p = tmp_path / f"w{i}.msgw"
        F.write_weights(p, _pwm(data, m, k, scales))
        back = F.read_weights(p)
        assert np.array_equal(back.data, data)
        if scales is not None:
            assert np.array_equal(np.asarray(back.scales.q), np.asarray(scales.q))
    X = rng.standard_normal((7, 3)).astype(np.float32)
    F.write_activations(tmp_path / "x.msga", X)
    assert np.array_equal(F.read_activations(tmp_path / "x.msga"), X)
    F.write_output(tmp_path / "y.msgy", X)
    assert np.array_equal(F.read_output(tmp_path / "y.msgy"), X)


def test_format_errors(tmp_path):
    p = tmp_path / "bad.msgw"
    p.write_bytes(b"XXXX" + bytes(26))
    with pytest.raises(F.FormatError):
        F.read_weights(p)
    p.write_bytes(bytes(5))
    with pytest.raises(F.FormatError):
        F.read_weights(p)
    data = orc.pack_rows(np.zeros((2, 4), np.uint8), 4)
    F.write_weights(p, _pwm(data, 2, 4))
    p.write_bytes(p.read_bytes()[:-1])
    with pytest.raises(F.FormatError):
        F.read_weights(p)


@pytest.mark.gpu
def test_load_weights_device_matches_host(tmp_path):
    import torch
    rng = np.random.default_rng(1)
    m, k = 1000, 3001
    data = orc.pack_rows(rng.integers(0, 16, (m, k), dtype=np.uint8), 4)
    p = tmp_path / "w.msgw"
    F.write_weights(p, _pwm(data, m, k))
    dev_pwm = F.load_weights_device(p, d=3)
    assert dev_pwm.data.is_cuda
    X = rng.standard_normal((k, 4)).astype(np.float16)
    y_dev = mg.msgemm(dev_pwm, torch.from_numpy(X).cuda(), 3).cpu().numpy()
    y_host = mg.msgemm(F.read_weights(p), X, 3)
    assert np.array_equal(y_dev.view(np.uint16), y_host.view(np.uint16))
    # against the oracle on the file's own bytes (not a self-comparison)
    W = orc.dense(data, k, 4, orc.int4_values())
    assert np.array_equal(np.asarray(dev_pwm.data.cpu()), data)
    assert orc.rel_error(y_dev, W, X) <= 2e-3
    Xi = rng.integers(-127, 128, (k, 2)).astype(np.int64)
    yi = mg.msgemm(dev_pwm, torch.from_numpy(Xi.astype(np.float16)).cuda(), 3,
                   table_dtype=np.float32, out_dtype=np.float32).cpu().numpy()
    assert np.array_equal(yi.astype(np.int64), orc.msgemm(data, m, k, 4, orc.int4_values(), Xi, 3))
