"""K3 (weight repack) layouts decoded on the host: every stored record must
reproduce the reference's group index (packing.py:201-228) under the layout's
fold and rotation, and the conflict-aware rotations of the rounds-of-4 layout
must cut the expected shared-memory wavefronts per LDS.128 phase below the
fixed rotation's (measured model: tools/microbench/lds_conflicts.cu)."""

import numpy as np
import pytest
import torch

import paper_2310_06178_b200 as mg
from oracle import msgemm_oracle as orc
from paper_2310_06178_b200 import _lib

pytestmark = pytest.mark.gpu


def _al256(v):
    return (v + 255) // 256 * 256


def _decode_rb4(buf, m, k, rpt=16):
    """lo/hi/rot planes of MSG_LAYOUT_RB4 (rpt 16) / RB4S (rpt 8) -> (f, sign,
    table) per (row, quad, position)."""
    nb = k // 3
    nq = (nb + 3) // 4
    mp = (m + 31) // 32 * 32
    lo_n = nq * mp
    hi_off = _al256(lo_n * 4)
    rot_off = hi_off + _al256(lo_n * 2)
    lo = np.frombuffer(buf[:lo_n * 4].tobytes(), np.uint32).reshape(nq, mp)
    hi = np.frombuffer(buf[hi_off:hi_off + lo_n * 2].tobytes(), np.uint16).reshape(nq, mp).astype(np.uint32)
    rot = np.frombuffer(buf[rot_off:rot_off + nq * (mp // rpt) * 4].tobytes(), np.uint32).reshape(nq, mp // rpt)
    f = np.stack([lo & 0x7FF, (lo >> 11) & 0x7FF, (lo >> 22) | ((hi & 1) << 10), (hi >> 1) & 0x7FF], -1)
    sg = np.stack([(hi >> (12 + s)) & 1 for s in range(4)], -1)
    rows = np.arange(mp)
    rho = (rot[:, rows // rpt] >> (2 * (rows % rpt))) & 3          # (nq, mp)
    table = (np.arange(4)[None, None, :] + rho[:, :, None]) % 4
    return f[:, :m], sg[:, :m], table[:, :m], rho[:, :m]


@pytest.mark.parametrize("rpt", [16, 8])
@pytest.mark.parametrize("m,k", [(8192, 96), (300, 3 * 41 + 2), (16384 + 64, 48)])
def test_rb4_layout_roundtrip_and_conflicts(m, k, rpt):
    rng = np.random.default_rng(m + k)
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, mg.int4_codebook())
    dev = _lib.require_device()
    lay = _lib.LAYOUT_RB4 if rpt == 16 else _lib.LAYOUT_RB4S
    buf = pwm.device_layout(dev, 3, lay, 1).cpu().numpy()
    f, sg, table, rho = _decode_rb4(buf, m, k, rpt)
    gidx = orc.group_indices(orc.pack_rows(codes, 4), k, 4, 3)     # (m, nb)
    nb = gidx.shape[1]
    nq = f.shape[0]
    # the record at (quad q, row i, position s) is group 4q + table[q, i, s]
    for q in range(nq):
        j = 4 * q + table[q]                                        # (m, 4)
        valid = j < nb
        want = np.where(valid, gidx[np.arange(m)[:, None], np.minimum(j, nb - 1)], 0)
        got = np.where(sg[q] == 1, f[q] ^ 0xFFF, f[q])
        assert np.array_equal(np.where(valid, got, 0), want)
        assert np.all(f[q][~valid] == 0) and np.all(sg[q][~valid] == 0)
    if m < 8192:
        return
    # expected LDS.128 wavefronts per phase: lanes u of an octet hold rows
    # base + rpt u + r; bank group of a lookup = 4 * (f & 1) + table
    ob = 8 * rpt
    blk = m // ob * ob
    bank = 4 * (f[:, :blk] & 1) + table[:, :blk]                    # (nq, rows, 4)
    b = bank.reshape(nq, blk // ob, 8, rpt, 4)                      # q, octet, u, r, s
    onehot = np.eye(8, dtype=np.int32)[b]                           # ... 8 bank groups
    cnt = onehot.sum(axis=2)                                        # q, octet, r, s, 8
    opt = cnt.max(-1).mean()
    fixed_table = (np.arange(4)[None, :] + (np.arange(blk) // rpt % 4)[:, None]) % 4
    # the same records under the fixed rotation rho = lane mod 4 (the parities
    # of the groups a lane would read at each position)
    fgrp = np.empty_like(f[:, :blk])
    for s in range(4):
        sel = (table[:, :blk] == s)
        fgrp[..., s] = np.where(sel, f[:, :blk], 0).sum(-1)
    par = fgrp & 1                                                  # parity per group
    fb = 4 * np.take_along_axis(par, np.broadcast_to(fixed_table[None], par.shape), -1) + fixed_table
    cnt_f = np.eye(8, dtype=np.int32)[fb.reshape(nq, blk // ob, 8, rpt, 4)].sum(axis=2)
    base = cnt_f.max(-1).mean()
    assert base > 1.85 and opt < 1.65, (base, opt)


@pytest.mark.parametrize("m,b", [(300, 8), (4096 + 33, 8), (11008, 16), (8192, 9)])
def test_rb4_row_variants_agree(m, b):
    """The 4096-row (RB4S) and 8192-row (RB4) kernels give the same results
    within the fp16 rule, and both match the oracle."""
    rng = np.random.default_rng(m * b)
    k = 3 * 97 + 1
    codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
    pwm = mg.from_codes(codes, mg.int4_codebook())
    X = rng.standard_normal((k, b)).astype(np.float16)
    W = orc.dense(np.asarray(pwm.data), k, 4, orc.int4_values())
    y16 = mg.msgemm(pwm, X, 3, _flags=_lib.FLAG_RB_ROWS16)
    y8 = mg.msgemm(pwm, X, 3, _flags=_lib.FLAG_RB_ROWS8)
    for y in (y16, y8):
        assert orc.rel_error(y.astype(np.float64), W, X) <= 2e-3
