"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
host-side planning, and the reference's host-side validation/error order
(all raised before any device work, so they run without a GPU)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2310_06178_b200 as mg
from paper_2310_06178_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        names |= set(re.findall(r"MSG_API\s+[\w\s\*]+?\b(msg_\w+)\s*\(", h.read_text()))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    decl = declared_symbols()
    assert decl, "no MSG_API declarations found"
    assert decl == set(_lib.EXPORTS)
    for name in decl:
        assert hasattr(lib, name), name
    assert lib.msg_version() >= 100


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _plan(m, k, b, d, dt=_lib.F16, flags=0, cb=None, scale=0, gs=0):
    lib = _lib.load_library()
    lay, sym, ws = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    vals = _lib.host_doubles((cb or mg.int4_codebook()).values)
    st = lib.msg_gemm_plan(m, k, 4 if cb is None else cb.width, vals, dt, b, d, scale, gs, flags,
                           ctypes.byref(lay), ctypes.byref(sym), ctypes.byref(ws))
    return st, lay.value, sym.value, ws.value


@pytest.mark.parametrize("m,k,b,d", [(1024, 1024, 1, 2), (4096, 4096, 1, 3),
                                     (11008, 4096, 16, 3), (8192, 8192, 256, 3),
                                     (65536, 8192, 8, 3)])
def test_plan_configs_take_fused_symmetric_path(m, k, b, d):
    st, lay, sym, ws = _plan(m, k, b, d)
    if d != 3:
        want = _lib.LAYOUT_QUAD
    elif b == 1:
        want = _lib.LAYOUT_LANE
    else:   # batched d = 3: the row-block kernel, rounds of 32 / min(b, 8) groups
        # (4096-row CTAs -- RB4S -- for m <= 16384 at b <= 16, 8192-row CTAs otherwise)
        want = _lib.LAYOUT_RB4S if (m <= 16384 and b <= 16) else _lib.LAYOUT_RB4
    assert st == 0 and lay == want and sym == 1 and ws > 0
    # the generic fused kernel remains selectable for every shape
    st, lay, sym, ws = _plan(m, k, b, d, flags=_lib.FLAG_NO_LANE | _lib.FLAG_NO_ROWBLOCK)
    assert st == 0 and lay == _lib.LAYOUT_QUAD


@pytest.mark.parametrize("b,want", [(2, 6), (3, 6), (4, 5), (5, 7), (7, 7), (8, 7), (16, 7), (64, 4)])
def test_plan_rowblock_round_width(b, want):
    st, lay, sym, ws = _plan(8192, 8192, b, 3)
    assert st == 0 and lay == want
    assert _plan(8192, 8192, b, 3, dt=_lib.F32)[1] == _lib.LAYOUT_QUAD     # fp32 X: fp32 tables
    assert _plan(8192, 8192, b, 3, flags=_lib.FLAG_F32_ENTRIES)[1] == _lib.LAYOUT_QUAD
    assert _plan(8192, 8192, b, 3, flags=_lib.FLAG_NO_SYMMETRY)[1] == _lib.LAYOUT_QUAD


def test_plan_routes_to_generic():
    assert _plan(64, 48, 3, 4)[1] == _lib.LAYOUT_NONE                    # d=4
    assert _plan(64, 48, 3, 2, dt=_lib.I64)[1] == _lib.LAYOUT_NONE       # integer X
    assert _plan(64, 48, 3, 2, scale=2, gs=4)[1] == _lib.LAYOUT_NONE     # per-group, 2 groups
    assert _plan(64, 48, 3, 2, scale=2, gs=8)[1] == _lib.LAYOUT_QUAD     # per-group, 1 quad
    assert _plan(64, 96, 1, 3, scale=2, gs=12)[1] == _lib.LAYOUT_QUAD    # b=1: not the lane kernel
    assert _plan(64, 40, 3, 2, scale=2, gs=16)[1] == _lib.LAYOUT_NONE    # k % group_size != 0
    assert _plan(64, 48, 3, 2, flags=_lib.FLAG_FORCE_GENERIC)[1] == _lib.LAYOUT_NONE
    assert _plan(64, 48, 3, 3, flags=_lib.FLAG_NO_SYMMETRY)[2] == 0
    custom = mg.custom_codebook([0, 1, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 17])
    st, lay, sym, _ = _plan(64, 48, 3, 3, cb=custom)
    assert st == 0 and lay == _lib.LAYOUT_QUAD and sym == 0            # not antisymmetric


def test_plan_errors_map_like_reference():
    assert _plan(4, 8, 1, 0)[0] == _lib.MSG_ERR_VALUE                   # d < 1
    assert _plan(4, 8, 1, 9)[0] == _lib.MSG_ERR_VALUE                   # d*width > 32
    assert _plan(4, 8, 1, 3, scale=2, gs=4)[0] == _lib.MSG_ERR_VALUE     # group 4 % 3
    assert _plan(4, 8, 1, 8)[0] == _lib.MSG_ERR_UNSUPPORTED             # > 2^28 entries
    assert _plan(4, 8, 1, 2, dt=_lib.BF16)[0] == _lib.MSG_ERR_UNSUPPORTED


def test_repacked_bytes():
    lib = _lib.load_library()
    assert lib.msg_repacked_bytes(4096, 4096, 3, _lib.LAYOUT_LANE) >= 4096 * 4096 // 2
    assert lib.msg_mma_layout_bytes(8192, 8192) == 8192 * 8192 // 2
    assert lib.msg_repacked_bytes(65536, 8192, 3, _lib.LAYOUT_QUAD) >= 65536 * 8192 // 2
    assert lib.msg_repacked_bytes(10, 10, 4, _lib.LAYOUT_QUAD) == -1
    assert lib.msg_repacked_bytes(10, 10, 2, _lib.LAYOUT_NONE) == 0


# ---- reference codebook semantics (test_codebook.py) : pure host ----

def test_codebook_semantics():
    cb = mg.int4_codebook()
    assert [cb.decode(c) for c in (0, 1, 7, 8, 15)] == [0, 1, 7, -8, -1]
    assert cb.zero_code == 0 and cb.encode(-1) == 0b1111
    with pytest.raises(ValueError):
        cb.encode(8)
    assert mg.uint4_codebook().decode(15) == 15
    c2 = mg.custom_codebook([0.0, 0.5, 1.0, 2.0])
    assert c2.width == 2 and c2.encode(2.0) == 3
    for bad in ([0, 0, 1, 2], [0, 1, 2], [float("nan")] * 4):
        with pytest.raises(ValueError):
            mg.custom_codebook(bad)
    assert cb.antisymmetric_offset() == -0.5
    assert mg.uint4_codebook().antisymmetric_offset() == 7.5


# ---- validation order of msgemm happens before any device call ----

def _pwm_host(m, k):
    data = np.zeros((m, (k + 1) // 2), dtype=np.uint8)
    return mg.PackedWeightMatrix(m=m, k=k, width=4, data=data, codebook=mg.int4_codebook())


def test_msgemm_validation_order_without_device():
    pwm = _pwm_host(4, 8)
    with pytest.raises(ValueError):
        mg.msgemm(pwm, np.zeros((8, 1, 1)), 2)
    with pytest.raises(ValueError):
        mg.msgemm(pwm, np.zeros(7, dtype=np.int64), 2)
    with pytest.raises(ValueError):
        mg.msgemm(pwm, np.zeros(8, dtype=np.int64), 0)
    with pytest.raises(ValueError):
        mg.msgemm(pwm, np.zeros(8, dtype=np.int64), 9)
    with pytest.raises(mg.TableBudgetError):
        mg.msgemm(pwm, np.zeros(8, dtype=np.int64), 4, budget=1024)
    q = np.ones((4, 2), dtype=np.int64)
    pg = mg.PackedWeightMatrix(m=4, k=8, width=4, data=pwm.data, codebook=pwm.codebook,
                               scales=mg.PerGroup(group_size=4, q=q))
    with pytest.raises(ValueError):
        mg.msgemm(pg, np.zeros(8, dtype=np.int64), 3)


def test_pwm_and_scale_validation():
    with pytest.raises(ValueError):
        mg.PackedWeightMatrix(m=2, k=4, width=4, data=np.zeros((2, 3), np.uint8),
                              codebook=mg.int4_codebook())
    with pytest.raises(ValueError):
        mg.PackedWeightMatrix(m=2, k=4, width=4, data=np.zeros((2, 2), np.uint8),
                              codebook=mg.int4_codebook(), scales=mg.PerRow(q=np.zeros(3)))
    with pytest.raises(ValueError):
        mg.PackedWeightMatrix(m=2, k=4, width=4, data=np.zeros((2, 2), np.uint8),
                              codebook=mg.int4_codebook(),
                              scales=mg.PerGroup(group_size=3, q=np.zeros((2, 1))))


def test_lut_validation_without_device():
    cb = mg.int4_codebook()
    with pytest.raises(ValueError):
        mg.build_lut(np.zeros((2, 2)), cb, 2)
    with pytest.raises(ValueError):
        mg.build_lut(np.zeros(8, np.float32), cb, 0)
    with pytest.raises(ValueError):
        mg.build_lut(np.zeros(8, np.float32), cb, 5)
    with pytest.raises(mg.TableBudgetError):
        mg.build_lut(np.zeros(8, np.float32), cb, 4, budget=1024)
    with pytest.raises(IndexError):
        mg.build_lut_block(np.zeros(4), cb, 2, 2)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mg.msgemm(_pwm_host(4, 8), np.zeros(8, np.float32), 2)


def test_package_never_imports_oracle():
    pat = re.compile(r"^\s*(from\s+oracle|import\s+oracle)", re.M)
    for p in (ROOT / "paper_2310_06178_b200").rglob("*.py"):
        assert not pat.search(p.read_text()), p
