"""MSGW / MSGA / MSGY files and the MSGW -> device loader.

Byte layouts are the reference's (formats.py:1-15, header structs at
formats.py:32-33): little-endian ``<4sIQQBBI`` weight header (magic "MSGW",
version 1, m, k, width, scale_mode 0/1/2, group_size) followed by the packed
rows and f32 scales; ``<4sIQQ`` matrix header (magic "MSGA"/"MSGY", version
1, rows, cols) followed by f32 column-major data.  Files written here are
byte-identical to the reference's (pinned by the golden MSGW hex in the
tests).

``load_weights_device`` is the new part: it reads the payload straight into
pinned host memory, uploads it once and (optionally) runs K3 for a given
depth, returning a device-resident PackedWeightMatrix ready for msgemm.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import _lib
from .codebook import Codebook, int4_codebook
from .packing import PackedWeightMatrix, PerGroup, PerRow, bytes_per_row

MAGIC_W, MAGIC_A, MAGIC_Y = b"MSGW", b"MSGA", b"MSGY"
VERSION = 1
_WHDR = struct.Struct("<4sIQQBBI")   # formats.py:32
_MHDR = struct.Struct("<4sIQQ")      # formats.py:33


class FormatError(ValueError):
    """Malformed or truncated msGeMM data file (formats.py:36-37)."""


def _scale_fields(scales):
    if scales is None:
        return 0, 0, np.empty(0, dtype="<f4")
    if isinstance(scales, PerRow):
        return 1, 0, np.asarray(scales.q, dtype="<f4").reshape(-1)
    if isinstance(scales, PerGroup):
        return 2, scales.group_size, np.ascontiguousarray(scales.q, dtype="<f4").reshape(-1)
    raise TypeError(f"unsupported scale spec: {scales!r}")


def write_weights(path, pwm: PackedWeightMatrix) -> None:
    """formats.py:40-57."""
    mode, gs, q = _scale_fields(pwm.scales)
    data = pwm.data.detach().cpu().numpy() if _lib.is_torch(pwm.data) else np.asarray(pwm.data)
    with open(path, "wb") as f:
        f.write(_WHDR.pack(MAGIC_W, VERSION, pwm.m, pwm.k, pwm.width, mode, gs))
        f.write(np.ascontiguousarray(data, dtype=np.uint8).tobytes())
        f.write(q.tobytes())


def _parse_weight_header(blob: bytes, path, codebook: Codebook | None):
    if len(blob) < _WHDR.size:
        raise FormatError(f"{path}: truncated weight header")
    magic, version, m, k, width, mode, gs = _WHDR.unpack_from(blob)
    if magic != MAGIC_W:
        raise FormatError(f"{path}: bad magic {magic!r}, expected {MAGIC_W!r}")
    if version != VERSION:
        raise FormatError(f"{path}: unsupported version {version}")
    if codebook is None:
        if width != 4:
            raise FormatError(f"{path}: width {width} needs an explicit codebook")
        codebook = int4_codebook()
    if codebook.width != width:
        raise FormatError(f"{path}: file width {width} != codebook width {codebook.width}")
    if mode == 0:
        nq = 0
    elif mode == 1:
        nq = m
    elif mode == 2:
        if gs == 0 or k % gs:
            raise FormatError(f"{path}: invalid group_size {gs} for k={k}")
        nq = m * (k // gs)
    else:
        raise FormatError(f"{path}: unknown scale_mode {mode}")
    nd = m * bytes_per_row(k, width)
    want = _WHDR.size + nd + 4 * nq
    if len(blob) != want:
        raise FormatError(f"{path}: expected {want} bytes, found {len(blob)}")
    return m, k, width, mode, gs, nd, nq, codebook


def _scales_from(blob, off, nd, nq, mode, gs, m, k):
    if not mode:
        return None
    q = np.frombuffer(blob, dtype="<f4", count=nq, offset=off + nd).copy()
    return PerRow(q=q) if mode == 1 else PerGroup(group_size=gs, q=q.reshape(m, k // gs))


def read_weights(path, codebook: Codebook | None = None) -> PackedWeightMatrix:
    """formats.py:60-100 (host arrays, reference-compatible)."""
    blob = Path(path).read_bytes()
    m, k, width, mode, gs, nd, nq, cb = _parse_weight_header(blob, path, codebook)
    data = np.frombuffer(blob, dtype=np.uint8, count=nd, offset=_WHDR.size)
    data = data.reshape(m, bytes_per_row(k, width)).copy()
    return PackedWeightMatrix(m=m, k=k, width=width, data=data, codebook=cb,
                              scales=_scales_from(blob, _WHDR.size, nd, nq, mode, gs, m, k))


def load_weights_device(path, codebook: Codebook | None = None, d: int | None = None,
                        device=None) -> PackedWeightMatrix:
    """MSGW file -> device-resident PackedWeightMatrix (data is a CUDA tensor).

    The packed payload is read into pinned memory and uploaded with one copy;
    if `d` is given, the fused kernels' weight layout (K3) is built right away
    so the first msgemm call does no re-layout.
    """
    t = _lib.torch()
    dev = device or _lib.require_device()
    blob = Path(path).read_bytes()
    m, k, width, mode, gs, nd, nq, cb = _parse_weight_header(blob, path, codebook)
    host = t.frombuffer(bytearray(blob[_WHDR.size:_WHDR.size + nd]), dtype=t.uint8)
    host = host.pin_memory() if host.numel() else host
    data = host.to(dev, non_blocking=True).reshape(m, bytes_per_row(k, width))
    pwm = PackedWeightMatrix(m=m, k=k, width=width, data=data, codebook=cb,
                             scales=_scales_from(blob, _WHDR.size, nd, nq, mode, gs, m, k))
    if d is not None and m and k >= d and width == 4:
        lib = _lib.lib()
        import ctypes
        lay, sym, ws = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _lib.check(lib.msg_gemm_plan(m, k, width, _lib.host_doubles(cb.values), _lib.F16, 1, d,
                                     0, 0, 0, ctypes.byref(lay), ctypes.byref(sym),
                                     ctypes.byref(ws)))
        if lay.value != _lib.LAYOUT_NONE:
            pwm.device_layout(dev, d, lay.value, sym.value)
    return pwm


def _write_matrix(path, magic, a) -> None:
    a = np.asarray(a)
    if a.ndim != 2:
        raise ValueError("expected a 2D matrix")
    with open(path, "wb") as f:
        f.write(_MHDR.pack(magic, VERSION, a.shape[0], a.shape[1]))
        f.write(np.asfortranarray(a, dtype="<f4").tobytes(order="F"))


def _read_matrix(path, magic) -> np.ndarray:
    blob = Path(path).read_bytes()
    if len(blob) < _MHDR.size:
        raise FormatError(f"{path}: truncated header")
    got, version, rows, cols = _MHDR.unpack_from(blob)
    if got != magic:
        raise FormatError(f"{path}: bad magic {got!r}, expected {magic!r}")
    if version != VERSION:
        raise FormatError(f"{path}: unsupported version {version}")
    want = _MHDR.size + 4 * rows * cols
    if len(blob) != want:
        raise FormatError(f"{path}: expected {want} bytes, found {len(blob)}")
    return np.frombuffer(blob, dtype="<f4", offset=_MHDR.size).reshape(
        (rows, cols), order="F").copy(order="F")


def write_activations(path, X) -> None:
    _write_matrix(path, MAGIC_A, X)


def read_activations(path) -> np.ndarray:
    return _read_matrix(path, MAGIC_A)


def write_output(path, Y) -> None:
    _write_matrix(path, MAGIC_Y, Y)


def read_output(path) -> np.ndarray:
    return _read_matrix(path, MAGIC_Y)
