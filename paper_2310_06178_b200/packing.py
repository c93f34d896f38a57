"""Packed int4 weight storage (mirror of reference packing.py:21-228).

The host-facing data model is the reference's: ``PackedWeightMatrix.data`` is
the row-major nibble array (column j in byte j//2, even j in the low nibble,
packing.py:99-114), so files and arrays are bit-compatible with the
reference.  The byte work -- packing, unpacking, value encoding, group-index
formation -- runs on the GPU through the C ABI (msg_pack_codes,
msg_unpack_codes, msg_encode_values, msg_group_indices).  Each matrix keeps a
cache of its device copy and of the repacked device layouts (K3) the fused
kernels read, so a weight is uploaded and repacked once.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .codebook import Codebook


@dataclass(frozen=True)
class PerRow:
    """One shared scale per row (packing.py:21-26)."""

    q: np.ndarray  # (m,)


@dataclass(frozen=True)
class PerGroup:
    """One shared scale per group of group_size consecutive columns (packing.py:29-34)."""

    group_size: int
    q: np.ndarray  # (m, k // group_size)


ScaleSpec = PerRow | PerGroup | None


def bytes_per_row(k: int, width: int) -> int:
    """packing.py:39-47."""
    if width == 4:
        return (k + 1) // 2
    if width == 2:
        return (k + 3) // 4
    return k


@dataclass(frozen=True)
class PackedWeightMatrix:
    """m x k packed codes with optional scales (packing.py:50-69).

    ``data`` may be a numpy array (host, reference-compatible) or a CUDA
    tensor (device-resident weights for serving); both have the reference's
    shape (m, bytes_per_row(k, width)) and dtype uint8.
    """

    m: int
    k: int
    width: int
    data: object
    codebook: Codebook
    scales: ScaleSpec = None

    def __post_init__(self) -> None:
        if self.m < 0 or self.k < 0:
            raise ValueError("matrix dimensions must be non-negative")
        if self.width != self.codebook.width:
            raise ValueError("width does not match codebook width")
        want = (self.m, bytes_per_row(self.k, self.width))
        if tuple(self.data.shape) != want:
            raise ValueError(f"packed data shape {tuple(self.data.shape)} != expected {want}")
        _validate_scales(self.scales, self.m, self.k)
        object.__setattr__(self, "_device_cache", {})

    # ---- device-side caches (not part of the reference surface) ----
    def device_data(self, dev):
        """The packed bytes on `dev` (uploaded once)."""
        cache = self._device_cache
        key = ("data", dev.index)
        if key not in cache:
            cache[key] = _lib.to_device(self.data, dev)
        return cache[key]

    def has_device_layout(self, dev, d: int, layout: int, symmetric: int) -> bool:
        """True once device_layout(...) has been built (by an earlier call)."""
        return ("layout", dev.index, d, layout, symmetric) in self._device_cache

    def device_layout(self, dev, d: int, layout: int, symmetric: int):
        """The K3-repacked layout for depth d on `dev` (built once)."""
        cache = self._device_cache
        key = ("layout", dev.index, d, layout, symmetric)
        if key not in cache:
            t = _lib.torch()
            nbytes = _lib.lib().msg_repacked_bytes(self.m, self.k, d, layout)
            if nbytes < 0:
                raise NotImplementedError(f"layout {layout} unsupported for d={d}")
            out = t.empty(max(int(nbytes), 1), dtype=t.uint8, device=dev)
            _lib.check(_lib.lib().msg_repack(
                _lib.ptr(self.device_data(dev)), self.m, self.k, d, layout, symmetric,
                _lib.ptr(out), _lib.stream_ptr()))
            _lib.layout_ready()
            cache[key] = out
        return cache[key]

    def device_mma_layout(self, dev):
        """The tensor-core tile layout of W (K4 comparison kernel), built once."""
        cache = self._device_cache
        key = ("mma", dev.index)
        if key not in cache:
            t = _lib.torch()
            nbytes = _lib.lib().msg_mma_layout_bytes(self.m, self.k)
            out = t.empty(max(int(nbytes), 1), dtype=t.uint8, device=dev)
            _lib.check(_lib.lib().msg_repack_mma(
                _lib.ptr(self.device_data(dev)), self.m, self.k,
                _lib.host_doubles(self.codebook.values), _lib.ptr(out), _lib.stream_ptr()))
            _lib.layout_ready()
            cache[key] = out
        return cache[key]

    def symmetric_conditioning(self, dev, d: int, beta: float):
        """Per-row conditioning ratio of the sign-symmetric tables (device
        float32 (m,), built once; csrc msg_row_conditioning): the expected
        half-table rounding error relative to the reference's tolerance bound
        sum_c |W_ic||x_c| (suites.py:106-124) at unit activations, +inf for
        rows without a nonzero weight."""
        cache = self._device_cache
        key = ("cond", dev.index, d, float(beta))
        if key not in cache:
            t = _lib.torch()
            out = t.empty(max(self.m, 1), dtype=t.float32, device=dev)
            _lib.check(_lib.lib().msg_row_conditioning(
                _lib.ptr(self.device_data(dev)), self.m, self.k, d,
                _lib.host_doubles(self.codebook.values), float(beta), _lib.ptr(out),
                _lib.stream_ptr()))
            cache[key] = out[: self.m]
        return cache[key]

    def ill_conditioned_rows(self, dev, d: int, beta: float, threshold: float):
        """Device int64 indices of the rows whose symmetric-table error could
        reach the tolerance (conditioning ratio above `threshold`), built once
        per threshold.  One host sync, at weight-preparation time."""
        cache = self._device_cache
        key = ("illrows", dev.index, d, float(beta), float(threshold))
        if key not in cache:
            t = _lib.torch()
            ratio = self.symmetric_conditioning(dev, d, beta)
            cache[key] = t.nonzero(ratio > threshold).reshape(-1).to(t.int64)
        return cache[key]

    def row_subset(self, dev, rows) -> "PackedWeightMatrix":
        """Device-resident matrix of the given rows (same k, codebook and the
        matching scale rows), gathered by msg_copy_rows; cached per row set."""
        cache = self._device_cache
        key = ("subset", dev.index, rows.data_ptr(), int(rows.numel()))
        if key not in cache:
            t = _lib.torch()
            n = int(rows.numel())
            src = self.device_data(dev)
            data = t.empty((n, src.shape[1]), dtype=t.uint8, device=dev)
            _lib.check(_lib.lib().msg_copy_rows(_lib.ptr(src), _lib.ptr(rows), n, int(src.shape[1]),
                                                _lib.ptr(data), 0, _lib.stream_ptr()))
            scales = None
            q = self.device_scales(dev)
            if q is not None:
                qd = q.contiguous()
                per = qd.numel() // max(self.m, 1)
                qs = t.empty((n, per) if qd.dim() == 2 else (n,), dtype=qd.dtype, device=dev)
                _lib.check(_lib.lib().msg_copy_rows(_lib.ptr(qd), _lib.ptr(rows), n,
                                                    per * qd.element_size(), _lib.ptr(qs), 0,
                                                    _lib.stream_ptr()))
                scales = (PerRow(q=qs) if isinstance(self.scales, PerRow)
                          else PerGroup(group_size=self.scales.group_size, q=qs))
            sub = PackedWeightMatrix(m=n, k=self.k, width=self.width, data=data,
                                     codebook=self.codebook, scales=scales)
            cache[key] = sub
        return cache[key]

    def device_scales(self, dev):
        cache = self._device_cache
        key = ("q", dev.index)
        if key not in cache:
            cache[key] = None if self.scales is None else _lib.to_device(self.scales.q, dev)
        return cache[key]


def _validate_scales(scales: ScaleSpec, m: int, k: int) -> None:
    """packing.py:72-87."""
    if scales is None:
        return
    if isinstance(scales, PerRow):
        shape = tuple(np.shape(scales.q))
        if shape != (m,):
            raise ValueError(f"PerRow scales must have shape ({m},), got {shape}")
    elif isinstance(scales, PerGroup):
        r = scales.group_size
        if r <= 0 or k % r != 0:
            raise ValueError(f"group_size {r} must be positive and divide k={k}")
        shape = tuple(np.shape(scales.q))
        if shape != (m, k // r):
            raise ValueError(f"PerGroup scales must have shape ({m}, {k // r}), got {shape}")
    else:
        raise TypeError(f"unsupported scale spec: {scales!r}")


def scale_grid(scales: ScaleSpec, m: int, k: int):
    """Per-element scale factors (m, k) or None (packing.py:90-96)."""
    if scales is None:
        return None
    q = np.asarray(scales.q)
    if isinstance(scales, PerRow):
        return np.broadcast_to(q[:, None], (m, k))
    return np.repeat(q, scales.group_size, axis=1)


def _host(arr):
    return arr.detach().cpu().numpy() if _lib.is_torch(arr) else arr


def _host_row(arr, i):
    """Row i on the host (a device matrix copies only that row)."""
    return arr[i].detach().cpu().numpy() if _lib.is_torch(arr) else arr[i]


def from_codes(codes, cb: Codebook, scales: ScaleSpec = None) -> PackedWeightMatrix:
    """Pack raw codes (packing.py:131-143), on the GPU (msg_pack_codes)."""
    on_device = _lib.is_torch(codes)
    c = codes if on_device else np.asarray(codes)
    if c.ndim != 2:
        raise ValueError("codes must be a 2D grid")
    if c.numel() if on_device else c.size:
        lo, hi = (int(c.min()), int(c.max()))
        if lo < 0 or hi >= cb.num_codes:
            raise ValueError("codes out of range for codebook width")
    m, k = (int(s) for s in c.shape)
    dev = _lib.require_device()
    t = _lib.torch()
    dc = _lib.to_device(c if on_device else np.ascontiguousarray(c, dtype=np.uint8), dev)
    if dc.dtype != t.uint8:
        dc = dc.to(t.uint8)
    out = t.empty((m, bytes_per_row(k, cb.width)), dtype=t.uint8, device=dev)
    _lib.check(_lib.lib().msg_pack_codes(_lib.ptr(dc), m, k, cb.width, _lib.ptr(out),
                                         _lib.stream_ptr()))
    data = out if on_device else out.cpu().numpy()
    pwm = PackedWeightMatrix(m=m, k=k, width=cb.width, data=data, codebook=cb, scales=scales)
    pwm._device_cache[("data", dev.index)] = out
    return pwm


def pack(weights, cb: Codebook, scales: ScaleSpec = None) -> PackedWeightMatrix:
    """Encode values to their nearest codebook codes (packing.py:146-169), on the GPU."""
    w = np.asarray(_host(weights))
    if w.ndim != 2:
        raise ValueError("weights must be a 2D grid")
    m, k = w.shape
    _validate_scales(scales, m, k)
    dev = _lib.require_device()
    t = _lib.torch()
    dw = t.from_numpy(np.ascontiguousarray(w, dtype=np.float64)).to(dev)
    grid = scale_grid(scales, m, k)
    dg = None if grid is None else t.from_numpy(np.ascontiguousarray(grid, dtype=np.float64)).to(dev)
    out = t.empty((m, bytes_per_row(k, cb.width)), dtype=t.uint8, device=dev)
    bad = t.empty(2, dtype=t.int64, device=dev)
    vals = _lib.host_doubles(cb.values)
    _lib.check(_lib.lib().msg_encode_values(_lib.ptr(dw), _lib.ptr(dg), m, k, cb.width, vals,
                                            _lib.ptr(out), _lib.ptr(bad), _lib.stream_ptr()))
    nbad, first = (int(v) for v in bad.cpu().tolist())
    if nbad:
        flat = (w / grid if grid is not None else w).astype(np.float64).reshape(-1)
        raise ValueError(f"weight {flat[first]!r} is not representable in the codebook")
    pwm = PackedWeightMatrix(m=m, k=k, width=cb.width, data=out.cpu().numpy(), codebook=cb,
                             scales=scales)
    pwm._device_cache[("data", dev.index)] = out
    return pwm


def _device_codes(pwm: PackedWeightMatrix, dev):
    t = _lib.torch()
    out = t.empty((pwm.m, pwm.k), dtype=t.uint8, device=dev)
    if pwm.m * pwm.k:
        _lib.check(_lib.lib().msg_unpack_codes(_lib.ptr(pwm.device_data(dev)), pwm.m, pwm.k,
                                               pwm.width, _lib.ptr(out), _lib.stream_ptr()))
    return out


def codes(pwm: PackedWeightMatrix):
    """All stored codes (m, k) uint8 (packing.py:172-174)."""
    dev = _lib.require_device()
    out = _device_codes(pwm, dev)
    return out if _lib.is_torch(pwm.data) else out.cpu().numpy()


def unpack(pwm: PackedWeightMatrix, i: int, j: int):
    """Decoded value at (i, j), scale NOT applied (packing.py:177-188)."""
    if not (0 <= i < pwm.m and 0 <= j < pwm.k):
        raise IndexError(f"({i}, {j}) out of bounds for {pwm.m}x{pwm.k}")
    row = _host_row(pwm.data, i)
    if pwm.width == 4:
        code = (int(row[j // 2]) >> (4 * (j % 2))) & 0xF
    elif pwm.width == 2:
        code = (int(row[j // 4]) >> (2 * (j % 4))) & 0x3
    else:
        code = int(row[j])
    return pwm.codebook.decode(code)


def dense(pwm: PackedWeightMatrix, apply_scales: bool = False) -> np.ndarray:
    """Decoded (m, k) weights, optionally scaled (packing.py:191-198).

    Codes are unpacked on the GPU; the value lookup and scale product keep
    numpy's dtype rules so the result is identical to the reference's.
    """
    c = codes(pwm)
    c = _host(c)
    w = pwm.codebook.value_array[c]
    if apply_scales:
        grid = scale_grid(pwm.scales, pwm.m, pwm.k)
        if grid is not None:
            w = w * grid
    return w


def group_index(pwm: PackedWeightMatrix, i: int, j: int, d: int) -> int:
    """Table index of block j of row i (packing.py:201-216)."""
    if d < 1:
        raise ValueError("depth d must be >= 1")
    if d * pwm.width > 32:
        raise ValueError(f"d*width = {d * pwm.width} exceeds 32-bit index limit")
    if not 0 <= i < pwm.m:
        raise IndexError(f"row {i} out of bounds")
    if not 0 <= j < pwm.k // d:
        raise IndexError(f"block {j} out of bounds for k={pwm.k}, d={d}")
    idx = 0
    row = _host_row(pwm.data, i)
    for r in range(d):
        col = j * d + r
        if pwm.width == 4:
            code = (int(row[col // 2]) >> (4 * (col % 2))) & 0xF
        elif pwm.width == 2:
            code = (int(row[col // 4]) >> (2 * (col % 4))) & 0x3
        else:
            code = int(row[col])
        idx |= code << (pwm.width * r)
    return idx


def group_indices(pwm: PackedWeightMatrix, d: int):
    """int64 (m, k // d) table indices, formed on the GPU (packing.py:219-228)."""
    if d < 1:
        raise ValueError("depth d must be >= 1")
    if d * pwm.width > 32:
        raise ValueError(f"d*width = {d * pwm.width} exceeds 32-bit index limit")
    dev = _lib.require_device()
    t = _lib.torch()
    nb = pwm.k // d
    out = t.empty((pwm.m, nb), dtype=t.int64, device=dev)
    if pwm.m * nb:
        _lib.check(_lib.lib().msg_group_indices(_lib.ptr(pwm.device_data(dev)), pwm.m, pwm.k,
                                                pwm.width, d, _lib.ptr(out), _lib.stream_ptr()))
    return out if _lib.is_torch(pwm.data) else out.cpu().numpy()
