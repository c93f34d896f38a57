"""Phase 1: look-up tables of all depth-d combinations (mirror of reference lut.py).

``build_lut`` / ``build_lut_block`` / ``block_entries`` build the table on
the GPU (msg_lut_build) with the reference's rounding order
(lut.py:59-72), so the entries are bit-identical to the reference's for
every activation dtype.  Inside ``msgemm`` the tables are never
materialised in HBM: the fused kernel builds them straight into shared
memory (see csrc/msg_fused.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import TableBudgetError
from .codebook import Codebook

#: default cap on materialized table size, in bytes (lut.py:23)
DEFAULT_BUDGET = 1 << 30

#: materialized tables are capped at this depth (lut.py:27)
MAX_MATERIALIZED_DEPTH = 4

__all__ = ["DEFAULT_BUDGET", "MAX_MATERIALIZED_DEPTH", "TableBudgetError", "LookupTable",
           "block_entries", "block_nbytes", "build_lut", "build_lut_block"]


@dataclass(frozen=True)
class LookupTable:
    """Block-major table: entries[j, idx] is the combination for block j (lut.py:34-41)."""

    d: int
    width: int
    num_blocks: int
    entries: object  # (num_blocks, 2**(width*d)), numpy or CUDA tensor


def _check_depth(cb: Codebook, d: int) -> None:
    """lut.py:75-81."""
    if d < 1:
        raise ValueError("depth d must be >= 1")
    if d > MAX_MATERIALIZED_DEPTH:
        raise ValueError(
            f"materialized tables are capped at depth {MAX_MATERIALIZED_DEPTH}, got {d}")


def block_nbytes(cb: Codebook, d: int, dtype) -> int:
    """lut.py:84-85."""
    return 2 ** (cb.width * d) * np.dtype(dtype).itemsize


def _itemsize(x) -> int:
    return x.element_size() if _lib.is_torch(x) else x.dtype.itemsize


def _device_table(xd, cb: Codebook, d: int, k: int, lo: int, hi: int):
    """Entries for blocks [lo, hi) of the contiguous device vector xd (k,)."""
    t = _lib.torch()
    n = 2 ** (cb.width * d)
    out = t.empty((hi - lo, n), dtype=xd.dtype, device=xd.device)
    if hi > lo:
        _lib.check(_lib.lib().msg_lut_build(
            _lib.ptr(xd), _lib.dtype_code(xd.dtype), k, 1, d, _lib.host_doubles(cb.values),
            cb.width, lo, hi, _lib.ptr(out), _lib.stream_ptr()))
    return out


def _as_vector_on_device(x, dev):
    t = _lib.torch()
    xd = _lib.to_device(x, dev)
    return xd.reshape(-1) if xd.dim() else xd


def block_entries(xb, cb: Codebook):
    """Entries for blocks given as an (nb, d) slice -> (nb, 2**(width*d)) (lut.py:59-72)."""
    on_device = _lib.is_torch(xb)
    a = xb if on_device else np.asarray(xb)
    nb, d = (int(s) for s in a.shape)
    dev = _lib.require_device()
    xd = _as_vector_on_device(a, dev)
    out = _device_table(xd, cb, d, nb * d, 0, nb)
    return out if on_device else out.cpu().numpy()


def build_lut_block(x, cb: Codebook, d: int, j: int):
    """Block j of the table (lut.py:88-95)."""
    on_device = _lib.is_torch(x)
    a = x if on_device else np.asarray(x)
    _check_depth(cb, d)
    nb = int(a.shape[0]) // d
    if not 0 <= j < nb:
        raise IndexError(f"block {j} out of range; k={a.shape[0]}, d={d} gives {nb} blocks")
    dev = _lib.require_device()
    xd = _as_vector_on_device(a[j * d:(j + 1) * d], dev)
    out = _device_table(xd, cb, d, d, 0, 1)[0]
    return out if on_device else out.cpu().numpy()


def build_lut(x, cb: Codebook, d: int, budget: int = DEFAULT_BUDGET,
              workers: int = 1) -> LookupTable:
    """Materialize the full table for activation vector x (lut.py:98-127).

    ``workers`` is accepted for signature compatibility; the GPU builds every
    block in one launch and the result does not depend on it.
    """
    on_device = _lib.is_torch(x)
    a = x if on_device else np.asarray(x)
    if a.ndim != 1:
        raise ValueError("x must be a 1D activation vector")
    _check_depth(cb, d)
    k = int(a.shape[0])
    nb = k // d
    nbytes = 2 ** (cb.width * d) * nb * _itemsize(a)
    if nbytes > budget:
        raise TableBudgetError(f"table of {nbytes} bytes exceeds budget of {budget} bytes")
    dev = _lib.require_device()
    xd = _as_vector_on_device(a, dev)
    out = _device_table(xd, cb, d, k, 0, nb)
    entries = out if on_device else out.cpu().numpy()
    return LookupTable(d=d, width=cb.width, num_blocks=nb, entries=entries)
