"""ctypes binding of the C-ABI library (include/msgemm_b200.h).

This is the only module that touches the shared library.  It fails loudly:
there is no CPU fallback anywhere in the package -- if the library or a CUDA
device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
# MSG_LIB_VARIANT=debug selects the debug-checks build (tests/test_gpu_debug_build.py)
# (MSG_LIB_PATH: an explicit library file, for experiment builds)
LIB_PATH = Path(os.environ["MSG_LIB_PATH"]) if os.environ.get("MSG_LIB_PATH") else \
    _PKG / "_lib" / ("libmsgemm_b200_debug.so" if os.environ.get("MSG_LIB_VARIANT") == "debug"
                     else "libmsgemm_b200.so")

# status codes / enums mirrored from include/msgemm_b200.h
MSG_OK = 0
MSG_ERR_VALUE, MSG_ERR_INDEX, MSG_ERR_BUDGET = -1, -2, -3
MSG_ERR_UNSUPPORTED, MSG_ERR_CUDA, MSG_ERR_WORKSPACE = -4, -5, -6
F32, F16, F64, I32, I64, U8, I8, I16, BF16 = range(9)
SCALE_NONE, SCALE_PER_ROW, SCALE_PER_GROUP = 0, 1, 2
FLAG_F32_ENTRIES, FLAG_NO_SYMMETRY, FLAG_FORCE_GENERIC, FLAG_LUT_PHASE_ONLY = 1, 2, 4, 8
FLAG_NO_LANE = 16
FLAG_NO_ROWBLOCK = 32
FLAG_STATIC_WEIGHTS = 64
FLAG_RB_ROWS8, FLAG_RB_ROWS16 = 128, 256
LAYOUT_NONE, LAYOUT_QUAD, LAYOUT_LANE = 0, 1, 2
LAYOUT_RB4, LAYOUT_RB8, LAYOUT_RB16, LAYOUT_RB4S = 4, 5, 6, 7

EXPORTS = (
    "msg_last_error", "msg_version", "msg_device_sm_count", "msg_pack_codes",
    "msg_unpack_codes", "msg_group_indices", "msg_encode_values", "msg_lut_build",
    "msg_repacked_bytes", "msg_repack", "msg_gemm_plan", "msg_gemm",
    "msg_dequant_mma_workspace_bytes", "msg_dequant_mma",
    "msg_mma_layout_bytes", "msg_repack_mma", "msg_row_conditioning", "msg_copy_rows",
    "msg_naive_gemm", "msg_graph_run", "msg_stream_sync", "msg_dequant_gemv",
    "msg_dequant_hmma", "msg_gemm_fanout", "msg_stage_copy",
)

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_vp = ctypes.c_void_p
_SIGS = {
    "msg_last_error": (ctypes.c_char_p, []),
    "msg_version": (_c_int, []),
    "msg_device_sm_count": (_c_int, []),
    "msg_pack_codes": (_c_int, [_vp, _c_i64, _c_i64, _c_int, _vp, _vp]),
    "msg_unpack_codes": (_c_int, [_vp, _c_i64, _c_i64, _c_int, _vp, _vp]),
    "msg_group_indices": (_c_int, [_vp, _c_i64, _c_i64, _c_int, _c_int, _vp, _vp]),
    "msg_encode_values": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_int, _vp, _vp, _vp, _vp]),
    "msg_lut_build": (_c_int, [_vp, _c_int, _c_i64, _c_i64, _c_int, _vp, _c_int, _c_i64,
                               _c_i64, _vp, _vp]),
    "msg_repacked_bytes": (_c_i64, [_c_i64, _c_i64, _c_int, _c_int]),
    "msg_repack": (_c_int, [_vp, _c_i64, _c_i64, _c_int, _c_int, _c_int, _vp, _vp]),
    "msg_gemm_plan": (_c_int, [_c_i64, _c_i64, _c_int, _vp, _c_int, _c_i64, _c_int, _c_int,
                               _c_i64, _c_int, _vp, _vp, _vp]),
    "msg_gemm": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_int, _vp, _vp, _c_int, _c_i64, _c_int,
                          _c_int, _c_i64, _vp, _c_int, _vp, _c_int, _vp, _c_i64, _c_int, _vp]),
    "msg_gemm_fanout": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_int, _vp, _vp, _c_int, _c_i64, _c_int,
                                 _c_int, _c_i64, _vp, _c_int, _vp, _c_int, _vp, _c_i64, _c_int, _vp,
                                 _vp, _c_int]),
    "msg_dequant_mma_workspace_bytes": (_c_i64, [_c_i64, _c_i64, _c_i64]),
    "msg_dequant_mma": (_c_int, [_vp, _c_i64, _c_i64, _vp, _vp, _c_int, _c_i64, _vp, _c_int,
                                 _vp, _c_i64, _vp]),
    "msg_mma_layout_bytes": (_c_i64, [_c_i64, _c_i64]),
    "msg_repack_mma": (_c_int, [_vp, _c_i64, _c_i64, _vp, _vp, _vp]),
    "msg_row_conditioning": (_c_int, [_vp, _c_i64, _c_i64, _c_int, _vp, ctypes.c_double, _vp,
                                      _vp]),
    "msg_copy_rows": (_c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _c_int, _vp]),
    "msg_naive_gemm": (_c_int, [_vp, _c_int, _vp, _c_int, _c_i64, _c_i64, _c_i64, _c_int, _vp,
                                _vp]),
    "msg_graph_run": (_c_int, [_vp, _vp, _c_int]),
    "msg_dequant_gemv": (_c_int, [_vp, _c_i64, _c_i64, _vp, _vp, _c_int, _c_i64, _vp, _c_int, _vp]),
    "msg_dequant_hmma": (_c_int, [_vp, _c_i64, _c_i64, _vp, _vp, _c_int, _c_i64, _vp, _c_int, _vp]),
    "msg_stage_copy": (_c_int, [_vp, _vp, _c_i64, _vp]),
    "msg_stream_sync": (_c_int, [_vp]),
}

_lib = None
_lock = threading.Lock()


class TableBudgetError(MemoryError):
    """The requested lookup table does not fit in the memory budget (lut.py:30-31)."""


def load_library(path: Path | None = None) -> ctypes.CDLL:
    """Load (once) and type the C-ABI library.  Raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"msgemm_b200 CUDA library not built ({p}); run "
                "`python -m paper_2310_06178_b200.build` -- there is no CPU fallback")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load_library()


def check(status: int) -> None:
    if status == MSG_OK:
        return
    msg = lib().msg_last_error().decode(errors="replace")
    if status == MSG_ERR_VALUE or status == MSG_ERR_WORKSPACE:
        raise ValueError(msg)
    if status == MSG_ERR_INDEX:
        raise IndexError(msg)
    if status == MSG_ERR_BUDGET:
        raise TableBudgetError(msg)
    if status == MSG_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"msgemm_b200 CUDA error: {msg}")


# --------------------------------------------------------------------------
# torch / device plumbing
# --------------------------------------------------------------------------

_torch = None
_Tensor = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    return _torch


_dev_ok = False
_devs = {}


def require_device():
    """The CUDA device this call runs on; raise loudly if there is none."""
    global _dev_ok
    t = torch()
    if not _dev_ok:
        if not t.cuda.is_available():
            raise RuntimeError("msgemm_b200 needs a CUDA device (B200, sm_100a); "
                               "there is no CPU fallback")
        lib()
        _dev_ok = True
    i = t.cuda.current_device()
    d = _devs.get(i)
    if d is None:
        d = _devs[i] = t.device("cuda", i)
    return d


def current_stream_handle(dev) -> int:
    """Raw cudaStream_t of the current stream on `dev` (an int).  Uses torch's
    raw-stream query when available (~10x cheaper than building a Stream)."""
    t = torch()
    get_raw = getattr(t._C, "_cuda_getCurrentRawStream", None)
    if get_raw is not None:
        return int(get_raw(dev.index))
    return int(t.cuda.current_stream(dev).cuda_stream)


def stream_ptr():
    return ctypes.c_void_p(torch().cuda.current_stream().cuda_stream)


def layout_ready() -> None:
    """A cached weight layout was just written on the current stream: wait for
    it once, so calls on any other stream (plans are per stream) never read a
    partial layout.  Skipped while a CUDA graph is being captured (the capture
    stream is the only stream then)."""
    t = torch()
    if not t.cuda.is_current_stream_capturing():
        t.cuda.current_stream().synchronize()


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def host_doubles(values) -> ctypes.Array:
    vals = [float(v) for v in values]
    return (ctypes.c_double * len(vals))(*vals)


_NP2CODE = {
    np.dtype(np.float32): F32, np.dtype(np.float16): F16, np.dtype(np.float64): F64,
    np.dtype(np.int32): I32, np.dtype(np.int64): I64, np.dtype(np.uint8): U8,
    np.dtype(np.int8): I8, np.dtype(np.int16): I16,
}


_T2CODE = None


def dtype_code(dt) -> int:
    """MSG_* element code of a numpy or torch dtype."""
    global _T2CODE
    t = torch()
    if isinstance(dt, t.dtype):
        if _T2CODE is None:
            _T2CODE = {t.float32: F32, t.float16: F16, t.float64: F64, t.int32: I32, t.int64: I64,
                       t.uint8: U8, t.int8: I8, t.int16: I16, t.bfloat16: BF16}
        if dt not in _T2CODE:
            raise NotImplementedError(f"dtype {dt} is not supported on the GPU path")
        return _T2CODE[dt]
    nd = np.dtype(dt)
    if nd not in _NP2CODE:
        raise NotImplementedError(f"dtype {nd} is not supported on the GPU path")
    return _NP2CODE[nd]


def torch_dtype_of(np_dtype):
    t = torch()
    return {np.dtype(np.float32): t.float32, np.dtype(np.float16): t.float16,
            np.dtype(np.float64): t.float64, np.dtype(np.int32): t.int32,
            np.dtype(np.int64): t.int64, np.dtype(np.uint8): t.uint8,
            np.dtype(np.int8): t.int8, np.dtype(np.int16): t.int16}[np.dtype(np_dtype)]


def is_torch(x) -> bool:
    global _Tensor
    if _Tensor is None:
        try:
            _Tensor = torch().Tensor
        except Exception:  # pragma: no cover
            return False
    return isinstance(x, _Tensor)


def to_device(x, dev, non_blocking: bool = False):
    """Contiguous device tensor view/copy of a numpy array or tensor."""
    t = torch()
    if is_torch(x):
        return x.to(dev, non_blocking=non_blocking).contiguous()
    a = np.ascontiguousarray(x)
    return t.from_numpy(a).to(dev, non_blocking=False)


_ws = {}


def workspace(nbytes: int, dev, kind: str = "scratch"):
    """Per-(device, stream, kind) scratch buffer, grown on demand, never freed on
    the hot path.  kind "lane": the b=1 kernel's self-cleaning accumulators
    (zero-filled here, left zero by every call), kept apart from the scratch
    the other kernels overwrite."""
    t = torch()
    key = (dev.index, t.cuda.current_stream(dev).cuda_stream, kind)
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = t.zeros(max(int(nbytes), 256), dtype=t.uint8, device=dev)
        _ws[key] = buf
    return buf


def reset_workspaces():
    """Zero the self-cleaning "lane" workspaces (needed only after LUT-phase-only
    measurement launches, which leave their row sums behind)."""
    for key, buf in _ws.items():
        if key[2] == "lane":
            buf.zero_()
