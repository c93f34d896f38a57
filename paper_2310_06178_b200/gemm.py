"""Phase 2: msGeMM on the GPU (mirror of reference gemm.py:24-231).

``msgemm`` keeps the reference's signature, validation order, output
dtype/shape and error types (gemm.py:89-153) and runs the CUDA path:

* widths 4, float16/float32 activations, d <= 3, no per-group scales: the
  fused kernel (K3 repack once per weight, then one launch that builds the
  tables in shared memory and gathers, plus a deterministic reduction);
* everything else the reference accepts (d up to 7, widths 2..8, int/f64
  activations, per-group scales): the generic global-memory-table kernels.

Numpy inputs give numpy outputs (the drop-in contract); CUDA tensors give
CUDA tensors with no host round trip.  There is no CPU fallback.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import TableBudgetError
from .lut import DEFAULT_BUDGET, block_nbytes, build_lut
from .codebook import Codebook
from .packing import PackedWeightMatrix, PerGroup, PerRow, group_indices

__all__ = ["OpCount", "msgemm", "msgemm_counted", "msgemm_traced", "naive_gemm",
           "naive_gemm_counted", "dequant_gemm"]


@dataclass(frozen=True)
class OpCount:
    """Arithmetic / memory-access counts for one execution (gemm.py:24-47)."""

    fma: int = 0
    add: int = 0
    mul: int = 0
    mem_weights: int = 0
    mem_activations: int = 0

    def __add__(self, other: "OpCount") -> "OpCount":
        return OpCount(self.fma + other.fma, self.add + other.add, self.mul + other.mul,
                       self.mem_weights + other.mem_weights,
                       self.mem_activations + other.mem_activations)


def _as_matrix(X, is_tensor=None):
    """(k, b) view of X and whether X was a vector (gemm.py:50-57)."""
    if _lib.is_torch(X) if is_tensor is None else is_tensor:
        if X.dim() == 1:
            return X[:, None], True
        if X.dim() != 2:
            raise ValueError("activations must be a vector or a (k, b) matrix")
        return X, False
    X = np.asarray(X)
    if X.ndim == 1:
        return X[:, None], True
    if X.ndim != 2:
        raise ValueError("activations must be a vector or a (k, b) matrix")
    return X, False


def _check_scales_for_depth(pwm, d: int) -> None:
    """gemm.py:60-67."""
    if isinstance(pwm.scales, PerGroup):
        r = pwm.scales.group_size
        if r < d or r % d != 0:
            raise ValueError(f"per-group scaling needs group_size >= d and divisible by d; "
                             f"got group_size={r}, d={d}")


_T2NP = None
_HOST_Y_DIRECT = __import__("os").environ.get("MSG_HOST_Y", "direct") != "copy"
# host X -> device staging inside the replayed graph: a copy kernel
# (msg_stage_copy) instead of a memcpy node, so the LUT kernel behind it starts
# under PDL and prefetches weights while X crosses PCIe (bench.py e2e: cfg4
# b = 1 40.9 -> 27.5 us, cfg2 32.5 -> 23.8 us, cfg5 255 -> 247 us).
# MSG_HOST_X=memcpy forces the copy node (A/B).
_HOST_X_KERNEL = __import__("os").environ.get("MSG_HOST_X", "kernel") != "memcpy"



def _np_dtype(X):
    global _T2NP
    if _lib.is_torch(X):
        if _T2NP is None:
            t = _lib.torch()
            _T2NP = {t.float32: np.float32, t.float16: np.float16, t.float64: np.float64,
                     t.int32: np.int32, t.int64: np.int64, t.uint8: np.uint8, t.int8: np.int8,
                     t.int16: np.int16}
        return _T2NP.get(X.dtype, None)
    return X.dtype


_FOREIGN = {}   # id(foreign pwm) -> (weakref to it, our wrapper, its scales, its codebook)


def _ensure_device_pwm(pwm):
    """Accept our PackedWeightMatrix or any duck-typed equivalent (e.g. the
    reference's).  A foreign object is wrapped once and the wrapper (with its
    device copies, layouts and call plans) reused while the object lives and
    still holds the same arrays, so a reference user's repeated calls do not
    repack the weights every time."""
    if isinstance(pwm, PackedWeightMatrix):
        return pwm
    ent = _FOREIGN.get(id(pwm))
    if ent is not None:
        ref, ours = ent[0], ent[1]
        if ref() is pwm and ours.data is pwm.data and ent[2] is pwm.scales and ent[3] is pwm.codebook:
            return ours
    cb = pwm.codebook
    if not isinstance(cb, Codebook):       # the reference's Codebook: same fields
        cb = Codebook(width=int(cb.width), values=tuple(cb.values))
    sc = pwm.scales
    if sc is not None and not isinstance(sc, (PerRow, PerGroup)):
        sc = (PerGroup(group_size=int(sc.group_size), q=sc.q) if hasattr(sc, "group_size")
              else PerRow(q=sc.q))
    ours = PackedWeightMatrix(m=pwm.m, k=pwm.k, width=pwm.width, data=pwm.data,
                              codebook=cb, scales=sc)
    try:
        import weakref
        key = id(pwm)
        ref = weakref.ref(pwm, lambda _r, key=key: _FOREIGN.pop(key, None))
        _FOREIGN[key] = (ref, ours, pwm.scales, pwm.codebook)
    except TypeError:        # not weak-referenceable: no caching
        pass
    return ours


def msgemm(pwm: PackedWeightMatrix, X, d: int, budget: int = DEFAULT_BUDGET,
           workers: int = 1, *, table_dtype=None, symmetric: bool = True,
           out_dtype=None, out=None, _flags: int = 0, _fan=None):
    """Two-phase GeMM Y = W @ X on the GPU (gemm.py:89-153).

    Returns (m, b), or (m,) for a vector X, in X's dtype.  ``budget`` keeps
    the reference's TableBudgetError contract (a single table block larger
    than the budget); ``workers`` is accepted and ignored (results never
    depend on it).  Keyword-only extensions:

    table_dtype: None (tables in X's dtype, as the reference) or
        "float32" (fp32 tables for fp16 X -- exact for integer-valued X).
    symmetric: use sign-symmetric half tables when the codebook allows.
    out_dtype: None (Y in X's dtype, as the reference) or a float dtype,
        e.g. float32 Y from fp16 X (the bit-exact integer check).
    out: optional preallocated CUDA tensor for Y (torch inputs only).
    _fan: device addresses (ints, at most 7) of the same Y region in other
        ranks' buffers (mapped peer memory): the finishing kernels store Y
        there as well (sharded.msgemm_sharded_fused).  Needs a CUDA ``out``.
    """
    # repeated host-path calls with the same X / out objects (a serving loop
    # reusing its pinned buffers): validation and plan lookup were done on
    # the first call; only the buffers' identity, shape and stream are checked
    fast = getattr(pwm, "_device_cache", None)
    if fast is None and id(pwm) in _FOREIGN:           # a wrapped reference-typed object
        fent = _FOREIGN[id(pwm)]
        if fent[0]() is pwm:
            fast = fent[1]._device_cache
    if fast is not None:
        ent = fast.get(("fast", id(X), id(out), d, budget, table_dtype, symmetric, out_dtype, _flags))
        if ent is not None:
            res = ent(X, out)
            if res is not None:
                return res
    pwm = _ensure_device_pwm(pwm)
    is_tensor = _lib.is_torch(X)
    Xm, was_vector = _as_matrix(X, is_tensor)
    if int(Xm.shape[0]) != pwm.k:
        raise ValueError(f"activation rows {Xm.shape[0]} != weight columns {pwm.k}")
    if d < 1:
        raise ValueError("depth d must be >= 1")
    _check_scales_for_depth(pwm, d)
    if d * pwm.width > 32:  # group_indices check, gemm.py:107 -> packing.py:221-224
        raise ValueError(f"d*width = {d * pwm.width} exceeds 32-bit index limit")
    itemsize = Xm.element_size() if is_tensor else Xm.dtype.itemsize
    if 2 ** (pwm.width * d) * itemsize > budget:
        raise TableBudgetError("a single table block exceeds the memory budget")

    dev = _lib.require_device()
    t = _lib.torch()
    m, k, b = pwm.m, pwm.k, int(Xm.shape[1])
    x_code = _lib.dtype_code(Xm.dtype)
    on_device = is_tensor and X.is_cuda
    stream = _lib.current_stream_handle(dev)
    call = _call_plan(pwm, dev, stream, b, x_code, Xm.dtype, d, table_dtype, symmetric,
                      out_dtype, int(_flags))
    y_dt = call.y_dtype
    host_out = dev_out = None
    if out is not None:
        shapes = ((m, b), (m,)) if was_vector else ((m, b),)
        if (not _lib.is_torch(out) or out.shape not in shapes or out.dtype != y_dt
                or not out.is_contiguous()):
            raise ValueError("out must be a contiguous tensor of Y's dtype and shape "
                             + ("(m,) or (m, 1)" if was_vector else "(m, b)"))
        if out.is_cuda:
            if out.device != dev:
                raise ValueError(f"out is on {out.device}, the call runs on {dev}")
            dev_out = out
        else:
            host_out = out
    if _fan:
        if dev_out is None or not on_device:
            raise ValueError("_fan needs CUDA activations and a CUDA out")
        if len(_fan) > 7:
            raise ValueError("at most 7 peer buffers")
    if on_device and host_out is None:  # device in, device out: no staging involved
        xd = call.device_x(Xm)
        Y = dev_out if dev_out is not None else t.empty((m, b), dtype=y_dt, device=dev)
        if m and b:
            call.launch(xd, Y, fan=_fan)
        return Y[:, 0] if (was_vector and dev_out is None) else Y
    # host activations and/or host output: the plan's pinned + device staging
    # buffers are shared by calls on this stream, so one call uses them at a time
    if not on_device and dev_out is None and m and b:
        res = _host_call(call, Xm, host_out, stream, is_tensor, was_vector)
        _register_fast(pwm, X, out, (d, budget, table_dtype, symmetric, out_dtype, _flags), call,
                       stream, dev, is_tensor, was_vector)
        return res
    with call.lock:
        xd = call.device_x(Xm) if on_device else call.stage_x(Xm)
        Y = dev_out if dev_out is not None else call.y_stage()
        if m and b:
            call.launch(xd, Y)
        if dev_out is not None:       # host X, device out: Y stays on the device
            return dev_out
        if host_out is not None:      # host tensor out (e.g. pinned): one D2H, synchronous
            host_out.copy_(Y.reshape(host_out.shape))
            return host_out
        Yh = call.y_host(Y)           # D2H into pinned staging, then a private copy
    Yh = Yh[:, 0] if was_vector else Yh
    return Yh if is_tensor else Yh.numpy()


def _host_call(call, Xm, host_out, stream, is_tensor, was_vector, pinned=None):
    """Host X in, host Y out through the plan's graph-replayed path."""
    with call.lock:
        Yh = call.run_host(Xm, host_out, stream, pinned)
        if host_out is not None:
            if Yh is not host_out:
                host_out.copy_(Yh.reshape(host_out.shape))
            return host_out
        Yh = Yh.clone() if is_tensor else Yh.numpy().copy()
    return Yh[:, 0] if was_vector else Yh


def _register_fast(pwm, X, out, opts, call, stream, dev, is_tensor, was_vector):
    """Remember a validated host-path call keyed by the identity of X and out.
    The entry re-checks that X / out are the same live objects with the same
    shape, dtype and data pointer and that the current stream is unchanged;
    anything else falls back to the full path (returns None)."""
    import weakref
    try:
        xref = weakref.ref(X)
        oref = weakref.ref(out) if out is not None else (lambda: None)
    except TypeError:           # e.g. a list: not weak-referenceable, no fast path
        return
    xshape, xdtype = X.shape, X.dtype
    xptr = X.data_ptr() if is_tensor else X.ctypes.data
    oshape = out.shape if out is not None else None
    optr = out.data_ptr() if out is not None else None
    key = ("fast", id(X), id(out)) + opts
    # Tensor.is_pinned() asks the driver (cudaPointerGetAttributes, ~4 us per
    # call): the answer cannot change while the same live tensor keeps the
    # same data pointer, so the entry remembers it
    pinned = (bool(is_tensor and X.is_pinned()), bool(out is not None and out.is_pinned()))

    def ent(X2, out2):
        if xref() is not X2 or X2.shape != xshape or X2.dtype != xdtype:
            return None
        if (X2.data_ptr() if is_tensor else X2.ctypes.data) != xptr:
            return None
        if out2 is not None and (oref() is not out2 or out2.shape != oshape or out2.data_ptr() != optr):
            return None
        if _lib.current_stream_handle(dev) != stream or _lib.torch().cuda.current_device() != dev.index:
            return None
        return _host_call(call, X2[:, None] if was_vector else X2, out2, stream, is_tensor, was_vector,
                          pinned)

    cache = pwm._device_cache
    if sum(1 for kk in cache if kk[0] == "fast") >= 8:
        for kk in [kk for kk in cache if kk[0] == "fast"]:
            del cache[kk]
    cache[key] = ent


# Sign-symmetric half tables (csrc msg_fused.cu / msg_lane.cu) round entries
# of sum_r (v - beta) x_r, so their error is relative to sum |v - beta||x|,
# not to the reference's bound sum |W||x| (suites.py:106-124).  Rows whose
# conditioning ratio (packing.symmetric_conditioning) exceeds
#     _SYM_MARGIN * rtol(X) / unit_roundoff(table entries)
# -- sparse rows, and every row without a nonzero weight, which the
# reference returns as exactly 0 (lut.py:59-72: the all-zero index is 0) --
# are recomputed with full tables; a matrix with more than 1/8 such rows
# runs on full tables altogether.
_SYM_MARGIN = 0.05
_RTOL = {_lib.F16: 2e-3, _lib.F32: 1e-5}
_UNIT = {2: 2.0 ** -11, 4: 2.0 ** -24}


def _symmetric_threshold(x_code: int, entry_bytes: int) -> float:
    return _SYM_MARGIN * _RTOL.get(x_code, 1e-5) / _UNIT[entry_bytes]


class _CallPlan:
    """Everything msgemm needs for one (weights, device, stream, shape, dtype,
    options) combination, prepared once: the C-ABI plan, the repacked layout,
    the codebook block, the workspace and the host/device staging buffers.
    Later calls only copy activations and launch."""

    def __init__(self, pwm, dev, stream, b, x_code, x_dtype, d, table_dtype, symmetric,
                 out_dtype, flags):
        t = _lib.torch()
        lib = _lib.lib()
        m, k = pwm.m, pwm.k
        self.m, self.b, self.dev = m, b, dev
        scale_mode, group_size, q_code = _lib.SCALE_NONE, 0, _lib.F64
        if isinstance(pwm.scales, PerRow):
            scale_mode = _lib.SCALE_PER_ROW
        elif isinstance(pwm.scales, PerGroup):
            scale_mode, group_size = _lib.SCALE_PER_GROUP, pwm.scales.group_size
        qd = pwm.device_scales(dev)
        if qd is not None:
            q_code = _lib.dtype_code(qd.dtype)
            if q_code == _lib.BF16:
                raise NotImplementedError("bfloat16 scales are not supported")
        if table_dtype is not None and np.dtype(table_dtype) == np.float32:
            flags |= _lib.FLAG_F32_ENTRIES
        if not symmetric:
            flags |= _lib.FLAG_NO_SYMMETRY
        self.vals = _lib.host_doubles(pwm.codebook.values)
        layout, sym = _lib.ctypes.c_int(0), _lib.ctypes.c_int(0)
        ws_bytes = _lib.ctypes.c_int64(0)

        def plan(fl):
            _lib.check(lib.msg_gemm_plan(m, k, pwm.width, self.vals, x_code, b, d, scale_mode,
                                         group_size, fl, _lib.ctypes.byref(layout),
                                         _lib.ctypes.byref(sym), _lib.ctypes.byref(ws_bytes)))
        plan(flags)
        self.fix = None
        if sym.value and m and b:
            entry = 4 if (x_code == _lib.F32 or flags & _lib.FLAG_F32_ENTRIES) else 2
            rows = pwm.ill_conditioned_rows(dev, d, pwm.codebook.antisymmetric_offset(),
                                            _symmetric_threshold(x_code, entry))
            n_ill = int(rows.numel())
            if n_ill * 8 > m:      # mostly sparse weights: full tables for every row
                flags |= _lib.FLAG_NO_SYMMETRY
                plan(flags)
            elif n_ill:            # a few sparse rows: recomputed on full tables
                sub = pwm.row_subset(dev, rows)
                self.fix = (_CallPlan(sub, dev, stream, b, x_code, x_dtype, d, table_dtype, False,
                                      out_dtype, flags), rows, n_ill)
        self.layout, self.symmetric = layout.value, sym.value
        x_t = x_dtype if isinstance(x_dtype, t.dtype) else _lib.torch_dtype_of(x_dtype)
        self.x_dtype = x_t
        self.y_dtype = x_t if out_dtype is None else _lib.torch_dtype_of(np.dtype(out_dtype))
        self.y_code = _lib.dtype_code(self.y_dtype)
        wrep = None
        if layout.value != _lib.LAYOUT_NONE and m and b:
            wrep = pwm.device_layout(dev, d, layout.value, sym.value)
            # the layout now exists before any later launch: the LUT kernel may
            # prefetch it under PDL (it is never written by the preceding kernel)
            flags |= _lib.FLAG_STATIC_WEIGHTS
        ws = _lib.workspace(ws_bytes.value, dev,
                            "lane" if layout.value == _lib.LAYOUT_LANE else "scratch")
        # a first call that built the layout must not prefetch it: it is not static yet
        self._first_flags = flags & ~_lib.FLAG_STATIC_WEIGHTS if wrep is not None else flags
        self._args_head = (_lib.ptr(pwm.device_data(dev)), _lib.ptr(wrep), m, k, pwm.width,
                           self.vals)
        self._args_mid = (x_code, b, d, scale_mode, group_size, _lib.ptr(qd), q_code)
        self._ws = (ws, _lib.ptr(ws), ws.numel())
        self._flags = flags
        self._stream = _lib.ctypes.c_void_p(stream)
        self._keep = (wrep, qd)
        self._xs = self._xh = self._ys = self._yh = None
        self._graphs, self._seen = {}, set()
        self._xh_view = None
        self._graph_run = lib.msg_graph_run
        self._fn = lib.msg_gemm
        self._launched = False
        self.lock = threading.Lock()

    def launch(self, xd, Y, stream=None, fan=None):
        flags = self._flags if self._launched else self._first_flags
        ws, wsp, wsn = self._ws
        st = self._stream if stream is None else _lib.ctypes.c_void_p(stream)
        if fan:   # Y also into the peers' buffers (msg_gemm_fanout)
            arr = (_lib.ctypes.c_void_p * len(fan))(*[int(a) for a in fan])
            _lib.check(_lib.lib().msg_gemm_fanout(
                *self._args_head, _lib.ctypes.c_void_p(xd.data_ptr()), *self._args_mid,
                _lib.ctypes.c_void_p(Y.data_ptr()), self.y_code, wsp, wsn, flags, st, arr, len(fan)))
        else:
            _lib.check(self._fn(*self._args_head, _lib.ctypes.c_void_p(xd.data_ptr()),
                                *self._args_mid, _lib.ctypes.c_void_p(Y.data_ptr()), self.y_code,
                                wsp, wsn, flags, st))
        self._launched = True
        if self.fix is not None:   # ill-conditioned rows: full tables, scattered into Y
            sub, rows, n = self.fix
            ys = sub.y_stage()
            sub.launch(xd, ys, stream)
            for dst in [Y.data_ptr()] + [int(a) for a in (fan or ())]:
                _lib.check(_lib.lib().msg_copy_rows(_lib.ctypes.c_void_p(ys.data_ptr()), _lib.ptr(rows),
                                                    n, self.b * Y.element_size(),
                                                    _lib.ctypes.c_void_p(dst), 1, st))

    def run_host(self, Xm, host_out, stream, pinned=None):
        """Host activations in, host Y out (the drop-in call): H2D -> kernels ->
        D2H -> one stream sync.  From the second call with the same host
        buffers on, the three steps replay as one CUDA graph launched and
        waited for in one C call (msg_graph_run) instead of a copy, two kernel
        launches, a copy and a sync: ~20 us less per GEMV-sized call.  Pinned
        torch buffers are used in place; anything else goes through the plan's
        pinned staging.  Returns the pinned tensor holding Y (host_out itself
        when it was used in place)."""
        xh = self._xh
        if xh is None or xh.shape != Xm.shape:
            t = _lib.torch()
            self._xs = t.empty(tuple(Xm.shape), dtype=self.x_dtype, device=self.dev)
            self._xh = xh = t.empty(tuple(Xm.shape), dtype=self.x_dtype, pin_memory=True)
            self._graphs.clear()
        if _lib.is_torch(Xm):
            if (Xm.dtype == self.x_dtype and Xm.is_contiguous()
                    and (pinned[0] if pinned is not None else Xm.is_pinned())):
                src = Xm
            else:
                src = xh
                src.copy_(Xm)
        else:
            src = xh
            np.copyto(self._xh_np(), Xm, casting="no")
        if (host_out is not None and host_out.dtype == self.y_dtype and host_out.is_contiguous()
                and (pinned[1] if pinned is not None else host_out.is_pinned())):
            dst = host_out
        else:
            if self._yh is None:
                self._yh = _lib.torch().empty((self.m, self.b), dtype=self.y_dtype, pin_memory=True)
            dst = self._yh
        key = (src.data_ptr(), dst.data_ptr())
        ex = self._graphs.get(key)
        if ex is None and key in self._seen and not _lib.torch().cuda.is_current_stream_capturing():
            ex = self._capture(src, dst)
        if ex is not None:
            _lib.check(self._graph_run(ex[1], stream, 1))
        else:
            self._seen.add(key)
            self._xs.copy_(src, non_blocking=True)
            self._launch_to_host(dst)
            _lib.check(_lib.lib().msg_stream_sync(_lib.ctypes.c_void_p(stream)))
        return dst

    def _launch_to_host(self, dst, stream=None):
        """Kernels -> Y in host memory.  The finishing kernels store Y straight
        into the pinned buffer (device-visible under UVA) with 16-byte stores,
        so no separate D2H copy trails the kernels (cfg5 e2e 272 -> 263 us;
        cfg4 b = 1 36.3 -> 32.8 us, cfg2 34.2 -> 25.7 us once the b = 1 finish
        wrote eight rows per store -- its former 2-byte stores were slower
        than a device Y plus one D2H copy).  MSG_HOST_Y=copy forces the copy
        (A/B).  Reading X in place from the pinned buffer instead of the H2D
        copy measured no gain when the caller rewrites X between calls (32.8 vs
        33.2 us, tools/fastpath_profile.py), so the copy node stays."""
        if _HOST_Y_DIRECT:
            self.launch(self._xs, dst.reshape(self.m, self.b), stream)
        else:
            ys = self.y_stage()
            self.launch(self._xs, ys, stream)
            dst.copy_(ys.reshape(dst.shape), non_blocking=True)

    def _xh_np(self):
        if self._xh_view is None or self._xh_view[0] is not self._xh:
            self._xh_view = (self._xh, self._xh.numpy())
        return self._xh_view[1]

    def _capture(self, src, dst):
        """Capture H2D -> kernels -> D2H for these host buffers (side stream)."""
        t = _lib.torch()
        if len(self._graphs) >= 4:
            self._graphs.pop(next(iter(self._graphs)))
        cur = t.cuda.current_stream(self.dev)
        side = t.cuda.Stream(self.dev)
        side.wait_stream(cur)
        ys = self.y_stage()
        g = t.cuda.CUDAGraph()
        with t.cuda.stream(side):
            with t.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
                if _HOST_X_KERNEL and src.data_ptr() % 16 == 0:
                    _lib.check(_lib.lib().msg_stage_copy(
                        _lib.ctypes.c_void_p(src.data_ptr()), _lib.ctypes.c_void_p(self._xs.data_ptr()),
                        src.numel() * src.element_size(), _lib.ctypes.c_void_p(side.cuda_stream)))
                else:
                    self._xs.copy_(src, non_blocking=True)
                self._launch_to_host(dst, side.cuda_stream)
        cur.wait_stream(side)
        ex = (g, _lib.ctypes.c_void_p(int(g.raw_cuda_graph_exec())))
        self._graphs[(src.data_ptr(), dst.data_ptr())] = ex
        return ex

    def device_x(self, Xm):
        """Contiguous device activations the kernels can read: the lane kernel
        stages X with 4-byte copies, so a misaligned view is copied first."""
        xd = Xm if Xm.is_contiguous() else Xm.contiguous()
        if xd.data_ptr() % 16:
            xd = xd.clone()
        return xd

    def stage_x(self, Xm):
        """Host activations -> device staging (pinned host tensors: one async H2D;
        numpy / pageable: through a cached pinned buffer)."""
        t = _lib.torch()
        shape = tuple(Xm.shape)
        if self._xs is None or tuple(self._xs.shape) != shape:
            self._xs = t.empty(shape, dtype=self.x_dtype, device=self.dev)
            self._xh = t.empty(shape, dtype=self.x_dtype, pin_memory=True)
            self._graphs.clear()
        if _lib.is_torch(Xm) and Xm.is_pinned():
            self._xs.copy_(Xm, non_blocking=True)
            return self._xs
        src = t.from_numpy(np.ascontiguousarray(Xm)) if not _lib.is_torch(Xm) else Xm
        self._xh.copy_(src)               # host memcpy into pinned memory
        self._xs.copy_(self._xh, non_blocking=True)
        return self._xs

    def y_stage(self):
        t = _lib.torch()
        if self._ys is None:
            self._ys = t.empty((self.m, self.b), dtype=self.y_dtype, device=self.dev)
        return self._ys

    def y_host(self, Y):
        t = _lib.torch()
        if self._yh is None:
            self._yh = t.empty((self.m, self.b), dtype=self.y_dtype, pin_memory=True)
        self._yh.copy_(Y)                 # D2H (synchronises the stream)
        return self._yh.clone()           # the caller owns its result


def _call_plan(pwm, dev, stream, b, x_code, x_dtype, d, table_dtype, symmetric, out_dtype,
               flags) -> _CallPlan:
    cache = pwm._device_cache
    key = ("call", dev.index, stream, b, x_code, d,
           None if table_dtype is None else np.dtype(table_dtype).str, bool(symmetric),
           None if out_dtype is None else np.dtype(out_dtype).str, flags)
    plan = cache.get(key)
    if plan is None:
        plan = _CallPlan(pwm, dev, stream, b, x_code, x_dtype, d, table_dtype, symmetric,
                         out_dtype, flags)
        cache[key] = plan
    return plan


def msgemm_counted(pwm: PackedWeightMatrix, X, d: int, budget: int = DEFAULT_BUDGET,
                   workers: int = 1):
    """msgemm plus shape-derived operation counts (gemm.py:156-183)."""
    Xm, _ = _as_matrix(X)
    if pwm.k % d != 0:
        raise ValueError("op counting requires k divisible by d")
    Y = msgemm(pwm, X, d, budget=budget, workers=workers)
    b = int(Xm.shape[1])
    nb = pwm.k // d
    mul = 0
    if isinstance(pwm.scales, PerRow):
        mul = pwm.m * b
    elif isinstance(pwm.scales, PerGroup):
        mul = pwm.m * (pwm.k // pwm.scales.group_size) * b
    return Y, OpCount(fma=2 ** (pwm.codebook.width * d) * d * nb * b,
                      add=(nb - 1) * pwm.m * b, mul=mul,
                      mem_weights=pwm.m * pwm.k * b, mem_activations=pwm.k * b)


def msgemm_traced(pwm: PackedWeightMatrix, x, d: int, budget: int = DEFAULT_BUDGET):
    """Matrix-vector msgemm with the lookup trace (gemm.py:186-203)."""
    if (x.dim() if _lib.is_torch(x) else np.asarray(x).ndim) != 1:
        raise ValueError("tracing is defined for a single activation vector")
    y = msgemm(pwm, x, d, budget=budget)
    idx = group_indices(pwm, d)
    table = build_lut(x, pwm.codebook, d, budget=budget)
    idx_h = idx.cpu().numpy() if _lib.is_torch(idx) else idx
    ent = table.entries.cpu().numpy() if _lib.is_torch(table.entries) else table.entries
    trace = [[(j, int(idx_h[i, j]), ent[j, idx_h[i, j]]) for j in range(idx_h.shape[1])]
             for i in range(pwm.m)]
    return y, trace


_NAIVE_MODES = {np.dtype(np.float16): 1, np.dtype(np.float32): 2, np.dtype(np.float64): 3}


def naive_gemm(W, X):
    """Dense reference W @ X (gemm.py:206-216) on the GPU (``msg_naive_gemm``).

    numpy's semantics: integer x integer -> int64 products and sums (wrapping,
    bit-exact); otherwise both operands go to ``np.result_type(W, X)`` --
    float16 sums exact products in fp32 in k order and rounds once (numpy's
    half loop, bit-exact); float32/float64 sum in fp64 in k order (numpy calls
    BLAS there; same values within rounding).
    """
    t = _lib.torch()
    on_device = _lib.is_torch(X) or _lib.is_torch(W)
    Wa = W if _lib.is_torch(W) else np.asarray(W)
    Xm, was_vector = _as_matrix(X)
    if Wa.ndim != 2 or Wa.shape[1] != Xm.shape[0]:
        raise ValueError(f"shape mismatch: W {tuple(Wa.shape)} x X {tuple(Xm.shape)}")
    wdt, xdt = _np_dtype(Wa), _np_dtype(Xm)
    wdt = None if wdt is None else np.dtype(wdt)
    xdt = None if xdt is None else np.dtype(xdt)
    if wdt is None or xdt is None or wdt.kind not in "iufb" or xdt.kind not in "iufb":
        raise NotImplementedError(f"naive_gemm: dtypes {wdt}, {xdt} are not supported on the GPU")
    if wdt.kind in "iub" and xdt.kind in "iub":
        mode, res = 0, np.dtype(np.int64)
    else:
        res = np.result_type(wdt, xdt)
        if res not in _NAIVE_MODES:
            raise NotImplementedError(f"naive_gemm: result dtype {res} is not supported on the GPU")
        mode = _NAIVE_MODES[res]
    dev = _lib.require_device()

    def operand(a, dt):
        if not _lib.is_torch(a) and (dt.kind == "b" or dt in (np.dtype(np.uint16), np.dtype(np.uint32),
                                                               np.dtype(np.uint64))):
            a = a.astype(np.uint8 if dt.kind == "b" else np.int64)   # same int64 wrap
        return _lib.to_device(a, dev).contiguous()

    wd, xd = operand(Wa, wdt), operand(Xm, xdt)
    m, k, b = int(wd.shape[0]), int(wd.shape[1]), int(xd.shape[1])
    Y = t.empty((m, b), dtype=_lib.torch_dtype_of(res), device=dev)
    _lib.check(_lib.lib().msg_naive_gemm(_lib.ptr(wd), _lib.dtype_code(wd.dtype), _lib.ptr(xd),
                                         _lib.dtype_code(xd.dtype), m, k, b, mode, _lib.ptr(Y),
                                         _lib.stream_ptr()))
    if was_vector:
        Y = Y[:, 0]
    return Y if on_device else Y.cpu().numpy()


def naive_gemm_counted(W, X):
    """naive_gemm plus the m*k*b FMA count (gemm.py:219-231)."""
    Wa = W if _lib.is_torch(W) else np.asarray(W)
    Xm, _ = _as_matrix(X)
    Y = naive_gemm(W, X)
    m, k = (int(s) for s in Wa.shape)
    b = int(Xm.shape[1])
    return Y, OpCount(fma=m * k * b, mem_weights=m * k, mem_activations=k * b)


_HMMA_MAX_B = 16   # dense baseline: weight-streaming mma.sync kernel up to b = 16, tcgen05 above
_GEMV_MAX_WEIGHTS = 1 << 25   # ... except b = 1 up to 32 M weights: the CUDA-core GEMV (8192^2: 12.8 vs 11.7 us)


def dequant_gemm(pwm: PackedWeightMatrix, X, out_dtype=np.float32, out=None, kernel="auto"):
    """Dense comparison baseline (K4): dequantise int4 W and multiply, fp32
    accumulation -- for b <= 16 a weight-streaming kernel straight from the
    packed layout (csrc/msg_dense_hmma.cu: in-register dequantise + mma.sync,
    split k over a thread-block cluster), else on the tcgen05 tensor cores
    (csrc/msg_mma.cu, accumulator in TMEM).

    X must be fp16 (k,) or (k, b) with b <= 256; int4/uint4 codebooks, no
    scales.  Same result contract as naive_gemm(dense(pwm), X) (gemm.py:206-216).
    kernel: "auto" | "hmma" (b <= 16, k % 32 == 0) | "gemv" (the CUDA-core
    variant, b <= 8, k % 32 == 0) | "mma".
    """
    pwm = _ensure_device_pwm(pwm)
    if pwm.scales is not None:
        raise NotImplementedError("dequant_gemm does not apply scales")
    if kernel not in ("auto", "hmma", "gemv", "mma"):
        raise ValueError(f"unknown dense kernel {kernel!r}")
    Xm, was_vector = _as_matrix(X)
    if int(Xm.shape[0]) != pwm.k:
        raise ValueError(f"activation rows {Xm.shape[0]} != weight columns {pwm.k}")
    dev = _lib.require_device()
    t = _lib.torch()
    lib = _lib.lib()
    m, k, b = pwm.m, pwm.k, int(Xm.shape[1])
    xd = _lib.to_device(Xm, dev)
    y_dt = _lib.torch_dtype_of(np.dtype(out_dtype))
    Y = out if out is not None else t.empty((m, b), dtype=y_dt, device=dev)
    cbv = [float(v) for v in pwm.codebook.values]
    nib = cbv == [float(c if c < 8 else c - 16) for c in range(16)] or cbv == [float(c) for c in range(16)]
    stream_ok = k % 32 == 0 and nib and xd.dtype == t.float16
    if kernel == "gemv" and not (stream_ok and b <= 8):
        raise NotImplementedError("the GEMV baseline needs b <= 8, k % 32 == 0, int4/uint4 and fp16 X")
    if kernel == "hmma" and not (stream_ok and b <= _HMMA_MAX_B):
        raise NotImplementedError("the HMMA baseline needs b <= 16, k % 32 == 0, int4/uint4 and fp16 X")
    if kernel == "auto":
        if stream_ok and b == 1 and m * k <= _GEMV_MAX_WEIGHTS:
            kernel = "gemv"    # tiny GEMVs: no cluster launch / DSMEM reduction (4096^2: 4.9 vs 7.3 us)
        else:
            kernel = "hmma" if stream_ok and b <= _HMMA_MAX_B else "mma"
    if m and b and kernel in ("hmma", "gemv"):
        fn = lib.msg_dequant_hmma if kernel == "hmma" else lib.msg_dequant_gemv
        _lib.check(fn(
            _lib.ptr(pwm.device_data(dev)), m, k, _lib.host_doubles(pwm.codebook.values),
            _lib.ptr(xd.contiguous()), _lib.dtype_code(xd.dtype), b, _lib.ptr(Y),
            _lib.dtype_code(y_dt), _lib.stream_ptr()))
    elif m and b:
        wt = pwm.device_mma_layout(dev)
        ws = _lib.workspace(lib.msg_dequant_mma_workspace_bytes(m, k, b), dev)
        _lib.check(lib.msg_dequant_mma(
            _lib.ptr(wt), m, k, _lib.host_doubles(pwm.codebook.values), _lib.ptr(xd),
            _lib.dtype_code(xd.dtype), b, _lib.ptr(Y), _lib.dtype_code(y_dt), _lib.ptr(ws),
            ws.numel(), _lib.stream_ptr()))
    if was_vector:
        Y = Y.reshape(m, b)[:, 0]
    return Y if _lib.is_torch(X) and X.is_cuda else Y.cpu().numpy()
