"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
writes small .npz fixtures next to this file.  The fixtures pin
``oracle/msgemm_oracle.py`` (CPU tests) and the CUDA path (GPU tests) to the
reference's own outputs; nothing at test time reads /root/reference.

Inputs are seeded numpy draws (same generator family as the reference's
suites.py:47-49) -- no external dataset is involved.
"""

from __future__ import annotations

import json
import sys
import zlib
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, str(REF))
    import msgemm  # noqa: F401  (the reference package)
    import msgemm.packing
    import msgemm.suites
    return msgemm


class Bank:
    """Accumulates named cases into one npz (flat keys, json metadata)."""

    def __init__(self):
        self.arrays = {}
        self.meta = []

    def add(self, kind, arrays, **meta):
        i = len(self.meta)
        for name, arr in arrays.items():
            self.arrays[f"c{i}_{name}"] = np.asarray(arr)
        meta["kind"] = kind
        meta["keys"] = sorted(arrays)
        self.meta.append(meta)

    def save(self, path):
        self.arrays["meta"] = np.frombuffer(json.dumps(self.meta).encode(), dtype=np.uint8)
        self.arrays["numpy_version"] = np.frombuffer(np.__version__.encode(), dtype=np.uint8)
        np.savez_compressed(path, **self.arrays)
        print(f"wrote {path} ({len(self.meta)} cases, {path.stat().st_size} bytes)")


def scale_meta(pwm):
    from msgemm import PerGroup, PerRow
    s = pwm.scales
    if s is None:
        return "none", 0, np.zeros(0)
    if isinstance(s, PerRow):
        return "per_row", 0, np.asarray(s.q)
    assert isinstance(s, PerGroup)
    return "per_group", s.group_size, np.asarray(s.q)


def add_gemm_case(bank, ms, pwm, X, d, tag, **extra):
    mode, gs, q = scale_meta(pwm)
    Y = ms.msgemm(pwm, X, d)
    W = ms.packing.dense(pwm, apply_scales=True)
    bank.add("gemm", {"data": pwm.data, "X": X, "Y": Y, "q": q, "W": W},
             m=pwm.m, k=pwm.k, width=pwm.width, d=d, scale_mode=mode, group_size=gs,
             values=[float(v) for v in pwm.codebook.values], tag=tag, **extra)


def main():
    ms = _ref()
    cb = ms.int4_codebook()

    # ---------------- packing / indices / LUT known answers ----------------
    pk = Bank()
    running = [
        [2, 4, 3, 5], [-1, 0, 1, -8], [7, -3, 2, 6], [0, 0, 0, 0],
        [1, 2, 3, 4], [-4, 5, -6, 7], [3, 3, 3, 3], [-8, -8, -8, -8],
        [6, 1, -2, 0], [5, -5, 5, -5], [0, 7, -1, 2], [-2, 4, 0, -7],
    ]
    pwm = ms.pack(running, cb)
    x = np.array([1, 10, 100, 1000], dtype=np.int64)
    y, trace = ms.msgemm_traced(pwm, x, 2)
    pk.add("running_example", {
        "W": np.asarray(running), "data": pwm.data, "x": x, "y": y,
        "trace_idx": np.array([[t[1] for t in row] for row in trace]),
        "trace_val": np.array([[t[2] for t in row] for row in trace]),
        "lut": ms.build_lut(x, cb, 2).entries,
        "gidx": ms.group_indices(pwm, 2),
    })
    rng = np.random.default_rng(123)
    for width, cbx in ((4, cb), (4, ms.uint4_codebook()), (2, ms.custom_codebook([0, 1, -1, 2])),
                       (8, ms.custom_codebook(list(range(-128, 128))))):
        for (m, k) in ((5, 12), (7, 11), (3, 1), (4, 17)):
            codes = rng.integers(0, cbx.num_codes, size=(m, k))
            p = ms.from_codes(codes, cbx)
            arrays = {"codes": codes.astype(np.uint8), "data": p.data,
                      "unpacked": ms.packing.codes(p)}
            for d in (1, 2, 3, 4):
                if d * width <= 32:
                    arrays[f"gidx_d{d}"] = ms.group_indices(p, d)
            pk.add("packing", arrays, width=width, m=m, k=k,
                   values=[float(v) for v in cbx.values])
    # pack() value encoding incl. scales
    w = rng.integers(-8, 8, size=(6, 8)).astype(np.float64)
    qrow = np.array([0.5, 2.0, 1.0, 0.25, 3.0, 1.5])
    p = ms.pack(w * qrow[:, None], cb, ms.PerRow(q=qrow))
    pk.add("pack_scaled", {"Wscaled": w * qrow[:, None], "q": qrow, "data": p.data}, mode="per_row")
    qg = rng.random((6, 4)) + 0.5
    p = ms.pack(w * np.repeat(qg, 2, axis=1), cb, ms.PerGroup(group_size=2, q=qg))
    pk.add("pack_scaled", {"Wscaled": w * np.repeat(qg, 2, axis=1), "q": qg, "data": p.data},
           mode="per_group", group_size=2)
    # LUTs for several dtypes and depths
    for dt in (np.int64, np.float32, np.float16, np.float64, np.int32):
        for d in (1, 2, 3, 4):
            k = 3 * d + 1
            if np.issubdtype(dt, np.integer):
                xv = rng.integers(-50, 50, size=k).astype(dt)
            else:
                xv = rng.standard_normal(k).astype(dt)
            tab = ms.build_lut(xv, cb, d).entries
            pk.add("lut", {"x": xv, "entries": tab, "block1": ms.build_lut_block(xv, cb, d, 1)},
                   d=d, dtype=np.dtype(dt).name)
    pk.save(OUT / "packing_lut.npz")

    # ---------------- msgemm vs reference on CaseGen + extra dtypes ----------------
    gb = Bank()
    for d in (1, 2, 3, 4):
        gen = ms.suites.CaseGen(seed=500 + d, depths=(d,))
        for _ in range(12):
            pwm, X, dd, seed = gen.draw()
            add_gemm_case(gb, ms, pwm, X, dd, f"exact_d{d}_seed{seed}")
    gen = ms.suites.CaseGen(seed=600, mode="f32")
    for _ in range(24):
        pwm, X, dd, seed = gen.draw()
        add_gemm_case(gb, ms, pwm, X, dd, f"f32_seed{seed}")
    # fp16 / fp64 / int32 / vector inputs (no reference test covers fp16; these
    # vectors are the only pin for that dtype)
    rng = np.random.default_rng(700)
    for i in range(16):
        d = int(rng.integers(1, 5))
        m = int(rng.integers(1, 70))
        k = int(rng.integers(d, 60))
        b = int(rng.integers(1, 9))
        pwm = ms.from_codes(rng.integers(0, 16, size=(m, k)), cb)
        X = rng.standard_normal((k, b)).astype(np.float16)
        add_gemm_case(gb, ms, pwm, X, d, f"f16_{i}")
    for i in range(6):
        d = int(rng.integers(1, 4))
        m, k = int(rng.integers(1, 40)), int(rng.integers(d, 40))
        pwm = ms.from_codes(rng.integers(0, 16, size=(m, k)), cb)
        add_gemm_case(gb, ms, pwm, rng.standard_normal(k), d, f"f64vec_{i}")
        add_gemm_case(gb, ms, pwm, rng.integers(-99, 99, size=(k, 3)).astype(np.int32), d,
                      f"i32_{i}")
    # uint4 codebook
    ucb = ms.uint4_codebook()
    for i in range(4):
        d = i % 3 + 1
        pwm = ms.from_codes(rng.integers(0, 16, size=(33, 25)), ucb)
        add_gemm_case(gb, ms, pwm, rng.standard_normal((25, 3)).astype(np.float32), d, f"u4_{i}")
    # config-shaped row slices (full k, few rows), seeded as bench.py seeds them
    shapes = [  # (m, k, b, d, dtype, tag)
        (64, 1024, 1, 2, np.float32, "cfg1"),
        (48, 4096, 1, 3, np.float16, "cfg2"),
        (16, 4096, 16, 3, np.float16, "cfg3"),
        (16, 8192, 8, 3, np.float16, "cfg5"),
    ]
    for m, k, b, d, dt, tag in shapes:
        rs = np.random.default_rng(zlib.crc32(tag.encode()))
        pwm = ms.from_codes(rs.integers(0, 16, size=(m, k), dtype=np.uint8), cb)
        X = rs.standard_normal((k, b), dtype=np.float32).astype(dt)
        add_gemm_case(gb, ms, pwm, X, d, tag)
    rs = np.random.default_rng(2002)
    pwm = ms.from_codes(rs.integers(0, 16, size=(48, 4096), dtype=np.uint8), cb)
    Xi = rs.integers(-127, 128, size=(4096, 1)).astype(np.int64)
    add_gemm_case(gb, ms, pwm, Xi, 3, "cfg2_int")
    gb.save(OUT / "gemm_cases.npz")


if __name__ == "__main__":
    main()
