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

import hashlib
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
    sparse_cases(ms)
    casegen_digests(ms)


def special_rows(rs, n, k, d):
    """Rows the sign-symmetric tables must not be trusted with: all-zero,
    single nonzero (random, +1, -1), 99% / 90% zero, only code 8 (-8), zero
    but for the k % d tail, two nonzeros in one group, all +1, one full group."""
    rows = []
    nb = k // d
    for t in range(n):
        r = np.zeros(k, dtype=np.uint8)
        kind = t % 11
        if kind == 1:
            r[rs.integers(0, k)] = rs.integers(1, 16)
        elif kind == 2:
            r[rs.integers(0, k)] = 1
        elif kind == 3:
            r[rs.integers(0, k)] = 15
        elif kind in (4, 5):
            frac = 0.01 if kind == 4 else 0.10
            mask = rs.random(k) < frac
            r[mask] = rs.integers(1, 16, size=int(mask.sum()))
        elif kind == 6:
            r[:] = 8
        elif kind == 7:
            r[nb * d:] = rs.integers(1, 16, size=k - nb * d)
        elif kind == 8:
            j = int(rs.integers(0, nb)) * d
            r[j] = rs.integers(1, 16)
            r[j + d - 1] = rs.integers(1, 16)
        elif kind == 9:
            r[:] = 1
        elif kind == 10:
            j = int(rs.integers(0, nb)) * d
            r[j:j + d] = rs.integers(1, 16, size=d)
        rows.append(r)
    return np.stack(rows)


def sparse_cases(ms):
    """Sparse / zero weight rows (round 2): the reference's bound
    |dy| <= rtol * sum_j |W_ij||x_j| (suites.py:104-124) is 0 for an all-zero
    row, whose all-zero index contributes exactly 0 (lut.py:59-72).
    Matrices: a mostly dense one with a few special rows, one made only of
    special rows, and a config-1-like d=2 one.  X is stored once per dtype at
    b=16; the b=1/4/8 cases use its first columns (b=1 as a vector)."""
    cb = ms.int4_codebook()
    sb = Bank()
    rs = np.random.default_rng(4242)
    mats = []
    dense = rs.integers(0, 16, size=(150, 8192), dtype=np.uint8)
    mixed = np.concatenate([dense[:75], special_rows(rs, 10, 8192, 3), dense[75:]])
    mats.append(("mixed", mixed, 3, (np.float16, np.float32)))
    mats.append(("special", special_rows(rs, 24, 4096, 3), 3, (np.float16, np.float32)))
    d1 = rs.integers(0, 16, size=(60, 1024), dtype=np.uint8)
    mats.append(("cfg1like", np.concatenate([d1[:30], special_rows(rs, 4, 1024, 2), d1[30:]]),
                 2, (np.float32,)))
    for name, codes, d, dts in mats:
        pwm = ms.from_codes(codes, cb)
        k = codes.shape[1]
        arrays = {"data": pwm.data}
        for dt in dts:
            X = rs.standard_normal((k, 16)).astype(dt)
            arrays[f"X_{np.dtype(dt).name}"] = X
            for b in (1, 4, 8, 16):
                Xb = X[:, 0].copy() if b == 1 else np.ascontiguousarray(X[:, :b])
                arrays[f"Y_{np.dtype(dt).name}_b{b}"] = ms.msgemm(pwm, Xb, d)
        Xi = rs.integers(-127, 128, size=(k, 8)).astype(np.int64)
        arrays["X_int"] = Xi
        arrays["Y_int_b1"] = ms.msgemm(pwm, Xi[:, 0].copy(), d)
        arrays["Y_int_b8"] = ms.msgemm(pwm, Xi, d)
        sb.add("sparse", arrays, name=name, m=pwm.m, k=k, width=4, d=d,
               dtypes=[np.dtype(dt).name for dt in dts],
               values=[float(v) for v in cb.values])
    sb.save(OUT / "sparse_cases.npz")


def casegen_digests(ms):
    """Digests of the reference's own CaseGen draws (suites.py:27-85) for the
    suites its tests run: acceptance criterion 1 (test_acceptance.py:50-61),
    test_suites.py:6-38 and the formula suite.  They pin the restatement in
    oracle/casegen.py, so the GPU replay of those suites runs the reference's
    exact cases.  For the exact suites the digest of the reference msgemm
    outputs is recorded too (int64, bit-exact)."""
    sys.path.insert(0, str(OUT.parents[1]))
    from oracle.casegen import Case
    suites = {
        "crit1_d1": (dict(seed=1001, depths=(1,)), 1000, {}),
        "crit1_d2": (dict(seed=1002, depths=(2,)), 1000, {}),
        "crit1_d3": (dict(seed=1003, depths=(3,)), 1000, {}),
        "crit1_d4": (dict(seed=1004, depths=(4,)), 1000, {}),
        "crit1_f32": (dict(seed=2000, mode="f32"), 1000, {}),
        "suite_exact_small": (dict(seed=1), 100, {}),
        "suite_f32_small": (dict(seed=2, mode="f32"), 100, {}),
        "formula": (dict(seed=5), 50, dict(divisible_only=True, scale_mode="none")),
    }
    out = {}
    for name, (kw, n, draw_kw) in suites.items():
        gen = ms.suites.CaseGen(**kw)
        hc, hy = hashlib.sha256(), hashlib.sha256()
        for _ in range(n):
            pwm, X, d, seed = gen.draw(**draw_kw)
            mode, gs, q = scale_meta(pwm)
            Case(seed, d, ms.packing.codes(pwm), X, mode, gs,
                 None if mode == "none" else q).digest_update(hc)
            if kw.get("mode", "exact") == "exact":
                hy.update(np.ascontiguousarray(ms.msgemm(pwm, X, d)).tobytes())
        out[name] = {"kwargs": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
                     "cases": n, "draw": draw_kw, "cases_sha256": hc.hexdigest(),
                     "Y_sha256": hy.hexdigest() if kw.get("mode", "exact") == "exact" else None}
    path = OUT / "casegen_digests.json"
    path.write_text(json.dumps({"numpy_version": np.__version__, "suites": out}, indent=1) + "\n")
    print(f"wrote {path}")


if __name__ == "__main__":
    if sys.argv[1:] == ["casegen"]:
        casegen_digests(_ref())
    else:
        main()
