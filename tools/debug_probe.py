"""Bitwise outputs of every kernel family on fixed seeded shapes, repeated.

    [MSG_LIB_VARIANT=debug] python tools/debug_probe.py OUT.npz [reps]

Run once with the release library and once with the debug-checks library
(device bounds asserts + race-provoking barrier jitter): a missing barrier or
an out-of-bounds index shows up as a trap, a non-repeatable result across the
reps, or a difference from the release bits (tests/test_gpu_debug_build.py).
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_06178_b200 as mg  # noqa: E402
from paper_2310_06178_b200 import _lib  # noqa: E402

CASES = [  # (m, k, b, d, dtype, kwargs)
    (97, 301, 1, 3, np.float16, {}),                        # lane GEMV, tail
    (700, 3000, 1, 3, np.float16, {}),                      # lane, many chunks / CTAs
    (9000, 700, 8, 3, np.float16, {}),                      # rb_tmem: two row blocks
    (300, 200, 16, 3, np.float16, {}),                      # rb_tmem: two column tiles
    (2100, 500, 4, 3, np.float16, {}),                      # rb_lut<4>
    (1100, 401, 2, 3, np.float16, {}),                      # rb_lut<2>
    (512, 600, 3, 2, np.float32, {}),                       # fused quad, fp32 X
    (300, 300, 8, 3, np.float16, {"table_dtype": np.float32}),
    (300, 300, 8, 3, np.float16, {"symmetric": False}),
    (40, 30, 2, 4, np.float64, {}),                         # generic
]


def main():
    out, reps = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rng = np.random.default_rng(99)
    res = {}
    for ci, (m, k, b, d, dt, kw) in enumerate(CASES):
        codes = rng.integers(0, 16, (m, k), dtype=np.uint8)
        codes[5::11] = 0                                    # zero rows (full-table fix-up path)
        pwm = mg.from_codes(codes, mg.int4_codebook())
        X = rng.standard_normal((k, b)).astype(dt)
        Xa = X[:, 0].copy() if b == 1 else X
        ys = [np.asarray(mg.msgemm(pwm, Xa, d, **kw)) for _ in range(reps)]
        for y in ys[1:]:
            assert y.tobytes() == ys[0].tobytes(), f"case {ci}: not repeatable"
        res[f"y{ci}"] = ys[0]
    pwm = mg.from_codes(rng.integers(0, 16, (384, 320), dtype=np.uint8), mg.int4_codebook())
    Xh = torch.from_numpy(rng.standard_normal((320, 24)).astype(np.float16)).cuda()
    ks = [mg.dequant_gemm(pwm, Xh).cpu().numpy() for _ in range(reps)]
    assert all(k.tobytes() == ks[0].tobytes() for k in ks), "dq_mma not repeatable"
    res["k4"] = ks[0]
    for nb in (1, 8, 13):                                   # dq_hmma: cluster split-k over DSMEM
        hs = [mg.dequant_gemm(pwm, Xh[:, :nb].contiguous(), kernel="hmma").cpu().numpy() for _ in range(reps)]
        assert all(h.tobytes() == hs[0].tobytes() for h in hs), "dq_hmma not repeatable"
        res[f"k4h{nb}"] = hs[0]
    torch.cuda.synchronize()
    np.savez(out, lib=np.frombuffer(str(_lib.LIB_PATH.name).encode(), dtype=np.uint8), **res)
    print(f"debug probe ok ({_lib.LIB_PATH.name}, {len(CASES)} cases x {reps})")


if __name__ == "__main__":
    main()
