"""Debug-checks build vs release build (stands in for compute-sanitizer,
which this GPU pool does not allow).

libmsgemm_b200_debug.so is the same sources compiled with MSG_DEBUG_CHECKS:
device-side bounds assertions on every shared-memory table address and TMA
batch, and a pseudo-random per-warp delay in front of every barrier and
mbarrier wait (csrc/msg_common.cuh).  tools/debug_probe.py runs every kernel
family on fixed shapes several times; the debug run must not trap, must be
bitwise repeatable under the jitter, and must reproduce the release bits.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _run(tmp_path, variant, reps):
    out = tmp_path / f"{variant}.npz"
    env = dict(os.environ)
    env["MSG_LIB_VARIANT"] = variant
    r = subprocess.run([sys.executable, "tools/debug_probe.py", str(out), str(reps)], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return np.load(out)


def test_debug_build_matches_release(tmp_path):
    lib = ROOT / "paper_2310_06178_b200" / "_lib" / "libmsgemm_b200_debug.so"
    assert lib.exists(), "debug library not built (__graft_entry__.build())"
    rel = _run(tmp_path, "release", 2)
    dbg = _run(tmp_path, "debug", 4)
    assert bytes(dbg["lib"]).decode() == "libmsgemm_b200_debug.so"
    keys = [k for k in rel.files if k != "lib"]
    assert keys and set(keys) == {k for k in dbg.files if k != "lib"}
    for k in keys:
        assert rel[k].tobytes() == dbg[k].tobytes(), k
