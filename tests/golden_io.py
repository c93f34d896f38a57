"""Loader for the reference-generated fixtures in tests/golden/ (see make_golden.py)."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    z = np.load(GOLDEN / name, allow_pickle=False)
    meta = json.loads(bytes(z["meta"]).decode())
    cases = []
    for i, m in enumerate(meta):
        arrs = {k: z[f"c{i}_{k}"] for k in m["keys"]}
        cases.append((m, arrs))
    return cases


def numpy_version(name):
    z = np.load(GOLDEN / name, allow_pickle=False)
    return bytes(z["numpy_version"]).decode()
