"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved; W is uniform int4 and X is
N(0,1) (or uniform integers for the exact variant), generated with numpy's
default_rng as the reference's own generators are (suites.py:47-49).  W is
drawn directly as packed bytes (two uniform nibbles per byte), which is the
same distribution as drawing codes and packing them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    k: int
    b: int
    d: int
    x_dtype: str          # "float32" | "float16" | "int"  (int: integer-valued, fp16 on device)
    seed: int
    note: str = ""


CONFIGS = {
    "cfg1": Config("cfg1", 1024, 1024, 1, 2, "float32", 1, "single GEMV, CPU-runnable case"),
    "cfg2": Config("cfg2", 4096, 4096, 1, 3, "float16", 2, "LLM decode GEMV"),
    "cfg2int": Config("cfg2int", 4096, 4096, 1, 3, "int", 2, "integer-valued X, bit-exact"),
    "cfg3": Config("cfg3", 11008, 4096, 16, 3, "float16", 3, "MLP up-projection, b=16"),
    "cfg4b1": Config("cfg4b1", 8192, 8192, 1, 3, "float16", 4, "batch sweep"),
    "cfg4b4": Config("cfg4b4", 8192, 8192, 4, 3, "float16", 4, "batch sweep"),
    "cfg4b16": Config("cfg4b16", 8192, 8192, 16, 3, "float16", 4, "batch sweep"),
    "cfg4b64": Config("cfg4b64", 8192, 8192, 64, 3, "float16", 4, "batch sweep"),
    "cfg4b256": Config("cfg4b256", 8192, 8192, 256, 3, "float16", 4, "batch sweep"),
    "cfg5": Config("cfg5", 65536, 8192, 8, 3, "float16", 5, "row-sharded large GEMM"),
    # not a BASELINE config: the cfg5 matrix as a GEMV -- a b = 1 kernel long enough
    # (268 MB of weights) for launch ramp and drain not to set its HBM fraction
    "cfg5b1": Config("cfg5b1", 65536, 8192, 1, 3, "float16", 5, "extra: cfg5's matrix at b = 1"),
}


def weights(cfg: Config) -> np.ndarray:
    """Packed (m, ceil(k/2)) uint8 in the reference layout (packing.py:99-114)."""
    rng = np.random.default_rng(cfg.seed)
    data = rng.integers(0, 256, size=(cfg.m, (cfg.k + 1) // 2), dtype=np.uint8)
    if cfg.k % 2:
        data[:, -1] &= 0x0F
    return data


def activations(cfg: Config, b: int | None = None) -> np.ndarray:
    """X (k, b): fp32/fp16 N(0,1), or integers in [-127, 127] (int64) for the exact variant."""
    b = cfg.b if b is None else b
    if cfg.name.startswith("cfg4"):
        rng = np.random.default_rng([4, b])
    else:
        rng = np.random.default_rng([cfg.seed, 1])
    if cfg.x_dtype == "int":
        return rng.integers(-127, 128, size=(cfg.k, b)).astype(np.int64)
    return rng.standard_normal((cfg.k, b), dtype=np.float32).astype(cfg.x_dtype)


def algorithmic_bytes(cfg: Config, x_itemsize: int = 2, y_itemsize: int = 4) -> int:
    """B = m*ceil(k/2) + k*b*s_x + m*b*s_y."""
    return cfg.m * ((cfg.k + 1) // 2) + cfg.k * cfg.b * x_itemsize + cfg.m * cfg.b * y_itemsize


def effective_ops(cfg: Config) -> int:
    """2*m*k*b -- the metric's 'effective' operation count."""
    return 2 * cfg.m * cfg.k * cfg.b
