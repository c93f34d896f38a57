"""Seeded case generator of the reference's oracle suites -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of ``CaseGen.draw`` (``/root/reference/pkg/src/msgemm/
suites.py:27-80``) returning plain arrays, so the reference's own acceptance
suites (criterion 1: 4 x 1000 exact + 1000 f32 cases,
``pkg/tests/test_acceptance.py:50-61``; the formula suite,
``suites.py:142-156``) can be replayed through the GPU package without
importing the reference.  The draw sequence (every ``rng`` call, its bounds
and its order) is the reference's, so a given ``seed`` yields the reference's
cases bit for bit; ``tests/golden/casegen_digests.json`` (written by
``tests/golden/make_golden.py`` from the reference itself) pins that.

Only ``tests/`` may import this module.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

#: suites.py:21-23 -- per-element relative tolerance of the f32 channel
F32_RTOL = 1e-5


@dataclass(frozen=True)
class Case:
    """One drawn case: codes (m, k) of the int4 codebook, optional scales, X."""

    case_seed: int
    d: int
    codes: np.ndarray
    X: np.ndarray
    scale_mode: str          # "none" | "per_row" | "per_group"
    group_size: int          # per_group only
    q: np.ndarray | None

    @property
    def m(self) -> int:
        return int(self.codes.shape[0])

    @property
    def k(self) -> int:
        return int(self.codes.shape[1])

    @property
    def b(self) -> int:
        return int(self.X.shape[1])

    def digest_update(self, h) -> None:
        """Feed the case into a hash (the layout make_golden.py uses)."""
        h.update(f"{self.case_seed},{self.d},{self.m},{self.k},{self.b},"
                 f"{self.scale_mode},{self.group_size};".encode())
        h.update(np.ascontiguousarray(self.codes, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(self.X).tobytes())
        if self.q is not None:
            h.update(np.ascontiguousarray(self.q).tobytes())


class CaseGen:
    """Restatement of suites.py:27-80 (same defaults, same draw order)."""

    def __init__(self, seed=0, m_range=(1, 64), k_max=48, b_range=(1, 8),
                 depths=(1, 2, 3, 4), scale_modes=("none", "per_row", "per_group"),
                 mode="exact"):
        if mode not in ("exact", "f32"):                      # suites.py:40-42
            raise ValueError(f"mode must be 'exact' or 'f32', got {mode!r}")
        self.seed, self.m_range, self.k_max, self.b_range = seed, m_range, k_max, b_range
        self.depths, self.scale_modes, self.mode = tuple(depths), tuple(scale_modes), mode
        self._rng = np.random.default_rng(seed)

    def _scale_values(self, crng, shape):                     # suites.py:82-85
        if self.mode == "exact":
            return crng.integers(1, 5, size=shape).astype(np.int64)
        return (0.25 + crng.random(shape)).astype(np.float32)

    def draw(self, d=None, divisible_only=False, scale_mode=None) -> Case:
        """suites.py:44-80: one case; every crng call in the reference's order."""
        case_seed = int(self._rng.integers(0, 2 ** 31))
        crng = np.random.default_rng(case_seed)
        if d is None:
            d = int(crng.choice(self.depths))
        m = int(crng.integers(self.m_range[0], self.m_range[1] + 1))
        k = int(crng.integers(d, self.k_max + 1))
        if scale_mode is None:
            scale_mode = str(crng.choice(self.scale_modes))
        if divisible_only or scale_mode == "per_group":
            k = max(d, k - k % d)
        b = int(crng.integers(self.b_range[0], self.b_range[1] + 1))
        codes = crng.integers(0, 16, size=(m, k))             # int4 codebook: 16 codes
        q, group_size = None, 0
        if scale_mode == "per_row":
            q = self._scale_values(crng, (m,))
        elif scale_mode == "per_group":
            multiples = [t for t in (1, 2, 4) if (t * d) <= k and k % (t * d) == 0]
            group_size = d * int(crng.choice(multiples))
            q = self._scale_values(crng, (m, k // group_size))
        if self.mode == "exact":
            X = crng.integers(-1000, 1001, size=(k, b)).astype(np.int64)
        else:
            X = crng.standard_normal((k, b)).astype(np.float32)
        return Case(case_seed, d, codes, X, scale_mode, group_size, q)


#: the five suites of acceptance criterion 1 (test_acceptance.py:50-61)
CRITERION1_SUITES = [dict(seed=1000 + d, depths=(d,)) for d in (1, 2, 3, 4)] + \
                    [dict(seed=2000, mode="f32")]


def suite_digest(cases) -> str:
    h = hashlib.sha256()
    for c in cases:
        c.digest_update(h)
    return h.hexdigest()
