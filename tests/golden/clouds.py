"""Deterministic synthetic clouds shared by the golden-vector generator and
the tests.  Recipes mirror the reference's own fixtures:

* ``uniform``  — ``io.py:209-210`` (``default_rng(seed).random((n, 3))``)
* ``ties``     — ``tests/test_fps_core.py:12-17`` (half the points duplicated)
* ``clusters`` — ``io.py:211-214`` (Gaussian blobs)
* ``*32``      — the same cloud rounded to float32 (the benchmark input
                 precision; the fp64 path sees the exact upcast)

NumPy's PCG64 ``random``/``integers``/``permutation`` streams are stable across
the NumPy versions in this image; the manifest stores a SHA-256 per generated
cloud so any drift fails loudly instead of producing silent mismatches.
"""

from __future__ import annotations

import hashlib

import numpy as np


def make_cloud(kind: str, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    base = kind[:-2] if kind.endswith("32") else kind
    if base == "uniform":
        pts = rng.random((n, 3))
    elif base == "ties":
        pts = rng.random((n, 3))
        if n >= 2:
            dup = pts[rng.integers(0, n, size=n // 2)]
            pts = np.vstack([pts[: n - n // 2], dup])[rng.permutation(n)]
    elif base == "clusters":
        centers = rng.random((4, 3))
        assign = rng.integers(0, 4, size=n)
        pts = centers[assign] + rng.normal(0.0, 0.05, size=(n, 3))
    else:
        raise ValueError(kind)
    if kind.endswith("32"):
        pts = pts.astype(np.float32).astype(np.float64)
    return np.ascontiguousarray(pts, dtype=np.float64)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
