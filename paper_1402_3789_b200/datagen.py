"""Synthetic Gaussian-blob inputs, bit-identical to the reference generator.

Restates ``parclust.dataio.generate_synthetic`` (dataio.py:124-145) so the
GPU box (where the reference is absent) produces the exact float64 inputs the
reference would; pinned by tests/golden/synthetic_sha256.csv.
"""

from __future__ import annotations

import numpy as np


def generate_synthetic(n: int, d: int, clusters: int, spread: float, seed: int):
    """Return (X float64 (n,d), labels int64 (n,)); rows grouped by blob."""
    if n < 1 or d < 1 or clusters < 1:
        raise ValueError(f"n, d, clusters must all be at least 1, got n={n} d={d} clusters={clusters}")
    if not spread >= 0.0:
        raise ValueError(f"spread must be nonnegative, got {spread}")
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-100.0, 100.0, size=(clusters, d))
    per = np.full(clusters, n // clusters, dtype=np.int64)
    per[: n % clusters] += 1
    labels = np.repeat(np.arange(clusters, dtype=np.int64), per)
    X = centers[labels] + rng.normal(0.0, spread, size=(n, d))
    return np.ascontiguousarray(X, dtype=np.float64), labels


def config_dataset(name: str):
    """Inputs for the BASELINE.json configs.  Returns X."""
    if name == "c1":
        return generate_synthetic(10_000, 8, 5, 1.0, seed=1)[0]
    if name == "c2":
        a = generate_synthetic(80_000, 25, 160, 1.0, seed=2)[0]
        b = generate_synthetic(20_000, 25, 400, 3.0, seed=3)[0]
        return np.ascontiguousarray(np.vstack([a, b]))
    if name == "c3":
        return generate_synthetic(500_000, 25, 1000, 1.0, seed=4)[0]
    if name in ("c4", "c5"):
        return generate_synthetic(2_000_000, 25, 4000, 1.0, seed=5)[0]
    raise ValueError(f"unknown config {name!r}")
