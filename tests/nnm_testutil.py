"""Test helpers shared by the suite (imported as a plain module from tests/)."""

from __future__ import annotations

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def canonical_labels(labels) -> np.ndarray:
    """Relabel clusters by first appearance (restates pkg/tests/conftest.py:16-22)."""
    labels = np.asarray(labels)
    mapping: dict = {}
    out = np.empty(labels.shape[0], dtype=np.int64)
    for i, v in enumerate(labels.tolist()):
        out[i] = mapping.setdefault(v, len(mapping))
    return out


def same_partition(x, y) -> bool:
    return np.array_equal(canonical_labels(x), canonical_labels(y))


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)
