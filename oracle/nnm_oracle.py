"""ctypes binding of the C oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Arrays in and out are numpy; argument conventions follow the reference:
constraints ``None`` = unset, metric names as in ``parclust.metrics.MetricKind``
(metrics.py:34-53).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libnnm_oracle.so")

METRIC_CODES = {"euclidean": 0, "squared-euclidean": 1, "manhattan": 2, "chebyshev": 3}
STOP_NAMES = {1: "kl1-reached", 2: "no-eligible-pairs", 3: "single-cluster"}


class _Merge(ctypes.Structure):
    _fields_ = [
        ("round", ctypes.c_int64),
        ("root_a", ctypes.c_int64),
        ("root_b", ctypes.c_int64),
        ("dist", ctypes.c_double),
        ("new_size", ctypes.c_int64),
        ("point_a", ctypes.c_int64),
        ("point_b", ctypes.c_int64),
    ]


MERGE_DTYPE = np.dtype(
    [
        ("round", np.int64),
        ("root_a", np.int64),
        ("root_b", np.int64),
        ("dist", np.float64),
        ("new_size", np.int64),
        ("point_a", np.int64),
        ("point_b", np.int64),
    ]
)
ROUND_DTYPE = np.dtype(
    [
        (k, np.int64)
        for k in ("round", "selected", "merged", "same_root", "kl2", "kl3", "unprocessed")
    ]
)

_lib = None


def build() -> str:
    """Compile the oracle with its own Makefile (needs gcc)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.POINTER
    d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
    lib.orc_internal_distance.restype = d
    lib.orc_internal_distance.argtypes = [i32, P(d), P(d), i32]
    lib.orc_pairwise.restype = None
    lib.orc_pairwise.argtypes = [i32, P(d), i64, P(d), i64, i32, P(d)]
    lib.orc_top_p.restype = i64
    lib.orc_top_p.argtypes = [P(d), i64, i32, i32, P(i64), P(i64), d, i64, i64, i64, i32,
                              P(d), P(i64), P(i64)]
    lib.orc_run.restype = i32
    lib.orc_run.argtypes = [P(d), i64, i32, i32, i64, i64, i64, i64, d, i64, i32,
                            ctypes.c_void_p, P(i64), P(i64), P(i64), P(i32),
                            ctypes.c_void_p, i64, P(i64)]
    lib.orc_single_linkage.restype = i32
    lib.orc_single_linkage.argtypes = [P(d), i64, i32, i32, i64, i64, i64, d,
                                       ctypes.c_void_p, P(i64), P(i64)]
    _lib = lib
    return lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _opt(v) -> int:
    return -1 if v is None else int(v)


def _metric(m) -> int:
    name = getattr(m, "value", m)
    return METRIC_CODES[str(name).strip().lower()]


def internal_pairwise(metric, x, y) -> np.ndarray:
    """scipy-order internal distances (metrics.py:67-73)."""
    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
    y = np.ascontiguousarray(np.atleast_2d(y), dtype=np.float64)
    out = np.empty((x.shape[0], y.shape[0]), dtype=np.float64)
    load().orc_pairwise(_metric(metric), _dp(x), x.shape[0], _dp(y), y.shape[0], x.shape[1],
                        _dp(out))
    return out


def top_p(X, roots, sizes, P, *, metric="euclidean", threshold=None, kl2=None, kl3=None,
          threads=None):
    """Exact top-P eligible pairs (pairgen.global_top_p / oracle_top_p semantics).

    ``threshold`` is in internal units (EligibilitySnapshot.threshold).
    Returns (dist, a, b) numpy arrays, ascending by (dist, a, b).
    """
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, d = X.shape
    roots = np.ascontiguousarray(roots, dtype=np.int64)
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    if P < 1:
        raise ValueError(f"P must be at least 1, got {P}")
    cap = max(1, min(P, n * (n - 1) // 2))
    od = np.empty(cap, np.float64)
    oa = np.empty(cap, np.int64)
    ob = np.empty(cap, np.int64)
    thr = math.nan if threshold is None else float(threshold)
    threads = threads or (os.cpu_count() or 1)
    ln = load().orc_top_p(_dp(X), n, d, _metric(metric), _ip(roots), _ip(sizes), thr,
                          _opt(kl2), _opt(kl3), int(P), int(threads), _dp(od), _ip(oa), _ip(ob))
    if ln < 0:
        raise ValueError("oracle top_p rejected its arguments")
    return od[:ln].copy(), oa[:ln].copy(), ob[:ln].copy()


@dataclass
class OracleRun:
    merges: np.ndarray  # MERGE_DTYPE records, step = index
    assignments: np.ndarray
    rounds: int
    stop_reason: str
    round_counters: np.ndarray  # ROUND_DTYPE records


def run(X, *, metric="euclidean", kl1=None, kl2=None, kl3=None, kl4=None, dmax=None, P=256,
        threads=None) -> OracleRun:
    """engine.run semantics (engine.py:154-199): top-P rounds + ordered live merging."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, d = X.shape
    merges = np.zeros(max(n - 1, 1), dtype=MERGE_DTYPE)
    assign = np.empty(n, np.int64)
    nm = ctypes.c_int64()
    rounds = ctypes.c_int64()
    stop = ctypes.c_int()
    ccap = n + 8
    counters = np.zeros(ccap, dtype=ROUND_DTYPE)
    nc = ctypes.c_int64()
    threads = threads or (os.cpu_count() or 1)
    rc = load().orc_run(_dp(X), n, d, _metric(metric), _opt(kl1), _opt(kl2), _opt(kl3),
                        _opt(kl4), math.nan if dmax is None else float(dmax), int(P),
                        int(threads), merges.ctypes.data, ctypes.byref(nm), _ip(assign),
                        ctypes.byref(rounds), ctypes.byref(stop), counters.ctypes.data, ccap,
                        ctypes.byref(nc))
    if rc != 0:
        raise ValueError("oracle run rejected its arguments")
    return OracleRun(merges[: nm.value].copy(), assign, rounds.value, STOP_NAMES[stop.value],
                     counters[: min(nc.value, ccap)].copy())


def single_linkage(X, *, metric="euclidean", kl1=None, kl2=None, kl3=None, dmax=None):
    """oracle_single_linkage (oracle.py:59-107): flat Kruskal with live checks."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, d = X.shape
    merges = np.zeros(max(n - 1, 1), dtype=MERGE_DTYPE)
    assign = np.empty(n, np.int64)
    nm = ctypes.c_int64()
    rc = load().orc_single_linkage(_dp(X), n, d, _metric(metric), _opt(kl1), _opt(kl2),
                                   _opt(kl3), math.nan if dmax is None else float(dmax),
                                   merges.ctypes.data, ctypes.byref(nm), _ip(assign))
    if rc != 0:
        raise ValueError("oracle single_linkage failed")
    return merges[: nm.value].copy(), assign
