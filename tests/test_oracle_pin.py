"""Pin the C oracle to the reference before trusting it (CPU only).

Two sources of truth:
  * the reference's own known-answer tests, restated here with the file:line
    they come from (pkg/tests/...);
  * golden fixtures made by importing the reference (tests/golden/make_golden.py).
"""

from __future__ import annotations

import hashlib
import math
import os

import numpy as np
import pytest

from oracle import nnm_oracle as orc
from nnm_testutil import GOLDEN, golden, same_partition


def _ones(n):
    return np.ones(n, np.int64)


# ---------------------------------------------------------------- metric KATs
class TestMetricKATs:
    # pkg/tests/test_metrics.py:41-55
    def test_345(self):
        D = orc.internal_pairwise("euclidean", [[0.0, 0.0]], [[3.0, 4.0]])
        assert D[0, 0] == 25.0

    def test_manhattan(self):
        assert orc.internal_pairwise("manhattan", [[1.0, 2.0]], [[4.0, -2.0]])[0, 0] == 7.0

    def test_chebyshev(self):
        assert orc.internal_pairwise("chebyshev", [[1.0, 2.0]], [[4.0, -2.0]])[0, 0] == 4.0

    def test_left_to_right_accumulation(self, rng):
        # pkg/tests/test_metrics.py:61-82: independent left-to-right loop, bit-equal
        x = rng.normal(size=(5, 11)) * 1e3
        y = rng.normal(size=(6, 11))
        D = orc.internal_pairwise("euclidean", x, y)
        for i in range(5):
            for j in range(6):
                acc = 0.0
                for k in range(11):
                    t = x[i, k] - y[j, k]
                    acc = acc + t * t
                assert D[i, j] == acc


def test_metric_tiles_match_scipy_bitwise():
    g = golden("metric_tiles.npz")
    for i in range(int(g["count"])):
        got = orc.internal_pairwise(str(g[f"metric_{i}"]), g[f"x_{i}"], g[f"y_{i}"])
        assert np.array_equal(got, g[f"D_{i}"]), f"tile {i} ({g[f'metric_{i}']})"


# ---------------------------------------------------------------- top-P
def test_topp_matches_reference_global_top_p():
    g = golden("topp_cases.npz")
    for i in range(int(g["count"])):
        kl2, kl3, P = (int(v) for v in g[f"args_{i}"])
        thr = float(g[f"thr_{i}"])
        d, a, b = orc.top_p(g[f"X_{i}"], g[f"roots_{i}"], g[f"sizes_{i}"], P,
                            metric=str(g[f"metric_{i}"]),
                            threshold=None if math.isnan(thr) else thr,
                            kl2=None if kl2 < 0 else kl2, kl3=None if kl3 < 0 else kl3,
                            threads=3)
        assert np.array_equal(d, g[f"dist_{i}"]), i
        assert np.array_equal(a, g[f"a_{i}"]), i
        assert np.array_equal(b, g[f"b_{i}"]), i


def test_topp_identical_points_order():
    # pkg/tests/test_pairgen.py:199-205: four identical points -> (0,1),(0,2),(0,3) at 0
    X = np.zeros((4, 2))
    d, a, b = orc.top_p(X, np.arange(4), _ones(4), 3)
    assert list(zip(a, b)) == [(0, 1), (0, 2), (0, 3)]
    assert np.all(d == 0.0)


def test_topp_dmax_excludes_everything():
    # pkg/tests/test_pairgen.py:207-213
    X = np.array([[0.0], [10.0], [20.0]])
    d, a, b = orc.top_p(X, np.arange(3), _ones(3), 5, threshold=1.0)
    assert len(d) == 0


# ---------------------------------------------------------------- full runs
def test_chain_kat():
    # pkg/tests/test_oracle.py:38-50
    m, _ = orc.single_linkage(np.array([[0.0], [10.0], [10.5], [30.0]]))
    assert [(r["point_a"], r["point_b"]) for r in m] == [(1, 2), (0, 1), (2, 3)]
    assert [r["dist"] for r in m] == [0.5, 10.0, 19.5]
    assert m[-1]["new_size"] == 4
    m, _ = orc.single_linkage(np.array([[0.0], [1.0], [2.0]]))
    assert (m[0]["point_a"], m[0]["point_b"]) == (0, 1)


def test_kl2_live_recheck_overshoot():
    # pkg/tests/test_engine.py:87-98 semantics: a cluster may overshoot kl2 by one union
    X = np.array([[0.0], [1.0], [2.0], [3.0]])
    r = orc.run(X, kl2=1, P=16)
    sizes = [int(m["new_size"]) for m in r.merges]
    assert max(sizes) <= 4


@pytest.mark.parametrize("threads", [1, 4])
def test_run_cases_match_reference_engine(threads):
    g = golden("run_cases.npz")
    for i in range(int(g["count"])):
        kl1, kl2, kl3, kl4, P = (int(v) for v in g[f"cons_{i}"])
        dm = float(g[f"dmax_{i}"])
        o = lambda v: None if v < 0 else v  # noqa: E731
        r = orc.run(g[f"X_{i}"], metric=str(g[f"metric_{i}"]), kl1=o(kl1), kl2=o(kl2),
                    kl3=o(kl3), kl4=o(kl4), dmax=None if math.isnan(dm) else dm, P=P,
                    threads=threads)
        want = g[f"merges_{i}"]
        assert len(r.merges) == len(want), i
        for f in ("round", "root_a", "root_b", "dist", "new_size", "point_a", "point_b"):
            assert np.array_equal(r.merges[f], want[f]), (i, f)
        assert np.array_equal(r.assignments, g[f"assign_{i}"]), i
        assert r.rounds == int(g[f"rounds_{i}"]), i
        assert r.stop_reason == str(g[f"stop_{i}"]), i
        rc = np.array(r.round_counters.tolist(), dtype=np.int64).reshape(-1, 7)
        assert np.array_equal(rc, g[f"counters_{i}"]), i
        if f"flat_{i}" in g:
            fm, fa = orc.single_linkage(
                g[f"X_{i}"], metric=str(g[f"metric_{i}"]), kl1=o(kl1), kl2=o(kl2),
                kl3=o(kl3), dmax=None if math.isnan(dm) else dm)
            flat = g[f"flat_{i}"]
            for f in ("root_a", "root_b", "dist", "new_size", "point_a", "point_b"):
                assert np.array_equal(fm[f], flat[f]), (i, f)


def test_c2_small_golden():
    p = os.path.join(GOLDEN, "c2_small_run.npz")
    if not os.path.exists(p):
        pytest.skip("c2 golden not generated")
    g = np.load(p)
    r = orc.run(g["X"], kl1=12, kl2=300, kl3=450, kl4=150, P=256)
    for f in ("round", "root_a", "root_b", "dist", "new_size", "point_a", "point_b"):
        assert np.array_equal(r.merges[f], g["merges"][f]), f
    assert r.rounds == int(g["rounds"])
    assert same_partition(r.assignments, g["assign"])
    assert np.array_equal(r.assignments, g["assign"])


def test_synthetic_generator_pinned():
    from paper_1402_3789_b200.datagen import generate_synthetic

    with open(os.path.join(GOLDEN, "synthetic_sha256.csv")) as fh:
        rows = fh.read().strip().splitlines()[1:]
    for row in rows:
        n, d, k, s, seed, hv, hl = row.split(",")
        if int(n) > 20_000:
            continue
        X, labels = generate_synthetic(int(n), int(d), int(k), float(s), int(seed))
        assert hashlib.sha256(X.tobytes()).hexdigest() == hv
        assert hashlib.sha256(labels.tobytes()).hexdigest() == hl
