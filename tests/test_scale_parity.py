"""Parity at the BASELINE scale (SURVEY.md 8(c) "Parity at 500k/2M").

The CUDA path (through the C ABI) against full-scale goldens of the pinned C oracle
(tests/golden/make_scale_golden.py; the oracle restates engine.run /
global_top_p, engine.py:154-199, pairgen.py:319-324, and tests/test_oracle_pin.py
pins it against the imported reference), plus identity checks between independent
GPU error models / algorithms at the full configs:

* C3 500k x 25 dmax=5 full run (tensor-core screen, pruned) == oracle;
  the same with the FP32 screen and no pruning (dense scans) == oracle;
* C4 X[::10] (200k x 25) full dendrograms, euclidean / manhattan / chebyshev == oracle;
* C2 100k x 25 kl1..kl4, P=256: merges, rounds and per-round counters == oracle;
* C4 2M x 25 round-1 global_top_p (P=256) == oracle;
* C4 2M x 25 full dendrogram: tensor-core screen == FP32 screen (NNM_TC=0), and the
  GPU merge replay == the sequential host replay.

Merge fields compare bit-exact (sha256 of the raw arrays); rounds are compared only
where they are part of parity (kl4).  All @gpu."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from nnm_testutil import GOLDEN

pytestmark = pytest.mark.gpu

FIELDS = ("root_a", "root_b", "dist", "new_size", "point_a", "point_b")
SCALE = os.path.join(GOLDEN, "scale")


def _golden(name):
    path = os.path.join(SCALE, f"{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{name} golden not generated (tests/golden/make_scale_golden.py {name})")
    with open(path) as f:
        return json.load(f)


def _digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def nnm():
    import paper_1402_3789_b200 as pkg
    from paper_1402_3789_b200 import _native

    _native.load()
    return pkg


@pytest.fixture(scope="module")
def c4():
    from paper_1402_3789_b200.datagen import config_dataset

    return config_dataset("c4")


def _check(res, g):
    arr = res.merges.array
    assert len(arr) == g["n_merges"]
    for row in g["sample"]:  # readable first mismatch
        i = row[0]
        got = [float(arr[i]["dist"]) if f == "dist" else int(arr[i][f]) for f in FIELDS]
        assert got == row[1:], (i, got, row[1:])
    for f in FIELDS:
        assert _digest(arr[f]) == g["digests"][f], f
    assert _digest(res.assignments) == g["digests"]["assignments"]
    assert res.stop_reason == g["stop_reason"]


class _Env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("mode", ["default", "fp32_dense"])
def test_c3_full_run_vs_oracle(nnm, mode):
    from paper_1402_3789_b200.datagen import config_dataset

    g = _golden("c3")
    X = config_dataset("c3")
    env = {} if mode == "default" else {"NNM_TC": "0", "NNM_PRUNE": "0"}
    with _Env(**env):
        res = nnm.fit(X, dmax=5.0)
    if mode == "default":
        assert res.device_stats["tc_items"] > 0
    else:
        assert res.device_stats["tc_items"] == 0
    _check(res, g)


@pytest.mark.parametrize("name,metric", [("c4sub", "euclidean"), ("c5msub", "manhattan"),
                                         ("c5csub", "chebyshev")])
def test_c4_subsample_vs_oracle(nnm, c4, name, metric):
    g = _golden(name)
    X = np.ascontiguousarray(c4[:: g["stride"]])
    _check(nnm.fit(X, metric=metric), g)


def test_c2_full_run_vs_oracle(nnm):
    from paper_1402_3789_b200.datagen import config_dataset

    g = _golden("c2")
    res = nnm.fit(config_dataset("c2"), pairs_per_batch=256, **g["constraints"])
    _check(res, g)
    assert res.rounds == g["rounds"]
    assert _digest(res.merges.array["round"]) == g["round_digest"]
    rc = [[c[k] for k in ("round", "selected", "merged", "same_root", "kl2", "kl3", "unprocessed")]
          for c in res.round_counters]
    assert rc == g["counters"]


def test_c2_without_kl4_fast_path_vs_oracle(nnm):
    """C2's data with kl1/kl2/kl3 and no kl4: the GPU's large-batch rounds reproduce the
    oracle's merge list (P-invariant without kl4) with >= 10x fewer rounds
    than the reference's round structure at P=256 (exact_rounds)."""
    from paper_1402_3789_b200.datagen import config_dataset

    g = _golden("c2nokl4")
    X = config_dataset("c2")
    res = nnm.fit(X, pairs_per_batch=256, **g["constraints"])
    _check(res, g)
    ref_rounds = nnm.fit(X, pairs_per_batch=256, exact_rounds=True, **g["constraints"]).rounds
    assert res.rounds * 10 <= ref_rounds, (res.rounds, ref_rounds)


def test_c4_round1_top256_vs_oracle(nnm, c4):
    from paper_1402_3789_b200.metrics import MetricKind
    from paper_1402_3789_b200.pairgen import EligibilitySnapshot, gpu_top_p

    g = _golden("c4top")
    n = c4.shape[0]
    snap = EligibilitySnapshot(np.arange(n, dtype=np.int64), np.ones(n, dtype=np.int64),
                               nnm.ConstraintSet(), None, MetricKind.EUCLIDEAN)
    buf = gpu_top_p(nnm.Dataset(values=c4), snap, 256)
    assert buf.dist.tolist() == g["dist"]
    assert buf.a.tolist() == g["a"]
    assert buf.b.tolist() == g["b"]


def _run_digest(nnm, X, **env):
    with _Env(**env):
        res = nnm.fit(X)
    arr = res.merges.array
    return [_digest(arr[f]) for f in FIELDS + ("round",)] + [_digest(res.assignments)], res


def test_c4_tensor_screen_equals_fp32_screen(nnm, c4):
    """Independent error models (TF32 tensor-core screen vs FP32 dot-form screen) give
    the identical 2M-point dendrogram."""
    a, ra = _run_digest(nnm, c4)
    b, rb = _run_digest(nnm, c4, NNM_TC="0")
    assert ra.device_stats["tc_items"] > 0 and rb.device_stats["tc_items"] == 0
    assert a[:-2] == b[:-2] and a[-1] == b[-1]  # Boruvka round numbering may differ


@pytest.mark.parametrize("env", [{"NNM_GPU_REPLAY": "0"}, {"NNM_REPLAY_LMAX": "4"},
                                 {"NNM_REPLAY_CHUNKS": "700"}, {"NNM_PINNED_OUT": "0"},
                                 {"NNM_REPLAY_LMAX": "4", "NNM_PINNED_OUT": "0"}])
def test_c4_gpu_replay_equals_host_replay(nnm, c4, env):
    """The component-parallel GPU replay == the sequential host replay at 2M (and the
    mixed case where the GPU stops early and the host finishes), with the records laid
    out by the GPU into page-locked outputs (default) or assembled on the host
    (NNM_PINNED_OUT=0)."""
    a, ra = _run_digest(nnm, c4)
    b, rb = _run_digest(nnm, c4, **env)
    # the last chunk (inter-blob edges: one component) is finished on the host
    assert ra.device_stats["replay_gpu_merges"] > 0.9 * len(ra.merges)
    if env.get("NNM_GPU_REPLAY") == "0":
        assert rb.device_stats["replay_gpu_merges"] == 0
    assert a == b


@pytest.fixture(scope="module")
def c4_full(nnm, c4):
    return nnm.fit(c4)


def test_c4_dmax_and_kl1_are_prefixes_of_the_full_dendrogram(nnm, c4, c4_full):
    """Single linkage: with dmax the merge list is the prefix of merges with height <= dmax
    (the MSF of the eligible graph, pairgen.py:197-198 / oracle.py:82-83); with kl1 it is
    the first n - kl1 merges (engine.py:139-142).  Checked at 2M against the full run."""
    full = c4_full.merges.array
    dmax = float(np.sqrt(full["dist"][1_500_000] * full["dist"][1_500_001]))  # between two merges
    part = nnm.fit(c4, dmax=dmax)
    k = int(np.searchsorted(full["dist"], dmax, side="right"))
    assert len(part.merges) == k
    for f in FIELDS:
        assert np.array_equal(part.merges.array[f], full[f][:k]), f
    kl1 = 4000
    trunc = nnm.fit(c4, kl1=kl1)
    assert len(trunc.merges) == c4.shape[0] - kl1
    for f in FIELDS:
        assert np.array_equal(trunc.merges.array[f], full[f][: c4.shape[0] - kl1]), f
    assert trunc.stop_reason == "kl1-reached" and len(np.unique(trunc.assignments)) == kl1


def test_c4_row_shuffled_same_dendrogram(nnm, c4, c4_full):
    """the row-shuffled C4 input (default_rng(seed + 100)) gives the same
    dendrogram: identical merge heights in order and the same point pairs (mapped back);
    blob data has no exact distance ties, so the order is fully determined."""
    perm = np.random.default_rng(5 + 100).permutation(c4.shape[0])
    res = nnm.fit(np.ascontiguousarray(c4[perm]))
    got, want = res.merges.array, c4_full.merges.array
    assert np.array_equal(got["dist"], want["dist"])
    a, b = perm[got["point_a"]], perm[got["point_b"]]
    pairs = np.stack([np.minimum(a, b), np.maximum(a, b)], 1)
    assert np.array_equal(pairs, np.stack([want["point_a"], want["point_b"]], 1))
    assert np.array_equal(got["new_size"], want["new_size"])


@pytest.mark.parametrize("metric", ["euclidean", "manhattan", "chebyshev"])
def test_dense_fp64_vs_pruned_screen_heavy_ties(nnm, metric, monkeypatch):
    """Two independent GPU algorithms on 48k points of an integer grid with duplicates
    (massive exact ties): the pruned, screened default path against the dense exact FP64
    Boruvka (NNM_SMALL=1, no screening, no pruning) -- identical merge logs and labels."""
    rng = np.random.default_rng(17)
    base = rng.integers(-20, 21, size=(24_000, 6)).astype(np.float64)
    X = np.ascontiguousarray(np.vstack([base, base[rng.permutation(len(base))]]))
    for cons in ({}, {"dmax": 2.0}, {"dmax": 0.0}, {"kl1": 300}):
        monkeypatch.setenv("NNM_SMALL", "0")
        a = nnm.fit(X, metric=metric, **cons)
        for mode in ("1", "2"):  # dense FP64; screened single launch (sweep 2 on ties)
            monkeypatch.setenv("NNM_SMALL", mode)
            b = nnm.fit(X, metric=metric, **cons)
            for f in FIELDS:
                assert np.array_equal(a.merges.array[f], b.merges.array[f]), (cons, mode, f)
            assert np.array_equal(a.assignments, b.assignments), (cons, mode)
            assert a.stop_reason == b.stop_reason
