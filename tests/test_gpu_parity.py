"""GPU parity: the CUDA path through the C ABI vs the reference's golden vectors
and the pinned C oracle.  Bit-exact for every key, label and index; merge heights
are compared bit-exact too (the FP64 keys are scipy-order exact).  All @gpu."""

from __future__ import annotations

import math

import numpy as np
import pytest

from nnm_testutil import golden, same_partition

pytestmark = pytest.mark.gpu

FIELDS = ("root_a", "root_b", "dist", "new_size", "point_a", "point_b")


@pytest.fixture(scope="module")
def nnm():
    import paper_1402_3789_b200 as pkg
    from paper_1402_3789_b200 import _native

    _native.load()
    return pkg


def _o(v):
    v = int(v)
    return None if v < 0 else v


def _records(merges):
    arr = getattr(merges, "array", None)
    if arr is not None:
        return arr
    return np.array([(e.round, e.root_a, e.root_b, e.dist, e.new_size, e.point_a, e.point_b)
                     for e in merges], dtype=[("round", np.int64), ("root_a", np.int64),
                                              ("root_b", np.int64), ("dist", np.float64),
                                              ("new_size", np.int64), ("point_a", np.int64),
                                              ("point_b", np.int64)])


def test_pairwise_bitwise_vs_scipy_golden(nnm):
    from paper_1402_3789_b200.metrics import MetricKind, internal_pairwise

    g = golden("metric_tiles.npz")
    for i in range(int(g["count"])):
        got = internal_pairwise(MetricKind.parse(str(g[f"metric_{i}"])), g[f"x_{i}"], g[f"y_{i}"])
        assert np.array_equal(got, g[f"D_{i}"]), i


def test_top_p_vs_reference_golden(nnm):
    from paper_1402_3789_b200.metrics import MetricKind
    from paper_1402_3789_b200.pairgen import EligibilitySnapshot, gpu_top_p

    g = golden("topp_cases.npz")
    for i in range(int(g["count"])):
        kl2, kl3, P = (int(v) for v in g[f"args_{i}"])
        thr = float(g[f"thr_{i}"])
        ds = nnm.Dataset(values=g[f"X_{i}"])
        snap = EligibilitySnapshot(g[f"roots_{i}"], g[f"sizes_{i}"],
                                   nnm.ConstraintSet(kl2=_o(kl2), kl3=_o(kl3)),
                                   None if math.isnan(thr) else thr,
                                   MetricKind.parse(str(g[f"metric_{i}"])))
        buf = gpu_top_p(ds, snap, P)
        assert np.array_equal(buf.dist, g[f"dist_{i}"]), i
        assert np.array_equal(buf.a, g[f"a_{i}"]), i
        assert np.array_equal(buf.b, g[f"b_{i}"]), i


@pytest.mark.parametrize("small", ["0", "auto"])
@pytest.mark.parametrize("exact_rounds", [False, True])
def test_run_vs_reference_engine_golden(nnm, exact_rounds, small, monkeypatch):
    """Every reference engine case; Boruvka-eligible cases run on the general pruned path
    (NNM_SMALL=0) and on the default selection (small inputs: the screened single launch)."""
    if small == "auto":
        monkeypatch.delenv("NNM_SMALL", raising=False)
    else:
        monkeypatch.setenv("NNM_SMALL", small)
    g = golden("run_cases.npz")
    for i in range(int(g["count"])):
        kl1, kl2, kl3, kl4, P = (int(v) for v in g[f"cons_{i}"])
        dm = float(g[f"dmax_{i}"])
        cfg = nnm.RunConfig(constraints=nnm.ConstraintSet(kl1=_o(kl1), kl2=_o(kl2), kl3=_o(kl3),
                                                          kl4=_o(kl4),
                                                          dmax=None if math.isnan(dm) else dm),
                            pairs_per_batch=P, metric=nnm.MetricKind.parse(str(g[f"metric_{i}"])),
                            exact_rounds=exact_rounds)
        res = nnm.run(nnm.Dataset(values=g[f"X_{i}"]), cfg)
        got, want = _records(res.merges), g[f"merges_{i}"]
        assert len(got) == len(want), i
        for f in FIELDS:
            assert np.array_equal(got[f], want[f]), (i, f)
        assert np.array_equal(res.assignments, g[f"assign_{i}"]), i
        assert res.stop_reason == str(g[f"stop_{i}"]), i
        if exact_rounds or kl4 >= 0:  # rounds are P-dependent, part of parity with kl4 (F3/F4)
            assert np.array_equal(got["round"], want["round"]), i
            assert res.rounds == int(g[f"rounds_{i}"]), i
            rc = np.array([[c[k] for k in ("round", "selected", "merged", "same_root", "kl2",
                                           "kl3", "unprocessed")] for c in res.round_counters],
                          dtype=np.int64).reshape(-1, 7)
            assert np.array_equal(rc, g[f"counters_{i}"]), i


@pytest.mark.parametrize("small", ["0", "1", "2"])
def test_c1_full_run_vs_reference(nnm, small, monkeypatch):
    """BASELINE config 1: 10k x 8, 5 blobs, unconstrained, P=256 (reference run here), on
    the general pruned path (0), the dense FP64 single launch (1) and the screened single
    launch (2, the default for C1)."""
    from paper_1402_3789_b200.datagen import config_dataset

    monkeypatch.setenv("NNM_SMALL", small)
    g = golden("c1_run.npz")
    res = nnm.run(nnm.Dataset(values=config_dataset("c1")), nnm.RunConfig(pairs_per_batch=256))
    got = _records(res.merges)
    for f in FIELDS:
        assert np.array_equal(got[f], g["merges"][f]), f
    assert np.array_equal(res.assignments, g["assign"])
    assert res.stop_reason == str(g["stop"])


def test_kl2_kl3_fast_path_rounds_drop(nnm):
    """kl2/kl3 without kl4: large GPU batches give the reference's merge list (P-invariant,
    SURVEY F3) in far fewer rounds than P=256."""
    from oracle import nnm_oracle as orc

    a = nnm.generate_synthetic(8000, 25, 16, 1.0, seed=2)[0]
    b = nnm.generate_synthetic(2000, 25, 40, 3.0, seed=3)[0]
    X = np.vstack([a, b])
    ref = orc.run(X, kl1=40, kl2=300, kl3=450, P=256)
    fast = nnm.fit(X, kl1=40, kl2=300, kl3=450, pairs_per_batch=256)
    exact = nnm.fit(X, kl1=40, kl2=300, kl3=450, pairs_per_batch=256, exact_rounds=True)
    got = _records(fast.merges)
    for f in FIELDS:
        assert np.array_equal(got[f], ref.merges[f]), f
    assert np.array_equal(fast.assignments, ref.assignments)
    assert exact.rounds == ref.rounds
    assert fast.rounds * 5 <= exact.rounds, (fast.rounds, exact.rounds)


def test_c2_analogue_rounds_vs_reference(nnm):
    g = golden("c2_small_run.npz")
    cfg = nnm.RunConfig(constraints=nnm.ConstraintSet(kl1=12, kl2=300, kl3=450, kl4=150),
                        pairs_per_batch=256)
    res = nnm.run(nnm.Dataset(values=g["X"]), cfg)
    got = _records(res.merges)
    for f in ("round",) + FIELDS:
        assert np.array_equal(got[f], g["merges"][f]), f
    assert res.rounds == int(g["rounds"])
    assert np.array_equal(res.assignments, g["assign"])


@pytest.mark.parametrize("small", ["0", "1", "2"])  # general pruned path / dense small-input path
@pytest.mark.parametrize("metric", ["euclidean", "squared-euclidean", "manhattan", "chebyshev"])
@pytest.mark.parametrize("kind", ["blobs", "ties", "dups"])
def test_boruvka_vs_oracle_flat(nnm, metric, kind, small, monkeypatch):
    monkeypatch.setenv("NNM_SMALL", small)
    from oracle import nnm_oracle as orc

    rng = np.random.default_rng(hash((metric, kind)) % 2**32)
    n = 1500
    if kind == "blobs":
        X = nnm.generate_synthetic(n, 7, 9, 1.0, seed=11)[0]
    elif kind == "ties":
        X = rng.integers(-4, 5, size=(n, 3)).astype(np.float64)
    else:
        X = np.repeat(rng.normal(size=(n // 3, 5)), 3, axis=0)
    for cons in ({}, {"dmax": 1.5}, {"kl1": 17}, {"dmax": 0.0}):
        m_or, a_or = orc.single_linkage(X, metric=metric, **cons)
        res = nnm.fit(X, metric=metric, **cons)
        got = _records(res.merges)
        assert len(got) == len(m_or), cons
        for f in FIELDS:
            assert np.array_equal(got[f], m_or[f]), (cons, f)
        assert np.array_equal(res.assignments, a_or), cons


def test_staged_dense_ranges_equal_single(nnm):
    """Emulate 3 ranks on one GPU with the dense staged scan (nnm_bv_scan): disjoint
    tile-pair ranges + the min-combine of keys give the single-GPU merge log."""
    import ctypes

    from paper_1402_3789_b200 import _native
    from paper_1402_3789_b200.distributed import shard_range

    X = nnm.generate_synthetic(3000, 6, 12, 1.0, seed=3)[0]
    want = nnm.fit(X)
    lib = _native.load()
    dd = _native.DeviceDataset(X)
    tp, rows = ctypes.c_int64(), ctypes.c_int64()
    _native.check(lib.nnm_bv_begin(dd.handle, 0, np.nan, ctypes.byref(tp), ctypes.byref(rows)))
    import torch

    n = X.shape[0]
    R = 3
    while True:
        parts = []
        for r in range(R):
            lo, hi = shard_range(tp.value, r, R)
            b1 = torch.empty(rows.value, dtype=torch.int64, device="cuda")
            b2 = torch.empty(rows.value, dtype=torch.int64, device="cuda")
            _native.check(lib.nnm_bv_scan(dd.handle, lo, hi, b1.data_ptr(), b2.data_ptr()))
            parts.append((b1, b2))
        torch.cuda.synchronize()
        g1 = torch.stack([p[0] for p in parts]).min(0).values
        c2 = []
        for b1, b2 in parts:
            out = torch.empty_like(b1)
            _native.check(lib.nnm_bv_second(dd.handle, b1.data_ptr(), b2.data_ptr(), g1.data_ptr(),
                                            out.data_ptr()))
            c2.append(out)
        g2 = torch.stack(c2).min(0).values
        torch.cuda.synchronize()
        added = ctypes.c_int64()
        _native.check(lib.nnm_bv_finish_round(dd.handle, g1.data_ptr(), g2.data_ptr(),
                                              ctypes.byref(added)))
        if added.value == 0:
            break
    merges = np.zeros(n - 1, dtype=_native.MERGE_DTYPE)
    assign = np.empty(n, np.int64)
    nm, rounds = ctypes.c_int64(), ctypes.c_int64()
    stop = ctypes.c_int32()
    _native.check(lib.nnm_bv_end(dd.handle, -1, merges.ctypes.data, ctypes.byref(nm),
                                 assign.ctypes.data, ctypes.byref(rounds), ctypes.byref(stop), None))
    for f in FIELDS + ("round",):
        assert np.array_equal(merges[: nm.value][f], want.merges.array[f]), f
    assert np.array_equal(assign, want.assignments)


@pytest.mark.parametrize("replicas", [2, 3, 4])
@pytest.mark.parametrize("kw", [{}, {"dmax": 4.0}, {"metric": "manhattan"}, {"kl1": 9}])
def test_multi_replica_run_equals_single(nnm, replicas, kw, monkeypatch):
    """RunConfig(n_gpus=R) through nnm_run_multi with R replicas on device 0 (NNM_DEVICES):
    sharded bound / phase-1 / phase-2 scans, caps / keys / cache combined by the peer
    kernels -- byte-identical to one replica, and the replicas together evaluate exactly
    the single run's pairs (each item scanned once)."""
    X = nnm.generate_synthetic(9000, 25, 30, 1.0, seed=41)[0]
    X = X[np.random.default_rng(6).permutation(len(X))]
    single = nnm.fit(X, **kw)
    monkeypatch.setenv("NNM_DEVICES", ",".join(["0"] * replicas))
    multi = nnm.fit(X, n_gpus=replicas, **kw)
    for f in FIELDS + ("round",):
        assert np.array_equal(multi.merges.array[f], single.merges.array[f]), f
    assert np.array_equal(multi.assignments, single.assignments)
    assert multi.stop_reason == single.stop_reason
    assert multi.device_stats["replicas"] == [0] * replicas
    assert multi.device_stats["pairs_evaluated"] == single.device_stats["pairs_evaluated"]


@pytest.mark.parametrize("small", ["0", "1", "2"])
@pytest.mark.parametrize("n", [1, 2, 3, 127, 129, 300, 2049])
def test_boruvka_small_and_ragged_sizes(nnm, n, small, monkeypatch):
    monkeypatch.setenv("NNM_SMALL", small)
    from oracle import nnm_oracle as orc

    rng = np.random.default_rng(n)
    X = rng.normal(size=(n, 3)) * 2.0
    for metric in ("euclidean", "manhattan"):
        m_or, a_or = orc.single_linkage(X, metric=metric)
        res = nnm.fit(X, metric=metric)
        got = _records(res.merges)
        assert len(got) == len(m_or)
        for f in FIELDS:
            assert np.array_equal(got[f], m_or[f]), (metric, f)
        assert np.array_equal(res.assignments, a_or)


@pytest.mark.parametrize("small", ["0", "1", "2"])
def test_boruvka_shuffled_blobs_vs_oracle(nnm, small, monkeypatch):
    """Row-shuffled blob data (SURVEY 8d asks for a shuffled variant): kd order + pruning
    (general path) and the dense small-input path."""
    monkeypatch.setenv("NNM_SMALL", small)
    from oracle import nnm_oracle as orc

    X = nnm.generate_synthetic(4000, 9, 23, 1.0, seed=7)[0]
    X = X[np.random.default_rng(107).permutation(len(X))]
    for cons in ({}, {"dmax": 4.0}, {"kl1": 5}):
        m_or, a_or = orc.single_linkage(X, **cons)
        res = nnm.fit(X, **cons)
        got = _records(res.merges)
        for f in FIELDS:
            assert np.array_equal(got[f], m_or[f]), (cons, f)
        assert np.array_equal(res.assignments, a_or)


def test_device_input_checks(nnm):
    """C-ABI input validation runs on the device (model.py:29-76 message, first bad row)."""
    from paper_1402_3789_b200 import _native
    from paper_1402_3789_b200.model import ValidationError

    X = np.zeros((5000, 4))
    X[3210, 2] = np.nan
    X[4000, 1] = np.inf
    with pytest.raises(ValidationError, match="non-finite feature value in row 3211"):
        _native.DeviceDataset(X)
    Y = np.ones((100, 3))
    Y[7, 0] = 3e18
    with pytest.raises(_native.NativeError, match="FP32 screening range"):
        _native.DeviceDataset(Y)


def test_round_path_reuse_equals_full_rescans():
    """Round path (kl1..kl4, P=256): reusing earlier row bounds (default) gives the same
    merges, rounds and counters as a full scan every round (NNM_ROUND_REUSE=0)."""
    import os
    import subprocess
    import sys

    from nnm_testutil import ROOT

    code = ("import hashlib, numpy as np, paper_1402_3789_b200 as nnm\n"
            "a = nnm.generate_synthetic(16000, 25, 32, 1.0, seed=2)[0]\n"
            "b = nnm.generate_synthetic(4000, 25, 80, 3.0, seed=3)[0]\n"
            "X = np.vstack([a, b])\n"
            "r = nnm.fit(X, kl1=80, kl2=300, kl3=450, kl4=150, pairs_per_batch=256)\n"
            "c = np.array([[v for v in d.values()] for d in r.round_counters])\n"
            "print(hashlib.sha256(r.merges.array.tobytes() + r.assignments.tobytes() + c.tobytes())"
            ".hexdigest(), r.rounds, r.device_stats['round_rescans'])\n")
    outs = []
    for flag in ("1", "0"):
        env = dict(os.environ, NNM_ROUND_REUSE=flag)
        p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(p.stdout.split())
    assert outs[0][0] == outs[1][0] and outs[0][1] == outs[1][1]
    assert int(outs[0][1]) > 20  # a multi-round run that exercised the reuse


@pytest.mark.parametrize("d", [29, 30, 48])
def test_high_dimension_paths_vs_oracle(nnm, d):
    """d <= 29 runs the tensor-core scan, d > 29 the FP32 dot-form scan: both exact."""
    from oracle import nnm_oracle as orc

    X = nnm.generate_synthetic(2500, d, 11, 1.5, seed=d)[0]
    X = X[np.random.default_rng(d).permutation(len(X))]
    res = nnm.fit(X)
    assert (res.device_stats["tc_items"] > 0) == (d <= 29)
    m_or, a_or = orc.single_linkage(X)
    got = _records(res.merges)
    for f in FIELDS:
        assert np.array_equal(got[f], m_or[f]), (d, f)
    assert np.array_equal(res.assignments, a_or)
