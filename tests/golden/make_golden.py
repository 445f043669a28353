"""Generate golden fixtures by importing the reference (parclust) in this container.

Run here (not on the GPU box; /root/reference only exists in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Every fixture records the exact reference call
that produced it, so tests can replay the same inputs through the oracle and
the CUDA path.  Reference call sites: metrics.internal_pairwise
(metrics.py:67-73), pairgen.global_top_p (pairgen.py:319-324), engine.run
(engine.py:154-199), oracle.oracle_single_linkage (oracle.py:59-107),
dataio.generate_synthetic (dataio.py:124-145).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from parclust import dataio, engine, metrics, oracle, pairgen  # noqa: E402
from parclust.model import ClusterForest, ConstraintSet, Dataset  # noqa: E402
from parclust.scheduler import PipelineConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
METRICS = ["euclidean", "squared-euclidean", "manhattan", "chebyshev"]
SERIAL = PipelineConfig(managers=1, workers_per_manager=1, input_buffers=1)


def _opt(v):
    return -1 if v is None else int(v)


def metric_tiles():
    rng = np.random.default_rng(101)
    out = {}
    idx = 0
    for d in (1, 3, 8, 25):
        for scale in (1e-3, 1.0, 1e3):
            for m in METRICS:
                x = rng.normal(size=(7, d)) * scale + rng.uniform(-100, 100, size=(1, d))
                y = rng.normal(size=(9, d)) * scale + rng.uniform(-100, 100, size=(1, d))
                D = metrics.internal_pairwise(metrics.MetricKind.parse(m), x, y)
                out[f"x_{idx}"] = x
                out[f"y_{idx}"] = y
                out[f"D_{idx}"] = D
                out[f"metric_{idx}"] = np.array(m)
                idx += 1
    out["count"] = np.array(idx)
    np.savez_compressed(os.path.join(OUT, "metric_tiles.npz"), **out)


def _random_forest(rng, n, merges):
    f = ClusterForest(n)
    for _ in range(merges):
        a, b = rng.integers(0, n, size=2)
        if f.find(int(a)) != f.find(int(b)):
            f.union(int(a), int(b))
    return f


def topp_cases():
    rng = np.random.default_rng(202)
    out = {}
    idx = 0
    for _ in range(48):
        n = int(rng.integers(2, 160))
        d = int(rng.integers(1, 9))
        m = METRICS[idx % 4]
        if idx % 5 == 0:
            X = rng.integers(-3, 4, size=(n, d)).astype(np.float64)  # heavy ties
        else:
            X = rng.normal(size=(n, d)) * 3.0
        f = _random_forest(rng, n, int(rng.integers(0, n)))
        kl2 = int(rng.integers(1, 6)) if rng.random() < 0.4 else None
        kl3 = (kl2 or 1) + int(rng.integers(1, 8)) if rng.random() < 0.4 else None
        dmax = float(rng.uniform(0.0, 4.0)) if rng.random() < 0.4 else None
        P = int(rng.choice([1, 2, 3, 7, 40, 10000]))
        con = ConstraintSet(kl2=kl2, kl3=kl3, dmax=dmax)
        kind = metrics.MetricKind.parse(m)
        snap = pairgen.make_snapshot(f, con, kind)
        ds = Dataset(values=X)
        plan = pairgen.plan_blocks(n, int(rng.integers(1, 5)))
        buf = pairgen.global_top_p(ds, snap, plan, P)
        out[f"X_{idx}"] = X
        out[f"roots_{idx}"] = snap.roots
        out[f"sizes_{idx}"] = snap.size_by_point
        out[f"args_{idx}"] = np.array([_opt(kl2), _opt(kl3), P])
        out[f"thr_{idx}"] = np.array(np.nan if snap.threshold is None else snap.threshold)
        out[f"metric_{idx}"] = np.array(m)
        out[f"dist_{idx}"] = buf.dist
        out[f"a_{idx}"] = buf.a
        out[f"b_{idx}"] = buf.b
        idx += 1
    out["count"] = np.array(idx)
    np.savez_compressed(os.path.join(OUT, "topp_cases.npz"), **out)


def _pack_run(res):
    m = np.array(
        [(e.step, e.round, e.root_a, e.root_b, e.dist, e.new_size, e.point_a, e.point_b)
         for e in res.merges],
        dtype=[("step", np.int64), ("round", np.int64), ("root_a", np.int64),
               ("root_b", np.int64), ("dist", np.float64), ("new_size", np.int64),
               ("point_a", np.int64), ("point_b", np.int64)],
    )
    keys = ("round", "selected", "merged", "same_root", "kl2", "kl3", "unprocessed")
    rc = np.array([[c[k] for k in keys] for c in res.round_counters], dtype=np.int64).reshape(
        -1, len(keys))
    return m, rc


def run_cases():
    rng = np.random.default_rng(303)
    out = {}
    idx = 0
    for _ in range(40):
        n = int(rng.integers(1, 120))
        d = int(rng.integers(1, 6))
        m = METRICS[idx % 4]
        if idx % 6 == 0:
            X = rng.integers(-2, 3, size=(n, d)).astype(np.float64)
        else:
            X = rng.normal(size=(n, d)) * 2.0
        kl1 = int(rng.integers(1, max(2, n // 3))) if rng.random() < 0.4 else None
        kl2 = int(rng.integers(1, 8)) if rng.random() < 0.4 else None
        kl3 = (kl2 or 1) + int(rng.integers(1, 10)) if rng.random() < 0.4 else None
        kl4 = int(rng.integers(1, 6)) if rng.random() < 0.4 else None
        dmax = float(rng.uniform(0.0, 3.0)) if rng.random() < 0.3 else None
        P = int(rng.choice([1, 3, 7, 64, 100000]))
        con = ConstraintSet(kl1=kl1, kl2=kl2, kl3=kl3, kl4=kl4, dmax=dmax)
        res = engine.run(Dataset(values=X), engine.RunConfig(
            constraints=con, pairs_per_batch=P, metric=metrics.MetricKind.parse(m),
            pipeline=SERIAL))
        mg, rc = _pack_run(res)
        out[f"X_{idx}"] = X
        out[f"cons_{idx}"] = np.array([_opt(kl1), _opt(kl2), _opt(kl3), _opt(kl4), P])
        out[f"dmax_{idx}"] = np.array(np.nan if dmax is None else dmax)
        out[f"metric_{idx}"] = np.array(m)
        out[f"merges_{idx}"] = mg
        out[f"assign_{idx}"] = res.assignments
        out[f"rounds_{idx}"] = np.array(res.rounds)
        out[f"stop_{idx}"] = np.array(res.stop_reason)
        out[f"counters_{idx}"] = rc
        if n <= 5000 and kl4 is None:
            ores = oracle.oracle_single_linkage(Dataset(values=X), con, metrics.MetricKind.parse(m))
            om, _ = _pack_run(engine.RunResult(ores.merges, ores.assignments, 0, "", None, []))
            out[f"flat_{idx}"] = om
        idx += 1
    out["count"] = np.array(idx)
    np.savez_compressed(os.path.join(OUT, "run_cases.npz"), **out)


def config_runs():
    """Full-run goldens on BASELINE config shapes the reference completes here."""
    # C1: generate_synthetic(10_000, 8, 5, 1.0, seed=1), unconstrained, P=256
    ds, _ = dataio.generate_synthetic(10_000, 8, 5, 1.0, seed=1)
    res = engine.run(ds, engine.RunConfig(pairs_per_batch=256))
    mg, rc = _pack_run(res)
    np.savez_compressed(os.path.join(OUT, "c1_run.npz"), merges=mg, assign=res.assignments,
                        rounds=np.array(res.rounds), stop=np.array(res.stop_reason),
                        counters=rc)
    # C2 analogue at 3k points: dense + diffuse blobs, kl1..kl4, P=256
    a, _ = dataio.generate_synthetic(2400, 25, 6, 1.0, seed=2)
    b, _ = dataio.generate_synthetic(600, 25, 12, 3.0, seed=3)
    X = np.vstack([a.values, b.values])
    con = ConstraintSet(kl1=12, kl2=300, kl3=450, kl4=150)
    res = engine.run(Dataset(values=X), engine.RunConfig(constraints=con, pairs_per_batch=256))
    mg, rc = _pack_run(res)
    np.savez_compressed(os.path.join(OUT, "c2_small_run.npz"), X=X, merges=mg,
                        assign=res.assignments, rounds=np.array(res.rounds),
                        stop=np.array(res.stop_reason), counters=rc)


def synthetic_hashes():
    """dataio.generate_synthetic bit patterns, so the in-repo generator can be pinned."""
    rows = []
    for (n, d, k, s, seed) in [(10_000, 8, 5, 1.0, 1), (3000, 25, 6, 1.0, 2), (777, 3, 4, 2.5, 9),
                               (50_000, 25, 100, 1.0, 4)]:
        ds, labels = dataio.generate_synthetic(n, d, k, s, seed)
        h = hashlib.sha256(ds.values.tobytes()).hexdigest()
        hl = hashlib.sha256(labels.tobytes()).hexdigest()
        rows.append(f"{n},{d},{k},{s},{seed},{h},{hl}")
    with open(os.path.join(OUT, "synthetic_sha256.csv"), "w") as fh:
        fh.write("n,d,clusters,spread,seed,values_sha256,labels_sha256\n")
        fh.write("\n".join(rows) + "\n")


if __name__ == "__main__":
    which = sys.argv[1:] or ["metric", "topp", "run", "config", "synth"]
    if "metric" in which:
        metric_tiles()
    if "topp" in which:
        topp_cases()
    if "run" in which:
        run_cases()
    if "synth" in which:
        synthetic_hashes()
    if "config" in which:
        config_runs()
    print("golden fixtures written to", OUT)
