"""Full-scale parity goldens for the BASELINE configs (SURVEY.md 8(c) "Parity at 500k/2M").

Run HERE (CPU container; hours of 8-core time, so one step at a time):

    python tests/golden/make_scale_golden.py c3 c4sub c5msub c5csub c2 c4top

Inputs come from ``paper_1402_3789_b200.datagen.config_dataset``, the restatement
of ``parclust.dataio.generate_synthetic`` (dataio.py:124-145) pinned bit-exact by
``tests/golden/synthetic_sha256.csv``.  Results come from the C oracle port
(``oracle/nnm_oracle.c``: ``orc_run`` restates engine.run, engine.py:154-199,
with order_batch / process_batch :73-143 and global_top_p, pairgen.py:319-324),
which ``tests/test_oracle_pin.py`` pins against the imported reference (48
``global_top_p`` cases, 40 ``engine.run`` cases with rounds and counters, the full
C1 run and a 3k C2 analogue).  The oracle is the checker, never the product.

Each step writes ``tests/golden/scale/<name>.json``: the exact call, the merge
count, stop reason, rounds (and the full per-round counters for the kl4 run, where
rounds are part of parity), sha256 digests of every merge field and of
the labels, and a strided sample of merge records for diagnosis.  Raw outputs are
not committed (2M merges are 112 MB).

Steps (P is part of the contract only with kl4; without it the merge list is
P-invariant, SURVEY F3 / test_acceptance.py:159-171, so the oracle runs with a
large P to finish in few rounds):
  c3     C3 500k x 25, dmax=5, full run (P=2^23)
  c4sub  C4 X[::10] (200k x 25) euclidean, full dendrogram (P=2^18)
  c5msub C4 X[::10] manhattan, full dendrogram
  c5csub C4 X[::10] chebyshev, full dendrogram
  c2     C2 100k x 25, kl1=400 kl2=300 kl3=450 kl4=150, P=256 (rounds + counters)
  c2nokl4  C2's X with kl1=400 kl2=300 kl3=450 (no kl4; merge list P-invariant, P=4096)
  c4top  C4 2M x 25 round-1 global_top_p with P=256 (singleton snapshot)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import nnm_oracle as orc  # noqa: E402
from paper_1402_3789_b200.datagen import config_dataset  # noqa: E402

OUT = os.path.join(HERE, "scale")
FIELDS = ("root_a", "root_b", "dist", "new_size", "point_a", "point_b")
SUB_STRIDE = 10


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def merge_digests(merges, assign) -> dict:
    out = {f: digest(merges[f]) for f in FIELDS}
    out["assignments"] = digest(assign)
    return out


def sample(merges, k: int = 64) -> list:
    m = len(merges)
    if m == 0:
        return []
    idx = sorted(set(np.linspace(0, m - 1, k).astype(np.int64).tolist()))
    return [[int(i)] + [float(merges[i]["dist"]) if f == "dist" else int(merges[i][f])
                        for f in FIELDS] for i in idx]


RUNS = {
    "c3": dict(config="c3", stride=1, metric="euclidean", cons=dict(dmax=5.0), P=1 << 23),
    "c4sub": dict(config="c4", stride=SUB_STRIDE, metric="euclidean", cons={}, P=1 << 18),
    "c5msub": dict(config="c4", stride=SUB_STRIDE, metric="manhattan", cons={}, P=1 << 18),
    "c5csub": dict(config="c4", stride=SUB_STRIDE, metric="chebyshev", cons={}, P=1 << 18),
    "c2": dict(config="c2", stride=1, metric="euclidean",
               cons=dict(kl1=400, kl2=300, kl3=450, kl4=150), P=256),
    # kl2/kl3 without kl4: P-invariant merge list (F3), so the oracle takes P = 4096
    "c2nokl4": dict(config="c2", stride=1, metric="euclidean",
                    cons=dict(kl1=400, kl2=300, kl3=450), P=4096),
}


def run_step(name: str) -> dict:
    if name == "c4top":
        X = config_dataset("c4")
        n = X.shape[0]
        t0 = time.time()
        d, a, b = orc.top_p(X, np.arange(n, dtype=np.int64), np.ones(n, dtype=np.int64), 256)
        return {"name": name, "config": "c4", "stride": 1, "metric": "euclidean", "P": 256,
                "call": "global_top_p(singleton snapshot of C4, P=256) == orc_top_p",
                "dist": [float(v) for v in d], "a": [int(v) for v in a], "b": [int(v) for v in b],
                "oracle_seconds": time.time() - t0, "threads": os.cpu_count()}
    spec = RUNS[name]
    X = np.ascontiguousarray(config_dataset(spec["config"])[:: spec["stride"]])
    t0 = time.time()
    r = orc.run(X, metric=spec["metric"], P=spec["P"], **spec["cons"])
    out = {"name": name, "config": spec["config"], "stride": spec["stride"], "n": int(X.shape[0]),
           "d": int(X.shape[1]), "metric": spec["metric"], "constraints": spec["cons"],
           "P": spec["P"], "call": "orc_run (engine.run semantics)",
           "n_merges": int(len(r.merges)), "stop_reason": r.stop_reason, "rounds": int(r.rounds),
           "digests": merge_digests(r.merges, r.assignments), "sample": sample(r.merges),
           "n_clusters": int(np.unique(r.assignments).shape[0]),
           "oracle_seconds": time.time() - t0, "threads": os.cpu_count()}
    if "kl4" in spec["cons"]:  # rounds and counters are part of parity
        out["round_digest"] = digest(r.merges["round"])
        out["counters"] = [[int(v) for v in row] for row in r.round_counters.tolist()]
    return out


def main(argv):
    os.makedirs(OUT, exist_ok=True)
    orc.load()
    for name in argv or ["c3", "c4sub", "c5msub", "c5csub", "c2", "c4top"]:
        t0 = time.time()
        res = run_step(name)
        with open(os.path.join(OUT, f"{name}.json"), "w") as f:
            json.dump(res, f, indent=1)
        print(f"{name}: {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
