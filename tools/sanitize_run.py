"""Small runs through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): TC Boruvka scan (euclidean), FP32 scans (manhattan, chebyshev), dmax, the
round path (kl1..kl4), top-P, pairwise, the GPU merge replay (forced on a small input)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_1402_3789_b200 as nnm  # noqa: E402

X = nnm.generate_synthetic(3000, 25, 12, 1.0, seed=5)[0]
for metric in ("euclidean", "manhattan", "chebyshev"):
    r = nnm.fit(X, metric=metric)
    print(metric, len(r.merges), r.device_stats["tc_items"], flush=True)
r = nnm.fit(X, dmax=4.0)
print("dmax", len(r.merges), r.stop_reason, flush=True)
r = nnm.fit(X[:1500], kl1=5, kl2=80, kl3=120, kl4=20, pairs_per_batch=64)
print("rounds", len(r.merges), r.rounds, flush=True)
Y = nnm.generate_synthetic(40000, 8, 20, 1.0, seed=3)[0]  # >= 32768 merges: GPU replay
r = nnm.fit(Y)
print("replay", len(r.merges), r.device_stats["replay_gpu_merges"], flush=True)
from paper_1402_3789_b200.metrics import MetricKind, internal_pairwise  # noqa: E402
print("pairwise", internal_pairwise(MetricKind.EUCLIDEAN, X[:50], X[50:90]).shape, flush=True)
