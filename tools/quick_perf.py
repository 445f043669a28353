"""Quick device timing of the NNM path (development aid, not the bench)."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.engine import run_arrays

for spec in sys.argv[1:]:
    n, d, k = (int(v) for v in spec.split("x"))
    X = nnm.generate_synthetic(n, d, k, 1.0, seed=5)[0]
    t0 = time.time(); dd = _native.DeviceDataset(X); t1 = time.time()
    m, a, r, stop, c, st = run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN)
    t2 = time.time()
    pe = st["pairs_evaluated"]
    print(json.dumps({"n": n, "d": d, "upload_s": round(t1 - t0, 3), "run_s": round(t2 - t1, 3),
                      "eval_pairs_per_s": pe / (st["scan_ms"] / 1e3),
                      "tflops_alg": pe * 3 * d / (st["scan_ms"] / 1e3) / 1e12,
                      "covered_pairs_per_s": st["pairs_covered"] / (t2 - t1), **st}), flush=True)
