"""A/B timing: runs each spec twice in-process (second run reported, dataset reused)."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.engine import run_arrays

for spec in sys.argv[1:]:
    n, d, k = (int(v) for v in spec.split("x"))
    X = nnm.generate_synthetic(n, d, k, 1.0, seed=5)[0]
    dd = _native.DeviceDataset(X)
    for rep in range(2):
        t1 = time.time()
        m, a, r, stop, c, st = run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN)
        t2 = time.time()
    pe = st["pairs_evaluated"]
    print(json.dumps({"spec": spec, "env": {k: v for k, v in os.environ.items() if k.startswith("NNM_")},
                      "run_s": round(t2 - t1, 3), "scan_s": round(st["scan_ms"] / 1e3, 3),
                      "eval_pairs_per_s": pe / (st["scan_ms"] / 1e3),
                      "frac_fp32": pe * 3 * d / (st["scan_ms"] / 1e3) / 74.3e12,
                      "pairs_evaluated": pe, "launches": st["kernel_launches"]}), flush=True)
