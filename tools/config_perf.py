"""Time the BASELINE configs through run_arrays (development aid)."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.datagen import config_dataset
from paper_1402_3789_b200.engine import run_arrays

CONS = {"c1": {}, "c2": dict(kl1=400, kl2=300, kl3=450, kl4=150), "c3": dict(dmax=5.0),
        "c4": {}, "c5m": {}, "c5c": {}}
MET = {"c5m": "manhattan", "c5c": "chebyshev"}
for name in sys.argv[1:]:
    X = config_dataset(name[:2] if name.startswith("c5") else name)
    dd = _native.DeviceDataset(X)
    metric = nnm.MetricKind.parse(MET.get(name, "euclidean"))
    for rep in range(2):
        t0 = time.time()
        m, a, r, stop, c, st = run_arrays(dd, nnm.ConstraintSet(**CONS[name]), 256, metric)
        t1 = time.time()
    print(json.dumps({"config": name, "n": X.shape[0], "run_s": round(t1 - t0, 3), "rounds": r,
                      "merges": len(m), "stop": stop, "scan_s": st["scan_ms"] / 1e3,
                      "path": st["path"], "pairs_evaluated": st["pairs_evaluated"],
                      "launches": st["kernel_launches"]}), flush=True)
