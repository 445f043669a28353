"""Repeat the bench's e2e call (run(Dataset(X_pinned))) and split each call's time."""
import sys, os, time, json, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.datagen import config_dataset
from paper_1402_3789_b200.engine import run_arrays
X = config_dataset(sys.argv[1] if len(sys.argv) > 1 else "c4")
Xh = torch.from_numpy(X).pin_memory().numpy()
if os.environ.get("NOGC"):
    gc.disable()
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    t = [time.perf_counter()]
    ds = nnm.Dataset(values=Xh); t.append(time.perf_counter())
    dd = _native.device_dataset(ds); t.append(time.perf_counter())
    m, a, r, stop, c, st = run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN); t.append(time.perf_counter())
    _ = float(m["dist"][-1]) + int(a[-1]); t.append(time.perf_counter())
    del ds, dd; t.append(time.perf_counter())
    print(json.dumps({"validate": round(t[1]-t[0], 4), "create": round(t[2]-t[1], 4), "run": round(t[3]-t[2], 4),
                      "touch": round(t[4]-t[3], 4), "destroy": round(t[5]-t[4], 4), "dev_total_ms": st["total_ms"],
                      "replay_ms": st["replay_ms"], "scan_ms": round(st["scan_ms"], 1)}), flush=True)
