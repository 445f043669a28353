"""Where does end-to-end time go (host API) for a config?"""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.datagen import config_dataset
from paper_1402_3789_b200.engine import run_arrays
X = config_dataset(sys.argv[1] if len(sys.argv) > 1 else "c4")
Xh = torch.from_numpy(X).pin_memory().numpy()
for rep in range(2):
    t = [time.perf_counter()]
    ds = nnm.Dataset(values=Xh); t.append(time.perf_counter())
    dd = _native.DeviceDataset(ds.values); t.append(time.perf_counter())
    m, a, r, stop, c, st = run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN); t.append(time.perf_counter())
    m2, a2, r2, stop2, c2, st2 = run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN); t.append(time.perf_counter())
    log = nnm.engine.MergeLog(m); _ = len(log); t.append(time.perf_counter())
    print(json.dumps({"dataset_validate_s": t[1]-t[0], "upload_prepare_s": t[2]-t[1], "first_run_s": t[3]-t[2],
                      "second_run_s": t[4]-t[3], "mergelog_s": t[5]-t[4], "first_total_ms": st["total_ms"],
                      "second_total_ms": st2["total_ms"], "scan_ms": st2["scan_ms"]}), flush=True)
