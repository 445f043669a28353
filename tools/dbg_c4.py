import os, sys, time, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.datagen import config_dataset
from paper_1402_3789_b200.engine import run_arrays
X = config_dataset("c4")
dd = _native.DeviceDataset(X)
cons = nnm.ConstraintSet()
for i in range(3):
    if i == 2: os.environ["NNM_DEBUG"] = "1"
    t = time.time(); r = run_arrays(dd, cons, 256, nnm.MetricKind.EUCLIDEAN); dt = time.time() - t
    print(i, dt, {k: r[5][k] for k in ("total_ms", "scan_ms", "replay_ms", "prep_ms")}, flush=True)
