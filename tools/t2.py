import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.datagen import config_dataset
from paper_1402_3789_b200.engine import run_arrays
cfg, small = sys.argv[1], sys.argv[2]
os.environ["NNM_SMALL"] = small
X = config_dataset(cfg)
dd = _native.DeviceDataset(X)
for i in range(3):
    t = time.time(); r = run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN); dt = time.time() - t
    print(cfg, small, i, round(dt * 1e3, 2), "ms", round(r[5]["total_ms"], 2), round(r[5]["scan_ms"], 2),
          r[5]["boruvka_rounds"], round(r[5]["replay_ms"], 2), r[5]["pairs_evaluated"], flush=True)
