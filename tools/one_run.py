"""One warm-up clustering of a config, then one measured run (ncu launch-list target)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.datagen import config_dataset
from paper_1402_3789_b200.engine import run_arrays
X = config_dataset(sys.argv[1] if len(sys.argv) > 1 else "c4")
dd = _native.DeviceDataset(X)
for _ in range(2):
    st = run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN)[5]
print(json.dumps(st))
