import os, sys
sys.path.insert(0, os.getcwd())
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.datagen import config_dataset
from paper_1402_3789_b200.engine import run_arrays
X = config_dataset(sys.argv[1] if len(sys.argv) > 1 else "c4")
dd = _native.DeviceDataset(X)
run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN)
os.environ["NNM_TC_TRACE"] = "gpurun_out/tc_trace.txt"
run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN)
