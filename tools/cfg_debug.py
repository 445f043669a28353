"""One run of a bench config with NNM_DEBUG output: python tools/cfg_debug.py c5m"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.datagen import config_dataset
from paper_1402_3789_b200.engine import run_arrays
from bench import CONFIGS
desc, cons, metric, data, P = CONFIGS[sys.argv[1]]
dd = _native.DeviceDataset(config_dataset(data))
for _ in range(2):
    out = run_arrays(dd, nnm.ConstraintSet(**cons), P, nnm.MetricKind.parse(metric))
    print({k: out[5][k] for k in ("scan_ms", "total_ms", "pairs_evaluated", "scans")}, flush=True)
