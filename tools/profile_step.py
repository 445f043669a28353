"""One device step of a bench config between cudaProfilerStart/Stop (ncu --profile-from-start off):
python tools/profile_step.py c4"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1402_3789_b200 as nnm  # noqa: E402
from paper_1402_3789_b200 import _native  # noqa: E402
from paper_1402_3789_b200.datagen import config_dataset  # noqa: E402
from paper_1402_3789_b200.engine import run_arrays  # noqa: E402

sys.path.insert(0, os.path.join(os.getcwd()))
from bench import CONFIGS  # noqa: E402

desc, cons, metric, data, P = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
dd = _native.DeviceDataset(config_dataset(data))
c = nnm.ConstraintSet(**cons)
m = nnm.MetricKind.parse(metric)
run_arrays(dd, c, P, m)
torch.cuda.synchronize()
torch.cuda.profiler.start()
out = run_arrays(dd, c, P, m)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(out[5])
