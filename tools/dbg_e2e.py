"""Timing breakdown of one end-to-end call (paper_1402_3789_b200.run on host arrays)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1402_3789_b200 as nnm  # noqa: E402
from paper_1402_3789_b200 import _native  # noqa: E402
from paper_1402_3789_b200.datagen import config_dataset  # noqa: E402
from paper_1402_3789_b200.engine import run_arrays  # noqa: E402

X = config_dataset(sys.argv[1] if len(sys.argv) > 1 else "c4")
Xp = torch.from_numpy(X).pin_memory().numpy()
for it in range(4):
    if it == 3:
        os.environ["NNM_DEBUG"] = "1"
    t0 = time.perf_counter()
    ds = nnm.Dataset(values=Xp)
    t1 = time.perf_counter()
    dd = _native.device_dataset(ds)
    t2 = time.perf_counter()
    out = run_arrays(dd, nnm.ConstraintSet(), 256, nnm.MetricKind.EUCLIDEAN)
    t3 = time.perf_counter()
    print(f"dataset {1e3*(t1-t0):.1f} ms, device_dataset {1e3*(t2-t1):.1f} ms, run {1e3*(t3-t2):.1f} ms "
          f"(total_ms {out[5]['total_ms']:.1f}, prep {out[5]['prep_ms']:.1f}, replay {out[5]['replay_ms']:.1f})",
          flush=True)
    del dd, ds
