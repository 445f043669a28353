"""Per-dataset preparation (upload, kd view, geometry, tables) of a config, for ncu
(--profile-from-start off) and wall timing: python tools/profile_prep.py c4 [reps]."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1402_3789_b200 import _native
from paper_1402_3789_b200.datagen import config_dataset
X = config_dataset(sys.argv[1] if len(sys.argv) > 1 else "c4")
Xh = torch.from_numpy(X).pin_memory().numpy()
lib = _native.load()
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    torch.cuda.synchronize()
    prof = rep == 1
    if prof:
        torch.cuda.profiler.start()
    t0 = time.perf_counter()
    dd = _native.DeviceDataset(Xh)
    t1 = time.perf_counter()
    tp, rows = ctypes.c_int64(), ctypes.c_int64()
    _native.check(lib.nnm_bv_begin(dd.handle, 0, np.nan, ctypes.byref(tp), ctypes.byref(rows)))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if prof:
        torch.cuda.profiler.stop()
    print(f"create {1e3*(t1-t0):.2f} ms, bv_begin {1e3*(t2-t1):.2f} ms", flush=True)
    del dd
