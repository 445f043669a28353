import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200.datagen import config_dataset
X = config_dataset("c2")
nnm.fit(X[:2000], kl1=4, kl2=300, kl3=450)
for P in (4096, 8192, 16384, 32768):
    os.environ["NNM_FAST_P"] = str(P)
    t = time.time(); r = nnm.fit(X, kl1=400, kl2=300, kl3=450); dt = time.time() - t
    print(P, r.rounds, round(dt, 3), r.device_stats["round_rescans"], round(r.device_stats["scan_ms"], 1), flush=True)
