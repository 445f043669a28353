"""Run C1 (or a config) through fit() a few times -- for ncu captures of the small path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_3789_b200 as nnm
from paper_1402_3789_b200.datagen import config_dataset
X = config_dataset(sys.argv[1] if len(sys.argv) > 1 else "c1")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    r = nnm.fit(X)
    print(r.device_stats["scan_ms"], r.device_stats["total_ms"], r.rounds, flush=True)
