import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1402_3789_b200 as nnm
for n in (1, 2, 5, 60, 300):
    X = np.random.default_rng(n).normal(size=(n, 3))
    try:
        r = nnm.fit(X)
        print(n, 'ok', len(r.merges), flush=True)
    except Exception as e:
        print(n, 'ERR', e, flush=True)
        break
