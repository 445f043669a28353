"""Functional test of the multi-process driver on the real kernels (@gpu).

Processes (torch.distributed, gloo) all drive device 0 through
paper_1402_3789_b200.distributed.run_boruvka_distributed: each rank runs the staged
pruned round on its shares (nnm_bv_round_bound / _phase1 / _phase2), the caps, keys
and this round's tile-pair cache entries are combined with all-reduces, and every rank
finishes the rounds identically.  The merge log and labels must equal the
single-process run byte for byte on every rank, and the ranks' evaluated pairs must add
up to the single run's (every item scanned by exactly one rank).  The ranks share one
GPU and only the host orchestrates the exchanges (no kernel waits on another); this
checks correctness of the sharded path, not timing.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, X, kwargs, out):
    import torch
    import torch.distributed as dist

    os.environ["NNM_DEVICE"] = "0"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_1402_3789_b200.distributed import run_boruvka_distributed

    merges, assign, rounds, stop, stats = run_boruvka_distributed(X, **kwargs)
    out[rank] = (merges.tobytes(), assign.tobytes(), rounds, stop, stats["pairs_evaluated"])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kwargs", [{}, {"dmax": 4.0}, {"metric": "manhattan"}])
def test_multi_rank_pruned_run_equals_single(kwargs, world):
    import torch.multiprocessing as mp

    import paper_1402_3789_b200 as nnm

    X = nnm.generate_synthetic(12000, 25, 40, 1.0, seed=31)[0]
    X = X[np.random.default_rng(5).permutation(len(X))]
    single = nnm.fit(X, **kwargs)
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, kwargs, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    want_m = single.merges.array.tobytes()
    want_a = single.assignments.tobytes()
    for r in range(world):
        m, a, rounds, stop, _ = out[r]
        assert m == want_m, r
        assert a == want_a, r
        assert stop == single.stop_reason
    # every phase-1 / phase-2 item was scanned by exactly one rank
    assert sum(out[r][4] for r in range(world)) == single.device_stats["pairs_evaluated"]


def test_tile_pair_cache_on_off_identical():
    """The tile-pair bound cache only prunes: NNM_TPCACHE=0 gives the same merge log and
    labels, and evaluates at least as many pairs."""
    import subprocess
    import sys

    from nnm_testutil import ROOT

    code = ("import hashlib, numpy as np, paper_1402_3789_b200 as nnm\n"
            "X = nnm.generate_synthetic(20000, 25, 60, 1.0, seed=8)[0]\n"
            "r = nnm.fit(X)\n"
            "print(hashlib.sha256(r.merges.array.tobytes() + r.assignments.tobytes()).hexdigest(),"
            " r.device_stats['pairs_evaluated'])\n")
    outs = []
    for flag in ("1", "0"):
        env = dict(os.environ, NNM_TPCACHE=flag)
        p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(p.stdout.split())
    assert outs[0][0] == outs[1][0]
    assert float(outs[1][1]) >= float(outs[0][1])
