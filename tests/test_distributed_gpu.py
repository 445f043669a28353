"""Functional test of the multi-GPU driver on the real kernels (@gpu).

Two processes (torch.distributed, gloo) both drive device 0 through
paper_1402_3789_b200.distributed.run_boruvka_distributed: each rank runs the
pruned scan on its phase-2 share (nnm_bv_scan_pruned), the keys are combined with
two all-reduce(MIN), and every rank finishes the rounds identically.  The merge log
and labels must equal the single-process run byte for byte, on both ranks.  This
checks correctness of the sharded path only (the ranks share one GPU; no timing).
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


@pytest.mark.parametrize("kwargs", [{}, {"dmax": 4.0}, {"metric": "manhattan"}])
def test_two_rank_pruned_run_equals_single(kwargs):
    import torch.multiprocessing as mp

    import paper_1402_3789_b200 as nnm

    X = nnm.generate_synthetic(12000, 25, 40, 1.0, seed=31)[0]
    X = X[np.random.default_rng(5).permutation(len(X))]
    single = nnm.fit(X, **kwargs)
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, X, kwargs, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    want_m = single.merges.array.tobytes()
    want_a = single.assignments.tobytes()
    for r in range(2):
        m, a, rounds, stop, _ = out[r]
        assert m == want_m, r
        assert a == want_a, r
        assert stop == single.stop_reason
