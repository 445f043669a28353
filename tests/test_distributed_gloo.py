"""Multi-process (world_size 2, gloo, CPU) test of the multi-GPU sharding logic.

The per-rank scan is emulated on the CPU by a numpy test double that produces
the same per-row keys the GPU kernel does over a tile-pair range
(fp32 bits << 32 | partner).  The test checks that the tile-pair partition
covers every pair exactly once and that the two all-reduce(MIN) steps of
paper_1402_3789_b200.distributed reproduce the single-rank best / second-best
keys exactly, for every world size.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

TILE = 128


def _decode(w, T):
    i = 0
    while (i + 1) * T - (i + 1) * i // 2 <= w:
        i += 1
    return i, i + (w - (i * T - i * (i - 1) // 2))


def _scan_range(X, lo, hi):
    """CPU test double of the GPU scan over tile pairs [lo, hi): per-row top-2 keys."""
    n = X.shape[0]
    T = (n + TILE - 1) // TILE
    none = np.iinfo(np.int64).max
    keys = [[] for _ in range(n)]
    for w in range(lo, hi):
        I, J = _decode(w, T)
        for i in range(I * TILE, min(n, (I + 1) * TILE)):
            for j in range(J * TILE, min(n, (J + 1) * TILE)):
                if I == J and j <= i:
                    continue
                v = np.float32(((X[i] - X[j]) ** 2).sum())
                bits = int(np.array(v, dtype=np.float32).view(np.uint32))
                keys[i].append((bits << 32) | j)
                keys[j].append((bits << 32) | i)
    b1 = np.full(n, none, np.int64)
    b2 = np.full(n, none, np.int64)
    for i, ks in enumerate(keys):
        ks = sorted(ks)
        if ks:
            b1[i] = ks[0]
        if len(ks) > 1:
            b2[i] = ks[1]
    return b1, b2


def _worker(rank, world, port, X, out):
    import torch
    import torch.distributed as dist

    from paper_1402_3789_b200.distributed import combine_second, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = X.shape[0]
    T = (n + TILE - 1) // TILE
    lo, hi = shard_range(T * (T + 1) // 2, rank, world)
    b1, b2 = _scan_range(X, lo, hi)
    g1 = torch.from_numpy(b1.copy())
    dist.all_reduce(g1, op=dist.ReduceOp.MIN)
    c2 = combine_second(torch.from_numpy(b1), torch.from_numpy(b2), g1)
    dist.all_reduce(c2, op=dist.ReduceOp.MIN)
    out[rank] = (g1.numpy().copy(), c2.numpy().copy(), hi - lo)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_two_rank_allreduce_reproduces_single_rank_keys(world):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(7)
    X = rng.integers(-3, 4, size=(300, 3)).astype(np.float64)  # many exact ties
    T = (300 + TILE - 1) // TILE
    ref1, ref2 = _scan_range(X, 0, T * (T + 1) // 2)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert sum(out[r][2] for r in range(world)) == T * (T + 1) // 2
    for r in range(world):
        assert np.array_equal(out[r][0], ref1)
        assert np.array_equal(out[r][1], ref2)


def test_shard_range_partitions_exactly():
    from paper_1402_3789_b200.distributed import shard_range

    for total in (0, 1, 7, 1000, 122078125):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
