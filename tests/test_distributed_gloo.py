"""Multi-process (gloo, CPU) tests of the multi-GPU exchange protocol.

paper_1402_3789_b200.distributed.boruvka_rounds is the production driver of the staged
pruned round (caps all-reduce MIN, key combine after phase 1, tile-pair cache all-reduce
MAX, key combine after phase 2).  Here it runs unchanged at world sizes 1, 2 and 4 over
gloo, with a numpy test double of the library's rank-local steps: identical item lists
on every rank, contiguous shares split as the library splits them, per-row top-2 keys
(fp32 bits << 32 | partner), component caps, a tile-pair lower-bound cache that prunes
the next round's phase-2 list, and a Kruskal replay.  Every rank of every world size
must produce the same merge log, labels and per-round item counts as world 1, and the
same total MST weight as a brute-force spanning tree.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

NONE = np.iinfo(np.int64).max


def _key(d32, j):
    return (int(np.array(d32, dtype=np.float32).view(np.uint32)) << 32) | int(j)


def _val(k):
    return float(np.array(np.uint32(k >> 32)).view(np.float32))


class NumpyBackend:
    """Test double of the library's staged round on a small point set (tiles of 8)."""

    def __init__(self, X, tile=8):
        self.X = np.asarray(X, dtype=np.float64)
        self.n = len(X)
        self.tile = tile
        self.T = -(-self.n // tile)
        self.comp = np.arange(self.n)
        self.edges = []
        self.cache = np.zeros(self.T * (self.T + 1) // 2)  # lower bounds of cross pairs
        self.D = np.sqrt(((self.X[:, None, :] - self.X[None, :, :]) ** 2).sum(-1)).astype(np.float32)
        self.items_log = []

    def _w(self, I, J):
        return I * self.T - I * (I - 1) // 2 + (J - I)

    def _pairs(self, I, J):
        for i in range(I * self.tile, min(self.n, (I + 1) * self.tile)):
            for j in range(J * self.tile, min(self.n, (J + 1) * self.tile)):
                if (I != J or i < j) and self.comp[i] != self.comp[j]:
                    yield i, j

    @staticmethod
    def _share(lst, rank, world):
        from paper_1402_3789_b200.distributed import shard_range

        lo, hi = shard_range(len(lst), rank, world)
        return lst[lo:hi]

    def _scan(self, items, b1, b2, caps=None):
        for I, J in items:
            lo = np.inf
            for i, j in self._pairs(I, J):
                d = self.D[i, j]
                lo = min(lo, d)
                for a, b in ((i, j), (j, i)):
                    if caps is not None and d > caps[self.comp[a]]:
                        continue
                    k = _key(d, b)
                    if k < b1[a]:
                        b1[a], b2[a] = k, b1[a]
                    elif k < b2[a] and k != b1[a]:
                        b2[a] = k
            w = self._w(I, J)
            if np.isfinite(lo):
                self.cache[w] = max(self.cache[w], lo)

    def components(self):
        return len(np.unique(self.comp))

    def same_single(self, I, J):
        ci = set(self.comp[I * self.tile:(I + 1) * self.tile])
        cj = set(self.comp[J * self.tile:(J + 1) * self.tile])
        return len(ci) == 1 and ci == cj

    def round_bound(self, rank, world):
        self.items1 = [(I, I) for I in range(self.T)] + [(I, I + 1) for I in range(self.T - 1)]
        self.items1 = sorted(it for it in self.items1 if not self.same_single(*it))
        caps = np.full(self.n, np.inf, dtype=np.float32)
        for I, J in self._share(self.items1, rank, world):
            for i, j in self._pairs(I, J):
                d = self.D[i, j]
                caps[self.comp[i]] = min(caps[self.comp[i]], d)
                caps[self.comp[j]] = min(caps[self.comp[j]], d)
        return caps.view(np.int32)  # fp32 bits: MIN over non-negative floats as integers

    def round_phase1(self, rank, world, caps):
        b1 = np.full(self.n, NONE, dtype=np.int64)
        b2 = b1.copy()
        cp = None if caps is None else np.asarray(caps).view(np.float32)
        self._scan(self._share(self.items1, rank, world), b1, b2, cp)
        return b1, b2

    def round_phase2(self, rank, world, g1, g2):
        b1, b2 = np.array(g1).copy(), np.array(g2).copy()
        ucomp = np.full(self.n, np.inf)
        for i in range(self.n):
            if b1[i] != NONE:
                ucomp[self.comp[i]] = min(ucomp[self.comp[i]], _val(int(b1[i])))
        umax = [max(ucomp[self.comp[i]] for i in range(I * self.tile, min(self.n, (I + 1) * self.tile)))
                for I in range(self.T)]
        p1 = set(self.items1)
        self.items2 = [(I, J) for I in range(self.T) for J in range(I, self.T)
                       if (I, J) not in p1 and not self.same_single(I, J)
                       and not self.cache[self._w(I, J)] > max(umax[I], umax[J])]
        self._scan(self._share(self.items2, rank, world), b1, b2)
        self._b1, self._b2 = b1, b2
        self.items_log.append((len(self.items1), len(self.items2)))
        self._all = self.items1 + self.items2
        if world == 1:
            return None
        self._buf = np.array([self.cache[self._w(I, J)] for I, J in self._all])
        return self._buf

    def cache_scatter(self):
        for (I, J), v in zip(self._all, self._buf):
            self.cache[self._w(I, J)] = v

    def keys(self):
        return self._b1, self._b2

    def copy(self, x):
        return np.array(x).copy()

    def second(self, b1, b2, g1):
        from paper_1402_3789_b200.distributed import combine_second

        return combine_second(np.asarray(b1), np.asarray(b2), np.asarray(g1))

    def finish_round(self, g1, g2):
        best = {}
        for i in range(self.n):
            k = int(g1[i])
            if k == NONE:
                continue
            j = k & 0xFFFFFFFF
            e = (_val(k), min(i, j), max(i, j))
            c = self.comp[i]
            if c not in best or e < best[c]:
                best[c] = e
        added = 0
        for d, a, b in sorted(set(best.values())):
            ca, cb = self.comp[a], self.comp[b]
            if ca == cb:
                continue
            keep, drop = min(ca, cb), max(ca, cb)
            self.comp[self.comp == drop] = keep
            self.edges.append((d, a, b))
            added += 1
        return added

    def end(self):
        par = np.arange(self.n)
        size = np.ones(self.n, dtype=np.int64)

        def find(x):
            while par[x] != x:
                x = par[x]
            return x

        log = []
        for d, a, b in sorted(self.edges):
            ra, rb = find(a), find(b)
            keep, drop = min(ra, rb), max(ra, rb)
            par[drop] = keep
            size[keep] += size[drop]
            log.append((keep, drop, d, int(size[keep]), a, b))
        return log, [find(i) for i in range(self.n)]


def _worker(rank, world, port, X, out):
    import torch
    import torch.distributed as dist

    from paper_1402_3789_b200.distributed import boruvka_rounds

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)

    def red(op):
        def f(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            dist.all_reduce(t, op=op)
            np.copyto(a, t.numpy())
        return f

    be = NumpyBackend(X)
    rounds = boruvka_rounds(be, rank, world, red(dist.ReduceOp.MIN), red(dist.ReduceOp.MAX))
    log, labels = be.end()
    out[rank] = (rounds, log, labels, be.items_log)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(X, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


@pytest.fixture(scope="module")
def points():
    rng = np.random.default_rng(7)
    centres = rng.uniform(-20, 20, size=(6, 3))
    X = np.vstack([c + rng.normal(size=(14, 3)) for c in centres])
    return X[rng.permutation(len(X))]


@pytest.fixture(scope="module")
def world1(points):
    return _run(points, 1)[0]


@pytest.mark.parametrize("world", [2, 4])
def test_protocol_world_sizes_identical(points, world1, world):
    res = _run(points, world)
    for r in range(world):
        assert res[r][0] == world1[0], r        # rounds
        assert res[r][1] == world1[1], r        # merge log (keep, drop, dist, size, a, b)
        assert res[r][2] == world1[2], r        # labels
        assert res[r][3] == world1[3], r        # per-round item counts (same lists everywhere)


def test_protocol_world1_is_a_spanning_tree(points, world1):
    from scipy.sparse.csgraph import minimum_spanning_tree

    n = len(points)
    D = np.sqrt(((points[:, None, :] - points[None, :, :]) ** 2).sum(-1)).astype(np.float32)
    mst = minimum_spanning_tree(D.astype(np.float64)).toarray()
    log = world1[1]
    assert len(log) == n - 1
    assert np.isclose(sum(e[2] for e in log), mst.sum(), rtol=1e-6)
    assert len(set(world1[2])) == 1


def test_shard_range_partitions_exactly():
    from paper_1402_3789_b200.distributed import shard_range

    for total in (0, 1, 7, 1000, 122078125):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
