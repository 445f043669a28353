"""Multi-GPU Boruvka driver: one process per GPU, torch.distributed for plumbing.

Partitioning: every rank holds the whole dataset (X64 +
FP32 tiles + tensor-core operand image).  Each Boruvka round is the staged pruned round
of the library (include/nnm.h, nnm_bv_round_*): both tile-pair item lists of the round
(phase 1: each tile's seed tiles; phase 2: every tile pair whose rigorous lower bound can
still reach a component bound) are derived identically on every rank, and every rank
scans a contiguous 1/world share of each.  Four exchanges per round, all small:

    caps   all-reduce MIN   per-component upper bounds from the bound pass   (4 B/row)
    keys   2 x all-reduce MIN  after phase 1: B1 = min_r B1_r,
                               B2 = min_r (B1_r == B1 ? B2_r : B1_r)           (16 B/row)
    cache  all-reduce MAX   this round's tile-pair cache entries only       (4 B/item)
    keys   2 x all-reduce MIN  after phase 2                                 (16 B/row)

(keys are u64 = fp32 bits << 32 | partner; NONE = INT64_MAX so signed and unsigned MIN
agree).  Every rank then finishes the round (FP64 certification, component minima,
hooking, pointer jumping) redundantly and deterministically, so labels and the merge log
are byte-identical on every rank and for every world size.

The protocol (`boruvka_rounds`) is written against a small backend interface so that the
CPU test double in tests/test_distributed_gloo.py runs the same exchange code with the
gloo backend at world sizes 1, 2 and 4.  In one process, `engine.run` with
RunConfig(n_gpus=N) reaches N GPUs through nnm_run_multi, where the same exchanges are
kernels reading the replicas' buffers through peer memory.
"""

from __future__ import annotations

import ctypes

import numpy as np

__all__ = ["shard_range", "combine_second", "boruvka_rounds", "LibBackend",
           "run_boruvka_distributed", "run_boruvka_distributed_handle"]


class _DeviceArray:
    """A library-owned device buffer seen through __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous equal-count share of [0, total) for `rank` (the library's split)."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi


def combine_second(b1_local, b2_local, b1_global):
    """Per-rank contribution to the global second-best key (numpy or torch arrays)."""
    if isinstance(b1_local, np.ndarray):
        return np.where(b1_local == b1_global, b2_local, b1_local)
    import torch

    return torch.where(b1_local == b1_global, b2_local, b1_local)


def boruvka_rounds(backend, rank: int, world: int, allreduce_min, allreduce_max) -> int:
    """The staged pruned Boruvka rounds with their four exchanges (module docstring).

    `backend` provides the rank-local steps (LibBackend on a GPU, a numpy double in the
    tests); `allreduce_min` / `allreduce_max` reduce an array in place across ranks.
    Returns the number of rounds run."""
    rounds = 0
    while backend.components() > 1:
        caps = backend.round_bound(rank, world)
        if caps is not None:
            allreduce_min(caps)
        b1, b2 = backend.round_phase1(rank, world, caps)
        g1, g2 = _combine_keys(backend, b1, b2, allreduce_min)
        cache = backend.round_phase2(rank, world, g1, g2)
        if cache is not None:
            allreduce_max(cache)
            backend.cache_scatter()
        b1, b2 = backend.keys()
        g1, g2 = _combine_keys(backend, b1, b2, allreduce_min)
        rounds += 1
        if backend.finish_round(g1, g2) == 0:
            break
    return rounds


def _combine_keys(backend, b1, b2, allreduce_min):
    g1 = backend.copy(b1)
    allreduce_min(g1)
    c2 = backend.second(b1, b2, g1)
    allreduce_min(c2)
    return g1, c2


class LibBackend:
    """Rank-local steps through libnnm's staged ABI on one resident DeviceDataset."""

    def __init__(self, dd, metric, dmax):
        import torch

        from . import _native
        from .metrics import metric_code

        self.torch = torch
        self.nat = _native
        self.lib = _native.load()
        self.dd = dd
        tp, rows = ctypes.c_int64(), ctypes.c_int64()
        _native.check(self.lib.nnm_bv_begin(dd.handle, metric_code(metric),
                                            np.nan if dmax is None else float(dmax),
                                            ctypes.byref(tp), ctypes.byref(rows)))
        self.rows = rows.value
        self.b1 = torch.empty(self.rows, dtype=torch.int64, device="cuda")
        self.b2 = torch.empty_like(self.b1)
        self.ncomp = dd.n
        self.added_total = 0

    def components(self) -> int:
        return self.dd.n - self.added_total

    def _view(self, ptr, count, typestr):
        return self.torch.as_tensor(_DeviceArray(ptr, count, typestr), device="cuda")

    def round_bound(self, rank, world):
        p, c = ctypes.POINTER(ctypes.c_uint32)(), ctypes.c_int64()
        self.nat.check(self.lib.nnm_bv_round_bound(self.dd.handle, rank, world, ctypes.byref(p),
                                                   ctypes.byref(c)))
        addr = ctypes.cast(p, ctypes.c_void_p).value
        return self._view(addr, c.value, "<i4") if addr and c.value else None

    def round_phase1(self, rank, world, caps):
        self.torch.cuda.synchronize()
        self.nat.check(self.lib.nnm_bv_round_phase1(
            self.dd.handle, rank, world, None if caps is None else caps.data_ptr(),
            self.b1.data_ptr(), self.b2.data_ptr()))
        return self.b1, self.b2

    def round_phase2(self, rank, world, g1, g2):
        self.torch.cuda.synchronize()
        p, c = ctypes.POINTER(ctypes.c_uint32)(), ctypes.c_int64()
        self.nat.check(self.lib.nnm_bv_round_phase2(self.dd.handle, rank, world, g1.data_ptr(),
                                                    g2.data_ptr(), self.b1.data_ptr(),
                                                    self.b2.data_ptr(), ctypes.byref(p),
                                                    ctypes.byref(c)))
        addr = ctypes.cast(p, ctypes.c_void_p).value
        return self._view(addr, c.value, "<i4") if addr and c.value else None

    def cache_scatter(self):
        self.torch.cuda.synchronize()
        self.nat.check(self.lib.nnm_bv_cache_scatter(self.dd.handle))

    def keys(self):
        return self.b1, self.b2

    def copy(self, x):
        return x.clone()

    def second(self, b1, b2, g1):
        out = self.torch.empty_like(b1)
        self.torch.cuda.synchronize()
        self.nat.check(self.lib.nnm_bv_second(self.dd.handle, b1.data_ptr(), b2.data_ptr(),
                                              g1.data_ptr(), out.data_ptr()))
        return out

    def finish_round(self, g1, g2):
        self.torch.cuda.synchronize()
        added = ctypes.c_int64()
        self.nat.check(self.lib.nnm_bv_finish_round(self.dd.handle, g1.data_ptr(), g2.data_ptr(),
                                                    ctypes.byref(added)))
        self.added_total += added.value
        return added.value

    def end(self, kl1):
        n = self.dd.n
        merges = self.nat.host_empty(max(n - 1, 1), self.nat.MERGE_DTYPE)
        assign = self.nat.host_empty(n, np.int64)
        nm, rounds = ctypes.c_int64(), ctypes.c_int64()
        stop = ctypes.c_int32()
        st = self.nat.Stats()
        self.nat.check(self.lib.nnm_bv_end(self.dd.handle, -1 if kl1 is None else int(kl1),
                                           merges.ctypes.data, ctypes.byref(nm),
                                           assign.ctypes.data, ctypes.byref(rounds),
                                           ctypes.byref(stop), ctypes.byref(st)))
        return (merges[: nm.value], assign, rounds.value, self.nat.STOP_NAMES[stop.value],
                st.as_dict())


def run_boruvka_distributed(X, *, metric="euclidean", dmax=None, kl1=None, group=None):
    """Full-dendrogram NNM on all ranks of `group` (NCCL); every rank returns the same
    (merges, assignments, rounds, stop_reason, stats).  Inputs are replicated."""
    import torch

    from . import _native

    dd = _native.DeviceDataset(np.ascontiguousarray(X, dtype=np.float64),
                               device=torch.cuda.current_device())
    return run_boruvka_distributed_handle(dd, metric=metric, dmax=dmax, kl1=kl1, group=group)


def run_boruvka_distributed_handle(dd, *, metric="euclidean", dmax=None, kl1=None, group=None):
    """As run_boruvka_distributed, on an already resident DeviceDataset."""
    import time

    import torch.distributed as dist

    t0 = time.perf_counter()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    be = LibBackend(dd, metric, dmax)

    def amin(t):
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)

    def amax(t):
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)

    if dd.n > 1 and not (kl1 is not None and dd.n <= kl1):
        boruvka_rounds(be, rank, world, amin, amax)
    merges, assign, rounds, stop, sd = be.end(kl1)
    sd["total_ms"] = 1e3 * (time.perf_counter() - t0)
    return merges, assign, rounds, stop, sd
