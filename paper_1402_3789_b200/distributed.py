"""Multi-GPU Boruvka driver: one process per GPU, torch.distributed for plumbing.

Partitioning: every rank holds the whole dataset (X64 + FP32
tiles, 600 MB at 2M x 25).  Each Boruvka round is the pruned scan of DESIGN.md
3.1: every rank evaluates the small phase-1 tile-pair list in full (so all
ranks derive the same component bounds and the same phase-2 list without an
exchange) and a contiguous equal-count 1/world share of the phase-2 tile pairs
(``nnm_bv_scan_pruned``).  ``pruned=False`` splits the dense upper-triangular
tile-pair space [0, T(T+1)/2) instead (``nnm_bv_scan``).  Each rank scans into
per-row keys (B1 best, B2 second best; u64 = fp32 bits << 32 | partner), then
two all-reduce(MIN) calls combine them:

    B1 = min_r B1_r
    B2 = min_r (B1_r == B1 ? B2_r : B1_r)      # second smallest of the union

and every rank finishes the round (FP64 certification, component minima,
hooking, pointer jumping) redundantly and deterministically, so labels and the
final merge log are byte-identical on every rank and for every world size.
The data path has exactly one exchange step per round; nothing else crosses
NVLink.
"""

from __future__ import annotations

import ctypes

import numpy as np

__all__ = ["shard_range", "combine_second", "run_boruvka_distributed",
           "run_boruvka_distributed_handle"]


class _DeviceArray:
    """A library-owned device buffer seen through __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous equal-count share of [0, total) for `rank`."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi


def combine_second(b1_local, b2_local, b1_global):
    """Per-rank contribution to the global second-best key (numpy or torch arrays)."""
    if isinstance(b1_local, np.ndarray):
        return np.where(b1_local == b1_global, b2_local, b1_local)
    import torch

    return torch.where(b1_local == b1_global, b2_local, b1_local)


def run_boruvka_distributed(X, *, metric="euclidean", dmax=None, kl1=None, group=None,
                            pruned=True):
    """Full-dendrogram NNM on all ranks of `group` (NCCL); every rank returns the same
    (merges, assignments, rounds, stop_reason, stats).  Inputs are replicated."""
    import torch

    from . import _native

    dd = _native.DeviceDataset(np.ascontiguousarray(X, dtype=np.float64),
                               device=torch.cuda.current_device())
    return run_boruvka_distributed_handle(dd, metric=metric, dmax=dmax, kl1=kl1, group=group,
                                          pruned=pruned)


def run_boruvka_distributed_handle(dd, *, metric="euclidean", dmax=None, kl1=None, group=None,
                                   pruned=True):
    """As run_boruvka_distributed, on an already resident DeviceDataset."""
    import time

    import torch
    import torch.distributed as dist

    from . import _native
    from .metrics import metric_code

    lib = _native.load()
    t0 = time.perf_counter()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    tp, rows = ctypes.c_int64(), ctypes.c_int64()
    _native.check(lib.nnm_bv_begin(dd.handle, metric_code(metric),
                                   np.nan if dmax is None else float(dmax), ctypes.byref(tp),
                                   ctypes.byref(rows)))
    n = dd.n
    # tile-pair bound cache (TC metric): kept identical on every rank by an all-reduce(MAX)
    # after each pruned scan, so the ranks keep deriving the same phase-2 lists
    cptr, ccount = ctypes.c_void_p(), ctypes.c_int64()
    _native.check(lib.nnm_bv_cache(dd.handle, 1 if (world > 1 and pruned) else 0,
                                   ctypes.byref(cptr), ctypes.byref(ccount)))
    cache = None
    if world > 1 and pruned and cptr.value and ccount.value > 0:
        cache = torch.as_tensor(_DeviceArray(cptr.value, ccount.value, "<i4"), device="cuda")
    lo, hi = shard_range(tp.value, rank, world)
    b1 = torch.empty(rows.value, dtype=torch.int64, device="cuda")
    b2 = torch.empty(rows.value, dtype=torch.int64, device="cuda")
    g1 = torch.empty_like(b1)
    c2 = torch.empty_like(b1)
    added = ctypes.c_int64()
    need = n > 1 and not (kl1 is not None and n <= kl1)
    while need:
        if pruned:
            _native.check(lib.nnm_bv_scan_pruned(dd.handle, rank, world, b1.data_ptr(),
                                                 b2.data_ptr()))
        else:
            _native.check(lib.nnm_bv_scan(dd.handle, lo, hi, b1.data_ptr(), b2.data_ptr()))
        torch.cuda.synchronize()
        if cache is not None:
            dist.all_reduce(cache, op=dist.ReduceOp.MAX, group=group)
        g1.copy_(b1)
        dist.all_reduce(g1, op=dist.ReduceOp.MIN, group=group)
        _native.check(lib.nnm_bv_second(dd.handle, b1.data_ptr(), b2.data_ptr(), g1.data_ptr(),
                                        c2.data_ptr()))
        dist.all_reduce(c2, op=dist.ReduceOp.MIN, group=group)
        _native.check(lib.nnm_bv_finish_round(dd.handle, g1.data_ptr(), c2.data_ptr(),
                                              ctypes.byref(added)))
        if added.value == 0:
            break
    merges = np.zeros(max(n - 1, 1), dtype=_native.MERGE_DTYPE)
    assign = np.empty(n, np.int64)
    nm, rounds = ctypes.c_int64(), ctypes.c_int64()
    stop = ctypes.c_int32()
    st = _native.Stats()
    _native.check(lib.nnm_bv_end(dd.handle, -1 if kl1 is None else int(kl1), merges.ctypes.data,
                                 ctypes.byref(nm), assign.ctypes.data, ctypes.byref(rounds),
                                 ctypes.byref(stop), ctypes.byref(st)))
    sd = st.as_dict()
    sd["total_ms"] = 1e3 * (time.perf_counter() - t0)
    return merges[: nm.value], assign, rounds.value, _native.STOP_NAMES[stop.value], sd
