"""Run seam mirroring parclust.engine (engine.py:1-199), executed on the GPU.

``run(dataset, config)`` has the reference's signature and result type.  It
makes ONE call into libnnm (``nnm_run``), which picks the algorithm:

* no kl2/kl3/kl4: exact Boruvka rounds on the GPU (fused FP32 screen + FP64
  exact keys), then a sort + union-find replay of the MST edges with kl1
  truncation.  The ordered merge list (root_a, root_b, dist, new_size,
  point_a, point_b) equals the reference's for every P;
  ``MergeEvent.round`` numbers Boruvka rounds instead.
* kl2 / kl3 / kl4 (or ``exact_rounds=True``): the reference's round structure
  with the caller's P -- exact top-P per round on the GPU, order_batch and
  process_batch with live re-checks -- so rounds, counters and the kl4-dependent
  partition match the reference exactly.

``order_batch`` / ``process_batch`` are kept as host utilities with the
reference's semantics (engine.py:73-143) for callers that drive rounds
themselves through ``scheduler.run_round``.
"""

from __future__ import annotations

import ctypes
import os
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .metrics import MetricKind, metric_code, reported
from .model import ClusterForest, ConstraintSet, Dataset, MergeEvent, ValidationError
from .pairgen import EligibilitySnapshot, TopPBuffer
from .scheduler import PipelineConfig, UtilizationStats

__all__ = ["RunConfig", "RunResult", "MergeLog", "order_batch", "process_batch", "run", "fit",
           "run_arrays", "run_arrays_multi", "replica_devices"]

DEFAULT_PAIRS_PER_BATCH = 256


@dataclass(frozen=True)
class RunConfig:
    """Everything a run needs besides the data (engine.py:35-54)."""

    constraints: ConstraintSet = ConstraintSet()
    pairs_per_batch: int = DEFAULT_PAIRS_PER_BATCH
    metric: MetricKind = MetricKind.EUCLIDEAN
    blocks: int | None = None
    pipeline: PipelineConfig = PipelineConfig()
    exact_rounds: bool = False  # force the reference's round structure for every constraint set
    n_gpus: int = 1  # replicas / GPUs of one process (nnm_run_multi); devices from NNM_DEVICES

    def __post_init__(self):
        if self.n_gpus < 1:
            raise ValidationError(f"n_gpus must be at least 1, got {self.n_gpus}")
        if self.pairs_per_batch < 1:
            raise ValidationError(
                f"pairs_per_batch must be at least 1, got {self.pairs_per_batch}")
        if self.blocks is not None and self.blocks < 1:
            raise ValidationError(f"blocks must be at least 1, got {self.blocks}")


class MergeLog(Sequence):
    """Sequence of MergeEvent backed by a structured array (no per-event objects
    until an element is touched; a 2M-point dendrogram stays cheap)."""

    def __init__(self, records: np.ndarray):
        self.array = records

    def __len__(self) -> int:
        return int(self.array.shape[0])

    def _event(self, i: int) -> MergeEvent:
        r = self.array[i]
        return MergeEvent(step=i, round=int(r["round"]), root_a=int(r["root_a"]),
                          root_b=int(r["root_b"]), dist=float(r["dist"]),
                          new_size=int(r["new_size"]), point_a=int(r["point_a"]),
                          point_b=int(r["point_b"]))

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._event(k) for k in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return self._event(i)

    def __eq__(self, other) -> bool:
        return list(self) == list(other)


@dataclass
class RunResult:
    """Merge log, final labels and accounting (engine.py:57-70)."""

    merges: Sequence
    assignments: np.ndarray
    rounds: int
    stop_reason: str
    stats: UtilizationStats
    round_counters: list = field(default_factory=list)
    device_stats: dict = field(default_factory=dict)

    @property
    def cluster_count(self) -> int:
        return int(np.unique(self.assignments).shape[0])


def order_batch(buffer: TopPBuffer, snapshot: EligibilitySnapshot, kl4):
    """kl4 stable partition by round-start sizes (engine.py:73-87)."""
    dist, a, b = buffer.dist, buffer.a, buffer.b
    if kl4 is not None and len(buffer) > 0:
        small = np.minimum(snapshot.size_by_point[a], snapshot.size_by_point[b])
        order = np.argsort(small >= kl4, kind="stable")
        dist, a, b = dist[order], a[order], b[order]
    return [(float(x), int(y), int(z)) for x, y, z in zip(dist, a, b)]


def process_batch(forest: ClusterForest, pairs, constraints: ConstraintSet, round_index: int, *,
                  metric: MetricKind, start_step: int = 0):
    """Sequential merge with live kl2/kl3 re-checks and the kl1 floor (engine.py:90-143)."""
    kl1, kl2, kl3 = constraints.kl1, constraints.kl2, constraints.kl3
    events: list[MergeEvent] = []
    skips = {"same_root": 0, "kl2": 0, "kl3": 0, "unprocessed": 0}
    stop = False
    for pos, (dist, a, b) in enumerate(pairs):
        ra, rb = forest.find(a), forest.find(b)
        if ra == rb:
            skips["same_root"] += 1
            continue
        sa, sb = forest.size_of_root(ra), forest.size_of_root(rb)
        if kl2 is not None and (sa > kl2 or sb > kl2):
            skips["kl2"] += 1
            continue
        if kl3 is not None and sa + sb > kl3:
            skips["kl3"] += 1
            continue
        keep, new_size = forest.union(ra, rb)
        events.append(MergeEvent(step=start_step + len(events), round=round_index, root_a=keep,
                                 root_b=rb if keep == ra else ra,
                                 dist=float(reported(metric, dist)), new_size=new_size,
                                 point_a=a, point_b=b))
        if forest.count == 1 or (kl1 is not None and forest.count <= kl1):
            stop = True
            skips["unprocessed"] = len(pairs) - pos - 1
            break
    return events, stop, skips


def _opt(v) -> int:
    return -1 if v is None else int(v)


def run_arrays(ddata, constraints: ConstraintSet, P: int, metric: MetricKind,
               exact_rounds: bool = False):
    """Low-level run on a resident device dataset; returns raw arrays.

    (merges structured array, assignments, rounds, stop_reason, counters array, stats dict)
    """
    n = ddata.n
    lib = _native.load()
    merges = _native.host_empty(max(n - 1, 1), _native.MERGE_DTYPE)
    assign = _native.host_empty(n, np.int64)
    ccap = n + 1
    counters = np.zeros(ccap, dtype=_native.COUNTER_DTYPE)
    nm, rounds, nc = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    stop = ctypes.c_int32()
    st = _native.Stats()
    cons = _native.Constraints(_opt(constraints.kl1), _opt(constraints.kl2),
                               _opt(constraints.kl3), _opt(constraints.kl4),
                               np.nan if constraints.dmax is None else float(constraints.dmax))
    flags = _native.FLAG_ROUNDS if exact_rounds else 0
    _native.check(lib.nnm_run(ddata.handle, metric_code(metric), ctypes.byref(cons), int(P), flags,
                              merges.ctypes.data, ctypes.byref(nm), assign.ctypes.data,
                              ctypes.byref(rounds), ctypes.byref(stop), counters.ctypes.data, ccap,
                              ctypes.byref(nc), ctypes.byref(st)))
    stats = st.as_dict()
    stats["round_log"] = _native.round_log(ddata.handle)
    return (merges[: nm.value], assign, rounds.value, _native.STOP_NAMES[stop.value],
            counters[: min(nc.value, ccap)], stats)


def replica_devices(n_gpus: int) -> list:
    """Devices of an n_gpus run: NNM_DEVICES (comma-separated, repeats allowed: several
    replicas on one device run the same exchange code) or 0 .. n_gpus-1."""
    env = os.environ.get("NNM_DEVICES")
    if env:
        devs = [int(x) for x in env.split(",") if x.strip()]
        if len(devs) < n_gpus:
            raise ValidationError(f"NNM_DEVICES lists {len(devs)} devices, n_gpus={n_gpus}")
        return devs[:n_gpus]
    return list(range(n_gpus))


def run_arrays_multi(dds, constraints: ConstraintSet, P: int, metric: MetricKind,
                     exact_rounds: bool = False):
    """run_arrays over several resident replicas (nnm_run_multi)."""
    if len(dds) == 1:
        return run_arrays(dds[0], constraints, P, metric, exact_rounds)
    n = dds[0].n
    lib = _native.load()
    merges = _native.host_empty(max(n - 1, 1), _native.MERGE_DTYPE)
    assign = _native.host_empty(n, np.int64)
    ccap = n + 1
    counters = np.zeros(ccap, dtype=_native.COUNTER_DTYPE)
    nm, rounds, nc = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    stop = ctypes.c_int32()
    st = _native.Stats()
    cons = _native.Constraints(_opt(constraints.kl1), _opt(constraints.kl2),
                               _opt(constraints.kl3), _opt(constraints.kl4),
                               np.nan if constraints.dmax is None else float(constraints.dmax))
    handles = (ctypes.c_void_p * len(dds))(*[d.handle for d in dds])
    flags = _native.FLAG_ROUNDS if exact_rounds else 0
    _native.check(lib.nnm_run_multi(handles, len(dds), metric_code(metric), ctypes.byref(cons),
                                    int(P), flags, merges.ctypes.data, ctypes.byref(nm),
                                    assign.ctypes.data, ctypes.byref(rounds), ctypes.byref(stop),
                                    counters.ctypes.data, ccap, ctypes.byref(nc),
                                    ctypes.byref(st)))
    stats = st.as_dict()
    stats["round_log"] = _native.round_log(dds[0].handle)
    stats["replicas"] = [d.device for d in dds]
    return (merges[: nm.value], assign, rounds.value, _native.STOP_NAMES[stop.value],
            counters[: min(nc.value, ccap)], stats)


def _replicas(dataset: Dataset, n_gpus: int) -> list:
    devs = replica_devices(n_gpus)
    cache = getattr(dataset, "_replica_cache", None)
    if cache is not None and cache[0] == tuple(devs):
        return cache[1]
    first = _native.device_dataset(dataset)
    reps = [first if first.device == devs[0] else _native.DeviceDataset(dataset.values, device=devs[0])]
    reps += [_native.DeviceDataset(dataset.values, device=dv) for dv in devs[1:]]
    object.__setattr__(dataset, "_replica_cache", (tuple(devs), reps))
    return reps


def run(dataset: Dataset, config: RunConfig) -> RunResult:
    """Cluster to completion on the GPU (engine.py:154-199); config.n_gpus > 1 runs the
    Boruvka path over that many GPU replicas in this process (nnm_run_multi)."""
    if not isinstance(dataset, Dataset):
        dataset = Dataset(values=np.asarray(dataset))
    if config.n_gpus > 1:
        merges, assign, rounds, stop, counters, dstats = run_arrays_multi(
            _replicas(dataset, config.n_gpus), config.constraints, config.pairs_per_batch,
            config.metric, config.exact_rounds)
    else:
        dd = _native.device_dataset(dataset)
        merges, assign, rounds, stop, counters, dstats = run_arrays(
            dd, config.constraints, config.pairs_per_batch, config.metric, config.exact_rounds)
    wall = dstats["total_ms"] / 1e3
    stats = UtilizationStats(worker_busy={"gpu0": dstats["scan_ms"] / 1e3},
                             worker_idle={"gpu0": max(0.0, wall - dstats["scan_ms"] / 1e3)},
                             manager_reduce={"gpu0": 0.0}, tasks_executed=[], wall_time=wall)
    rc = [{k: int(r[k]) for k in _native.COUNTER_KEYS} for r in counters]
    return RunResult(merges=MergeLog(merges), assignments=assign, rounds=rounds, stop_reason=stop,
                     stats=stats, round_counters=rc, device_stats=dstats)


def fit(X, *, metric="euclidean", kl1=None, kl2=None, kl3=None, kl4=None, dmax=None,
        pairs_per_batch: int = DEFAULT_PAIRS_PER_BATCH, exact_rounds: bool = False,
        n_gpus: int = 1) -> RunResult:
    """Convenience entry: fit on an (n, d) float array with the paper's constraints."""
    kind = MetricKind.parse(metric) if isinstance(metric, str) else metric
    cfg = RunConfig(constraints=ConstraintSet(kl1=kl1, kl2=kl2, kl3=kl3, kl4=kl4, dmax=dmax),
                    pairs_per_batch=pairs_per_batch, metric=kind, exact_rounds=exact_rounds,
                    n_gpus=n_gpus)
    return run(Dataset(values=np.asarray(X, dtype=np.float64)), cfg)
