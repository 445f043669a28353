"""Round seam mirroring parclust.scheduler (scheduler.py:1-335).

The reference's two-level manager/worker thread pipeline (the paper's
"first/second level managers") exists to keep CPU cores busy with block-pair
tasks.  On the B200 the CTA scheduler does that load balancing: one fused
kernel covers every tile pair of the round on one stream.  ``PipelineConfig``
is accepted (and validated exactly like the reference) so callers need no
changes; its sizing has no effect on the result, which the reference also
guarantees for its own pipeline (scheduler.py:16-20).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field, replace

from .model import ValidationError
from .pairgen import TopPBuffer, gpu_top_p

__all__ = ["PipelineConfig", "UtilizationStats", "WorkerError", "run_round", "report_utilization"]

_THREAD_CAP_ENV = "PARCLUST_THREADS"


class WorkerError(RuntimeError):
    """A device task failed (scheduler.py:45-46)."""


@dataclass(frozen=True)
class PipelineConfig:
    managers: int = 4
    workers_per_manager: int | None = None
    input_buffers: int = 12
    output_buffers: int = 12
    buffers_per_worker: int = 3

    def __post_init__(self):
        for name in ("managers", "input_buffers", "output_buffers", "buffers_per_worker"):
            v = getattr(self, name)
            if v < 1:
                raise ValidationError(f"{name} must be at least 1, got {v}")
        if self.workers_per_manager is not None and self.workers_per_manager < 1:
            raise ValidationError(
                f"workers_per_manager must be at least 1, got {self.workers_per_manager}")
        if self.input_buffers < self.managers:
            raise ValidationError(
                f"input_buffers ({self.input_buffers}) must be >= managers ({self.managers})")

    def resolve(self) -> "PipelineConfig":
        """Same derivation as the reference (scheduler.py:78-107)."""
        cap = None
        raw = os.environ.get(_THREAD_CAP_ENV)
        if raw is not None and raw.strip():
            try:
                cap = int(raw)
            except ValueError as exc:
                raise ValidationError(f"{_THREAD_CAP_ENV} must be an integer, got {raw!r}") from exc
            if cap < 1:
                raise ValidationError(f"{_THREAD_CAP_ENV} must be at least 1, got {cap}")
        managers = min(self.managers, cap) if cap is not None else self.managers
        workers = self.workers_per_manager
        if workers is None:
            workers = max(1, (os.cpu_count() or 1) // managers)
        if cap is not None:
            workers = max(1, min(workers, cap // managers))
        return replace(self, managers=managers, workers_per_manager=workers,
                       input_buffers=max(self.input_buffers, managers))


@dataclass
class UtilizationStats:
    """Timing ledger (scheduler.py:110-143); the device is reported as one worker "gpu0"."""

    worker_busy: dict = field(default_factory=dict)
    worker_idle: dict = field(default_factory=dict)
    manager_reduce: dict = field(default_factory=dict)
    tasks_executed: list = field(default_factory=list)
    wall_time: float = 0.0

    def absorb(self, other: "UtilizationStats") -> None:
        for mine, theirs in ((self.worker_busy, other.worker_busy),
                             (self.worker_idle, other.worker_idle),
                             (self.manager_reduce, other.manager_reduce)):
            for k, v in theirs.items():
                mine[k] = mine.get(k, 0.0) + v
        self.tasks_executed.extend(other.tasks_executed)
        self.wall_time += other.wall_time

    def as_dict(self) -> dict:
        return {
            "worker_busy_s": dict(sorted(self.worker_busy.items())),
            "worker_idle_s": dict(sorted(self.worker_idle.items())),
            "manager_reduce_s": dict(sorted(self.manager_reduce.items())),
            "tasks_executed": len(self.tasks_executed),
            "wall_time_s": self.wall_time,
        }


def report_utilization(stats: UtilizationStats) -> str:
    def pct(b, i):
        return 100.0 * b / (b + i) if b + i > 0 else 0.0

    lines = [f"worker {k}: busy {stats.worker_busy[k]:.3f}s idle {stats.worker_idle.get(k, 0.0):.3f}s "
             f"util {pct(stats.worker_busy[k], stats.worker_idle.get(k, 0.0)):.1f}%"
             for k in sorted(stats.worker_busy)]
    lines += [f"manager {k}: reduce {v:.3f}s" for k, v in sorted(stats.manager_reduce.items())]
    b, i = sum(stats.worker_busy.values()), sum(stats.worker_idle.values())
    lines.append(f"aggregate: busy {b:.3f}s idle {i:.3f}s util {pct(b, i):.1f}% over "
                 f"{len(stats.tasks_executed)} tasks, wall {stats.wall_time:.3f}s")
    return "\n".join(lines)


def run_round(dataset, snapshot, plan, P: int, config: PipelineConfig):
    """One round's top-P buffer, computed on the GPU (scheduler.py:268-335).

    Returns (TopPBuffer, UtilizationStats); the buffer equals the reference's
    global_top_p for any plan / config.
    """
    config.resolve()  # same validation as the reference
    if P < 1:
        raise ValidationError(f"P must be at least 1, got {P}")
    t0 = time.perf_counter()
    try:
        buf = gpu_top_p(dataset, snapshot, P)
    except ValidationError:
        raise
    except Exception as exc:  # noqa: BLE001 - uniform failure contract (scheduler.py:327-334)
        raise WorkerError(f"GPU scan of all tile pairs failed: {exc}") from exc
    wall = time.perf_counter() - t0
    st = UtilizationStats(worker_busy={"gpu0": wall}, worker_idle={"gpu0": 0.0},
                          manager_reduce={"gpu0": 0.0}, tasks_executed=list(plan.tasks),
                          wall_time=wall)
    return buf, st


__all__ += ["TopPBuffer"]
