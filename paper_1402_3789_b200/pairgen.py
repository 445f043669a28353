"""Pair selection mirroring parclust.pairgen (pairgen.py:1-324).

The block plan is kept for API compatibility but is invisible in results
(the reference asserts this itself, test_pairgen.py:170-186): the GPU scans
the whole upper triangle in 128x128 tiles regardless of ``plan``.
``global_top_p`` runs on the GPU through libnnm ``nnm_top_p`` and returns a
buffer bit-identical to the reference's serial fold.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .metrics import MetricKind, effective_threshold, metric_code
from .model import CandidatePair, ClusterForest, ConstraintSet, ValidationError

__all__ = ["BlockPlan", "TopPBuffer", "EligibilitySnapshot", "plan_blocks", "suggested_blocks",
           "make_snapshot", "pair_eligible", "reduce_topp", "global_top_p", "gpu_top_p"]

_TARGET_BLOCK_POINTS = 4096


@dataclass(frozen=True)
class BlockPlan:
    n: int
    bounds: np.ndarray
    tasks: tuple

    @property
    def num_blocks(self) -> int:
        return self.bounds.shape[0] - 1

    def block_range(self, i: int) -> tuple[int, int]:
        return int(self.bounds[i]), int(self.bounds[i + 1])


def plan_blocks(n: int, blocks: int) -> BlockPlan:
    """Contiguous blocks, remainder to the first ones; tasks (i, j), i <= j (pairgen.py:64-78)."""
    if n < 1:
        raise ValidationError(f"need at least one point, got n={n}")
    if blocks < 1:
        raise ValidationError(f"need at least one block, got {blocks}")
    B = min(blocks, n)
    sizes = np.full(B, n // B, dtype=np.int64)
    sizes[: n % B] += 1
    bounds = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    bounds.setflags(write=False)
    tasks = tuple((i, j) for i in range(B) for j in range(i, B))
    return BlockPlan(n=n, bounds=bounds, tasks=tasks)


def suggested_blocks(n: int) -> int:
    return max(1, -(-n // _TARGET_BLOCK_POINTS))


@dataclass(frozen=True, eq=False)
class TopPBuffer:
    """Up to P pairs ascending by (dist, a, b); dist in internal units (pairgen.py:85-131)."""

    dist: np.ndarray
    a: np.ndarray
    b: np.ndarray

    def __len__(self) -> int:
        return int(self.dist.shape[0])

    def __eq__(self, other) -> bool:
        if not isinstance(other, TopPBuffer):
            return NotImplemented
        return (np.array_equal(self.dist, other.dist) and np.array_equal(self.a, other.a)
                and np.array_equal(self.b, other.b))

    __hash__ = None  # type: ignore[assignment]

    @classmethod
    def empty(cls) -> "TopPBuffer":
        return cls(np.empty(0, np.float64), np.empty(0, np.int64), np.empty(0, np.int64))

    @classmethod
    def from_candidates(cls, dist, a, b, P: int) -> "TopPBuffer":
        dist = np.asarray(dist, dtype=np.float64)
        a = np.asarray(a, dtype=np.int64)
        b = np.asarray(b, dtype=np.int64)
        order = np.lexsort((b, a, dist))[:P]
        return cls(dist[order], a[order], b[order])

    def pairs(self) -> list[CandidatePair]:
        return [CandidatePair(a=int(x), b=int(y), dist=float(d))
                for d, x, y in zip(self.dist, self.a, self.b)]


@dataclass(frozen=True)
class EligibilitySnapshot:
    """Frozen per-round roots / sizes / threshold (pairgen.py:134-147)."""

    roots: np.ndarray
    size_by_point: np.ndarray
    constraints: ConstraintSet
    threshold: float | None
    metric: MetricKind


def make_snapshot(forest: ClusterForest, constraints: ConstraintSet,
                  metric: MetricKind) -> EligibilitySnapshot:
    roots = forest.roots_snapshot()
    sizes = forest.sizes_by_point(roots)
    roots.setflags(write=False)
    sizes.setflags(write=False)
    thr = None if constraints.dmax is None else effective_threshold(metric, constraints.dmax)
    return EligibilitySnapshot(roots, sizes, constraints, thr, metric)


def pair_eligible(snapshot: EligibilitySnapshot, a: int, b: int, dist: float) -> bool:
    """Scalar eligibility predicate (pairgen.py:169-187)."""
    if snapshot.roots[a] == snapshot.roots[b]:
        return False
    if snapshot.threshold is not None and dist > snapshot.threshold:
        return False
    sa, sb = int(snapshot.size_by_point[a]), int(snapshot.size_by_point[b])
    c = snapshot.constraints
    if c.kl2 is not None and (sa > c.kl2 or sb > c.kl2):
        return False
    if c.kl3 is not None and sa + sb > c.kl3:
        return False
    return True


def reduce_topp(lhs: TopPBuffer, rhs: TopPBuffer, P: int) -> TopPBuffer:
    """Associative merge of two buffers keeping the P smallest keys (pairgen.py:301-316)."""
    if len(lhs) == 0 and len(rhs) <= P:
        return rhs
    if len(rhs) == 0 and len(lhs) <= P:
        return lhs
    return TopPBuffer.from_candidates(np.concatenate([lhs.dist, rhs.dist]),
                                      np.concatenate([lhs.a, rhs.a]),
                                      np.concatenate([lhs.b, rhs.b]), P)


def gpu_top_p(dataset, snapshot: EligibilitySnapshot, P: int) -> TopPBuffer:
    """Exact top-P eligible pairs on the GPU (libnnm nnm_top_p)."""
    if P < 1:
        raise ValidationError(f"P must be at least 1, got {P}")
    dd = _native.device_dataset(dataset)
    n = dataset.n
    cap = max(1, min(P, n * (n - 1) // 2))
    dist = np.empty(cap, np.float64)
    a = np.empty(cap, np.int64)
    b = np.empty(cap, np.int64)
    roots = np.ascontiguousarray(snapshot.roots, dtype=np.int64)
    sizes = np.ascontiguousarray(snapshot.size_by_point, dtype=np.int64)
    c = snapshot.constraints
    thr = np.nan if snapshot.threshold is None else float(snapshot.threshold)
    import ctypes

    ln = ctypes.c_int64()
    lib = _native.load()
    _native.check(lib.nnm_top_p(dd.handle, metric_code(snapshot.metric), roots.ctypes.data,
                                sizes.ctypes.data, thr, -1 if c.kl2 is None else int(c.kl2),
                                -1 if c.kl3 is None else int(c.kl3), int(min(P, cap)),
                                dist.ctypes.data, a.ctypes.data, b.ctypes.data, ctypes.byref(ln)))
    k = ln.value
    return TopPBuffer(dist[:k].copy(), a[:k].copy(), b[:k].copy())


def global_top_p(dataset, snapshot: EligibilitySnapshot, plan: BlockPlan, P: int) -> TopPBuffer:
    """Same contract as the reference's serial fold (pairgen.py:319-324), on the GPU."""
    return gpu_top_p(dataset, snapshot, P)
