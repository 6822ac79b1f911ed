"""Execution context accepted by the phase functions.

The reference schedules item ranges on a fork/thread pool
(engine.py:147-168).  Here the unit of parallelism is the GPU: a phase runs
its items on this process's GPU in one launch, and a multi-GPU job is one
process per GPU (torch.distributed) sharded by ``dist.partition_ranges``,
the reference's partition rule.  ``Engine`` keeps the reference's
constructor and ``partition`` so existing call sites still work; its pool
fields are recorded but never fork (CUDA contexts do not survive fork).
"""

from __future__ import annotations

import contextlib
import warnings
from dataclasses import dataclass, field

import numpy as np

from .dist import partition_ranges

__all__ = ["Engine", "TaskPlan", "TimingLog", "partition", "EngineTaskError", "log_phase", "nvtx_range"]


class EngineTaskError(RuntimeError):
    def __init__(self, task_id: int, cause: BaseException):
        super().__init__(f"task {task_id} failed: {cause!r}")
        self.task_id = task_id


@dataclass(frozen=True)
class TaskPlan:
    total_items: int
    nb_tasks: int
    ranges: tuple
    phase: str = ""


def partition(total: int, nb: int, phase: str = "") -> TaskPlan:
    """Contiguous ranges, sizes within 1 (engine.py:65-81)."""
    if total < 1:
        raise ValueError(f"need at least one item, got {total}")
    if nb < 1:
        raise ValueError(f"need at least one task, got {nb}")
    if nb > total:
        warnings.warn(f"nb_tasks={nb} exceeds {total} items; clamping", stacklevel=2)
        nb = total
    return TaskPlan(total, nb, tuple(partition_ranges(total, nb)), phase)


@dataclass
class TimingLog:
    """Per-task durations (engine.py:126-144): rows of (phase, task_id, seconds).

    The reference's task is one item range on one pool worker; here it is one
    phase launch on this rank's GPU -- a date's label launch ("calc"), a
    date's AdaBoost or regression ("class" / "reg"), the pricing launch
    ("mc") -- timed on the device (CUDA events) where the date loop is
    device-resident, and task_id is the date index (the rank for "mc")."""

    rows: list = field(default_factory=list)

    def record(self, phase: str, task_id: int, seconds: float) -> None:
        self.rows.append((phase, int(task_id), float(seconds)))

    def phase_seconds(self, phase: str) -> float:
        return sum(s for p, _, s in self.rows if p == phase)

    def straggler_ratio(self, phase: str) -> float:
        """max / median of the phase's task durations (1.0 if degenerate)."""
        times = [s for p, _, s in self.rows if p == phase]
        if not times:
            return 1.0
        med = float(np.median(times))
        return float(max(times) / med) if med > 0.0 else 1.0


def log_phase(engine, phase: str, seconds_by_task) -> None:
    """Append (phase, task_id, seconds) rows to ``engine.timing`` when the
    caller passed an engine with a timing log (this package's or the
    reference's: both keep ``rows``)."""
    rows = getattr(getattr(engine, "timing", None), "rows", None)
    if rows is not None:
        rows.extend((phase, int(t), float(s)) for t, s in seconds_by_task)


@contextlib.contextmanager
def nvtx_range(name: str):
    """NVTX range around a phase's launches (visible in nsys / ncu --nvtx);
    a no-op without a CUDA build of torch."""
    try:
        import torch
        nvtx = torch.cuda.nvtx if torch.cuda.is_available() else None
    except Exception:  # pragma: no cover - torch is part of the image
        nvtx = None
    if nvtx is None:
        yield
        return
    nvtx.range_push(name)
    try:
        yield
    finally:
        nvtx.range_pop()


@dataclass
class Engine:
    workers: int = 1
    nb_tasks: int | None = None
    pool: str = "process"
    timing: TimingLog = field(default_factory=TimingLog)

    def plan(self, total: int, phase: str = "") -> TaskPlan:
        return partition(total, self.nb_tasks or self.workers, phase)
