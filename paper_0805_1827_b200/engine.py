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

import warnings
from dataclasses import dataclass, field

from .dist import partition_ranges

__all__ = ["Engine", "TaskPlan", "partition", "EngineTaskError"]


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
class Engine:
    workers: int = 1
    nb_tasks: int | None = None
    pool: str = "process"
    timing: list = field(default_factory=list)

    def plan(self, total: int, phase: str = "") -> TaskPlan:
        return partition(total, self.nb_tasks or self.workers, phase)
