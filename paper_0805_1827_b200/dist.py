"""Multi-GPU sharding: one process per GPU, torch.distributed for the plumbing.

Replaces the reference's master-worker pool (engine.py:65-123): items
(probes, training points, 4096-path blocks) are split into contiguous rank
ranges with the reference's partition rule (sizes within 1, engine.py:65-81),
every rank runs its range on its own GPU, and the per-date exchange is one
collective:

* labels / probe levels: all-gather (each rank contributes its range);
* pricing: all-reduce of the zero-padded per-block (count, sum, sumsq)
  table, which is exact (x + 0 == x), so the fold in block order gives the
  same bits for any GPU count, like the reference's ordered merge
  (pricer.py:190-191).

The fits (AdaBoost, least squares) are deterministic device kernels, so
every rank runs them on the gathered data and gets the same rule; no
broadcast is needed.  With world size 1 every collective is a no-op and
torch.distributed is never touched.

``virtual_shards(n)`` runs the same decomposition inside one process: every
phase is executed range by range for all n partitions (the reference's task
partition, engine.py:65-81, with nb_tasks = n) and nothing is exchanged.  It
is how the reference CLI's determinism bench (cli.py:281-319) checks that a
price does not depend on the partition, on a box with one GPU.
"""

from __future__ import annotations

import contextlib
import threading
from dataclasses import dataclass

import numpy as np

__all__ = ["Shard", "current", "partition_ranges", "virtual_shards"]


def partition_ranges(total: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous ranges with sizes within 1, first ranges larger (engine.py:65-81)."""
    if total < 0 or parts < 1:
        raise ValueError(f"bad partition total={total} parts={parts}")
    base, extra = divmod(total, parts)
    out, lo = [], 0
    for i in range(parts):
        hi = lo + base + (1 if i < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


@dataclass
class Shard:
    rank: int = 0
    world: int = 1
    group: object = None
    virtual: bool = False  # all partitions run in this process, one after another

    @property
    def distributed(self) -> bool:
        """True when ranks are processes that exchange data through collectives."""
        return self.world > 1 and not self.virtual

    def range(self, total: int) -> tuple[int, int]:
        return partition_ranges(total, self.world)[self.rank]

    def local_ranges(self, total: int) -> list[tuple[int, int]]:
        """The item ranges this process computes, in item order: its own rank's
        range, or every partition's range under ``virtual_shards``."""
        if self.virtual:
            return partition_ranges(total, self.world)
        return [self.range(total)]

    def all_gather_rows(self, local, total: int):
        """Concatenate each rank's contiguous rows (torch tensors on this rank's GPU)."""
        if not self.distributed:
            return local
        import torch
        import torch.distributed as dist
        ranges = partition_ranges(total, self.world)
        width = max(hi - lo for lo, hi in ranges)
        shape = (width,) + tuple(local.shape[1:])
        pad = torch.zeros(shape, dtype=local.dtype, device=local.device)
        pad[:local.shape[0]] = local
        parts = [torch.empty(shape, dtype=local.dtype, device=local.device) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        return torch.cat([parts[r][:hi - lo] for r, (lo, hi) in enumerate(ranges)], dim=0)

    def all_reduce_sum(self, t):
        if self.distributed:
            import torch.distributed as dist
            dist.all_reduce(t, group=self.group)
        return t

    def barrier(self):
        if self.distributed:
            import torch.distributed as dist
            dist.barrier(group=self.group)


_local = threading.local()


@contextlib.contextmanager
def virtual_shards(world: int):
    """Run every phase as ``world`` contiguous partitions in this process."""
    if world < 1:
        raise ValueError(f"need at least one partition, got {world}")
    prev = getattr(_local, "shard", None)
    _local.shard = Shard(0, int(world), None, virtual=True)
    try:
        yield _local.shard
    finally:
        _local.shard = prev


def current() -> Shard:
    """The shard of this process (torch.distributed world if initialised)."""
    v = getattr(_local, "shard", None)
    if v is not None:
        return v
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return Shard(dist.get_rank(), dist.get_world_size(), None)
    except Exception:
        pass
    return Shard()
