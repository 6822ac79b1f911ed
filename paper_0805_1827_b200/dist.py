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
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Shard", "current", "partition_ranges"]


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

    @property
    def distributed(self) -> bool:
        return self.world > 1

    def range(self, total: int) -> tuple[int, int]:
        return partition_ranges(total, self.world)[self.rank]

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


def current() -> Shard:
    """The shard of this process (torch.distributed world if initialised)."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return Shard(dist.get_rank(), dist.get_world_size(), None)
    except Exception:
        pass
    return Shard()
