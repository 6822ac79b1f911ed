"""Final pricing under a fixed exercise rule (phase [mc]), on the device.

Drop-in for the reference's ``price`` (pricer.py:167-202): same signature,
same stream convention (PATH_BLOCK = 4096 paths per block, block b on
StreamKey(seed, PRICING, b), pricer.py:30-32, 161), same per-block (count,
sum, sumsq) fold in block order and the same PriceEstimate.  Blocks are
sharded over the GPUs of the job (dist.py) and each GPU walks its blocks in
one kernel launch.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import backend as _be
from .dist import current as _current_shard
from .engine import log_phase, nvtx_range
from .packs import RulePack, pack_market

__all__ = ["PATH_BLOCK", "EuropeanRule", "ImmediateAtDate", "IzRule", "CmcScoreRule", "PriceEstimate", "price",
           "pool_moments", "block_stats"]

PATH_BLOCK = 4096


@dataclass(frozen=True)
class EuropeanRule:
    kind = "european"

    def pack(self, spec) -> RulePack:
        return RulePack.european(_call_like(spec))


@dataclass(frozen=True)
class ImmediateAtDate:
    date_index: int
    kind = "immediate"

    def pack(self, spec) -> RulePack:
        if not 1 <= self.date_index <= spec.n_dates:
            raise ValueError(f"date index {self.date_index} outside 1..{spec.n_dates}")
        return RulePack.immediate(self.date_index, _call_like(spec))


@dataclass(frozen=True)
class IzRule:
    boundary: object
    kind = "iz"

    def pack(self, spec) -> RulePack:
        return self.boundary.pack()


@dataclass(frozen=True)
class CmcScoreRule:
    rule: object
    kind = "cmc"

    def pack(self, spec) -> RulePack:
        return self.rule.pack()


def _call_like(spec) -> bool:
    from .market import is_call_like
    return is_call_like(spec.payoff_kind)


@dataclass(frozen=True)
class PriceEstimate:
    price: float
    variance: float
    ci95: float
    n_paths: int
    timings: dict = field(default_factory=dict)
    rule_kind: str = ""
    unconverged_points: int = 0

    @property
    def std_error(self) -> float:
        return float(np.sqrt(self.variance / self.n_paths)) if self.n_paths else 0.0

    def to_json_dict(self) -> dict:
        return {"price": self.price, "variance": self.variance, "ci95": self.ci95, "n_paths": self.n_paths,
                "timings": dict(self.timings), "rule_kind": self.rule_kind,
                "unconverged_points": self.unconverged_points}


def pool_moments(counts, sums, sumsqs) -> tuple[float, float, int]:
    """Fold per-block (count, sum, sumsq) in block order (pricer.py:136-151)."""
    n = int(np.sum(counts))
    # numpy's cumsum is the sequential chain ((x0 + x1) + x2) + ...: the same fp64 adds, in block
    # order, as the reference's Python loop (unlike np.sum, which adds pairwise)
    s = float(np.cumsum(np.asarray(sums, dtype=np.float64))[-1]) if len(sums) else 0.0
    ss = float(np.cumsum(np.asarray(sumsqs, dtype=np.float64))[-1]) if len(sumsqs) else 0.0
    mean = s / n
    var = (ss - s * s / n) / (n - 1) if n > 1 else 0.0
    return mean, max(var, 0.0), n


def block_stats(mp, rp, n_paths: int, seed: int, mode=None, shard=None):
    """Per-block stats of every block, gathered across the job's GPUs -> numpy [n_blocks, 3]."""
    shard = shard or _current_shard()
    n_blocks = (n_paths + PATH_BLOCK - 1) // PATH_BLOCK
    if shard.world == 1:
        return _be.price_blocks(mp, rp, n_paths, seed, 0, n_blocks, mode=mode)
    if shard.virtual:  # every partition in this process, block ranges in order
        table = np.empty((n_blocks, 3))
        for lo, hi in shard.local_ranges(n_blocks):
            if hi > lo:
                _be.price_blocks(mp, rp, n_paths, seed, lo, hi, out=table[lo:hi], mode=mode)
        return table
    import torch
    lo, hi = shard.range(n_blocks)
    table = torch.zeros((n_blocks, 3), dtype=torch.float64, device="cuda")
    if hi > lo:
        ctx_stream = torch.cuda.current_stream()
        from .context import get_context
        get_context(mp, rp, mode=mode).set_stream(ctx_stream)
        _be.price_blocks(mp, rp, n_paths, seed, lo, hi, out=table[lo:hi], mode=mode)
    shard.all_reduce_sum(table)  # zero-padded: exact, same bits for any GPU count
    return table.cpu().numpy()


def price(params, spec, rule, n_paths: int, seed: int, engine=None, backend=None, build_timings: dict | None = None,
          unconverged_points: int = 0, *, mode=None) -> PriceEstimate:
    """Monte Carlo price under ``rule`` (pricer.py:167-202); deterministic in (seed, n_paths).

    ``engine`` and ``backend`` are accepted for signature compatibility; the
    work runs on this process's GPU(s)."""
    if n_paths < 1:
        raise ValueError(f"need at least one path, got {n_paths}")
    spec.validate_against(params)
    mp = pack_market(params, spec)
    rp = rule.pack(spec)
    t0 = time.perf_counter()
    with nvtx_range("mc"):
        stats = block_stats(mp, rp, n_paths, seed, mode=mode)
    pricing_seconds = time.perf_counter() - t0
    log_phase(engine, "mc", [(_current_shard().rank, pricing_seconds)])
    mean, var, n = pool_moments(stats[:, 0], stats[:, 1], stats[:, 2])
    timings = dict(build_timings or {})
    timings["pricing"] = pricing_seconds
    return PriceEstimate(price=mean, variance=var, ci95=1.96 * float(np.sqrt(var / n)), n_paths=n, timings=timings,
                         rule_kind=getattr(rule, "kind", type(rule).__name__),
                         unconverged_points=unconverged_points)
