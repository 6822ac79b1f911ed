"""Flat market/rule packs: the data contract of the C ABI.

Same fields and evaluation conventions as the reference packs
(pkg/src/bermuda/_kernels/packs.py:44-193) so that reference-built packs
can be handed to this engine unchanged, plus ``iz_space`` on rule packs
(0 = the reference's price-space argmax surfaces, 1 = log-space surface of
the last asset, used for the geometric put).  Arrays are computed with the
same numpy expressions as the reference so the engine consumes
bit-identical step tables.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .market import payoff_code

__all__ = ["MarketPack", "RulePack", "pack_market", "n_quad_basis", "quad_basis",
           "RULE_EUROPEAN", "RULE_IMMEDIATE", "RULE_IZ", "RULE_CMC"]

RULE_EUROPEAN, RULE_IMMEDIATE, RULE_IZ, RULE_CMC = 0, 1, 2, 3


@dataclass(frozen=True, eq=False)
class MarketPack:
    d: int
    n_dates: int
    strike: float
    payoff_kind: int
    step_mu: np.ndarray
    step_vol: np.ndarray
    chol: np.ndarray
    disc_steps: np.ndarray
    s0: np.ndarray


def pack_market(params, spec) -> MarketPack:
    """Per-step drift/vol and discount tables (reference packs.py:57-71)."""
    spec.validate_against(params)
    dt = spec.dt
    steps = np.arange(spec.n_dates + 1, dtype=np.float64)
    return MarketPack(
        d=int(params.d), n_dates=int(spec.n_dates), strike=float(spec.strike),
        payoff_kind=payoff_code(spec.payoff_kind),
        step_mu=np.ascontiguousarray(params.log_drift * dt),
        step_vol=np.ascontiguousarray(params.sigma * np.sqrt(dt)),
        chol=np.ascontiguousarray(params.corr_factor),
        disc_steps=np.exp(-params.r * dt * steps),
        s0=np.ascontiguousarray(params.s0))


def n_quad_basis(k: int) -> int:
    """|[1, z_a, z_a z_b (a <= b)]| over k coordinates."""
    return 1 + k + k * (k + 1) // 2


def quad_basis(z: np.ndarray) -> np.ndarray:
    """Design rows [1, z_a, z_a z_b (a <= b)] (upper triangle, row-major)."""
    z = np.atleast_2d(np.asarray(z, dtype=np.float64))
    n, k = z.shape
    out = np.empty((n, n_quad_basis(k)))
    out[:, 0] = 1.0
    out[:, 1:1 + k] = z
    col = 1 + k
    for a in range(k):
        width = k - a
        out[:, col:col + width] = z[:, a:a + 1] * z[:, a:]
        col += width
    return out


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int32)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


@dataclass(frozen=True, eq=False)
class RulePack:
    """Exercise rule flattened for the kernels (unused fields are dummies)."""

    kind: int
    call_like: int
    imm_date: int = 0
    iz_coeffs: np.ndarray = field(default_factory=lambda: np.zeros((1, 1, 1)))
    iz_lo: np.ndarray = field(default_factory=lambda: np.zeros(1))
    iz_hi: np.ndarray = field(default_factory=lambda: np.ones(1))
    cmc_starts: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int32))
    cmc_counts: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int32))
    cmc_feat: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    cmc_thr: np.ndarray = field(default_factory=lambda: np.zeros(0))
    cmc_pol: np.ndarray = field(default_factory=lambda: np.zeros(0))
    cmc_alpha: np.ndarray = field(default_factory=lambda: np.zeros(0))
    cmc_intercept: np.ndarray = field(default_factory=lambda: np.zeros(1))
    iz_space: int = 0

    @classmethod
    def european(cls, call_like: bool = True) -> "RulePack":
        return cls(RULE_EUROPEAN, int(call_like))

    @classmethod
    def immediate(cls, date_index: int, call_like: bool = True) -> "RulePack":
        return cls(RULE_IMMEDIATE, int(call_like), imm_date=int(date_index))

    @classmethod
    def from_surfaces(cls, coeffs, lo, hi, call_like: bool, iz_space: int = 0) -> "RulePack":
        """coeffs[(n_dates+1), d, nbasis]; rows of date 0 and the last date unused."""
        return cls(RULE_IZ, int(call_like), iz_coeffs=_f64(coeffs), iz_lo=_f64(lo), iz_hi=_f64(hi),
                   iz_space=int(iz_space))

    @classmethod
    def from_stumps(cls, n_dates: int, per_date: dict, call_like: bool) -> "RulePack":
        """per_date[m] = (feat, thr, pol, alpha, intercept); other dates score -1."""
        starts = np.zeros(n_dates + 1, np.int32)
        counts = np.zeros(n_dates + 1, np.int32)
        icept = np.full(n_dates + 1, -1.0)
        cols = ([], [], [], [])
        pos = 0
        for m in sorted(per_date):
            feat, thr, pol, alpha, c0 = per_date[m]
            starts[m], counts[m], icept[m] = pos, len(feat), c0
            for dst, src in zip(cols, (feat, thr, pol, alpha)):
                dst.extend(np.asarray(src).tolist())
            pos += len(feat)
        return cls(RULE_CMC, int(call_like), cmc_starts=starts, cmc_counts=counts, cmc_intercept=icept,
                   cmc_feat=_i32(cols[0]), cmc_thr=_f64(cols[1]), cmc_pol=_f64(cols[2]),
                   cmc_alpha=_f64(cols[3]))
