"""Option and market configuration objects (host side, no compute).

Mirrors the reference's config surface (pkg/src/bermuda/market.py:36-169):
``ConfigError``, ``PayoffKind``, ``MarketParams``, ``BermudanSpec`` with the
same constructor arguments, validation messages and derived fields, so a
caller of the reference builds the same objects here.  Two payoffs are added
for BASELINE.json configs 2 and 4, which the reference cannot express:
``GEO_PUT`` (put on the geometric average) and ``BASKET_PUT`` (put on the
arithmetic average).  The engine's phase functions also accept the
reference's own objects (duck-typed on these attributes).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

__all__ = ["ConfigError", "PayoffKind", "MarketParams", "BermudanSpec", "payoff_code", "is_call_like"]


class ConfigError(ValueError):
    """Invalid market or contract configuration (reference market.py:36)."""


class PayoffKind(str, Enum):
    MAX_CALL = "maxcall"
    PUT_1D = "put"
    CALL_1D = "call"
    GEO_PUT = "geoput"
    BASKET_PUT = "basketput"

    @property
    def call_like(self) -> bool:
        return self in (PayoffKind.MAX_CALL, PayoffKind.CALL_1D)

    @property
    def one_dimensional(self) -> bool:
        return self in (PayoffKind.PUT_1D, PayoffKind.CALL_1D)


_CODES = {"maxcall": 0, "put": 1, "call": 2, "geoput": 3, "basketput": 4}


def payoff_code(kind) -> int:
    """Kernel payoff code of a PayoffKind (ours or the reference's)."""
    return _CODES[getattr(kind, "value", kind)]


def is_call_like(kind) -> bool:
    return payoff_code(kind) in (0, 2)


def _vector(x, d: int, name: str) -> np.ndarray:
    v = np.asarray(x, dtype=np.float64)
    if v.ndim == 0:
        v = np.full(d, float(v))
    if v.shape != (d,):
        raise ConfigError(f"{name} must be a scalar or length-{d} vector, got shape {v.shape}")
    return v


def _factor(rho: np.ndarray) -> np.ndarray:
    """Cholesky factor, or an eigen square root on the semidefinite boundary."""
    try:
        return np.linalg.cholesky(rho)
    except np.linalg.LinAlgError:
        w, v = np.linalg.eigh(rho)
        if w.min() < -1e-10:
            raise ConfigError(
                f"correlation matrix is not positive semidefinite (min eigenvalue {w.min():.3e})") from None
        return v * np.sqrt(np.clip(w, 0.0, None))


class MarketParams:
    """Risk-neutral GBM market: d assets, spots, rate, vols, yields, correlation."""

    def __init__(self, d: int, s0, r: float, sigma, delta=0.0, rho=None):
        if d < 1:
            raise ConfigError(f"need at least one asset, got d={d}")
        self.d = int(d)
        self.s0 = _vector(s0, self.d, "s0")
        self.r = float(r)
        self.sigma = _vector(sigma, self.d, "sigma")
        self.delta = _vector(delta, self.d, "delta")
        if np.any(self.s0 <= 0.0):
            raise ConfigError("spot prices must be positive")
        if np.any(self.sigma <= 0.0):
            raise ConfigError("volatilities must be positive")
        if rho is None:
            rho = np.eye(self.d)
        elif np.isscalar(rho):
            rho = np.full((self.d, self.d), float(rho)) + (1.0 - float(rho)) * np.eye(self.d)
        rho = np.asarray(rho, dtype=np.float64)
        if rho.shape != (self.d, self.d):
            raise ConfigError(f"rho must be {self.d}x{self.d}, got {rho.shape}")
        if not np.allclose(rho, rho.T, atol=1e-12):
            raise ConfigError("rho must be symmetric")
        if not np.allclose(np.diag(rho), 1.0, atol=1e-12):
            raise ConfigError("rho must have a unit diagonal")
        self.rho = rho
        self.corr_factor = _factor(rho)

    @property
    def log_drift(self) -> np.ndarray:
        """r - delta - sigma^2/2 per asset."""
        return self.r - self.delta - 0.5 * self.sigma ** 2

    def __repr__(self) -> str:
        return f"MarketParams(d={self.d}, r={self.r}, s0={self.s0.tolist()}, sigma={self.sigma.tolist()})"


@dataclass(frozen=True)
class BermudanSpec:
    """Strike, maturity and n_dates equally spaced exercise dates t_m = m T / n."""

    strike: float
    maturity: float
    n_dates: int
    payoff_kind: PayoffKind = PayoffKind.MAX_CALL

    def __post_init__(self):
        if self.strike <= 0.0:
            raise ConfigError("strike must be positive")
        if self.maturity <= 0.0:
            raise ConfigError("maturity must be positive")
        if self.n_dates < 1:
            raise ConfigError("need at least one exercise date")

    @property
    def dt(self) -> float:
        return self.maturity / self.n_dates

    @property
    def date_times(self) -> np.ndarray:
        return np.arange(1, self.n_dates + 1, dtype=np.float64) * self.maturity / self.n_dates

    def validate_against(self, params) -> None:
        kind = PayoffKind(getattr(self.payoff_kind, "value", self.payoff_kind))
        if kind.one_dimensional and params.d != 1:
            raise ConfigError(f"{kind.value} payoff requires d=1, got d={params.d}")
