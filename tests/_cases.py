"""Shared market/rule builders for the parity tests (no reference import)."""
from __future__ import annotations

import numpy as np

from paper_0805_1827_b200.market import BermudanSpec, MarketParams, PayoffKind
from paper_0805_1827_b200.packs import RulePack, n_quad_basis, pack_market


def maxcall(d=5, n_dates=9, rho=None, sigma=0.2):
    p = MarketParams(d=d, s0=100.0, r=0.05, sigma=sigma, delta=0.1, rho=rho)
    s = BermudanSpec(100.0, 3.0, n_dates, PayoffKind.MAX_CALL)
    return p, s


def put1d(n_dates=10):
    p = MarketParams(d=1, s0=40.0, r=0.06, sigma=0.2)
    s = BermudanSpec(40.0, 1.0, n_dates, PayoffKind.PUT_1D)
    return p, s


def geoput(d=5, n_dates=10):
    p = MarketParams(d=d, s0=100.0, r=0.03, sigma=0.4)
    s = BermudanSpec(100.0, 1.0, n_dates, PayoffKind.GEO_PUT)
    return p, s


def basketput(d=40, n_dates=20, seed=1827):
    sig = np.random.default_rng(seed).uniform(0.2, 0.4, d)
    p = MarketParams(d=d, s0=100.0, r=0.05, sigma=sig, rho=0.3)
    s = BermudanSpec(100.0, 1.0, n_dates, PayoffKind.BASKET_PUT)
    return p, s


def random_stumps(d, n_dates, per_date=40, seed=0, lo=70.0, hi=140.0, call_like=True):
    rng = np.random.default_rng(seed)
    nf = d + 1 if d > 1 else 1
    per = {}
    for m in range(1, n_dates):
        feat = rng.integers(0, nf, per_date)
        thr = rng.uniform(lo, hi, per_date)
        pol = rng.choice([-1.0, 1.0], per_date)
        alpha = rng.uniform(0.05, 1.0, per_date)
        per[m] = (feat, thr, pol, alpha, 0.0)
    return RulePack.from_stumps(n_dates, per, call_like)


def random_surfaces(d, n_dates, strike, seed=0, iz_space=0, call_like=True):
    lvl = (1.1, 1.4) if call_like else (0.8, 0.95)
    rng = np.random.default_rng(seed)
    k = max(d - 1, 0)
    nb = n_quad_basis(k)
    coeffs = np.zeros((n_dates + 1, d, nb))
    if iz_space == 1:
        # log x* = c0 - sum log z  (geometric boundary g* = exp(c0/d)) + small curvature
        for m in range(1, n_dates):
            g = np.log(strike * rng.uniform(0.8, 0.95))
            coeffs[m, :, 0] = d * g
            coeffs[m, :, 1:1 + k] = -1.0
            coeffs[m, :, 1 + k:] = rng.normal(scale=1e-3, size=nb - 1 - k)
        lo, hi = np.full(k, np.log(0.5 * strike)), np.full(k, np.log(2.5 * strike))
    else:
        for m in range(1, n_dates):
            coeffs[m, :, 0] = strike * rng.uniform(*lvl)
            if k:
                coeffs[m, :, 1:1 + k] = rng.normal(scale=0.05, size=(d, k))
                coeffs[m, :, 1 + k:] = rng.normal(scale=2e-4, size=(d, nb - 1 - k))
        lo, hi = np.full(max(k, 1), 0.5 * strike), np.full(max(k, 1), 2.5 * strike)
        if k == 0:
            lo, hi = lo[:0], hi[:0]
    coeffs[n_dates, :, 0] = strike
    return RulePack.from_surfaces(coeffs, lo, hi, call_like, iz_space)


def packs(p, s):
    return pack_market(p, s)
