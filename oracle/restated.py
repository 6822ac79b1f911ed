"""Restated CPU pricers for the configs the reference cannot express (C2, C4).

TEST / BASELINE INFRASTRUCTURE ONLY: the
reference package has no geometric-average or arithmetic-basket put
(market.py:40-47), so the CPU baseline of configs 2 and 4 is this
restatement -- the C walker of oracle/bermuda_oracle.c, run over every host
core (POSIX threads, one item per task), driven by the same algorithm as the
engine:

* C2 (I&Z, geometric put, d = 5): per date, bisection solves of every probe
  (orc_iz_bisect_batch, common random numbers), the log-space quadratic
  regression (numpy lstsq, boundary_iz.py:250-276 restated), then final
  pricing over 4096-path blocks (orc_price_blocks).
* C4 (CMC, arithmetic-basket put, d = 40): per date, forward-sampled training
  points (orc_sample_points), labels under the later dates' rule
  (orc_cmc_labels_mt), the numpy AdaBoost restatement (oracle.fit_ensemble),
  then final pricing.

Results are labelled "restated, not reference" wherever they are reported.
The market and rule packs are restated here from the reference's conventions
(packs.py:57-71, 133-182) so this module does not import the engine.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from types import SimpleNamespace

import numpy as np

from . import oracle as O

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_up = C.POINTER(C.c_uint64)
_lib = O._lib
_lib.orc_threads.restype = C.c_int
_lib.orc_threads.argtypes = []
for _name, _args in {
    "orc_cmc_labels_mt": [C.POINTER(O.OrcCtx), _dp, C.c_int64, C.c_int, C.c_int, _up, _up, C.c_uint64, _dp],
    "orc_iz_bisect_batch": [C.POINTER(O.OrcCtx), _dp, C.c_int, _ip, C.c_int64, C.c_int, C.c_int, C.c_double,
                            C.c_double, C.c_double, C.c_int, C.c_uint64, C.c_int64, _dp, _ip, _ip],
    "orc_price_blocks": [C.POINTER(O.OrcCtx), _dp, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, _dp],
}.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = C.c_int

PAY = {"maxcall": 0, "put": 1, "call": 2, "geoput": 3, "basketput": 4}


def threads() -> int:
    return int(_lib.orc_threads())


def market_pack(d, s0, r, sigma, delta, rho, strike, maturity, n_dates, payoff):
    """MarketPack restated (packs.py:57-71; market.py:59-75 correlation factor)."""
    sigma = np.broadcast_to(np.asarray(sigma, dtype=np.float64), (d,)).copy()
    delta = np.broadcast_to(np.asarray(delta, dtype=np.float64), (d,)).copy()
    if rho is None:
        corr = np.eye(d)
    else:
        corr = np.full((d, d), float(rho)) + (1.0 - float(rho)) * np.eye(d)
    dt = maturity / n_dates
    return SimpleNamespace(d=d, n_dates=n_dates, strike=float(strike), payoff_kind=PAY[payoff],
                           step_mu=(r - delta - 0.5 * sigma ** 2) * dt, step_vol=sigma * math.sqrt(dt),
                           chol=np.linalg.cholesky(corr), disc_steps=np.exp(-r * dt * np.arange(n_dates + 1)),
                           s0=np.full(d, float(s0)), log_drift=r - delta - 0.5 * sigma ** 2, sigma=sigma,
                           r=r, maturity=maturity)


def _rule(kind, call_like, n_dates, d, **kw):
    z = np.zeros(1)
    zi = np.zeros(n_dates + 1, np.int32)
    rp = SimpleNamespace(kind=kind, call_like=int(call_like), imm_date=-1, iz_space=0,
                         iz_coeffs=z, iz_lo=z, iz_hi=z, cmc_starts=zi, cmc_counts=zi, cmc_feat=np.zeros(1, np.int32),
                         cmc_thr=z, cmc_pol=z, cmc_alpha=z, cmc_intercept=np.full(n_dates + 1, -1.0))
    for k, v in kw.items():
        setattr(rp, k, v)
    return rp


def cmc_rule(n_dates, per_date, call_like):
    """RulePack.from_stumps restated (packs.py:149-182)."""
    starts = np.zeros(n_dates + 1, np.int32)
    counts = np.zeros(n_dates + 1, np.int32)
    icept = np.full(n_dates + 1, -1.0)
    cols = ([], [], [], [])
    pos = 0
    for m in sorted(per_date):
        feat, thr, pol, alpha, c0 = per_date[m]
        starts[m], counts[m], icept[m] = pos, len(feat), c0
        for dst, src in zip(cols, (feat, thr, pol, alpha)):
            dst.extend(list(src))
        pos += len(feat)
    f = np.asarray(cols[0] or [0], np.int32)
    return _rule(3, call_like, n_dates, 0, cmc_starts=starts, cmc_counts=counts, cmc_intercept=icept, cmc_feat=f,
                 cmc_thr=np.asarray(cols[1] or [0.0]), cmc_pol=np.asarray(cols[2] or [0.0]),
                 cmc_alpha=np.asarray(cols[3] or [0.0]))


def quad_basis(z):
    z = np.atleast_2d(z)
    n, k = z.shape
    cols = [np.ones(n)] + [z[:, a] for a in range(k)] + [z[:, a] * z[:, b] for a in range(k) for b in range(a, k)]
    return np.stack(cols, axis=1)


def price(mp, rp, n_paths, seed):
    ctx = O.Ctx(mp, rp)
    n_blocks = (n_paths + 4095) // 4096
    out = np.empty((n_blocks, 3))
    s0 = np.ascontiguousarray(mp.s0)
    _lib.orc_price_blocks(ctx.ref, s0.ctypes.data_as(_dp), n_paths, seed, 0, n_blocks, out.ctypes.data_as(_dp))
    mean, var, n = O.pool_moments(out[:, 0], out[:, 1], out[:, 2])
    return mean, 1.96 * math.sqrt(var / n)


def build_price_iz_geoput(cfg, seed, j_points=None):
    """C2: I&Z bisection over a uniform log-price probe grid, log-space surface
    of the last asset (the engine's algorithm), then final pricing."""
    d, nd, K = cfg["d"], cfg["n_dates"], cfg["strike"]
    J = j_points or cfg["j_points"]
    mp = market_pack(d, cfg["s0"], cfg["r"], cfg["sigma"], cfg["delta"], cfg["rho"], K, cfg["maturity"], nd,
                     cfg["payoff"])
    k = d - 1
    lo, hi = math.log(0.5 * K), math.log(2.5 * K)
    pts = np.exp(lo + np.random.default_rng(seed).random((J, k)) * (hi - lo))
    design = quad_basis(np.log(pts))
    nb = design.shape[1]
    coeffs = np.zeros((nd + 1, d, nb))
    coeffs[nd, :, 0] = K
    box_lo, box_hi = np.full(k, lo), np.full(k, hi)
    assets = np.full(J, d - 1, np.int32)
    lvl, its, cv = np.empty(J), np.empty(J, np.int32), np.empty(J, np.int32)
    seeds = np.ascontiguousarray(pts)
    (blo, bhi), tol = cfg["bracket"], cfg["tol"]
    evals = 0
    for m in range(nd - 1, 0, -1):
        rp = _rule(2, False, nd, d, iz_coeffs=coeffs.copy(), iz_lo=box_lo, iz_hi=box_hi, iz_space=1)
        ctx = O.Ctx(mp, rp)
        _lib.orc_iz_bisect_batch(ctx.ref, seeds.ctypes.data_as(_dp), k, assets.ctypes.data_as(_ip), J, m,
                                 cfg["n_inner"], blo, bhi, tol, 1000, seed, 0, lvl.ctypes.data_as(_dp),
                                 its.ctypes.data_as(_ip), cv.ctypes.data_as(_ip))
        evals += int(its.sum()) * (nd - m)
        c = O.regress(design, np.log(lvl))
        coeffs[m, :] = c
    rp = _rule(2, False, nd, d, iz_coeffs=coeffs, iz_lo=box_lo, iz_hi=box_hi, iz_space=1)
    p, ci = price(mp, rp, cfg["n_paths"], seed)
    return p, ci, float(evals) * cfg["n_inner"] / max(J, 1), J


def build_price_cmc(cfg, seed, n_train, n_label, n_paths):
    """C4 (and any CMC config): forward-sampled points, labels under the later
    rule, numpy AdaBoost, final pricing -- at the given (scaled) sizes."""
    d, nd, K = cfg["d"], cfg["n_dates"], cfg["strike"]
    sigma = cfg["sigma"]
    if sigma == "u[0.2,0.4]":
        sigma = np.random.default_rng(1827).uniform(0.2, 0.4, d)
    mp = market_pack(d, cfg["s0"], cfg["r"], sigma, cfg["delta"], cfg["rho"], K, cfg["maturity"], nd, cfg["payoff"])
    call_like = cfg["payoff"] in ("maxcall", "call")
    per_date = {}
    params = SimpleNamespace(s0=mp.s0, log_drift=mp.log_drift, sigma=mp.sigma)
    spec = SimpleNamespace(maturity=cfg["maturity"], dt=cfg["maturity"] / nd, n_dates=nd)
    for m in range(nd - 1, 0, -1):
        later = cmc_rule(nd, per_date, call_like)
        ctx = O.Ctx(mp, later)
        pts, keys, streams = O.sample_points(ctx, params, spec, m, seed, n_train, 0, mode=1)
        beta = np.empty(n_train)
        _lib.orc_cmc_labels_mt(ctx.ref, np.ascontiguousarray(pts).ctypes.data_as(_dp), n_train, m, n_label,
                               keys.ctypes.data_as(_up), streams.ctypes.data_as(_up), m * d,
                               beta.ctypes.data_as(_dp))
        agg = pts.mean(axis=1) if cfg["payoff"] == "basketput" else pts.max(axis=1)
        xs = np.hstack([pts, agg[:, None]])
        f, t, p, a, ic = O.fit_ensemble(xs, beta, cfg["rounds"])
        per_date[m] = (f, t, p, a, ic)
    p, ci = price(mp, cmc_rule(nd, per_date, call_like), n_paths, seed)
    return p, ci


def time_config(cfg, scale: float = 1.0, seed: int = 1827) -> dict:
    """Wall time of one restated build + price on every host core, and its
    nominal path-steps (paths x remaining dates) at the sizes it ran."""
    t0 = time.perf_counter()
    nd = cfg["n_dates"]
    if cfg["method"] == "iz":
        _, _, _, _ = build_price_iz_geoput(cfg, seed)
        n_train = None
        iters = math.ceil(math.log2((cfg["bracket"][1] - cfg["bracket"][0]) / cfg["tol"]))
        work = sum(cfg["j_points"] * iters * cfg["n_inner"] * (nd - m) for m in range(1, nd)) + cfg["n_paths"] * nd
        sample = (f"{cfg['name']}: full config (J={cfg['j_points']}, n_inner={cfg['n_inner']}, "
                  f"n_paths={cfg['n_paths']})")
    else:
        # the training points and final paths are scaled; the label paths per
        # point stay full so the walker / AdaBoost share stays that of the config
        n_train = max(int(cfg["n_train"] * scale), 64)
        n_label = cfg["n_label"]
        n_paths = max(int(cfg["n_paths"] * scale), 1 << 14)
        build_price_cmc(cfg, seed, n_train, n_label, n_paths)
        work = sum(n_train * n_label * (nd - m) for m in range(1, nd)) + n_paths * nd
        sample = (f"{cfg['name']} at scale: n_train={n_train}, n_label={n_label}, n_paths={n_paths}, "
                  f"rounds={cfg['rounds']} (full: {cfg['n_train']}, {cfg['n_label']}, {cfg['n_paths']})")
    dt = time.perf_counter() - t0
    return {"seconds": dt, "path_steps": float(work), "value": work / dt, "threads": threads(), "sample": sample}
