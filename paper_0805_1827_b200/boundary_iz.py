"""I&Z exercise-boundary parameterisation (phases [glp], [calc], [reg]) on the device.

Drop-in for the reference's ``build_iz_boundary`` (boundary_iz.py:296-360):
backward over dates, every probe (item asset*J + j, stream
StreamKey(seed, IZ_CALC, item, m), boundary_iz.py:287-288) is solved for the
critical price of its asset, and a quadratic surface is regressed through
the J levels of each asset.  On each GPU one cluster launch solves the GPU's
range of probes (brm_iz_solve: a thread-block cluster per probe iterates the
fixed-point map of _core.pyx:433-512 or, for BASELINE.json configs 1-2, a
bisection with common random numbers, without leaving the kernel); the
levels are all-gathered and every GPU runs the device least-squares fit.

Beyond the reference: the geometric-average put (BASELINE config 2) uses a
log-space surface of the last asset over the other log prices (iz_space 1,
probes on a uniform log grid); the reference rejects d>1 puts
(boundary_iz.py:309-310).
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import backend as _be
from .dist import current as _current_shard
from .engine import log_phase, nvtx_range
from .lowdisc import SeedGrid, default_box, generate_glp, uniform_log_grid
from .market import ConfigError, is_call_like, payoff_code
from .packs import RulePack, n_quad_basis, pack_market, quad_basis

__all__ = ["BoundaryPointJob", "PointResult", "IzBoundary", "IzBuildReport", "continuation_value",
           "solve_boundary_point", "regress_boundary", "build_iz_boundary"]


@dataclass(frozen=True)
class BoundaryPointJob:
    date_index: int
    asset_index: int
    seed_point: np.ndarray
    n_inner: int
    epsilon: float = 0.01
    max_iter: int = 100

    def __post_init__(self):
        if self.n_inner < 1:
            raise ConfigError(f"need at least one inner path, got {self.n_inner}")
        if self.epsilon <= 0.0:
            raise ConfigError(f"epsilon must be positive, got {self.epsilon}")


@dataclass(frozen=True)
class PointResult:
    level: float
    iterations: int
    converged: bool


class IzBoundary:
    """coeffs[m, i] = quadratic-basis coefficients of asset i's boundary at date m.

    iz_space 0 (the reference's): level of the argmax asset over the other
    prices clamped into ``box``, floored at K for calls / capped for puts.
    iz_space 1: log level of the last asset over the other log prices."""

    def __init__(self, strike: float, d: int, n_dates: int, call_like: bool, coeffs, box, iz_space: int = 0):
        nb = n_quad_basis(max(d - 1, 0))
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        if coeffs.shape != (n_dates + 1, d, nb):
            raise ValueError(f"coefficient block has shape {coeffs.shape}, expected {(n_dates + 1, d, nb)}")
        self.strike, self.d, self.n_dates = float(strike), int(d), int(n_dates)
        self.call_like, self.iz_space = bool(call_like), int(iz_space)
        self.coeffs = coeffs
        self.box = np.asarray(box, dtype=np.float64).reshape(-1, 2)
        self._pack = None

    @classmethod
    def terminal_only(cls, spec, d: int, box, iz_space: int = 0) -> "IzBoundary":
        coeffs = np.zeros((spec.n_dates + 1, d, n_quad_basis(max(d - 1, 0))))
        coeffs[spec.n_dates, :, 0] = spec.strike
        return cls(spec.strike, d, spec.n_dates, is_call_like(spec.payoff_kind), coeffs, box, iz_space)

    def level(self, m: int, asset: int, others) -> float:
        z = np.asarray(others, dtype=np.float64).reshape(1, -1)
        if self.iz_space == 1:
            z = np.clip(np.log(z), self.box[:, 0], self.box[:, 1])
            return float(np.exp(quad_basis(z) @ self.coeffs[m, asset]))
        if z.size:
            z = np.clip(z, self.box[:, 0], self.box[:, 1])
        raw = float(quad_basis(z) @ self.coeffs[m, asset]) if z.size else float(self.coeffs[m, asset, 0])
        return max(raw, self.strike) if self.call_like else min(raw, self.strike)

    def crossed(self, m: int, values) -> bool:
        v = np.asarray(values, dtype=np.float64)
        if self.d == 1:
            b = self.level(m, 0, v[:0])
            return v[0] >= b if self.call_like else v[0] <= b
        if self.iz_space == 1:
            return v[-1] <= self.level(m, self.d - 1, v[:-1])
        i = int(np.argmax(v))
        return v[i] >= self.level(m, i, np.delete(v, i))

    def pack(self) -> RulePack:
        if self._pack is None:
            lo = self.box[:, 0] if self.d > 1 else np.zeros(0)
            hi = self.box[:, 1] if self.d > 1 else np.zeros(0)
            self._pack = RulePack.from_surfaces(self.coeffs, lo, hi, self.call_like, self.iz_space)
        return self._pack

    def to_json_dict(self) -> dict:
        doc = {"version": 1, "strike": self.strike, "d": self.d, "n_dates": self.n_dates,
               "call_like": self.call_like, "box": self.box.tolist(), "coeffs": self.coeffs.tolist()}
        if self.iz_space:
            doc["iz_space"] = self.iz_space
        return doc

    @classmethod
    def from_json_dict(cls, doc: dict) -> "IzBoundary":
        if doc.get("version") != 1:
            raise ValueError(f"unsupported boundary document version {doc.get('version')!r}")
        return cls(doc["strike"], doc["d"], doc["n_dates"], doc["call_like"], np.asarray(doc["coeffs"]),
                   np.asarray(doc["box"], dtype=np.float64), int(doc.get("iz_space", 0)))

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict())

    @classmethod
    def from_json(cls, text: str) -> "IzBoundary":
        return cls.from_json_dict(json.loads(text))


@dataclass
class IzBuildReport:
    glp_seconds: float = 0.0
    calc_seconds: float = 0.0
    reg_seconds: float = 0.0
    per_date: list = field(default_factory=list)
    unconverged_points: int = 0
    iteration_counts: list = field(default_factory=list)

    def iteration_spread(self) -> dict:
        if not self.iteration_counts:
            return {"min": 0, "median": 0.0, "max": 0}
        a = np.asarray(self.iteration_counts)
        return {"min": int(a.min()), "median": float(np.median(a)), "max": int(a.max())}

    def to_json_dict(self) -> dict:
        return {"phases": {"glp": self.glp_seconds, "calc": self.calc_seconds, "reg": self.reg_seconds},
                "per_date": self.per_date, "unconverged_points": self.unconverged_points,
                "iteration_spread": self.iteration_spread()}


def _key(key):
    return key.words() if hasattr(key, "words") else key


def continuation_value(x: float, job: BoundaryPointJob, later: IzBoundary, params, spec, key, draw_base: int = 0,
                       backend=None, mode=None) -> float:
    """Mean of n_inner stopped paths from the probe state at level x (boundary_iz.py:198-220)."""
    mp = pack_market(params, spec)
    d = params.d
    others = np.where(job.seed_point > x, x - 0.01 * spec.strike, job.seed_point)
    start = np.insert(np.asarray(others, dtype=np.float64), job.asset_index, x) if d > 1 else np.array([x])
    k, s = _key(key)
    tot, _ = _be.stopped_sums(mp, later.pack(), start, job.date_index, job.n_inner, k, s, draw_base, mode=mode)
    return tot / job.n_inner


def solve_boundary_point(job: BoundaryPointJob, later: IzBoundary, params, spec, key, backend=None,
                         avg_window: int = 5, mode=None) -> PointResult:
    """Fixed-point probe solve (boundary_iz.py:223-247)."""
    mp = pack_market(params, spec)
    k, s = _key(key)
    lv, it, cv = _be.iz_solve(mp, later.pack(), job.seed_point, job.asset_index, job.date_index, job.n_inner,
                              job.epsilon, job.max_iter, avg_window, k, s, mode=mode)
    return PointResult(lv, it, cv)


def regress_boundary(grid: SeedGrid, levels, log_space: bool = False) -> np.ndarray:
    """Least-squares quadratic surface through the levels (boundary_iz.py:250-276), on the device.

    log_space fits log(level) on the basis of log(points)."""
    levels = np.asarray(levels, dtype=np.float64)
    pts = np.log(grid.points) if log_space else grid.points
    design = quad_basis(pts) if pts.shape[1] else np.ones((levels.size, 1))
    n, nb = design.shape
    if n < nb:
        raise ConfigError(f"need at least {nb} probe points for the quadratic fit, got {n}")
    coeffs, deficient = _be.lstsq(design, np.log(levels) if log_space else levels, pts.shape[1])
    if deficient:
        import warnings
        warnings.warn("rank-deficient boundary design; dropping cross terms")
    return coeffs


def _default_bracket(spec, iz_space: int, call_like: bool, lo_mult: float, hi_mult: float):
    K = spec.strike
    if iz_space == 1 or not call_like:
        return lo_mult * K, K
    return K, hi_mult * K


def _torch_cuda():
    try:
        import torch
        return torch if torch.cuda.is_available() else None
    except ImportError:
        return None


def _build_device_loop(params, spec, n_inner, epsilon, max_iter, seed, solver, lo_b, hi_b, tol, mode, shard, torch,
                       mp, d, call_like, iz_space, box, reg_pts, assets_per_item, item_asset, item_seed, j_points,
                       report):
    """The backward date loop with no host round trip until the end: per date
    the probe clusters write their levels to HBM, the level exchange is a
    device collective, and brm_iz_fit regresses the surface(s) on the device
    straight into the rule image the next (earlier) date's probes read.
    Per-date times are CUDA-event times on torch's current stream."""
    from .context import Context
    nd = spec.n_dates
    stream = torch.cuda.current_stream()
    boundary0 = IzBoundary.terminal_only(spec, d, box, iz_space)
    ctx = Context(mp, boundary0.pack(), mode=mode)  # private image, surfaces filled date by date
    ctx.set_stream(stream)
    f64, i32 = torch.float64, torch.int32
    pts = np.log(reg_pts) if iz_space == 1 else reg_pts
    design_h = quad_basis(pts) if pts.shape[1] else np.ones((j_points, 1))
    J, nb = design_h.shape
    if J < nb:
        raise ConfigError(f"need at least {nb} probe points for the quadratic fit, got {J}")
    n_items = item_asset.size
    n_fits = 1 if iz_space == 1 else d
    design = torch.from_numpy(np.ascontiguousarray(design_h)).to("cuda")
    seeds_dev = torch.from_numpy(np.ascontiguousarray(item_seed, dtype=np.float64)).to("cuda")
    assets_dev = torch.from_numpy(np.ascontiguousarray(item_asset, dtype=np.int32)).to("cuda")
    levels = torch.zeros((nd + 1, n_items), dtype=f64, device="cuda")
    iters = torch.zeros((nd + 1, n_items), dtype=i32, device="cuda")
    conv = torch.zeros((nd + 1, n_items), dtype=i32, device="cuda")
    coeffs = torch.zeros((nd + 1, n_fits, nb), dtype=f64, device="cuda")
    ranks = torch.zeros((nd + 1, n_fits), dtype=i32, device="cuda")
    marks = []
    for m in range(nd - 1, 0, -1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        with nvtx_range(f"iz.calc[date {m}]"):
            for lo, hi in shard.local_ranges(n_items):
                if hi > lo:
                    _be.iz_solve_batch(mp, None, seeds_dev[lo:hi] if d > 1 else None, assets_dev[lo:hi], m, n_inner,
                                       solver=solver, epsilon=epsilon, max_iter=max_iter, avg_window=5, lo=lo_b,
                                       hi=hi_b, tol=tol, seed=seed, item_lo=lo, mode=mode, ctx=ctx,
                                       out=(levels[m, lo:hi], iters[m, lo:hi], conv[m, lo:hi]))
            if shard.distributed:  # disjoint rows, zero elsewhere: the sum is an exact gather
                for t in (levels[m], iters[m], conv[m]):
                    shard.all_reduce_sum(t)
        ev[1].record(stream)
        # levels[m] is [n_fits * J]: fit g regresses asset g's probes (one fit in log space)
        with nvtx_range(f"iz.reg[date {m}]"):
            ctx.iz_fit(m, design, J, nb, pts.shape[1], levels[m], n_fits, iz_space == 1, coeffs[m], ranks[m])
        ev[2].record(stream)
        marks.append((m, ev))
    host = {"levels": levels.cpu().numpy(), "iters": iters.cpu().numpy(), "conv": conv.cpu().numpy(),
            "coeffs": coeffs.cpu().numpy(), "ranks": ranks.cpu().numpy()}  # the build's one synchronisation
    ctx.close()
    full = boundary0.coeffs.copy()
    for m, ev in marks:
        if iz_space == 1:
            full[m, :] = host["coeffs"][m, 0]
        else:
            for a_idx, asset in enumerate(assets_per_item):
                full[m, asset] = host["coeffs"][m, a_idx]
        if np.any(host["ranks"][m] < nb):
            import warnings
            warnings.warn("rank-deficient boundary design; dropping cross terms")
        its = host["iters"][m].astype(int)
        n_unconv = int(np.sum(host["conv"][m] == 0))
        calc_s, reg_s = ev[0].elapsed_time(ev[1]) / 1e3, ev[1].elapsed_time(ev[2]) / 1e3
        report.calc_seconds += calc_s
        report.reg_seconds += reg_s
        report.unconverged_points += n_unconv
        report.iteration_counts.extend(its.tolist())
        report.per_date.append({"date_index": m, "calc_seconds": calc_s, "reg_seconds": reg_s,
                                "unconverged": n_unconv, "iterations": its.tolist()})
    report.per_date.reverse()
    return IzBoundary(spec.strike, d, nd, call_like, full, box, iz_space), report


def build_iz_boundary(params, spec, j_points: int, n_inner: int, epsilon: float = 0.01, max_iter: int = 100,
                      seed: int = 0, engine=None, lo_mult: float = 0.5, hi_mult: float = 2.5, backend=None, *,
                      solver: str = "fixed_point", bracket=None, tol: float = 1e-4, grid: str | None = None,
                      mode=None, device_loop=None) -> tuple[IzBoundary, IzBuildReport]:
    """Backward induction over dates (boundary_iz.py:296-360).

    device_loop: keep the date loop on the device (default when a GPU is
    visible): probe levels, the level exchange and the regression stay in
    HBM and the surfaces are written into the rule image without a host
    round trip; False regresses each date on the host path (brm_lstsq)."""
    spec.validate_against(params)
    code = payoff_code(spec.payoff_kind)
    d = params.d
    call_like = is_call_like(spec.payoff_kind)
    if code == 4:
        raise ConfigError("I&Z boundaries are not defined for the arithmetic basket put; use CMC")
    iz_space = 1 if code == 3 and d > 1 else 0
    if code == 3 and d == 1:
        raise ConfigError("geometric put needs d > 1 (use the 1-D put)")
    if solver not in ("fixed_point", "bisection"):
        raise ValueError(f"unknown solver {solver!r}")
    shard = _current_shard()
    report = IzBuildReport()
    t0 = time.perf_counter()
    dim = max(d - 1, 1)
    grid = grid or ("uniform_log" if iz_space == 1 else "glp")
    if grid == "uniform_log":
        sg = uniform_log_grid(j_points, dim, spec.strike, seed, lo_mult, hi_mult)
    else:
        sg = generate_glp(j_points, dim, default_box(spec.strike, dim, lo_mult, hi_mult))
    report.glp_seconds = time.perf_counter() - t0
    box = sg.box if d > 1 else sg.box[:0]
    boundary = IzBoundary.terminal_only(spec, d, box, iz_space)
    seeds = sg.points if d > 1 else np.zeros((j_points, 0))
    reg_grid = sg if d > 1 else SeedGrid(points=seeds, box=box)
    assets_per_item = [d - 1] if iz_space == 1 else list(range(d))
    n_items = len(assets_per_item) * j_points
    item_asset = np.repeat(np.asarray(assets_per_item, dtype=np.int32), j_points)
    item_seed = np.tile(seeds, (len(assets_per_item), 1))
    lo_b, hi_b = bracket if bracket is not None else _default_bracket(spec, iz_space, call_like, lo_mult, hi_mult)
    mp = pack_market(params, spec)
    torch = _torch_cuda()
    if device_loop is None:
        device_loop = torch is not None
    if device_loop:
        if torch is None:
            raise RuntimeError("device_loop=True needs a CUDA device")
        boundary, report = _build_device_loop(params, spec, n_inner, epsilon, max_iter, seed, solver, lo_b, hi_b, tol,
                                              mode, shard, torch, mp, d, call_like, iz_space, box, reg_grid.points,
                                              assets_per_item, item_asset, item_seed, j_points, report)
        _log_report(engine, report)
        return boundary, report
    for m in range(spec.n_dates - 1, 0, -1):
        later = boundary.pack()
        t0 = time.perf_counter()
        res = np.zeros((n_items, 3))
        for lo, hi in shard.local_ranges(n_items):
            if hi > lo:
                lv, it, cv = _be.iz_solve_batch(mp, later, item_seed[lo:hi], item_asset[lo:hi], m, n_inner,
                                                solver=solver, epsilon=epsilon, max_iter=max_iter, avg_window=5,
                                                lo=lo_b, hi=hi_b, tol=tol, seed=seed, item_lo=lo, mode=mode)
                res[lo:hi] = np.stack([lv, it, cv], axis=1)
        if shard.distributed:
            import torch
            t = torch.from_numpy(res).cuda()
            shard.all_reduce_sum(t)  # disjoint rows: exact gather
            res = t.cpu().numpy()
        calc_s = time.perf_counter() - t0
        levels, iters, conv = res[:, 0], res[:, 1].astype(int), res[:, 2].astype(bool)
        t0 = time.perf_counter()
        coeffs = boundary.coeffs.copy()
        for a_idx, asset in enumerate(assets_per_item):
            lv = levels[a_idx * j_points:(a_idx + 1) * j_points]
            c = regress_boundary(reg_grid, lv, log_space=iz_space == 1)
            if iz_space == 1:
                coeffs[m, :] = c  # every row carries the surface of the last asset
            else:
                coeffs[m, asset] = c
        reg_s = time.perf_counter() - t0
        boundary = IzBoundary(spec.strike, d, spec.n_dates, call_like, coeffs, box, iz_space)
        n_unconv = int(np.sum(~conv))
        report.calc_seconds += calc_s
        report.reg_seconds += reg_s
        report.unconverged_points += n_unconv
        report.iteration_counts.extend(iters.tolist())
        report.per_date.append({"date_index": m, "calc_seconds": calc_s, "reg_seconds": reg_s,
                                "unconverged": n_unconv, "iterations": iters.tolist()})
    report.per_date.reverse()
    _log_report(engine, report)
    return boundary, report


def _log_report(engine, report) -> None:
    """Per-date phase times into the caller's timing log (engine.py:126-144, :167)."""
    log_phase(engine, "calc", [(r["date_index"], r["calc_seconds"]) for r in report.per_date])
    log_phase(engine, "reg", [(r["date_index"], r["reg_seconds"]) for r in report.per_date])
