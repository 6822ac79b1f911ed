"""CMC exercise-region classification (phases [calc] and [class]) on the device.

Drop-in for the reference's ``build_cmc_rule`` (boundary_cmc.py:230-281):
backward over dates m = n_dates-1 .. 1, each date samples n_train points,
labels them with beta = payoff - continuation under the rule of the later
dates, and fits a boosted-stump classifier.  Per date, on each GPU:

  brm_cmc_calc      sampler + classifier features + labels for the GPU's
                    contiguous range of training points (one kernel walk,
                    one CTA per point, draws continuing each point's stream)
  all-gather        features and labels of every range (NCCL, dist.py)
  brm_fit_ensemble  the AdaBoost kernel on the full training set (every
                    GPU fits the same deterministic ensemble)

Streams are the reference's: point i of date m uses StreamKey(seed,
CMC_CALC, i, m), the sampler draws 0..2d-1 and the labels continue at 2d
(boundary_cmc.py:164-177, 220-226).  ``sampler="forward"`` steps points
forward from S0 instead (BASELINE.json), labels then start at draw m*d.
"""

from __future__ import annotations

import json
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import backend as _be
from .boosting import StumpEnsemble, ensemble_from_arrays
from .context import get_context
from .dist import current as _current_shard
from .engine import log_phase, nvtx_range
from .market import ConfigError, is_call_like
from .packs import RulePack, pack_market

__all__ = ["CmcRule", "CmcBuildConfig", "CmcBuildReport", "build_cmc_rule", "classifier_features",
           "n_classifier_features", "bridge_scalars", "sample_training_points", "label_points"]


def n_classifier_features(d: int) -> int:
    return d + 1 if d > 1 else 1


def classifier_features(values, d: int, payoff_kind=0) -> np.ndarray:
    """[S_0..S_{d-1}, aggregate] (boundary_cmc.py:38-52): max for the max-call,
    arithmetic / geometric mean for the basket / geometric puts."""
    v = np.atleast_2d(np.asarray(values, dtype=np.float64))
    if d == 1:
        return v
    from .market import payoff_code
    code = payoff_code(payoff_kind) if not isinstance(payoff_kind, int) else payoff_kind
    if code == 3:
        agg = np.exp(np.log(v).sum(axis=1) / d)
    elif code == 4:
        agg = v.sum(axis=1) / d
    else:
        agg = v.max(axis=1)
    return np.hstack([v, agg[:, None]])


class CmcRule:
    """Per-date stump ensembles; the final date exercises on payoff alone."""

    def __init__(self, d: int, n_dates: int, call_like: bool, ensembles: dict):
        want = n_classifier_features(d)
        for m, ens in ensembles.items():
            if not 1 <= m < n_dates:
                raise ValueError(f"ensemble date {m} outside 1..{n_dates - 1}")
            if ens.dim != want:
                raise ValueError(f"ensemble at date {m} has feature dim {ens.dim}, expected {want}")
        self.d, self.n_dates, self.call_like = int(d), int(n_dates), bool(call_like)
        self.ensembles = dict(sorted(ensembles.items()))
        self._pack = None

    @classmethod
    def empty(cls, d: int, n_dates: int, call_like: bool = True) -> "CmcRule":
        return cls(d, n_dates, call_like, {})

    def score(self, m: int, values, payoff_kind=0) -> float:
        ens = self.ensembles.get(m)
        if ens is None:
            return -1.0
        return float(ens.score(classifier_features(values, self.d, payoff_kind)[0]))

    def restricted_after(self, m: int) -> "CmcRule":
        return CmcRule(self.d, self.n_dates, self.call_like, {k: v for k, v in self.ensembles.items() if k > m})

    def pack(self) -> RulePack:
        if self._pack is None:
            per = {m: (*e.arrays(), e.intercept) for m, e in self.ensembles.items()}
            self._pack = RulePack.from_stumps(self.n_dates, per, self.call_like)
        return self._pack

    def to_json_dict(self) -> dict:
        return {"version": 1, "d": self.d, "n_dates": self.n_dates, "call_like": self.call_like,
                "dates": {str(m): e.to_json_dict() for m, e in self.ensembles.items()}}

    @classmethod
    def from_json_dict(cls, doc: dict) -> "CmcRule":
        if doc.get("version") != 1:
            raise ValueError(f"unsupported rule document version {doc.get('version')!r}")
        ens = {int(m): StumpEnsemble.from_json_dict(e) for m, e in doc["dates"].items()}
        return cls(doc["d"], doc["n_dates"], doc["call_like"], ens)

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict())

    @classmethod
    def from_json(cls, text: str) -> "CmcRule":
        return cls.from_json_dict(json.loads(text))


@dataclass(frozen=True)
class CmcBuildConfig:
    n_train: int
    n_label: int
    boost_rounds: int = 100

    def __post_init__(self):
        if self.n_train < 1 or self.n_label < 1:
            raise ConfigError("training and labeling path counts must be positive")
        if self.boost_rounds < 1:
            raise ConfigError("need at least one boosting round")


@dataclass
class CmcBuildReport:
    calc_seconds: float = 0.0
    class_seconds: float = 0.0
    per_date: list = field(default_factory=list)
    one_class_dates: list = field(default_factory=list)

    def to_json_dict(self) -> dict:
        return {"phases": {"calc": self.calc_seconds, "class": self.class_seconds}, "per_date": self.per_date,
                "one_class_dates": self.one_class_dates}


def bridge_scalars(params, spec, m: int) -> np.ndarray:
    """Host scalars of the reference sampler, formed as market.py:180-220 forms them."""
    T = spec.maturity
    t = m * spec.dt
    sd = math.sqrt((t - 0.0) * (T - t) / (T - 0.0)) if m < spec.n_dates else 0.0
    return np.concatenate([params.log_drift * T, params.sigma * math.sqrt(T), np.log(params.s0),
                           params.sigma * sd, [(t - 0.0) / (T - 0.0)]])


def sample_training_points(params, spec, m: int, n_points: int, seed: int, sampler: str = "bridge",
                           mode=None) -> np.ndarray:
    """Training points at date m, one stream per point (boundary_cmc.py:180-189), on the device."""
    if not 1 <= m <= spec.n_dates:
        raise ValueError(f"date index {m} outside 1..{spec.n_dates}")
    mp = pack_market(params, spec)
    rp = RulePack.european(is_call_like(spec.payoff_kind))
    return _be.sample_points(mp, rp, m, seed, 0, n_points, bridge=bridge_scalars(params, spec, m), sampler=sampler,
                             mode=mode)


def label_points(params, spec, points, m: int, n_label: int, later: CmcRule, seed: int, item_lo: int = 0,
                 draw_base: int | None = None, mode=None) -> np.ndarray:
    """beta for given points on StreamKey(seed, CMC_CALC, item_lo + i, m) (boundary_cmc.py:192-207)."""
    mp = pack_market(params, spec)
    db = 2 * params.d if draw_base is None else draw_base
    return _be.cmc_labels_keyed(mp, later.pack(), np.asarray(points, dtype=np.float64), m, n_label, seed, item_lo,
                                db, mode=mode)


def _torch_cuda():
    """torch when a CUDA device is visible (device-resident buffers), else None."""
    try:
        import torch
        return torch if torch.cuda.is_available() else None
    except ImportError:
        return None


# Largest slotted rule image (shared memory of every walker CTA) for which the
# device-resident date loop is used; beyond it the per-date host-built images
# are smaller and keep the walker's occupancy.
_SLOT_IMAGE_LIMIT = 96 * 1024


def slot_image_bytes(n_dates: int, capacity: int, n_features: int, fast: bool) -> int:
    """Shared-memory bytes of a brm_ctx_create_cmc image (brm_internal.h SlotDims)."""
    per_date_dbl = 2 * capacity + 2 * capacity + capacity + n_features  # thr, ap, thresholds, table values
    n_dbl = (n_dates + 1) * per_date_dbl + 64
    n_int = (n_dates + 1) * (capacity + 3 * n_features + 2)
    return (4 if fast else 8) * n_dbl + 4 * n_int


def _build_device_loop(params, spec, cfg, seed, sampler, mode, shard, torch, stream, mp, F, call_like):
    """The backward date loop with every date's work enqueued on one stream and
    no host round trip until the end: the fitted stumps stay in HBM and
    brm_ctx_set_ensemble writes them into the rule image the next (earlier)
    date labels under.  Per-date times are CUDA-event times."""
    from .context import Context
    nd, R = spec.n_dates, cfg.boost_rounds
    ctx = Context.cmc_slots(mp, call_like, R, mode=mode)
    ctx.set_stream(stream)
    f64, i32 = torch.float64, torch.int32
    out = {"feat": torch.zeros((nd + 1, R), dtype=i32, device="cuda"),
           "thr": torch.zeros((nd + 1, R), dtype=f64, device="cuda"),
           "pol": torch.zeros((nd + 1, R), dtype=f64, device="cuda"),
           "alpha": torch.zeros((nd + 1, R), dtype=f64, device="cuda"),
           "err": torch.zeros((nd + 1, R), dtype=f64, device="cuda"),
           "count": torch.zeros((nd + 1,), dtype=i32, device="cuda"),
           "intercept": torch.full((nd + 1,), -1.0, dtype=f64, device="cuda")}
    n_pos = torch.zeros((nd + 1,), dtype=i32, device="cuda")
    marks = []
    for m in range(nd - 1, 0, -1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        with nvtx_range(f"cmc.calc[date {m}]"):
            ranges = shard.local_ranges(cfg.n_train)
            rows = sum(hi - lo for lo, hi in ranges)
            feats = torch.empty((rows, F), dtype=f64, device="cuda")
            betas = torch.empty((rows,), dtype=f64, device="cuda")
            off = 0
            # one rank, one range: the fit below reads this very tensor, so its column sort can run
            # beside the label walk (brm_fit_presort); BRM_NO_PRESORT=1 keeps it inside the fit
            ctx.set_presort(not shard.distributed and len(ranges) == 1 and rows == cfg.n_train
                            and not os.environ.get("BRM_NO_PRESORT"))
            for lo, hi in ranges:
                if hi > lo:
                    _be.cmc_calc(mp, None, m, seed, lo, hi - lo, cfg.n_label, bridge_scalars(params, spec, m),
                                 sampler, feats[off:off + hi - lo], betas[off:off + hi - lo], mode=mode, ctx=ctx)
                off += hi - lo
            feats = shard.all_gather_rows(feats, cfg.n_train)
            betas = shard.all_gather_rows(betas, cfg.n_train)
        ev[1].record(stream)
        with nvtx_range(f"cmc.class[date {m}]"):
            date_out = {k: (v[m] if v.dim() == 2 else v[m:m + 1]) for k, v in out.items()}
            date_out["n_pos"] = n_pos[m:m + 1]
            _be.fit_ensemble_device(feats, betas, R, date_out, mode=mode, stream=stream)
            ctx.set_ensemble(m, date_out["feat"], date_out["thr"], date_out["pol"], date_out["alpha"],
                             date_out["count"], date_out["intercept"])
        ev[2].record(stream)
        marks.append((m, ev))
    host = {k: v.cpu().numpy() for k, v in out.items()}  # the build's one synchronisation
    # np.mean(betas > 0.0) (boundary_cmc.py:275): count / n in fp64
    pos_h = n_pos.cpu().numpy().astype(np.float64) / cfg.n_train
    ensembles, report = {}, CmcBuildReport()
    for m, ev in marks:
        c = int(host["count"][m])
        ens = ensemble_from_arrays(F, host["feat"][m, :c], host["thr"][m, :c], host["pol"][m, :c],
                                   host["alpha"][m, :c], float(host["intercept"][m]))
        ensembles[m] = ens
        if not ens.rounds:
            report.one_class_dates.append(m)
        calc_s, class_s = ev[0].elapsed_time(ev[1]) / 1e3, ev[1].elapsed_time(ev[2]) / 1e3
        report.calc_seconds += calc_s
        report.class_seconds += class_s
        report.per_date.append({"date_index": m, "calc_seconds": calc_s, "class_seconds": class_s,
                                "positive_fraction": float(pos_h[m]), "rounds": len(ens.rounds)})
    report.per_date.reverse()
    return CmcRule(params.d, nd, call_like, ensembles), report


def build_cmc_rule(params, spec, cfg: CmcBuildConfig, seed: int = 0, engine=None, backend=None, *,
                   sampler: str = "bridge", mode=None, device_loop=None) -> tuple[CmcRule, CmcBuildReport]:
    """Fit the per-date classifiers by backward induction (boundary_cmc.py:230-281).

    device_loop: enqueue every date without host round trips (default: on a
    GPU when the slotted rule image fits, see ``slot_image_bytes``); False
    rebuilds the rule image on the host per date.  Both give the same rule."""
    spec.validate_against(params)
    if sampler not in ("bridge", "forward"):
        raise ValueError(f"unknown sampler {sampler!r}")
    shard = _current_shard()
    mp = pack_market(params, spec)
    d = params.d
    F = n_classifier_features(d)
    call_like = is_call_like(spec.payoff_kind)
    rule = CmcRule.empty(d, spec.n_dates, call_like)
    report = CmcBuildReport()
    torch = _torch_cuda()
    stream = torch.cuda.current_stream() if torch is not None else None
    if device_loop is None:
        from .context import resolve_mode
        fast = resolve_mode(mode) == 1
        device_loop = (torch is not None and cfg.boost_rounds <= 1024
                       and slot_image_bytes(spec.n_dates, cfg.boost_rounds, F, fast) <= _SLOT_IMAGE_LIMIT)
    if device_loop:
        if torch is None:
            raise RuntimeError("device_loop=True needs a CUDA device")
        rule, report = _build_device_loop(params, spec, cfg, seed, sampler, mode, shard, torch, stream, mp, F,
                                          call_like)
        _log_report(engine, report)
        return rule, report
    for m in range(spec.n_dates - 1, 0, -1):
        later = rule.pack()
        bridge = bridge_scalars(params, spec, m)
        t0 = time.perf_counter()
        ranges = shard.local_ranges(cfg.n_train)
        if torch is not None:
            # device-resident date step: features and labels stay in HBM, every
            # launch (sampler, walker, AdaBoost) is ordered on torch's stream
            date_ctx = get_context(mp, later, mode=mode)
            date_ctx.set_stream(stream)
            rows = sum(hi - lo for lo, hi in ranges)
            # (as in the device loop: the fit's column sort beside the label walk)
            date_ctx.set_presort(not shard.distributed and len(ranges) == 1 and rows == cfg.n_train
                                 and not os.environ.get("BRM_NO_PRESORT"))
            feats = torch.empty((rows, F), dtype=torch.float64, device="cuda")
            betas = torch.empty((rows,), dtype=torch.float64, device="cuda")
            off = 0
            for lo, hi in ranges:
                if hi > lo:
                    _be.cmc_calc(mp, later, m, seed, lo, hi - lo, cfg.n_label, bridge, sampler,
                                 feats[off:off + hi - lo], betas[off:off + hi - lo], mode=mode)
                off += hi - lo
            feats = shard.all_gather_rows(feats, cfg.n_train)
            betas = shard.all_gather_rows(betas, cfg.n_train)
        else:
            feats, betas = _be.cmc_calc(mp, later, m, seed, 0, cfg.n_train, cfg.n_label, bridge, sampler, mode=mode)
        calc_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        f, t, p, a, _, icept = _be.fit_ensemble_arrays(feats, betas, cfg.boost_rounds, mode=mode, stream=stream)
        ens = ensemble_from_arrays(F, f, t, p, a, icept)
        class_s = time.perf_counter() - t0
        pos = float((betas > 0).double().mean().item()) if torch is not None else float(np.mean(betas > 0.0))
        if not ens.rounds:
            report.one_class_dates.append(m)
        ensembles = dict(rule.ensembles)
        ensembles[m] = ens
        rule = CmcRule(d, spec.n_dates, call_like, ensembles)
        report.calc_seconds += calc_s
        report.class_seconds += class_s
        report.per_date.append({"date_index": m, "calc_seconds": calc_s, "class_seconds": class_s,
                                "positive_fraction": pos, "rounds": len(ens.rounds)})
    report.per_date.reverse()
    _log_report(engine, report)
    return rule, report


def _log_report(engine, report) -> None:
    """Per-date phase times into the caller's timing log (engine.py:126-144, :167)."""
    log_phase(engine, "calc", [(r["date_index"], r["calc_seconds"]) for r in report.per_date])
    log_phase(engine, "class", [(r["date_index"], r["class_seconds"]) for r in report.per_date])
