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
import time
from dataclasses import dataclass, field

import numpy as np

from . import backend as _be
from .boosting import StumpEnsemble, ensemble_from_arrays
from .context import get_context
from .dist import current as _current_shard
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


def build_cmc_rule(params, spec, cfg: CmcBuildConfig, seed: int = 0, engine=None, backend=None, *,
                   sampler: str = "bridge", mode=None) -> tuple[CmcRule, CmcBuildReport]:
    """Fit the per-date classifiers by backward induction (boundary_cmc.py:230-281)."""
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
    for m in range(spec.n_dates - 1, 0, -1):
        later = rule.pack()
        bridge = bridge_scalars(params, spec, m)
        t0 = time.perf_counter()
        lo, hi = shard.range(cfg.n_train)
        if torch is not None:
            # device-resident date step: features and labels stay in HBM, every
            # launch (sampler, walker, AdaBoost) is ordered on torch's stream
            get_context(mp, later, mode=mode).set_stream(stream)
            feats = torch.empty((hi - lo, F), dtype=torch.float64, device="cuda")
            betas = torch.empty((hi - lo,), dtype=torch.float64, device="cuda")
            if hi > lo:
                _be.cmc_calc(mp, later, m, seed, lo, hi - lo, cfg.n_label, bridge, sampler, feats, betas, mode=mode)
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
    return rule, report
