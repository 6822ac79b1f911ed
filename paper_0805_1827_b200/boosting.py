"""Boosted decision stumps, fitted on the device.

Same public surface as the reference's boosting module (boosting.py:28-211:
``Stump``, ``StumpEnsemble``, ``TrainingSet``, ``fit_stump``,
``fit_ensemble``, ``score``) and the same JSON v1 format.  The fit itself is
the cooperative AdaBoost kernel of libbermuda_b200.so (brm_fit_ensemble):
columns sorted once per fit, numpy's cumsum / pairwise-sum orders and the
reference tie rules in parity mode.
"""

from __future__ import annotations

import json
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import backend as _be

__all__ = ["Stump", "StumpEnsemble", "TrainingSet", "fit_stump", "fit_ensemble", "score"]


@dataclass(frozen=True)
class Stump:
    """Votes ``polarity`` where x[feature] > threshold, else -polarity."""

    feature: int
    threshold: float
    polarity: float
    alpha: float = 1.0

    def predict(self, xs: np.ndarray) -> np.ndarray:
        return np.where(np.asarray(xs)[:, self.feature] > self.threshold, self.polarity, -self.polarity)


@dataclass(frozen=True)
class TrainingSet:
    """Points xs[n, F] with raw labels betas[n]; ys = +1 where beta > 0."""

    xs: np.ndarray
    betas: np.ndarray
    ys: np.ndarray = field(init=False)

    def __post_init__(self):
        xs = np.ascontiguousarray(self.xs, dtype=np.float64)
        betas = np.asarray(self.betas, dtype=np.float64)
        if xs.ndim != 2 or betas.shape != (xs.shape[0],):
            raise ValueError(f"inconsistent training set shapes {xs.shape}, {betas.shape}")
        object.__setattr__(self, "xs", xs)
        object.__setattr__(self, "betas", betas)
        object.__setattr__(self, "ys", np.where(betas > 0.0, 1.0, -1.0))


@dataclass(frozen=True)
class StumpEnsemble:
    dim: int
    rounds: tuple = ()
    intercept: float = 0.0

    def score(self, x) -> float:
        x = np.asarray(x, dtype=np.float64)
        s = self.intercept
        for st in self.rounds:
            s += st.alpha * (st.polarity if x[st.feature] > st.threshold else -st.polarity)
        return s

    def score_many(self, xs) -> np.ndarray:
        xs = np.asarray(xs, dtype=np.float64)
        out = np.full(xs.shape[0], self.intercept)
        for st in self.rounds:
            out += st.alpha * st.predict(xs)
        return out

    def decisions(self, xs) -> np.ndarray:
        return np.where(self.score_many(xs) > 0.0, 1.0, -1.0)

    def arrays(self):
        """(feat, thr, pol, alpha) columns for a rule pack."""
        r = self.rounds
        return ([s.feature for s in r], [s.threshold for s in r], [s.polarity for s in r], [s.alpha for s in r])

    def to_json_dict(self) -> dict:
        return {"version": 1, "dim": self.dim, "intercept": self.intercept,
                "rounds": [{"feature": s.feature, "threshold": None if np.isneginf(s.threshold) else s.threshold,
                            "polarity": s.polarity, "alpha": s.alpha} for s in self.rounds]}

    @classmethod
    def from_json_dict(cls, doc: dict) -> "StumpEnsemble":
        if doc.get("version") != 1:
            raise ValueError(f"unsupported ensemble document version {doc.get('version')!r}")
        rounds = tuple(Stump(int(r["feature"]), float("-inf") if r["threshold"] is None else float(r["threshold"]),
                             float(r["polarity"]), float(r["alpha"])) for r in doc["rounds"])
        return cls(dim=int(doc["dim"]), rounds=rounds, intercept=float(doc["intercept"]))

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict())

    @classmethod
    def from_json(cls, text: str) -> "StumpEnsemble":
        return cls.from_json_dict(json.loads(text))


def fit_stump(xs, ys, weights, mode=None) -> tuple[Stump, float]:
    """Best single stump under weighted 0-1 loss (boosting.py:126-171), on the device."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    f, t, p, _, e, _ = _be.fit_ensemble_arrays(xs, np.asarray(ys, dtype=np.float64), 1, mode=mode,
                                               weights=np.asarray(weights, dtype=np.float64), single=True)
    return Stump(int(f[0]), float(t[0]), float(p[0])), float(e[0])


def ensemble_from_arrays(dim, feat, thr, pol, alpha, intercept) -> StumpEnsemble:
    cols = [np.asarray(c).tolist() for c in (feat, thr, pol, alpha)]  # Python scalars in one pass per column
    rounds = tuple(Stump(int(f), float(t), float(p), float(a)) for f, t, p, a in zip(*cols))
    return StumpEnsemble(dim=int(dim), rounds=rounds, intercept=float(intercept))


def fit_ensemble(ts: TrainingSet, rounds: int, mode=None, stream=None) -> StumpEnsemble:
    """Discrete AdaBoost with ``rounds`` stumps (boosting.py:174-206), on the device.

    ``ts`` may also be a pair (xs, betas) of device tensors (no host copy)."""
    if rounds < 1:
        raise ValueError(f"need at least one round, got {rounds}")
    xs, betas = (ts.xs, ts.betas) if isinstance(ts, TrainingSet) else ts
    f, t, p, a, _, icept = _be.fit_ensemble_arrays(xs, betas, rounds, mode=mode, stream=stream)
    if len(f) == 0 and isinstance(ts, TrainingSet) and np.unique(ts.ys).size > 1:
        warnings.warn("no stump beat random guessing; falling back to majority sign")
    return ensemble_from_arrays(xs.shape[1], f, t, p, a, icept)


def score(ensemble: StumpEnsemble, x) -> float:
    return ensemble.score(x)
