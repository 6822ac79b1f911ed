"""Probe grids for the I&Z boundary search (host side, microseconds of work).

``generate_glp`` is the reference's Korobov rank-1 lattice in the price box
(lowdisc.py:26-110: same multiplier table semantics, same mapping), so
``build_iz_boundary`` probes the reference's points.  ``uniform_log_grid``
draws J points uniformly in the log-price box from the keyed Philox stream
StreamKey(seed, GLP, 0, 0) (BASELINE.json config 2: "64 boundary points per
date drawn uniformly in the reduced (d-1)-dim log-price box").
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

__all__ = ["SeedGrid", "generate_glp", "default_box", "korobov_multiplier", "uniform_log_grid"]

# Korobov multipliers a(J, dim) selected by the P2 figure of merit; the same
# values the reference tabulates (lowdisc.py:26-37).
_TABLE = {
    8: (3, 3, 3, 3), 16: (7, 3, 3, 3), 32: (7, 3, 3, 5), 64: (19, 5, 3, 5), 128: (47, 25, 21, 3),
    256: (75, 37, 39, 21), 512: (149, 119, 115, 151), 1024: (275, 149, 27, 189),
    2048: (791, 495, 137, 453), 4096: (1557, 751, 791, 755),
}


@dataclass(frozen=True)
class SeedGrid:
    points: np.ndarray  # (J, dim)
    box: np.ndarray     # (dim, 2)

    @property
    def j_count(self) -> int:
        return self.points.shape[0]

    @property
    def dim(self) -> int:
        return self.points.shape[1]


def korobov_multiplier(j_points: int, dim: int) -> int:
    if dim == 1:
        return 1
    row = _TABLE.get(j_points)
    if row is not None and 2 <= dim <= 5:
        return row[dim - 2]
    a = max(3, int(round(j_points * (math.sqrt(5.0) - 1.0) / 2.0)) | 1)
    while math.gcd(a, j_points) != 1:
        a += 2
    warnings.warn(f"no tabulated lattice multiplier for J={j_points}, dim={dim}; using default a={a}",
                  stacklevel=2)
    return a


def default_box(strike: float, dim: int, lo_mult: float = 0.5, hi_mult: float = 2.5) -> np.ndarray:
    if not 0.0 <= lo_mult < hi_mult:
        raise ValueError(f"need 0 <= lo_mult < hi_mult, got {lo_mult}, {hi_mult}")
    return np.tile([lo_mult * strike, hi_mult * strike], (dim, 1)).astype(np.float64)


def generate_glp(j_points: int, dim: int, box) -> SeedGrid:
    """x_j = frac(j (1, a, a^2, ...) / J) mapped affinely into ``box``."""
    if j_points < 1:
        raise ValueError(f"need at least one point, got J={j_points}")
    if dim < 1:
        raise ValueError(f"need dim >= 1, got {dim}")
    box = np.asarray(box, dtype=np.float64)
    if box.ndim == 1:
        box = np.tile(box, (dim, 1))
    if box.shape != (dim, 2) or np.any(box[:, 0] >= box[:, 1]):
        raise ValueError(f"box must be (dim, 2) rows [lo, hi], got {box!r}")
    a = korobov_multiplier(j_points, dim)
    gen = np.ones(dim, dtype=np.int64)
    for k in range(1, dim):
        gen[k] = (gen[k - 1] * a) % j_points
    unit = (np.outer(np.arange(j_points, dtype=np.int64), gen) % j_points) / float(j_points)
    return SeedGrid(points=box[:, 0] + unit * (box[:, 1] - box[:, 0]), box=box)


def uniform_log_grid(j_points: int, dim: int, strike: float, seed: int, lo_mult: float = 0.5,
                     hi_mult: float = 2.5) -> SeedGrid:
    """J points with log-prices uniform in [log(lo_mult K), log(hi_mult K)]^dim.

    Uniforms are the 53-bit words j*dim .. j*dim+dim-1 of StreamKey(seed, GLP,
    0, 0) from the device generator; the returned box is the log box (clamp box
    of the log-space boundary surface)."""
    from . import backend
    lo, hi = math.log(lo_mult * strike), math.log(hi_mult * strike)
    k, s = backend.derive_words(seed, 0, 0, 0)  # one GLP-phase stream for the whole grid
    w = backend.raw_uint64(k, s, 0, j_points * dim).reshape(j_points, dim)
    u = ((w >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    pts = np.exp(lo + u * (hi - lo))
    return SeedGrid(points=pts, box=np.tile([lo, hi], (dim, 1)).astype(np.float64))
