"""The log-price walker instance (csrc/brm_walk_log.cuh: max-call payoff, CMC
rule, independent assets, parity draws) against the CPU oracle's price
stepper (reference _core.pyx:290-323) on identical draws.

Bar (north star): stop dates bit-exact, per-path values within
1e-12 * max(|ref|, K).  The cases aim at what the instance adds: search
trees over log-thresholds (clustered thresholds, -inf and non-positive
thresholds, ties, empty dates, trees of different depths), the exact
stump-order fallback when the trees do not fit in shared memory, a
single-date contract, and start states other than s0.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests import _cases as CS

pytestmark = pytest.mark.gpu

O = pytest.importorskip("oracle.oracle")
from paper_0805_1827_b200 import backend as G  # noqa: E402
from paper_0805_1827_b200.packs import RulePack  # noqa: E402

TOL = 1e-12


def _close(a, b, K):
    return np.all(np.abs(a - b) <= TOL * np.maximum(np.abs(b), K))


def _clustered_rule(d, n_dates, per_date, seed, heavy_feature_share=0.4):
    """Random stumps the way AdaBoost leaves them: the derived feature carries a large share,
    thresholds cluster within 1e-12 relative of one another, a few are -inf / non-positive,
    one date is empty and one is one-class."""
    rng = np.random.default_rng(seed)
    per = {}
    for m in range(1, n_dates):
        n = per_date
        feat = np.where(rng.random(n) < heavy_feature_share, d, rng.integers(0, d, n))
        thr = np.where(rng.random(n) < 0.5, 118.0 * (1 + 1e-12 * rng.integers(0, 40, n)), rng.uniform(70, 170, n))
        thr[:2] = -np.inf
        thr[2] = 0.0
        thr[3] = -5.0
        per[m] = (feat, thr, rng.choice([-1.0, 1.0], n), rng.uniform(0.05, 1.0, n), rng.normal(scale=0.3))
    per[2] = (np.array([], np.int64), np.array([]), np.array([]), np.array([]), -1.0)  # never stop
    per[n_dates - 2] = (np.array([], np.int64), np.array([]), np.array([]), np.array([]), 1.0)  # always stop
    return RulePack.from_stumps(n_dates, per, True)


@pytest.mark.parametrize("d", [2, 3, 5, 10])
@pytest.mark.parametrize("m_start", [0, 3])
def test_log_walker_vs_oracle(d, m_start):
    p, s = CS.maxcall(d)
    mp = CS.packs(p, s)
    rp = _clustered_rule(d, s.n_dates, 70, seed=20 + d)
    n = 4096
    k, st = O.derive_words(1827, 2, 31 + d, m_start)
    base = 2 * d  # even: the instance's draw-index requirement for even d (the label launches' base)
    rng = np.random.default_rng(d)
    for start in (mp.s0, 100.0 * np.exp(0.3 * rng.normal(size=d)), np.full(d, 117.99999999)):
        gv, gs = G.path_values(mp, rp, start, m_start, n, k, st, base, mode="parity")
        ov, os_ = O.path_values(O.Ctx(mp, rp), start, m_start, n, k, st, base)
        assert np.array_equal(gs, os_), f"stop dates differ on {np.sum(gs != os_)} paths"
        assert _close(gv, ov, mp.strike)
        assert len(set(gs.tolist())) >= 3  # the rule does stop paths at several dates


def test_log_walker_trees_too_large_use_exact_sums():
    """700 distinct thresholds per date on the derived feature need depth-10 trees (16 KB per
    date): more than the shared-memory budget, so every decision is the stump-order sum."""
    d = 5
    p, s = CS.maxcall(d)
    mp = CS.packs(p, s)
    rng = np.random.default_rng(8)
    per = {}
    for m in range(1, s.n_dates):
        n = 700
        per[m] = (np.full(n, d), rng.uniform(90, 180, n), rng.choice([-1.0, 1.0], n), rng.uniform(0.01, 0.1, n),
                  rng.normal(scale=0.1))
    rp = RulePack.from_stumps(s.n_dates, per, True)
    k, st = O.derive_words(7, 2, 5, 0)
    gv, gs = G.path_values(mp, rp, mp.s0, 0, 1024, k, st, 0, mode="parity")
    ov, os_ = O.path_values(O.Ctx(mp, rp), mp.s0, 0, 1024, k, st, 0)
    assert np.array_equal(gs, os_)
    assert _close(gv, ov, mp.strike)


def test_log_walker_single_date():
    """One exercise date (no stump date at all, depth-0 trees): the walk is the in-the-money test
    at expiry, from a start far from and a start next to the strike."""
    d = 2
    p, s = CS.maxcall(d, n_dates=1)
    mp = CS.packs(p, s)
    rp = RulePack.from_stumps(1, {}, True)
    k, st = O.derive_words(3, 2, 1, 0)
    for start in (np.array([100.0, 60.0]), np.array([99.999999999999, 99.999999999999])):
        gv, gs = G.path_values(mp, rp, start, 0, 8192, k, st, 0, mode="parity")
        ov, os_ = O.path_values(O.Ctx(mp, rp), start, 0, 8192, k, st, 0)
        assert np.array_equal(gs, os_)
        assert _close(gv, ov, mp.strike)


_AB = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from tests import _cases as CS
from tests.test_gpu_logwalk import _clustered_rule
from paper_0805_1827_b200 import backend as G
p, s = CS.maxcall(10)
mp = CS.packs(p, s)
rp = _clustered_rule(10, s.n_dates, 100, seed=77)
k, st = G.derive_words(1827, 2, 9, 0)
v, m = G.path_values(mp, rp, mp.s0, 0, 20000, k, st, 20, mode="parity")
np.savez({out!r}, v=v, m=m)
"""


def test_log_walker_equals_price_stepper(tmp_path):
    """The same launch through the price-stepping instance (BRM_WALK_LOG=0, walk_paths in
    brm_walk.cuh): stop dates equal, values within 1e-13 K."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        out = str(tmp_path / f"ab{flag}.npz")
        env = dict(os.environ, BRM_WALK_LOG=flag)
        subprocess.run([sys.executable, "-c", _AB.format(root=root, out=out)], check=True, env=env, cwd=root)
        outs.append(np.load(out))
    assert np.array_equal(outs[0]["m"], outs[1]["m"])
    assert np.all(np.abs(outs[0]["v"] - outs[1]["v"]) <= 1e-13 * 100.0)


@pytest.mark.parametrize("d", [2, 5])
def test_geoput_probe_bisection_log_walker_and_draw_cache(d, monkeypatch):
    """The geometric put's probe clusters on log-prices (iz_probes<.., 2 / 3>): sequential bisection
    (tree off) with the draw cache -- first pass records the increments, the others replay them --
    returns the bits of the re-simulating kernel, and both agree with the oracle's price-space
    bisection (iteration counts and flags equal, levels to 1e-9 K)."""
    p, s = CS.geoput(d)
    mp = CS.packs(p, s)
    rp = CS.random_surfaces(d, s.n_dates, 100.0, seed=6, iz_space=1, call_like=False)
    n = 6
    seeds = np.random.default_rng(4).uniform(60, 140, size=(n, d - 1))
    keys, strs = zip(*[O.derive_words(5, 1, i, 3) for i in range(n)])
    monkeypatch.setenv("BRM_IZ_NO_TREE", "1")
    args = dict(solver="bisection", lo=50.0, hi=100.0, tol=1e-4, max_iter=100, keys=keys, streams=strs,
                mode="parity")
    cached = G.iz_solve_batch(mp, rp, seeds, [d - 1] * n, 3, 1500, **args)
    monkeypatch.setenv("BRM_IZ_NO_CACHE", "1")
    plain = G.iz_solve_batch(mp, rp, seeds, [d - 1] * n, 3, 1500, **args)
    for a, b in zip(cached, plain):
        assert np.array_equal(a, b)
    octx = O.Ctx(mp, rp)
    for i in range(n):
        ol, oi, oc = O.iz_bisect(octx, seeds[i], d - 1, 3, 1500, 50.0, 100.0, 1e-4, 100, keys[i], strs[i])
        assert cached[1][i] == oi and cached[2][i] == oc
        assert abs(cached[0][i] - ol) <= 1e-9 * max(abs(ol), mp.strike)
