"""CUDA path vs the CPU oracle on identical seeded inputs (runs on a B200).

Bar (north star): per-path values within 1e-12 * max(|ref|, K) (fp64 parity
mode; the reference's own two backends differ by up to ~1e-15 K), exercise
decisions / stop dates and label signs bit-exact, raw words and central
normals bit-exact.
"""
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


@pytest.mark.parametrize("start,count", [(0, 1), (3, 1001), (2**40 + 1, 4097)])
def test_rng_words_bit_exact(start, count):
    k, s = O.derive_words(11, 3, 5, 0)
    assert (k, s) == G.derive_words(11, 3, 5, 0)
    assert np.array_equal(G.raw_uint64(k, s, start, count), O.raw_uint64(k, s, start, count))


def test_rng_normals():
    k, s = O.derive_words(1827, 2, 77, 4)
    a = G.normals(k, s, 5, 300001)
    b = O.normals(k, s, 5, 300001)
    central = np.abs(b) <= 1.0364  # |q| <= 0.425: IEEE ops only -> bit-exact
    assert np.array_equal(a[central], b[central])
    assert np.max(np.abs(a - b)) <= 4e-15 * np.max(np.abs(b))  # tails go through log (<= 1 ulp apart)


CASES = {
    "maxcall5_european": lambda: (CS.maxcall(5), RulePack.european(True)),
    "maxcall5_immediate": lambda: (CS.maxcall(5), RulePack.immediate(4, True)),
    "maxcall5_cmc": lambda: (CS.maxcall(5), CS.random_stumps(5, 9, 60, seed=3)),
    "maxcall3_iz": lambda: (CS.maxcall(3), CS.random_surfaces(3, 9, 100.0, seed=2)),
    "maxcall10_cmc": lambda: (CS.maxcall(10), CS.random_stumps(10, 9, 40, seed=4)),
    "maxcall4_cmc_dyn": lambda: (CS.maxcall(4), CS.random_stumps(4, 9, 30, seed=5)),
    "put1d_iz": lambda: (CS.put1d(), CS.random_surfaces(1, 10, 40.0, seed=1, call_like=False)),
    "put1d_european": lambda: (CS.put1d(), RulePack.european(False)),
    "geoput5_iz_log": lambda: (CS.geoput(5), CS.random_surfaces(5, 10, 100.0, seed=6, iz_space=1, call_like=False)),
    "basket40_cmc": lambda: (CS.basketput(40, 20), CS.random_stumps(40, 20, 30, seed=7, lo=80, hi=110,
                                                                     call_like=False)),
    "maxcall2_corr_cmc": lambda: (CS.maxcall(2, rho=0.5), CS.random_stumps(2, 9, 30, seed=8)),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("m_start", [0, 3])
def test_path_values_vs_oracle(case, m_start):
    (p, s), rp = CASES[case]()
    mp = CS.packs(p, s)
    n = 2048 if p.d < 40 else 256
    k, st = O.derive_words(99, 3, 7, m_start)
    base = 13
    gv, gs = G.path_values(mp, rp, mp.s0, m_start, n, k, st, base, mode="parity")
    ov, os_ = O.path_values(O.Ctx(mp, rp), mp.s0, m_start, n, k, st, base)
    assert np.array_equal(gs, os_), f"stop dates differ on {np.sum(gs != os_)} paths"
    assert _close(gv, ov, mp.strike)
    gsum, gsq = G.stopped_sums(mp, rp, mp.s0, m_start, n, k, st, base, mode="parity")
    osum, osq = O.stopped_sums(O.Ctx(mp, rp), mp.s0, m_start, n, k, st, base)
    assert abs(gsum - osum) <= 1e-12 * max(abs(osum), 1.0)
    assert abs(gsq - osq) <= 1e-12 * max(abs(osq), 1.0)


def test_supplied_normals_fixed_input():
    (p, s), rp = CASES["maxcall5_cmc"]()
    mp = CS.packs(p, s)
    n = 500
    z = np.random.default_rng(5).normal(size=n * 9 * 5)
    gv, gs = G.path_values(mp, rp, mp.s0, 0, n, 0, 0, 0, mode="parity", normals_in=z)
    ov, os_ = O.path_values(O.Ctx(mp, rp, normals=z), mp.s0, 0, n, 0, 0, 0)
    assert np.array_equal(gs, os_)
    assert _close(gv, ov, mp.strike)


def test_decisions_bit_exact():
    for key in ("maxcall5_cmc", "maxcall3_iz", "geoput5_iz_log", "put1d_iz"):
        (p, s), rp = CASES[key]()
        mp = CS.packs(p, s)
        rng = np.random.default_rng(3)
        states = mp.s0 * np.exp(0.3 * rng.normal(size=(4000, p.d)))
        for m in (1, 4, s.n_dates):
            g = G.decisions(mp, rp, states, m, mode="parity")
            octx = O.Ctx(mp, rp)
            o = np.array([O.decision(octx, m, x) for x in states])
            assert np.array_equal(g, o), (key, m)


def test_decisions_bucket_overflow_and_edge_thresholds():
    """Step-table lookups where buckets hold many thresholds (clustered within one key, so the
    date takes the bucket-scan path), thresholds at -inf (all-constant majority stumps), ties
    between a state and a threshold, and states far outside the thresholds' key range: decisions
    equal the oracle's stump-order sum bit for bit."""
    from paper_0805_1827_b200.packs import RulePack
    p, s = CS.maxcall(5)
    mp = CS.packs(p, s)
    rng = np.random.default_rng(12)
    per = {}
    for m in range(1, s.n_dates):
        n = 60
        feat = rng.integers(0, 6, n)
        thr = np.where(rng.random(n) < 0.5, 100.0 * (1 + 1e-12 * rng.integers(0, 50, n)),  # one key
                       rng.uniform(60, 160, n))
        thr[:3] = -np.inf
        per[m] = (feat, thr, rng.choice([-1.0, 1.0], n), rng.uniform(0.05, 1.0, n), rng.normal(scale=0.3))
    rp = RulePack.from_stumps(s.n_dates, per, True)
    states = mp.s0 * np.exp(0.3 * rng.normal(size=(3000, p.d)))
    states[:200] = 100.0 * (1 + 1e-12 * rng.integers(0, 50, (200, p.d)))  # on / between clustered thresholds
    states[200:220] = 1e-300
    states[220:240] = 1e300
    octx = O.Ctx(mp, rp)
    for m in (1, 4, 7):
        g = G.decisions(mp, rp, states, m, mode="parity")
        o = np.array([O.decision(octx, m, x) for x in states])
        assert np.array_equal(g, o), m


def test_cmc_labels_vs_oracle():
    (p, s), rp = CASES["maxcall5_cmc"]()
    mp = CS.packs(p, s)
    rng = np.random.default_rng(9)
    pts = 100 * np.exp(0.25 * rng.normal(size=(300, 5)))
    keys = rng.integers(0, 2**63, 300, dtype=np.uint64)
    strs = rng.integers(0, 2**63, 300, dtype=np.uint64)
    g = G.cmc_labels(mp, rp, pts, 3, 500, keys, strs, 10, mode="parity")
    o = O.cmc_labels(O.Ctx(mp, rp), pts, 3, 500, keys, strs, 10)
    assert np.array_equal(g > 0, o > 0)
    assert _close(g, o, mp.strike)


def test_cmc_labels_keyed_matches_explicit_keys():
    (p, s), rp = CASES["maxcall5_cmc"]()
    mp = CS.packs(p, s)
    pts = 100 * np.exp(0.25 * np.random.default_rng(2).normal(size=(64, 5)))
    keys, strs = zip(*[O.derive_words(1827, 2, 10 + i, 3) for i in range(64)])
    a = G.cmc_labels(mp, rp, pts, 3, 200, np.array(keys), np.array(strs), 10, mode="parity")
    b = G.cmc_labels_keyed(mp, rp, pts, 3, 200, 1827, 10, 10, mode="parity")
    assert np.array_equal(a, b)


@pytest.mark.parametrize("case,asset", [("maxcall3_iz", 1), ("put1d_iz", 0), ("geoput5_iz_log", 4)])
def test_iz_fixed_point_vs_oracle(case, asset):
    (p, s), rp = CASES[case]()
    mp = CS.packs(p, s)
    seeds = np.random.default_rng(4).uniform(60, 140, size=(6, max(p.d - 1, 0)))
    keys, strs = zip(*[O.derive_words(5, 1, i, 4) for i in range(6)])
    lv, it, cv = G.iz_solve_batch(mp, rp, seeds, [asset] * 6, 4, 700, epsilon=0.01, max_iter=60, avg_window=5,
                                  keys=keys, streams=strs, mode="parity")
    octx = O.Ctx(mp, rp)
    for i in range(6):
        ol, oi, oc = O.iz_solve(octx, seeds[i], asset, 4, 700, 0.01, 60, 5, keys[i], strs[i])
        assert it[i] == oi and cv[i] == oc
        assert abs(lv[i] - ol) <= 1e-10 * max(abs(ol), mp.strike)


@pytest.mark.parametrize("case,asset,lo,hi", [("put1d_iz", 0, 20.0, 40.0), ("geoput5_iz_log", 4, 50.0, 100.0)])
def test_iz_bisection_vs_oracle(case, asset, lo, hi):
    (p, s), rp = CASES[case]()
    mp = CS.packs(p, s)
    seeds = np.random.default_rng(4).uniform(60, 140, size=(4, max(p.d - 1, 0)))
    keys, strs = zip(*[O.derive_words(5, 1, i, 4) for i in range(4)])
    lv, it, cv = G.iz_solve_batch(mp, rp, seeds, [asset] * 4, 4, 2000, solver="bisection", lo=lo, hi=hi, tol=1e-4,
                                  max_iter=100, keys=keys, streams=strs, mode="parity")
    octx = O.Ctx(mp, rp)
    for i in range(4):
        ol, oi, oc = O.iz_bisect(octx, seeds[i], asset, 4, 2000, lo, hi, 1e-4, 100, keys[i], strs[i])
        assert it[i] == oi and cv[i] == oc
        assert abs(lv[i] - ol) <= 1e-9 * max(abs(ol), mp.strike)


def test_price_blocks_vs_oracle():
    (p, s), rp = CASES["maxcall5_cmc"]()
    mp = CS.packs(p, s)
    n = 3 * 4096 + 100
    g = G.price_blocks(mp, rp, n, 1827, mode="parity")
    o = O.price_blocks(O.Ctx(mp, rp), n, 1827)
    assert np.array_equal(g[:, 0], o[:, 0])
    assert np.all(np.abs(g[:, 1:] - o[:, 1:]) <= 1e-12 * np.abs(o[:, 1:]))


def test_sampler_bridge_vs_oracle():
    p, s = CS.maxcall(5)
    mp = CS.packs(p, s)
    rp = RulePack.european(True)
    for m in (1, 4, 9):
        xs, _, _ = O.sample_points(O.Ctx(mp, rp), p, s, m, 1827, 500, item_lo=0, mode=0)
        g = G.sample_points(mp, rp, m, 1827, 0, 500, bridge=O.bridge_scalars(p, s, m), mode="parity")
        assert np.max(np.abs(g / xs - 1.0)) <= 1e-14


def test_sampler_forward_vs_oracle():
    p, s = CS.maxcall(3)
    mp = CS.packs(p, s)
    rp = RulePack.european(True)
    xs, _, _ = O.sample_points(O.Ctx(mp, rp), p, s, 5, 7, 300, mode=1)
    g = G.sample_points(mp, rp, 5, 7, 0, 300, sampler="forward", mode="parity")
    assert np.max(np.abs(g / xs - 1.0)) <= 1e-14


@pytest.mark.parametrize("case", ["maxcall5_cmc", "basket40_cmc"])
def test_fast_mode_statistical(case):
    """fp32 Box-Muller mode: price within 4 combined SE of the fp64 parity walker (d=40: the
    correlated factor and the shared-memory path state of the large-d fast walker)."""
    (p, s), rp = CASES[case]()
    mp = CS.packs(p, s)
    n = 1 << 18
    g = G.price_blocks(mp, rp, n, 1827, mode="fast")
    o = G.price_blocks(mp, rp, n, 1828, mode="parity")
    mg, vg, _ = O.pool_moments(g[:, 0], g[:, 1], g[:, 2])
    mo, vo, _ = O.pool_moments(o[:, 0], o[:, 1], o[:, 2])
    se = np.sqrt(vg / n + vo / n)
    assert abs(mg - mo) < 4 * se, (mg, mo, se)


@pytest.mark.parametrize("n,F,rounds,seed", [(500, 6, 30, 1), (5000, 6, 150, 2), (3000, 11, 60, 3), (1000, 1, 20, 4)])
def test_fit_ensemble_vs_oracle(n, F, rounds, seed):
    rng = np.random.default_rng(seed)
    X = 100 * np.exp(0.2 * rng.normal(size=(n, F)))
    X[:, -1] = X.max(axis=1) if F > 1 else X[:, -1]
    beta = (X[:, 0] - 100) + 0.5 * (X[:, -1] - 110) + 5 * rng.normal(size=n)
    gf, gt, gp, ga, _, gi = G.fit_ensemble_arrays(X, beta, rounds, mode="parity")
    of, ot, op, oa, oi = O.fit_ensemble(X, beta, rounds)
    assert len(gf) == len(of) and gi == oi
    assert np.array_equal(gf, of) and np.array_equal(gt, ot) and np.array_equal(gp, op)
    assert np.allclose(ga, oa, rtol=1e-12, atol=0)


def test_fit_ensemble_one_class_and_constant():
    X = np.ones((50, 3))
    f, t, p, a, _, i = G.fit_ensemble_arrays(X, np.ones(50), 5)
    assert len(f) == 0 and i == 1.0
    beta = np.where(np.arange(50) < 20, 1.0, -1.0)
    f, t, p, a, _, i = G.fit_ensemble_arrays(X, beta, 5)
    of, ot, op, oa, oi = O.fit_ensemble(X, beta, 5)
    assert list(f) == of and list(p) == op and np.allclose(a, oa, rtol=1e-12) and i == oi


@pytest.mark.parametrize("k,J", [(0, 8), (2, 16), (4, 64)])
def test_lstsq_vs_numpy(k, J):
    from paper_0805_1827_b200.packs import quad_basis
    rng = np.random.default_rng(k)
    z = rng.uniform(50, 250, size=(J, k))
    design = quad_basis(z) if k else np.ones((J, 1))
    levels = 120 + (z.sum(axis=1) * 0.1 if k else 0) + rng.normal(size=J)
    g, deficient = G.lstsq(design, levels, k)
    o = O.regress(design, levels)
    assert not deficient
    assert np.allclose(design @ g, design @ o, rtol=1e-9, atol=1e-9)


def test_branch_free_math_is_bit_identical():
    """exp_nb / div_nb / log_nb / sqrt_nb (brm_rng.cuh) return the bits of CUDA's exp / __ddiv_rn / log /
    __dsqrt_rn on the walker's ranges."""
    from paper_0805_1827_b200 import _native as N
    rng = np.random.default_rng(11)
    n = 1 << 22
    x = np.concatenate([rng.uniform(-40, 40, n), rng.normal(scale=0.3, size=n), rng.uniform(-700, 700, 1 << 16)])

    def run(kind, a, b=None):
        out = np.empty(a.size)
        N.check(N.lib.brm_selftest_math(0, kind, N.ptr(a), N.ptr(b), a.size, N.ptr(out)))
        return out

    assert np.array_equal(run(0, x).view(np.int64), run(1, x).view(np.int64))
    # AS241 central quotients plus generic well-scaled operands
    q = rng.uniform(-0.425, 0.425, n)
    r = 0.180625 - q * q
    num = q * (3.387 + 133.1 * r + 1971.6 * r * r)
    den = 1.0 + 42.3 * r + 687.2 * r * r
    a = np.concatenate([num, rng.normal(size=n) * np.exp(rng.uniform(-300, 300, n))])
    b = np.concatenate([den, rng.normal(size=n) * np.exp(rng.uniform(-300, 300, n))])
    assert np.array_equal(run(2, a, b).view(np.int64), run(3, a, b).view(np.int64))
    # log / sqrt of the AS241 tail: log of u or 1-u in [2^-54, 0.075], sqrt of -log in [2.5, 37.5]
    u = np.concatenate([rng.uniform(0, 0.075, n), np.exp(rng.uniform(np.log(2.0 ** -54), np.log(0.075), n)),
                        np.array([2.0 ** -54, 0.075, 0.5, 1.0, 1.5, 2.0 ** 500, np.sqrt(0.5), np.sqrt(2.0)])])
    assert np.array_equal(run(4, u).view(np.int64), run(5, u).view(np.int64))
    s = np.concatenate([rng.uniform(2.5, 37.5, n), np.exp(rng.uniform(-600, 600, n))])
    assert np.array_equal(run(6, s).view(np.int64), run(7, s).view(np.int64))


def test_exact_scan_is_bit_identical_to_sequential_cumsum():
    """AdaBoost's block-parallel exact scan (brm_boost_exact.cuh, kind 10) equals the one-thread
    sequential np.cumsum chain bit for bit: AdaBoost-like weights, wide dynamic ranges, zeros,
    exact ties (dyadic weights), long and short chains."""
    from paper_0805_1827_b200 import _native as N
    rng = np.random.default_rng(23)

    def run(kind, a):
        out = np.empty(a.size)
        N.check(N.lib.brm_selftest_math(0, kind, N.ptr(a), N.ptr(None), a.size, N.ptr(out)))
        return out

    cases = []
    for n in (1, 2, 31, 257, 1000, 9900, 20000):
        w = rng.random(n) * np.exp(rng.normal(scale=2.0, size=n))
        cases.append(w / w.sum())
    w = np.exp(rng.uniform(-60, 0, 12000))
    cases.append(w)
    w = rng.integers(0, 64, 8000).astype(float) * 2.0 ** -20      # dyadic: many exact ties
    cases.append(w)
    w = np.where(rng.random(8000) < 0.3, 0.0, rng.random(8000))   # zeros
    cases.append(w)
    w = np.concatenate([np.full(100, 1e-300), rng.random(3000), np.full(50, 5e-324)])  # tiny and subnormal
    cases.append(w)
    cases.append(np.sort(rng.random(5000))[::-1].copy())           # decreasing
    for a in cases:
        a = np.ascontiguousarray(a)
        seq, ex = run(8, a), run(10, a)
        assert np.array_equal(seq.view(np.int64), ex.view(np.int64)), a.size
        assert np.array_equal(seq, np.cumsum(a))


def test_fast_mode_adaboost_deterministic_and_equivalent():
    """Fixed-point fast fit: deterministic, same first stump as the exact fit on a clear split,
    training error within 1% of the exact fit."""
    rng = np.random.default_rng(5)
    n, F = 6000, 6
    X = 100 * np.exp(0.2 * rng.normal(size=(n, F)))
    X[:, -1] = X.max(axis=1)
    beta = (X[:, -1] - 118) + 3 * rng.normal(size=n)
    a = G.fit_ensemble_arrays(X, beta, 60, mode="fast")
    b = G.fit_ensemble_arrays(X, beta, 60, mode="fast")
    for u, v in zip(a, b):
        assert np.array_equal(np.asarray(u), np.asarray(v))
    p = G.fit_ensemble_arrays(X, beta, 60, mode="parity")
    assert (a[0][0], a[1][0], a[2][0]) == (p[0][0], p[1][0], p[2][0])

    def train_err(fit):
        f, t, pol, al, _, ic = fit
        s = np.full(n, ic)
        for k in range(len(f)):
            s += al[k] * np.where(X[:, f[k]] > t[k], pol[k], -pol[k])
        return np.mean((s > 0) != (beta > 0))

    assert abs(train_err(a) - train_err(p)) < 0.01
