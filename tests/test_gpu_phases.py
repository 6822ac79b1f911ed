"""Phase-level parity: this engine's price / build_* vs the reference package.

The reference (``bermuda``, built unmodified into oracle/_ref by
oracle/build_ref.sh) runs on the CPU with its Cython backend; the engine runs
on the B200 in parity mode with the same seeds.  Where the reference has the
algorithm, results must match to rounding (I&Z, identical draws) or within 3
combined standard errors (CMC: training points differ in the last ulp
between numpy's and CUDA's exp/log).  Configs the reference cannot express
are checked against closed-form / lattice values.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

O = pytest.importorskip("oracle.oracle")
R = pytest.importorskip("oracle.reference")  # the built reference package, or skip
import paper_0805_1827_b200 as E  # noqa: E402


def _ref():
    return R.bermuda()


def test_iz_put_1d_matches_reference():
    B = _ref()
    args = dict(d=1, s0=40.0, r=0.06, sigma=0.2)
    spec_args = (40.0, 1.0, 10)
    pr, sr = B.MarketParams(**args), B.BermudanSpec(*spec_args, B.PayoffKind.PUT_1D)
    pe, se = E.MarketParams(**args), E.BermudanSpec(*spec_args, E.PayoffKind.PUT_1D)
    bref, rep_ref = B.build_iz_boundary(pr, sr, 1, 2000, seed=1827)
    beng, rep_eng = E.build_iz_boundary(pe, se, 1, 2000, seed=1827, mode="parity")
    assert rep_ref.iteration_counts == rep_eng.iteration_counts
    assert np.allclose(beng.coeffs, bref.coeffs, rtol=1e-12, atol=1e-12)
    n = 1 << 16
    ref = B.price(pr, sr, B.IzRule(bref), n, 1827)
    eng = E.price(pe, se, E.IzRule(beng), n, 1827, mode="parity")
    assert abs(eng.price - ref.price) <= 1e-12 * ref.price
    assert abs(eng.variance - ref.variance) <= 1e-9 * ref.variance


def test_iz_maxcall_d3_matches_reference():
    B = _ref()
    pr, sr = B.MarketParams(d=3, s0=100.0, r=0.05, sigma=0.2, delta=0.1), B.BermudanSpec(100.0, 3.0, 9)
    pe, se = E.MarketParams(d=3, s0=100.0, r=0.05, sigma=0.2, delta=0.1), E.BermudanSpec(100.0, 3.0, 9)
    bref, rref = B.build_iz_boundary(pr, sr, 16, 300, max_iter=40, seed=4)
    beng, reng = E.build_iz_boundary(pe, se, 16, 300, max_iter=40, seed=4, mode="parity")
    assert rref.iteration_counts == reng.iteration_counts
    # levels agree to rounding; the lstsq solvers differ (LAPACK gelsd vs device QR)
    assert np.allclose(beng.coeffs, bref.coeffs, rtol=1e-7, atol=1e-9)
    n = 1 << 15
    ref = B.price(pr, sr, B.IzRule(bref), n, 7)
    eng = E.price(pe, se, E.IzRule(beng), n, 7, mode="parity")
    assert abs(eng.price - ref.price) <= 1e-6 * ref.price


def test_cmc_maxcall_d5_statistical():
    B = _ref()
    pr, sr = B.MarketParams(d=5, s0=100.0, r=0.05, sigma=0.2, delta=0.1), B.BermudanSpec(100.0, 3.0, 9)
    pe, se = E.MarketParams(d=5, s0=100.0, r=0.05, sigma=0.2, delta=0.1), E.BermudanSpec(100.0, 3.0, 9)
    rr, _ = B.build_cmc_rule(pr, sr, B.CmcBuildConfig(500, 100, 20), seed=11)
    re, _ = E.build_cmc_rule(pe, se, E.CmcBuildConfig(500, 100, 20), seed=11, mode="parity")
    # most dates fit the same stumps (points differ only in the last ulp)
    same = sum(tuple(s.feature for s in rr.ensembles[m].rounds) == tuple(s.feature for s in re.ensembles[m].rounds)
               for m in rr.ensembles)
    assert same >= len(rr.ensembles) - 2
    n = 1 << 16
    ref = B.price(pr, sr, B.CmcScoreRule(rr), n, 5)
    eng = E.price(pe, se, E.CmcScoreRule(re), n, 5, mode="parity")
    se_ = np.sqrt(ref.variance / n + eng.variance / n)
    assert abs(eng.price - ref.price) < 3 * se_


def test_cmc_shared_rule_prices_bitwise():
    """Same rule + same seed: the device price equals the reference's to rounding."""
    B = _ref()
    pr, sr = B.MarketParams(d=5, s0=100.0, r=0.05, sigma=0.2, delta=0.1), B.BermudanSpec(100.0, 3.0, 9)
    pe, se = E.MarketParams(d=5, s0=100.0, r=0.05, sigma=0.2, delta=0.1), E.BermudanSpec(100.0, 3.0, 9)
    rr, _ = B.build_cmc_rule(pr, sr, B.CmcBuildConfig(400, 50, 15), seed=3)
    re = E.CmcRule.from_json(rr.to_json())
    n = 1 << 16
    ref = B.price(pr, sr, B.CmcScoreRule(rr), n, 9)
    eng = E.price(pe, se, E.CmcScoreRule(re), n, 9, mode="parity")
    assert abs(eng.price - ref.price) <= 1e-12 * ref.price


def test_cmc_labels_on_reference_points_bit_exact_signs():
    """Fixed inputs: the reference's own training points and rule -> same labels."""
    B = _ref()
    from bermuda._kernels import get_backend
    from bermuda._kernels.packs import pack_market
    pr, sr = B.MarketParams(d=5, s0=100.0, r=0.05, sigma=0.2, delta=0.1), B.BermudanSpec(100.0, 3.0, 9)
    rr, _ = B.build_cmc_rule(pr, sr, B.CmcBuildConfig(300, 60, 10), seed=2)
    mp = pack_market(pr, sr)
    later = rr.restricted_after(3).pack()
    xs = B.sample_training_points(pr, sr, 3, 400, 2)
    keys, strs = zip(*[B.StreamKey(2, B.Phase.CMC_CALC, i, 3).words() for i in range(400)])
    ref = get_backend("cython").cmc_labels(mp, later, xs, 3, 300, np.array(keys), np.array(strs), 10)
    from paper_0805_1827_b200 import backend as G
    eng = G.cmc_labels(mp, later, xs, 3, 300, np.array(keys), np.array(strs), 10, mode="parity")
    assert np.array_equal(eng > 0, ref > 0)
    assert np.all(np.abs(eng - ref) <= 1e-12 * np.maximum(np.abs(ref), 100.0))


def test_fit_stump_with_weights_matches_reference():
    B = _ref()
    rng = np.random.default_rng(3)
    X = rng.normal(size=(800, 4))
    ys = np.where(X[:, 1] + 0.4 * rng.normal(size=800) > 0, 1.0, -1.0)
    w = rng.uniform(0.1, 1.0, 800)
    w /= w.sum()
    sr, er = B.fit_stump(X, ys, w)
    se_, ee = E.fit_stump(X, ys, w)
    assert (se_.feature, se_.threshold, se_.polarity) == (sr.feature, sr.threshold, sr.polarity)
    assert ee == er


def test_geoput_iz_bisection_vs_lattice():
    """Config-2 shape at small size: geometric put on d=5 iid assets == 1-D put on G."""
    d, sig = 5, 0.4
    pe, se = E.MarketParams(d=d, s0=100.0, r=0.03, sigma=sig), E.BermudanSpec(100.0, 1.0, 10, E.PayoffKind.GEO_PUT)
    b, rep = E.build_iz_boundary(pe, se, 32, 2000, seed=1827, solver="bisection", mode="parity")
    est = E.price(pe, se, E.IzRule(b), 1 << 18, 1827, mode="parity")
    sg = sig / np.sqrt(d)
    dg = 0.5 * sig ** 2 - 0.5 * sg ** 2
    exact = O.crr_bermudan(100.0, 100.0, 0.03, dg, sg, 1.0, 10, 5000, put=True)
    # a boundary-rule price is a lower bound: within 3 SE below, a few SE of rule error above
    assert exact - 3 * est.std_error - 0.05 <= est.price <= exact + 3 * est.std_error


def test_put_1d_bisection_near_lattice():
    pe, se = E.MarketParams(d=1, s0=40.0, r=0.06, sigma=0.2), E.BermudanSpec(40.0, 1.0, 10, E.PayoffKind.PUT_1D)
    b, rep = E.build_iz_boundary(pe, se, 1, 2000, seed=1827, solver="bisection", bracket=(20.0, 40.0), mode="parity")
    assert all(it == 18 for it in rep.iteration_counts)
    est = E.price(pe, se, E.IzRule(b), 1 << 18, 1827, mode="parity")
    exact = O.crr_bermudan(40.0, 40.0, 0.06, 0.0, 0.2, 1.0, 10, 5000, put=True)
    assert abs(est.price - exact) < 4 * est.std_error + 0.01


def test_builders_fill_the_engine_timing_log():
    """Per-date device times land in the caller's engine.timing (engine.py:126-144, :167) under the
    reference's phase names, for both builders and the pricer."""
    from tests import _cases as CS
    eng = E.Engine(workers=1)
    p, s = CS.maxcall(3, n_dates=4)
    rule, rep = E.build_cmc_rule(p, s, E.CmcBuildConfig(300, 64, 10), seed=3, engine=eng)
    est = E.price(p, s, E.CmcScoreRule(rule), 1 << 14, 3, engine=eng)
    phases = [r[0] for r in eng.timing.rows]
    assert phases.count("calc") == 3 and phases.count("class") == 3 and phases.count("mc") == 1
    assert abs(eng.timing.phase_seconds("calc") - rep.calc_seconds) < 1e-9
    assert eng.timing.straggler_ratio("calc") >= 1.0
    assert est.timings["pricing"] > 0.0
    p1, s1 = CS.put1d(n_dates=4)
    eng2 = E.Engine(workers=1)
    E.build_iz_boundary(p1, s1, 8, 256, seed=2, engine=eng2)
    assert [r[0] for r in eng2.timing.rows].count("reg") == 3
