"""Host-side logic (CPU only): config objects, packs, rule formats, partitioning, bench bookkeeping."""
import json

import numpy as np
import pytest

from tests import golden_io as GI
import paper_0805_1827_b200 as E
from paper_0805_1827_b200.dist import partition_ranges
from paper_0805_1827_b200.packs import RulePack, n_quad_basis, pack_market, quad_basis


def test_market_validation_messages():
    with pytest.raises(E.ConfigError):
        E.MarketParams(d=0, s0=1.0, r=0.0, sigma=0.2)
    with pytest.raises(E.ConfigError):
        E.MarketParams(d=2, s0=[1.0, -1.0], r=0.0, sigma=0.2)
    with pytest.raises(E.ConfigError):
        E.BermudanSpec(100.0, 1.0, 0)
    with pytest.raises(E.ConfigError):
        E.BermudanSpec(100.0, 1.0, 4, E.PayoffKind.PUT_1D).validate_against(E.MarketParams(d=2, s0=1.0, r=0,
                                                                                            sigma=0.2))
    # semidefinite correlation falls back to the eigen square root
    p = E.MarketParams(d=3, s0=100.0, r=0.05, sigma=0.2, rho=1.0)
    assert np.allclose(p.corr_factor @ p.corr_factor.T, np.ones((3, 3)))


def test_pack_market_matches_reference_numbers():
    g = GI.G()
    mp_ref, _ = GI.packs("path.maxcall5_cmc")
    mp = pack_market(E.MarketParams(d=5, s0=100.0, r=0.05, sigma=0.2, delta=0.1), E.BermudanSpec(100.0, 3.0, 9))
    for f in ("step_mu", "step_vol", "chol", "disc_steps", "s0"):
        assert np.array_equal(getattr(mp, f), getattr(mp_ref, f)), f
    assert np.array_equal(quad_basis(g["quad_basis.z"]), g["quad_basis.design"])
    assert n_quad_basis(4) == 15


def test_rule_formats_round_trip_reference_json():
    rule = E.CmcRule.from_json(GI.text("cmc_rule.json"))
    assert json.loads(rule.to_json()) == GI.doc("cmc_rule.json")
    b = E.IzBoundary.from_json(GI.text("iz_boundary.json"))
    assert json.loads(b.to_json()) == GI.doc("iz_boundary.json")
    _, rp_ref = GI.packs("path.maxcall5_cmc")
    rp = rule.pack()
    for f in ("cmc_starts", "cmc_counts", "cmc_feat", "cmc_thr", "cmc_pol", "cmc_alpha", "cmc_intercept"):
        assert np.array_equal(getattr(rp, f), getattr(rp_ref, f)), f
    _, rp_iz = GI.packs("path.maxcall3_iz")
    assert np.array_equal(b.pack().iz_coeffs, rp_iz.iz_coeffs)


def test_glp_and_partition_match_reference():
    g = GI.G()
    grid = E.generate_glp(64, 4, E.default_box(100.0, 4))
    assert np.array_equal(grid.points, g["glp.64x4"])
    assert [tuple(r) for r in g["partition.17x5"]] == partition_ranges(17, 5)
    assert E.partition(17, 5).ranges == tuple(partition_ranges(17, 5))


def test_pool_moments_is_the_reference_fold():
    counts = np.array([4096, 4096, 100.0])
    sums = np.array([1.0e4, 2.5e4, 3.0])
    sq = np.array([1e6, 2e6, 30.0])
    mean, var, n = E.pool_moments(counts, sums, sq)
    s = 1.0e4 + 2.5e4 + 3.0
    assert n == 8292 and mean == s / n and var == (3e6 + 30.0 - s * s / n) / (n - 1)


def test_bridge_scalars_match_reference_sampler_inputs():
    import math
    from paper_0805_1827_b200.boundary_cmc import bridge_scalars
    p, s = E.MarketParams(d=2, s0=[90.0, 110.0], r=0.05, sigma=[0.2, 0.3], delta=0.1), E.BermudanSpec(100, 3.0, 9)
    b = bridge_scalars(p, s, 4)
    t = 4 * s.dt
    assert np.array_equal(b[:2], p.log_drift * 3.0)
    assert np.array_equal(b[2:4], p.sigma * math.sqrt(3.0))
    assert np.array_equal(b[6:8], p.sigma * math.sqrt(t * (3.0 - t) / 3.0))
    assert b[8] == t / 3.0


def test_rulepack_from_stumps_layout():
    rp = RulePack.from_stumps(5, {3: ([0, 1], [1.0, 2.0], [1.0, -1.0], [0.5, 0.25], 0.0),
                                  1: ([2], [3.0], [1.0], [1.0], -0.5)}, True)
    assert list(rp.cmc_starts) == [0, 0, 0, 1, 0, 0] and list(rp.cmc_counts) == [0, 1, 0, 2, 0, 0]
    assert list(rp.cmc_intercept) == [-1.0, -0.5, -1.0, 0.0, -1.0, -1.0]
    assert list(rp.cmc_feat) == [2, 0, 1]


def test_bench_nominal_work_and_sample():
    import bench
    c5 = bench.CONFIGS["c5"]
    assert bench.nominal_path_steps(c5) == 10000 * 2000 * 36 + (1 << 24) * 9
    c1 = bench.CONFIGS["c1"]
    assert bench.nominal_path_steps(c1) == 1 * 18 * 2000 * 45 + (1 << 18) * 10
    s = bench.reference_sample(c5)
    assert s["n_label"] == c5["n_label"] and s["n_train"] < c5["n_train"]


def test_timing_log_matches_reference_semantics():
    """TimingLog (engine.py:126-144): phase totals and the max / median straggler ratio."""
    from paper_0805_1827_b200.engine import Engine, TimingLog, log_phase
    log = TimingLog()
    assert log.straggler_ratio("calc") == 1.0 and log.phase_seconds("calc") == 0.0
    eng = Engine(workers=1)
    log_phase(eng, "calc", [(8, 0.5), (7, 1.5), (6, 1.0)])
    log_phase(eng, "class", [(8, 0.0)])
    log_phase(None, "calc", [(1, 1.0)])  # no engine, no log: ignored
    assert eng.timing.rows[:2] == [("calc", 8, 0.5), ("calc", 7, 1.5)]
    assert eng.timing.phase_seconds("calc") == 3.0
    assert eng.timing.straggler_ratio("calc") == 1.5
    assert eng.timing.straggler_ratio("class") == 1.0  # zero median


def test_nvtx_range_is_a_noop_without_cuda():
    from paper_0805_1827_b200.engine import nvtx_range
    with nvtx_range("phase"):
        pass


def test_column_constant_factor_is_detected_in_fp32_only():
    """numpy's factor of the equicorrelated matrix is constant below the diagonal only after
    rounding to fp32 (the fp64 entries differ in the last bits), which is the image the fast
    walkers read (brm_capi.cu: chol_colconst)."""
    from tests import _cases as CS
    L = CS.basketput(40, 20)[0].corr_factor
    L32 = L.astype(np.float32)
    assert all(L32[i, a] == L32[a + 1, a] for a in range(38) for i in range(a + 2, 40))
