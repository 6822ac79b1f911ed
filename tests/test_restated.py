"""The restated CPU baseline for configs the reference cannot express (C2, C4):
its threaded batch entry points equal the oracle's serial ones bit for bit,
and the restated pricers run end to end."""
import numpy as np
import pytest

O = pytest.importorskip("oracle.oracle")
from oracle import restated as RS  # noqa: E402


def _geo_ctx(d=3, nd=6):
    mp = RS.market_pack(d, 100.0, 0.03, 0.4, 0.0, None, 100.0, 1.0, nd, "geoput")
    nb = 1 + (d - 1) + (d - 1) * d // 2
    coeffs = np.zeros((nd + 1, d, nb))
    coeffs[nd, :, 0] = 100.0
    coeffs[3:nd, :, 0] = np.log(80.0)
    rp = RS._rule(2, False, nd, d, iz_coeffs=coeffs, iz_lo=np.full(d - 1, np.log(50.0)),
                  iz_hi=np.full(d - 1, np.log(250.0)), iz_space=1)
    return mp, rp


def test_threaded_batches_equal_serial_oracle():
    mp, rp = _geo_ctx()
    ctx = O.Ctx(mp, rp)
    # labels
    pts = np.abs(100 + 15 * np.random.default_rng(1).normal(size=(37, mp.d)))
    keys = np.array([O.derive_words(5, 2, i, 2)[0] for i in range(37)], dtype=np.uint64)
    strs = np.array([O.derive_words(5, 2, i, 2)[1] for i in range(37)], dtype=np.uint64)
    ser = O.cmc_labels(ctx, pts, 2, 50, keys, strs, 6)
    par = np.empty(37)
    RS._lib.orc_cmc_labels_mt(ctx.ref, pts.ctypes.data_as(RS._dp), 37, 2, 50, keys.ctypes.data_as(RS._up),
                              strs.ctypes.data_as(RS._up), 6, par.ctypes.data_as(RS._dp))
    assert np.array_equal(ser.view(np.int64), par.view(np.int64))
    # pricing blocks
    n = 3 * 4096 + 17
    ser = O.price_blocks(ctx, n, 9)
    par = np.empty_like(ser)
    s0 = np.ascontiguousarray(mp.s0)
    RS._lib.orc_price_blocks(ctx.ref, s0.ctypes.data_as(RS._dp), n, 9, 0, ser.shape[0], par.ctypes.data_as(RS._dp))
    assert np.array_equal(ser, par)
    # bisection solves
    seeds = np.abs(100 + 20 * np.random.default_rng(2).normal(size=(5, mp.d - 1)))
    assets = np.full(5, mp.d - 1, np.int32)
    lv, it, cv = np.empty(5), np.empty(5, np.int32), np.empty(5, np.int32)
    RS._lib.orc_iz_bisect_batch(ctx.ref, seeds.ctypes.data_as(RS._dp), mp.d - 1, assets.ctypes.data_as(RS._ip), 5, 2,
                                200, 50.0, 100.0, 1e-3, 100, 7, 0, lv.ctypes.data_as(RS._dp),
                                it.ctypes.data_as(RS._ip), cv.ctypes.data_as(RS._ip))
    for j in range(5):
        k, s = O.derive_words(7, 1, j, 2)
        want = O.iz_bisect(ctx, seeds[j], mp.d - 1, 2, 200, 50.0, 100.0, 1e-3, 100, k, s)
        assert (lv[j], it[j], bool(cv[j])) == want


def test_restated_pricers_run():
    c2 = dict(method="iz", d=3, payoff="geoput", s0=100.0, strike=100.0, r=0.03, sigma=0.4, delta=0.0, rho=None,
              maturity=1.0, n_dates=5, j_points=8, n_inner=200, bracket=(50.0, 100.0), tol=1e-2, n_paths=1 << 13,
              name="c2-tiny")
    p, ci, _, _ = RS.build_price_iz_geoput(c2, 3)
    assert 0.0 < p < 100.0 and ci > 0.0
    c4 = dict(method="cmc", d=6, payoff="basketput", s0=100.0, strike=100.0, r=0.05, sigma="u[0.2,0.4]", delta=0.0,
              rho=0.3, maturity=1.0, n_dates=4, n_train=60, n_label=40, rounds=5, n_paths=1 << 13, name="c4-tiny")
    p, ci = RS.build_price_cmc(c4, 3, 60, 40, 1 << 13)
    assert 0.0 < p < 100.0 and ci > 0.0
    r = RS.time_config(c4, scale=1.0)
    assert r["value"] > 0 and r["threads"] >= 1
