"""Device-resident backward induction: rule images
filled on the device (brm_ctx_create_cmc / brm_ctx_set_ensemble) and the
build_cmc_rule date loop with no host round trip per date must reproduce the
host-built images and the host-driven loop exactly."""
import numpy as np
import pytest

from tests import _cases as CS

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_0805_1827_b200 as E  # noqa: E402
from paper_0805_1827_b200 import backend as G  # noqa: E402
from paper_0805_1827_b200.context import Context  # noqa: E402
from paper_0805_1827_b200.packs import RulePack  # noqa: E402


def _per_date(rp, m):
    s, c = int(rp.cmc_starts[m]), int(rp.cmc_counts[m])
    return (rp.cmc_feat[s:s + c], rp.cmc_thr[s:s + c], rp.cmc_pol[s:s + c], rp.cmc_alpha[s:s + c],
            float(rp.cmc_intercept[m]), c)


def _slot_ctx_from_pack(mp, rp, capacity, mode, device_inputs):
    ctx = Context.cmc_slots(mp, bool(rp.call_like), capacity, mode=mode)
    for m in range(1, int(mp.n_dates)):
        f, t, p, a, ic, c = _per_date(rp, m)
        arrs = [np.zeros(capacity, np.int32), np.zeros(capacity), np.zeros(capacity), np.zeros(capacity)]
        for dst, src in zip(arrs, (f, t, p, a)):
            dst[:c] = src
        cnt, icp = np.array([c], np.int32), np.array([ic])
        if device_inputs:
            arrs = [torch.from_numpy(x).cuda() for x in arrs]
            cnt, icp = torch.from_numpy(cnt).cuda(), torch.from_numpy(icp).cuda()
        ctx.set_ensemble(m, *arrs, cnt, icp)
    return ctx


@pytest.mark.parametrize("mode", ["parity", "fast"])
@pytest.mark.parametrize("device_inputs", [False, True])
def test_slotted_image_decides_like_the_host_image(mode, device_inputs):
    d, nd = 5, 7
    mp = CS.packs(*CS.maxcall(d, n_dates=nd))
    per = {}
    rng = np.random.default_rng(5)
    for m in range(1, nd):
        c = int(rng.integers(0, 30))
        feat = rng.integers(0, d + 1, c)
        thr = np.round(rng.uniform(70.0, 140.0, c), 1)  # repeated thresholds
        per[m] = (feat, thr, rng.choice([-1.0, 1.0], c), rng.uniform(0.05, 1.0, c), 0.0 if c else -1.0)
    per[3] = (np.array([], np.int64), np.array([]), np.array([]), np.array([]), 1.0)  # one-class date
    rp = RulePack.from_stumps(nd, per, True)
    slot = _slot_ctx_from_pack(mp, rp, 32, mode, device_inputs)
    states = 100 * np.exp(0.25 * np.random.default_rng(1).normal(size=(20000, d)))
    for m in range(1, nd + 1):
        want = G.decisions(mp, rp, states, m, mode=mode)
        got = G.decisions(mp, rp, states, m, mode=mode, ctx=slot)
        assert np.array_equal(want, got), m


def test_slotted_image_prices_like_the_host_image():
    mp = CS.packs(*CS.maxcall(5))
    rp = CS.random_stumps(5, 9, 25, seed=8)
    slot = _slot_ctx_from_pack(mp, rp, 25, "parity", True)
    n = 3 * 4096 + 17
    want = G.price_blocks(mp, rp, n, 41, mode="parity")
    from paper_0805_1827_b200 import _native as N
    got = np.empty_like(want)
    N.check(N.lib.brm_price_blocks(slot.handle, n, 41, 0, want.shape[0], N.ptr(got)))
    assert np.array_equal(want, got)


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_device_loop_reproduces_host_loop(mode):
    p, s = CS.maxcall(5)
    cfg = E.CmcBuildConfig(700, 60, 12)
    a, ra = E.build_cmc_rule(p, s, cfg, seed=7, mode=mode, device_loop=True)
    b, rb = E.build_cmc_rule(p, s, cfg, seed=7, mode=mode, device_loop=False)
    assert a.ensembles.keys() == b.ensembles.keys()
    for m in a.ensembles:
        assert a.ensembles[m].rounds == b.ensembles[m].rounds, m
        assert a.ensembles[m].intercept == b.ensembles[m].intercept, m
    assert [r["rounds"] for r in ra.per_date] == [r["rounds"] for r in rb.per_date]
    assert [r["positive_fraction"] for r in ra.per_date] == [r["positive_fraction"] for r in rb.per_date]
    assert ra.one_class_dates == rb.one_class_dates
    assert ra.calc_seconds > 0 and ra.class_seconds > 0


def test_device_fit_matches_synchronous_fit():
    rng = np.random.default_rng(3)
    n, F, R = 900, 4, 15
    X = rng.normal(size=(n, F))
    beta = rng.normal(size=n) + 0.3 * X[:, 1]
    want = G.fit_ensemble_arrays(X, beta, R, mode="parity")
    out = {"feat": torch.zeros(R, dtype=torch.int32, device="cuda"), "count": torch.zeros(1, dtype=torch.int32,
                                                                                           device="cuda")}
    for k in ("thr", "pol", "alpha", "err"):
        out[k] = torch.zeros(R, dtype=torch.float64, device="cuda")
    out["intercept"] = torch.zeros(1, dtype=torch.float64, device="cuda")
    xs, bs = torch.from_numpy(X).cuda(), torch.from_numpy(beta).cuda()
    G.fit_ensemble_device(xs, bs, R, out, mode="parity", stream=torch.cuda.current_stream())
    c = int(out["count"].item())
    assert c == len(want[0])
    assert np.array_equal(out["feat"].cpu().numpy()[:c], want[0])
    for k, w in zip(("thr", "pol", "alpha", "err"), want[1:5]):
        assert np.array_equal(out[k].cpu().numpy()[:c], w), k
    assert float(out["intercept"].item()) == want[5]
    # one class and no-better-than-chance: the intercepts come from the device
    for betas, ic in ((np.full(n, -1.0), -1.0), (np.full(n, 2.0), 1.0)):
        G.fit_ensemble_device(xs, torch.from_numpy(betas).cuda(), R, out, mode="parity",
                              stream=torch.cuda.current_stream())
        assert int(out["count"].item()) == 0 and float(out["intercept"].item()) == ic


def test_set_ensemble_rejects_bad_calls():
    mp = CS.packs(*CS.maxcall(3))
    plain = G.get_context(mp, RulePack.european(True), mode="parity")
    z = np.zeros(4)
    with pytest.raises(ValueError):
        plain.set_ensemble(1, np.zeros(4, np.int32), z, z, z, np.array([0], np.int32), np.array([1.0]))
    slot = Context.cmc_slots(mp, True, 4, mode="parity")
    with pytest.raises(ValueError):
        slot.set_ensemble(int(mp.n_dates), np.zeros(4, np.int32), z, z, z, np.array([0], np.int32), np.array([1.0]))
    with pytest.raises(ValueError):
        Context.cmc_slots(mp, True, 0, mode="parity")


IZ_CASES = [
    # (d, payoff, J, n_inner, solver, kwargs): C1-like put, d=3 max-call, C2-like geometric put
    (1, "put", 1, 2000, "bisection", dict(bracket=(20.0, 40.0), tol=1e-4)),
    (1, "put", 4, 500, "fixed_point", dict(max_iter=40)),
    (3, "maxcall", 16, 300, "fixed_point", dict(max_iter=30)),
    (5, "geoput", 32, 400, "bisection", dict(bracket=(50.0, 100.0), tol=1e-3)),
]


def _iz_objects(d, payoff):
    if payoff == "put":
        return E.MarketParams(d=1, s0=40.0, r=0.06, sigma=0.2), E.BermudanSpec(40.0, 1.0, 10, E.PayoffKind.PUT_1D)
    if payoff == "geoput":
        return (E.MarketParams(d=d, s0=100.0, r=0.03, sigma=0.4),
                E.BermudanSpec(100.0, 1.0, 10, E.PayoffKind.GEO_PUT))
    return E.MarketParams(d=d, s0=100.0, r=0.05, sigma=0.2, delta=0.1), E.BermudanSpec(100.0, 3.0, 9)


@pytest.mark.parametrize("case", IZ_CASES, ids=lambda c: f"{c[1]}-d{c[0]}-{c[4]}")
def test_iz_device_loop_equals_host_loop(case):
    """The device-resident I&Z date loop (levels, exchange and regression in HBM,
    surfaces written into the rule image by brm_iz_fit) reproduces the
    host-driven loop bit for bit: levels, iteration counts, coefficients, price."""
    d, payoff, J, n_inner, solver, kw = case
    params, spec = _iz_objects(d, payoff)
    a, ra = E.build_iz_boundary(params, spec, J, n_inner, seed=11, solver=solver, mode="parity", device_loop=True, **kw)
    b, rb = E.build_iz_boundary(params, spec, J, n_inner, seed=11, solver=solver, mode="parity", device_loop=False,
                                **kw)
    assert ra.iteration_counts == rb.iteration_counts
    assert ra.unconverged_points == rb.unconverged_points
    assert np.array_equal(a.coeffs, b.coeffs)
    pa = E.price(params, spec, E.IzRule(a), 1 << 14, 3, mode="parity")
    pb = E.price(params, spec, E.IzRule(b), 1 << 14, 3, mode="parity")
    assert pa.price == pb.price


def test_bisection_tree_equals_sequential_bisection(monkeypatch):
    """The bisection tree (2^L - 1 midpoints per pass on as many clusters)
    takes exactly the sequential bisection's decisions: same levels, iteration
    counts and convergence flags, for one probe (C1: the tree is used) and for
    many (the tree is off when the probes fill the GPU)."""
    for d, payoff, J, n_inner, kw in [(1, "put", 1, 2000, dict(bracket=(20.0, 40.0), tol=1e-4)),
                                      (1, "put", 3, 700, dict(bracket=(20.0, 40.0), tol=1e-6)),
                                      (5, "geoput", 24, 300, dict(bracket=(50.0, 100.0), tol=1e-4))]:
        params, spec = _iz_objects(d, payoff)
        monkeypatch.delenv("BRM_IZ_NO_TREE", raising=False)
        a, ra = E.build_iz_boundary(params, spec, J, n_inner, seed=5, solver="bisection", mode="parity", **kw)
        monkeypatch.setenv("BRM_IZ_NO_TREE", "1")
        b, rb = E.build_iz_boundary(params, spec, J, n_inner, seed=5, solver="bisection", mode="parity", **kw)
        assert ra.iteration_counts == rb.iteration_counts
        assert np.array_equal(a.coeffs, b.coeffs), payoff


def test_partitions_give_identical_bits_at_c2_probe_count():
    """Any item partition (1, 2, 3, 8 GPUs' worth, dist.virtual_shards) gives the
    same boundary and price bits at C2's full probe count (64 probes, 5000
    inner paths): the probe clusters fold their paths in fixed 256-path
    chunks, so the continuation value does not depend on how many probes
    share a launch (cluster size) -- and the bisection tree's decisions equal
    the sequential ones."""
    from paper_0805_1827_b200.dist import virtual_shards
    params = E.MarketParams(d=5, s0=100.0, r=0.03, sigma=0.4)
    spec = E.BermudanSpec(100.0, 1.0, 10, E.PayoffKind.GEO_PUT)
    out = []
    for parts in (1, 2, 3, 8):
        with virtual_shards(parts):
            b, rep = E.build_iz_boundary(params, spec, 64, 5000, seed=1827, solver="bisection",
                                         bracket=(50.0, 100.0), tol=1e-4, mode="parity")
            est = E.price(params, spec, E.IzRule(b), 1 << 16, 1827, mode="parity")
        out.append((b.coeffs, rep.iteration_counts, est.price))
    for coeffs, its, p in out[1:]:
        assert np.array_equal(coeffs, out[0][0])
        assert its == out[0][1]
        assert p == out[0][2]


def test_fit_presort_on_a_side_stream_gives_the_same_ensemble():
    """brm_fit_presort (the column sort ahead of its fit, on another stream): the fit that finds it
    returns the stumps of a fit that sorts itself, in both modes; a sort nobody uses is dropped."""
    import torch
    from paper_0805_1827_b200 import _native as N
    from paper_0805_1827_b200 import backend as G
    rng = np.random.default_rng(12)
    n, F = 3000, 6
    X = 100 * np.exp(0.2 * rng.normal(size=(n, F)))
    X[:, -1] = X[:, :-1].max(axis=1)
    beta = (X[:, -1] - 125) + 0.4 * (X[:, 0] - 100) + 6 * rng.normal(size=n)
    xs, bs = torch.from_numpy(X).cuda(), torch.from_numpy(beta).cuda()
    side = torch.cuda.Stream()
    for mode in ("parity", "fast"):
        plain = G.fit_ensemble_arrays(xs, bs, 40, mode=mode)
        for _ in range(2):  # the first sort is replaced by the second, which the fit takes
            N.check(N.lib.brm_fit_presort(0, N.stream_handle(side), N.ptr(xs), n, F))
        pre = G.fit_ensemble_arrays(xs, bs, 40, mode=mode)
        again = G.fit_ensemble_arrays(xs, bs, 40, mode=mode)  # nothing left to take: sorts itself
        for a, b, c in zip(plain, pre, again):
            assert np.array_equal(np.asarray(a), np.asarray(b)) and np.array_equal(np.asarray(a), np.asarray(c))
    N.check(N.lib.brm_fit_presort(0, N.stream_handle(side), N.ptr(xs), n, F))  # left unused on purpose
    torch.cuda.synchronize()
    with pytest.raises(Exception):
        N.check(N.lib.brm_fit_presort(0, N.stream_handle(side), N.ptr(X), n, F))  # host matrix: refused
