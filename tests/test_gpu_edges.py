"""Edge cases the reference handles (errors, empty / ragged inputs, size limits), on the B200."""
import numpy as np
import pytest

from tests import _cases as CS

pytestmark = pytest.mark.gpu

O = pytest.importorskip("oracle.oracle")
from paper_0805_1827_b200 import backend as G  # noqa: E402
from paper_0805_1827_b200.packs import RulePack  # noqa: E402
import paper_0805_1827_b200 as E  # noqa: E402


def _mc(d=5):
    p, s = CS.maxcall(d)
    return CS.packs(p, s)


def test_no_remaining_dates_raises_value_error():
    mp = _mc()
    rp = RulePack.european(True)
    k, s = O.derive_words(1, 3, 0, 0)
    # _core.pyx:406-407, 445-446, 524-525
    with pytest.raises(ValueError, match="no remaining exercise dates"):
        G.stopped_sums(mp, rp, mp.s0, 9, 10, k, s)
    with pytest.raises(ValueError):
        G.cmc_labels(mp, rp, np.full((2, 5), 100.0), 9, 10, [1, 2], [3, 4], 0)
    with pytest.raises(ValueError):
        G.iz_solve(mp, RulePack.european(True), np.full(4, 90.0), 0, 9, 10, 0.01, 10, 5, k, s)


def test_zero_and_single_paths():
    mp = _mc()
    rp = CS.random_stumps(5, 9, 20, seed=1)
    k, s = O.derive_words(1, 3, 0, 0)
    assert G.stopped_sums(mp, rp, mp.s0, 0, 0, k, s) == (0.0, 0.0)
    g = G.stopped_sums(mp, rp, mp.s0, 0, 1, k, s, 7)
    o = O.stopped_sums(O.Ctx(mp, rp), mp.s0, 0, 1, k, s, 7)
    assert abs(g[0] - o[0]) <= 1e-12 * max(abs(o[0]), 100.0)


@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 3 * 4096 + 1])
def test_ragged_pricing_blocks(n):
    mp = _mc()
    rp = CS.random_stumps(5, 9, 20, seed=2)
    g = G.price_blocks(mp, rp, n, 1827, mode="parity")
    o = O.price_blocks(O.Ctx(mp, rp), n, 1827)
    assert np.array_equal(g[:, 0], o[:, 0])
    assert np.all(np.abs(g[:, 1:] - o[:, 1:]) <= 1e-12 * np.maximum(np.abs(o[:, 1:]), 1.0))


def test_price_blocks_subrange_equals_slice():
    mp = _mc()
    rp = CS.random_stumps(5, 9, 20, seed=2)
    full = G.price_blocks(mp, rp, 10 * 4096 + 5, 3, mode="parity")
    part = G.price_blocks(mp, rp, 10 * 4096 + 5, 3, 4, 11, mode="parity")
    assert np.array_equal(full[4:11], part)


@pytest.mark.parametrize("d", [4, 7, 12])
def test_runtime_dimension_kernels(d):
    """Dimensions without a specialised kernel use the runtime-d instantiation."""
    p, s = CS.maxcall(d, rho=0.2)
    mp = CS.packs(p, s)
    rp = CS.random_stumps(d, 9, 25, seed=d)
    k, st = O.derive_words(9, 3, d, 0)
    gv, gs = G.path_values(mp, rp, mp.s0, 1, 700, k, st, 3, mode="parity")
    ov, os_ = O.path_values(O.Ctx(mp, rp), mp.s0, 1, 700, k, st, 3)
    assert np.array_equal(gs, os_)
    assert np.all(np.abs(gv - ov) <= 1e-12 * np.maximum(np.abs(ov), 100.0))


def test_large_label_count_multiple_chunks():
    """n_label above the 4096-path chunk: a unit is folded from several chunks."""
    mp = _mc()
    rp = CS.random_stumps(5, 9, 20, seed=4)
    pts = 100 * np.exp(0.2 * np.random.default_rng(1).normal(size=(3, 5)))
    keys = np.array([11, 12, 13], dtype=np.uint64)
    strs = np.array([21, 22, 23], dtype=np.uint64)
    g = G.cmc_labels(mp, rp, pts, 2, 9000, keys, strs, 10, mode="parity")
    o = O.cmc_labels(O.Ctx(mp, rp), pts, 2, 9000, keys, strs, 10)
    assert np.array_equal(g > 0, o > 0)
    assert np.all(np.abs(g - o) <= 1e-12 * np.maximum(np.abs(o), 100.0))


def test_one_class_and_tiny_training_sets():
    X = np.array([[1.0], [2.0], [3.0]])
    f, t, p, a, _, ic = G.fit_ensemble_arrays(X, np.array([-1.0, -2.0, -3.0]), 5)
    assert len(f) == 0 and ic == -1.0
    for n in (2, 5, 9, 130):
        rng = np.random.default_rng(n)
        X = rng.normal(size=(n, 2))
        beta = rng.normal(size=n)
        gf = G.fit_ensemble_arrays(X, beta, 4, mode="parity")
        of = O.fit_ensemble(X, beta, 4)
        assert list(gf[0]) == of[0] and list(gf[1]) == of[1] and gf[5] == of[4]


def test_invalid_configs_raise_config_errors():
    with pytest.raises(E.ConfigError):
        E.CmcBuildConfig(0, 10)
    with pytest.raises(E.ConfigError):
        E.build_iz_boundary(*CS.basketput(4, 4), 4, 10)
    with pytest.raises(ValueError):
        E.price(*CS.maxcall(2), E.EuropeanRule(), 0, 1)


def test_price_deterministic_across_calls_and_block_splits():
    p, s = CS.maxcall(5)
    a = E.price(p, s, E.EuropeanRule(), 3 * 4096 + 9, 77, mode="parity")
    b = E.price(p, s, E.EuropeanRule(), 3 * 4096 + 9, 77, mode="parity")
    assert a.price == b.price and a.variance == b.variance
    mp = CS.packs(p, s)
    rp = RulePack.european(True)
    parts = np.vstack([G.price_blocks(mp, rp, 3 * 4096 + 9, 77, lo, lo + 1, mode="parity") for lo in range(4)])
    assert E.pool_moments(parts[:, 0], parts[:, 1], parts[:, 2])[0] == a.price
