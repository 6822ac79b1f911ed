"""Pin the CPU oracle (oracle/) against the reference's golden vectors (CPU only).

The golden vectors come from the unmodified reference (tests/golden/
make_golden.py); the oracle must reproduce them bit for bit wherever both
use the same libm (everything but the numpy-vectorised sampler, which differs
from glibc exp/log in the last ulp).
"""
import numpy as np
import pytest

from tests import golden_io as GI

O = pytest.importorskip("oracle.oracle")


def test_stream_words_and_draws():
    g = GI.G()
    for j, (seed, phase, item, date) in enumerate(g["rng.fields"]):
        k, s = O.derive_words(int(seed), int(phase), int(item), int(date))
        assert (k, s) == tuple(g["rng.words"][j])
        assert np.array_equal(O.raw_uint64(k, s, 3 + j, 257), g[f"rng.raw.{j}"])
        assert np.array_equal(O.normals(k, s, 1000 * j + 1, 4099), g[f"rng.normals.{j}"])


@pytest.mark.parametrize("case", GI.PATH_CASES)
def test_path_values_bit_exact(case):
    g = GI.G()
    mp, rp = GI.packs(case)
    k, s = g[f"{case}.key"]
    ref = g[f"{case}.values"]
    vals, _ = O.path_values(O.Ctx(mp, rp), mp.s0, int(g[f"{case}.m_start"]), ref.size, k, s,
                            int(g[f"{case}.draw_base"]))
    assert np.array_equal(vals, ref)
    sums = O.stopped_sums(O.Ctx(mp, rp), mp.s0, int(g[f"{case}.m_start"]), ref.size, k, s,
                          int(g[f"{case}.draw_base"]))
    assert sums == tuple(g[f"{case}.sums"])


def test_labels_bit_exact():
    g = GI.G()
    mp, _ = GI.packs("path.maxcall5_cmc")
    from paper_0805_1827_b200.boundary_cmc import CmcRule
    rule = CmcRule.from_json(GI.text("cmc_rule.json")).restricted_after(3)
    betas = O.cmc_labels(O.Ctx(mp, rule.pack()), g["labels.points"], 3, 200, g["labels.keys"][:, 0],
                         g["labels.keys"][:, 1], 10)
    assert np.array_equal(betas, g["labels.beta"])


def test_iz_solve_bit_exact():
    g = GI.G()
    mp, rp = GI.packs("path.maxcall3_iz")
    for j in range(3):
        k, s = O.derive_words(4, 1, j, 4)
        lv, it, cv = O.iz_solve(O.Ctx(mp, rp), g["iz_solve.seeds"][j], j % 3, 4, 300, 0.01, 60, 5, k, s)
        assert [lv, it, cv] == list(g["iz_solve.result"][j])


def test_sampler_within_one_ulp_of_numpy():
    g = GI.G()
    from tests import _cases as CS
    from paper_0805_1827_b200.packs import RulePack
    p, s = CS.maxcall(5)
    xs, _, _ = O.sample_points(O.Ctx(CS.packs(p, s), RulePack.european()), p, s, 4, 1827, 16)
    assert np.max(np.abs(xs / g["sampler.points"] - 1.0)) <= 4.5e-16


def test_boosting_bit_exact():
    g = GI.G()
    f, t, p, a, icept = O.fit_ensemble(g["boost.X"], g["boost.beta"], 25)
    assert np.array_equal(np.column_stack([f, t, p, a]), g["boost.stumps"])
    ys = np.where(g["boost.beta"] > 0, 1.0, -1.0)
    assert list(O.fit_stump(g["boost.X"], ys, g["fit_stump.w"])) == list(g["fit_stump.result"])


def test_pairwise_sum_is_numpy_order():
    rng = np.random.default_rng(0)
    for n in (1, 7, 8, 9, 127, 128, 129, 1000, 10007):
        a = rng.random(n) * np.exp(rng.normal(size=n) * 4)
        assert O.pairwise_sum(a) == np.sum(a)


def test_price_and_lattice_known_answers():
    g = GI.G()
    assert O.crr_bermudan(40.0, 40.0, 0.06, 0.0, 0.2, 1.0, 10, 5000) == pytest.approx(float(g["crr.put1"]), abs=0)
    assert abs(float(g["crr.put1"]) - 2.292914) < 1e-6


def test_regression_matches_reference():
    g = GI.G()
    from paper_0805_1827_b200.packs import quad_basis
    assert np.array_equal(quad_basis(g["quad_basis.z"]), g["quad_basis.design"])
    coeffs = O.regress(quad_basis(g["glp.64x4"]), g["regress.levels"])
    assert np.array_equal(coeffs, g["regress.coeffs"])
