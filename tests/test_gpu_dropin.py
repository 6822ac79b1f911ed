"""The drop-in exercised from the reference side, on the GPU.

1. The reference's OWN phase builders (``build_cmc_rule``, boundary_cmc.py:230-281;
   ``build_iz_boundary``, boundary_iz.py:296-360; ``price``, pricer.py:167-202)
   run unchanged with ``backend="cuda"`` registered by ``refshim.register``:
   every kernel call (``cmc_labels``, ``iz_solve``, ``stopped_sums``) goes
   through this package's backend module to the B200.  Their results must
   equal this package's device-resident phase builders.
2. The reference's own config objects (``MarketParams``, ``BermudanSpec``,
   ``CmcBuildConfig``, ``CmcScoreRule``, ``IzRule``) go straight into this
   package's ``build_*`` / ``price``, and the results convert to the
   reference's own result types.
3. The reference CLI entry point (cli.py:402) runs ``price`` and the ``bench``
   determinism check (exit 2 on a price change, cli.py:303-309) with
   ``--backend cuda``.
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

R = pytest.importorskip("oracle.reference")
import paper_0805_1827_b200 as E  # noqa: E402
from paper_0805_1827_b200 import refshim  # noqa: E402


@pytest.fixture(scope="module")
def B():
    mod = R.bermuda()
    refshim.register(mod)
    yield mod
    refshim.unregister(mod)


def _mc5(B):
    return B.MarketParams(d=5, s0=100.0, r=0.05, sigma=0.2, delta=0.1), B.BermudanSpec(100.0, 3.0, 9)


def test_reference_cmc_builder_on_cuda_backend(B):
    """boundary_cmc.build_cmc_rule of the reference with every label on the GPU
    == this package's device build (same stumps; points differ by <= 1 ulp)."""
    params, spec = _mc5(B)
    cfg = B.CmcBuildConfig(400, 64, 15)
    eng = B.Engine(workers=1)
    rule_ref, rep_ref = B.build_cmc_rule(params, spec, cfg, seed=3, engine=eng, backend=B._kernels.get_backend("cuda"))
    rule_eng, rep_eng = E.build_cmc_rule(params, spec, cfg, seed=3, mode="parity")
    assert [d["positive_fraction"] for d in rep_ref.per_date] == [d["positive_fraction"] for d in rep_eng.per_date]
    for m, ens in rule_ref.ensembles.items():
        mine = rule_eng.ensembles[m]
        assert len(ens.rounds) == len(mine.rounds), m
        for a, b in zip(ens.rounds, mine.rounds):
            assert (a.feature, a.polarity) == (b.feature, b.polarity)
            assert abs(a.threshold - b.threshold) <= 1e-12 * abs(a.threshold)
            assert abs(a.alpha - b.alpha) <= 1e-12 * abs(a.alpha)
    # the reference's pricer, one stopped_sums call per 4096-path block on the GPU
    n = 1 << 15
    p_ref = B.price(params, spec, B.CmcScoreRule(rule_ref), n, 11, engine=eng, backend=B._kernels.get_backend("cuda"))
    p_eng = E.price(params, spec, E.CmcScoreRule(rule_eng), n, 11, mode="parity")
    assert abs(p_ref.price - p_eng.price) <= 1e-12 * abs(p_eng.price)
    assert type(p_ref).__module__ == "bermuda.pricer"


def test_reference_iz_builder_on_cuda_backend(B):
    """boundary_iz.build_iz_boundary of the reference, one kern.iz_solve per probe
    on the GPU: iteration counts equal this package's batched solve."""
    params = B.MarketParams(d=3, s0=100.0, r=0.05, sigma=0.2, delta=0.1)
    spec = B.BermudanSpec(100.0, 3.0, 9)
    eng = B.Engine(workers=1, pool="thread")
    b_ref, r_ref = B.build_iz_boundary(params, spec, 16, 200, max_iter=30, seed=4, engine=eng,
                                       backend=B._kernels.get_backend("cuda"))
    b_eng, r_eng = E.build_iz_boundary(params, spec, 16, 200, max_iter=30, seed=4, mode="parity")
    assert r_ref.iteration_counts == r_eng.iteration_counts
    # levels are bit-identical; the fits are LAPACK gelsd (reference) vs the device QR
    assert np.allclose(b_ref.coeffs, b_eng.coeffs, rtol=1e-7, atol=1e-9)


def test_reference_config_objects_into_engine(B):
    """The reference's own objects in, the reference's own types out."""
    params, spec = _mc5(B)
    cfg = B.CmcBuildConfig(300, 40, 12)
    rule, rep = E.build_cmc_rule(params, spec, cfg, seed=5, mode="parity")
    ref_rule = refshim.to_reference(rule, B)
    ref_rep = refshim.to_reference(rep, B)
    assert type(ref_rule).__name__ == "CmcRule" and type(ref_rule).__module__ == "bermuda.boundary_cmc"
    assert type(ref_rep).__module__ == "bermuda.boundary_cmc"
    assert ref_rep.to_json_dict()["per_date"] == rep.to_json_dict()["per_date"]
    # the converted rule, wrapped in the reference's CmcScoreRule, prices identically
    n = 1 << 14
    a = E.price(params, spec, B.CmcScoreRule(ref_rule), n, 9, mode="parity")
    b = E.price(params, spec, E.CmcScoreRule(rule), n, 9, mode="parity")
    assert a.price == b.price and a.variance == b.variance
    ref_est = refshim.to_reference(a, B)
    assert type(ref_est).__module__ == "bermuda.pricer" and ref_est.price == a.price
    # I&Z with the reference's objects and its IzRule
    p3 = B.MarketParams(d=3, s0=100.0, r=0.05, sigma=0.2, delta=0.1)
    bnd, _ = E.build_iz_boundary(p3, spec, 16, 150, max_iter=20, seed=2, mode="parity")
    ref_bnd = refshim.to_reference(bnd, B)
    assert np.array_equal(ref_bnd.coeffs, bnd.coeffs)
    c = E.price(p3, spec, B.IzRule(ref_bnd), n, 3, mode="parity")
    d = E.price(p3, spec, E.IzRule(bnd), n, 3, mode="parity")
    assert c.price == d.price


def test_reference_cli_price_and_bench_on_cuda(B, tmp_path):
    import importlib
    cli = importlib.import_module("bermuda.cli")
    out = tmp_path / "price.json"
    common = ["--backend", "cuda", "--method", "cmc", "--d", "5", "--n1", "400", "--n2", "64",
              "--boost-rounds", "12", "--n-paths", "32768", "--seed", "7"]
    assert cli.main(["price", *common, "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["backend"] == "cuda"
    assert doc["estimate"]["n_paths"] == 32768
    # the same run through this package's API directly
    rc = cli.RunConfig.from_sources(None, {"method": "cmc", "d": 5, "n1": 400, "n2": 64, "boost_rounds": 12,
                                           "n_paths": 32768, "seed": 7, "backend": "cuda"})
    est, _ = refshim.build_and_price(B, rc)
    assert doc["estimate"]["price"] == est.price
    # determinism across item partitions: 1, 2 and 3 partitions give the same price bits (exit 0, not 2)
    csv = tmp_path / "bench.csv"
    assert cli.main(["bench", *common, "--worker-counts", "1,2,3", "--out", str(csv)]) == 0
    iz = ["--backend", "cuda", "--method", "iz", "--d", "3", "--j-points", "16", "--n1", "200",
          "--n-paths", "32768", "--seed", "5"]
    assert cli.main(["bench", *iz, "--worker-counts", "1,3", "--out", str(tmp_path / "iz.csv")]) == 0
