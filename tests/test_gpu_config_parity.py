"""Parity at the BASELINE.json config sizes against the unmodified reference.

Fixtures: tests/golden/make_config_golden.py ran the reference's own
``build_cmc_rule`` + ``price`` (boundary_cmc.py:230-281, pricer.py:167-202) at
full C5 (10000 x 2000, 100 rounds, 2^24 paths) and full C3 (5000 x 500,
150 rounds, 2^20 paths), bridge sampler, seeds 1827..1830, and the I&Z
fixed-point build of C1 -- on the build container's 8 cores.  Per run they hold
the rule (JSON v1), the price, its variance and ci95, the per-date report, and
for seed 1827 the label vector of every date.

(a) the reference's rule priced on the GPU == the reference's price (1e-12);
(b) the GPU parity build reproduces the reference's rule stump by stump
    (match rate reported) and its price;
(c) fast mode (fp32 Box-Muller stepping, fixed-point AdaBoost) is within 3
    combined standard errors of the reference over 4 build seeds each (the
    seed-to-seed spread carries the rule noise);
(d) labels of every date at full size, under the reference's rule, equal the
    reference's labels (signs exact).
"""
import gzip
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_0805_1827_b200 as E  # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden"


def _doc(name):
    with gzip.open(GOLD / f"cfg_{name}.json.gz", "rt") as fh:
        return json.load(fh)


def _objects(c):
    params = E.MarketParams(d=c["d"], s0=c["s0"], r=c["r"], sigma=c["sigma"], delta=c["delta"])
    spec = E.BermudanSpec(c["strike"], c["maturity"], c["n_dates"])
    return params, spec


def _se(run):
    return float(np.sqrt(run["variance"] / run["n_paths"]))


@pytest.mark.parametrize("name", ["c5", "c3"])
def test_reference_rules_priced_on_gpu(name):
    """(a) every seed's reference rule, priced by the GPU parity walker."""
    doc = _doc(name)
    params, spec = _objects(doc["params"])
    for run in doc["runs"]:
        rule = E.CmcRule.from_json_dict(run["rule"])
        est = E.price(params, spec, E.CmcScoreRule(rule), run["n_paths"], run["seed"], mode="parity")
        assert est.n_paths == run["n_paths"]
        assert abs(est.price - run["price"]) <= 1e-12 * run["price"], (run["seed"], est.price, run["price"])
        assert abs(est.variance - run["variance"]) <= 1e-9 * run["variance"]


def _stump_match(ref_rule, eng_rule):
    """(matching stumps, total) in order per date; a date stops matching at its first difference."""
    same = total = 0
    per_date = {}
    for m, ens in ref_rule.ensembles.items():
        mine = eng_rule.ensembles.get(m)
        k = 0
        if mine is not None:
            for a, b in zip(ens.rounds, mine.rounds):
                ok = (a.feature == b.feature and a.polarity == b.polarity
                      and (a.threshold == b.threshold or abs(a.threshold - b.threshold) <= 1e-12 * abs(a.threshold))
                      and abs(a.alpha - b.alpha) <= 1e-12 * abs(a.alpha))
                if not ok:
                    break
                k += 1
        per_date[m] = (k, len(ens.rounds))
        same += k
        total += len(ens.rounds)
    return same, total, per_date


@pytest.mark.parametrize("name", ["c5", "c3"])
def test_parity_build_reproduces_reference_rule(name):
    """(b) the full-size GPU parity build (bridge sampler, the reference's streams)."""
    doc = _doc(name)
    c = doc["params"]
    params, spec = _objects(c)
    run = doc["runs"][0]
    rule, rep = E.build_cmc_rule(params, spec, E.CmcBuildConfig(c["n_train"], c["n_label"], c["rounds"]),
                                 seed=run["seed"], sampler="bridge", mode="parity")
    ref_rule = E.CmcRule.from_json_dict(run["rule"])
    same, total, per_date = _stump_match(ref_rule, rule)
    rate = same / total
    print(f"\n{name}: {same}/{total} stumps identical to the reference ({rate:.4f}); per date {per_date}")
    pos_ref = [d["positive_fraction"] for d in run["report"]["per_date"]]
    pos_eng = [d["positive_fraction"] for d in rep.per_date]
    print(f"{name}: positive fractions ref {pos_ref} engine {pos_eng}")
    est = E.price(params, spec, E.CmcScoreRule(rule), c["n_paths"], run["seed"], mode="parity")
    se = np.hypot(_se(run), est.std_error)
    print(f"{name}: engine {est.price!r} reference {run['price']!r} ({(est.price - run['price']) / se:+.2f} SE)")
    assert abs(est.price - run["price"]) <= 3 * se
    assert rate >= 0.9


def test_labels_at_full_size_match_reference():
    """(d) C5 labels of every date at full size under the reference's rule, on
    the GPU's sampler points (<= 1 ulp from numpy's): signs exact."""
    doc = _doc("c5")
    c = doc["params"]
    params, spec = _objects(c)
    run = doc["runs"][0]
    betas = np.load(GOLD / "cfg_c5_betas.npz")
    rule = E.CmcRule.from_json_dict(run["rule"])
    K = c["strike"]
    worst = 0.0
    for m in range(1, c["n_dates"]):
        ref = betas[f"beta_m{m}"]
        pts = E.boundary_cmc.sample_training_points(params, spec, m, c["n_train"], run["seed"], "bridge",
                                                    mode="parity")
        got = E.boundary_cmc.label_points(params, spec, pts, m, c["n_label"], rule.restricted_after(m), run["seed"],
                                          mode="parity")
        assert np.array_equal(got > 0.0, ref > 0.0), (m, int(np.sum((got > 0.0) != (ref > 0.0))))
        worst = max(worst, float(np.max(np.abs(got - ref))) / K)
    print(f"\nworst |beta_gpu - beta_ref| / K over 8 dates x 10000 points: {worst:.3e}")
    assert worst <= 1e-9


def _fast_runs(name, seeds, sampler):
    doc = _doc(name)
    c = doc["params"]
    params, spec = _objects(c)
    out = []
    for seed in seeds:
        rule, _ = E.build_cmc_rule(params, spec, E.CmcBuildConfig(c["n_train"], c["n_label"], c["rounds"]),
                                   seed=seed, sampler=sampler, mode="fast")
        est = E.price(params, spec, E.CmcScoreRule(rule), c["n_paths"], seed, mode="fast")
        out.append((est.price, est.std_error))
    return out


@pytest.mark.parametrize("name,sampler", [("c5", "bridge"), ("c3", "bridge"), ("c3", "forward")])
def test_fast_mode_within_3se_of_reference(name, sampler):
    """(c) fp32 fast mode vs the reference, 4 build seeds each side."""
    doc = _doc(name)
    ref = np.array([r["price"] for r in doc["runs"]])
    ref_se = np.array([_se(r) for r in doc["runs"]])
    fast = _fast_runs(name, [r["seed"] for r in doc["runs"]], sampler)
    fp = np.array([p for p, _ in fast])
    fse = np.array([s for _, s in fast])
    # variance of a seed mean: the seed-to-seed spread (rule + pricing noise),
    # never below the pricing variance alone
    v_ref = max(np.var(ref, ddof=1), np.mean(ref_se ** 2)) / ref.size
    v_fast = max(np.var(fp, ddof=1), np.mean(fse ** 2)) / fp.size
    se = float(np.sqrt(v_ref + v_fast))
    z = (fp.mean() - ref.mean()) / se
    print(f"\n{name} fast ({sampler}): {fp.mean():.5f} (seeds {np.round(fp, 5).tolist()}) vs reference "
          f"{ref.mean():.5f} (seeds {np.round(ref, 5).tolist()}): {z:+.2f} combined SE")
    assert abs(z) <= 3.0
