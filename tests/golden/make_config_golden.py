"""Config-scale fixtures from the UNMODIFIED reference package (test infrastructure).

Runs the reference's own ``build_cmc_rule`` + ``price`` (boundary_cmc.py:230-281,
pricer.py:167-202) and ``build_iz_boundary`` (boundary_iz.py:296-360) at the
BASELINE.json config sizes, with the reference's own algorithm (bridge sampler,
raw+max features, fixed-point I&Z solver), on every core of the build
container.  Run where oracle/build_ref.sh has installed the reference into
oracle/_ref:

    python tests/golden/make_config_golden.py [c5] [c3] [c1] [--seeds 1827,1828,1829,1830]

Writes, per config, ``tests/golden/cfg_<name>.json.gz`` (prices, variances, ci95,
per-date report, rule JSON v1 for every seed) and for the first seed
``cfg_<name>_betas.npz`` (the label vector of every date, captured from the
TrainingSet the reference hands to its own ``fit_ensemble``).  Nothing in the
reference is modified: the capture wraps the module attribute in memory.
"""

from __future__ import annotations

import argparse
import gzip
import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import reference as R  # noqa: E402

B = R.bermuda()
import bermuda.boundary_cmc as bcmc  # noqa: E402

CFG = {
    # BASELINE.json configs[4] (C5) and configs[2] (C3) with the reference's own sampler and features
    "c5": dict(d=10, s0=100.0, strike=100.0, r=0.05, sigma=0.2, delta=0.10, maturity=3.0, n_dates=9,
               n_train=10000, n_label=2000, rounds=100, n_paths=1 << 24),
    "c3": dict(d=5, s0=100.0, strike=100.0, r=0.05, sigma=0.2, delta=0.10, maturity=3.0, n_dates=9,
               n_train=5000, n_label=500, rounds=150, n_paths=1 << 20),
    # configs[0] (C1) with the reference's fixed-point solver, J = 1
    "c1": dict(d=1, s0=40.0, strike=40.0, r=0.06, sigma=0.2, delta=0.0, maturity=1.0, n_dates=10,
               j_points=1, n_inner=2000, n_paths=1 << 18),
}


def run_cmc(name, c, seed, engine, capture):
    params = B.MarketParams(d=c["d"], s0=c["s0"], r=c["r"], sigma=c["sigma"], delta=c["delta"])
    spec = B.BermudanSpec(c["strike"], c["maturity"], c["n_dates"])
    seen = []
    orig = bcmc.fit_ensemble

    def fit(ts, rounds):
        seen.append(np.array(ts.beta if hasattr(ts, "beta") else ts.betas, dtype=np.float64))
        return orig(ts, rounds)

    bcmc.fit_ensemble = fit
    try:
        t0 = time.perf_counter()
        rule, rep = B.build_cmc_rule(params, spec, B.CmcBuildConfig(c["n_train"], c["n_label"], c["rounds"]),
                                     seed=seed, engine=engine)
        t1 = time.perf_counter()
    finally:
        bcmc.fit_ensemble = orig
    est = B.price(params, spec, B.CmcScoreRule(rule), c["n_paths"], seed, engine=engine)
    t2 = time.perf_counter()
    out = {"seed": seed, "price": est.price, "variance": est.variance, "ci95": est.ci95, "n_paths": est.n_paths,
           "build_seconds": t1 - t0, "price_seconds": t2 - t1, "report": rep.to_json_dict(),
           "rule": json.loads(rule.to_json())}
    betas = None
    if capture:
        # dates are fitted m = n_dates-1 .. 1 (boundary_cmc.py:248)
        betas = {f"beta_m{c['n_dates'] - 1 - i}": b for i, b in enumerate(seen)}
    return out, betas


def run_iz(name, c, seed, engine):
    params = B.MarketParams(d=c["d"], s0=c["s0"], r=c["r"], sigma=c["sigma"], delta=c["delta"])
    spec = B.BermudanSpec(c["strike"], c["maturity"], c["n_dates"], B.PayoffKind.PUT_1D)
    t0 = time.perf_counter()
    b, rep = B.build_iz_boundary(params, spec, c["j_points"], c["n_inner"], seed=seed, engine=engine)
    t1 = time.perf_counter()
    est = B.price(params, spec, B.IzRule(b), c["n_paths"], seed, engine=engine,
                  unconverged_points=rep.unconverged_points)
    t2 = time.perf_counter()
    return {"seed": seed, "price": est.price, "variance": est.variance, "ci95": est.ci95, "n_paths": est.n_paths,
            "build_seconds": t1 - t0, "price_seconds": t2 - t1,
            "iteration_counts": [int(v) for v in rep.iteration_counts],
            "boundary": json.loads(b.to_json())}, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c3", "c5"])
    ap.add_argument("--seeds", default="1827,1828,1829,1830")
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    args = ap.parse_args()
    seeds = [int(s) for s in args.seeds.split(",")]
    engine = B.Engine(workers=args.workers, pool="process")
    for name in args.configs:
        c = CFG[name]
        runs = []
        for i, seed in enumerate(seeds):
            if name == "c1":
                res, betas = run_iz(name, c, seed, engine)
            else:
                res, betas = run_cmc(name, c, seed, engine, capture=(i == 0))
            runs.append(res)
            if betas:
                np.savez_compressed(HERE / f"cfg_{name}_betas.npz", **betas)
            print(f"{name} seed {seed}: {res['price']:.6f} +- {res['ci95']:.6f} "
                  f"(build {res['build_seconds']:.1f} s, price {res['price_seconds']:.1f} s)", flush=True)
            doc = {"config": name, "params": c, "workers": args.workers, "cpu_count": os.cpu_count(),
                   "numpy": np.__version__, "glibc": platform.libc_ver()[1], "python": platform.python_version(),
                   "reference": "bermuda " + B.__version__ + " (oracle/_ref, cython backend, Engine(pool='process'))",
                   "runs": runs}
            with gzip.open(HERE / f"cfg_{name}.json.gz", "wt") as fh:
                json.dump(doc, fh)


if __name__ == "__main__":
    main()
