"""Time the parity walker on C5 work (diagnostic, GPU): final pricing of the
reference's C5 rule (2^24 paths) and the date-1 label launch (10000 points x
2000 paths under the reference rule).  BRM_LIB_PATH selects a library variant.

    python tools/walk_bench.py [reps]
"""
import gzip
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_0805_1827_b200 as E  # noqa: E402
from paper_0805_1827_b200 import _native as N  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    with gzip.open(ROOT / "tests/golden/cfg_c5.json.gz", "rt") as fh:
        doc = json.load(fh)
    c = doc["params"]
    params = E.MarketParams(d=c["d"], s0=c["s0"], r=c["r"], sigma=c["sigma"], delta=c["delta"])
    spec = E.BermudanSpec(c["strike"], c["maturity"], c["n_dates"])
    run = doc["runs"][0]
    rule = E.CmcRule.from_json_dict(run["rule"])
    pts = E.boundary_cmc.sample_training_points(params, spec, 1, c["n_train"], run["seed"], "bridge", mode="parity")
    later = rule.restricted_after(1)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        N.profile_reset()
        N.profile_enable(True)
        for _ in range(reps):
            out = fn()
        torch.cuda.synchronize()
        N.profile_enable(False)
        prof = N.profile_read()
        return prof["walk"][0] / reps, prof["walk"][2] / reps, out

    ms_p, steps_p, est = timed(lambda: E.price(params, spec, E.CmcScoreRule(rule), c["n_paths"], run["seed"],
                                               mode="parity"))
    ms_l, steps_l, beta = timed(lambda: E.boundary_cmc.label_points(params, spec, pts, 1, c["n_label"], later,
                                                                    run["seed"], mode="parity"))
    lib = os.environ.get("BRM_LIB_PATH", "default")
    for name, ms, steps in (("pricing", ms_p, steps_p), ("labels m=1", ms_l, steps_l)):
        rate = steps * c["d"] / (ms / 1e3)
        print(f"{lib}: {name}: {ms:.3f} ms, {rate:.4g} asset-steps/s, frac(70 ops) {rate * 70 / 18.61e12:.3f}")
    print(f"{lib}: price {est.price!r} (reference {run['price']!r}); beta checksum {float(np.sum(beta))!r}")


if __name__ == "__main__":
    main()
