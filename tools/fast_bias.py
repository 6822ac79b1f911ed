"""Separate rule noise from walker bias in fast mode (diagnostic, GPU).

For build seeds s: parity rule P_s and fast rule F_s (full config), each
priced in parity and in fast mode on the same 2^24-path seed.  A biased fast
WALKER shows as price_fast(R) - price_parity(R) != 0 for a fixed rule R
(independent draws, so ~N(0, 2 SE^2)); a different RULE quality shows as
price_parity(F_s) - price_parity(P_s).

    python tools/fast_bias.py [c5|c3] [n_seeds]
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_0805_1827_b200 as E  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    n_seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    cfg = dict(bench.CONFIGS[name])
    params, spec = bench.build_objects(cfg, E)
    bc = E.CmcBuildConfig(cfg["n_train"], cfg["n_label"], cfg["rounds"])
    rows = []
    for seed in range(1827, 1827 + n_seeds):
        rules = {}
        for mode in ("parity", "fast"):
            rules[mode], _ = E.build_cmc_rule(params, spec, bc, seed=seed, sampler="bridge", mode=mode)
        row = {"seed": seed}
        for rmode, rule in rules.items():
            for pmode in ("parity", "fast"):
                est = E.price(params, spec, E.CmcScoreRule(rule), cfg["n_paths"], seed, mode=pmode)
                row[f"rule_{rmode}/price_{pmode}"] = (est.price, est.std_error)
        rows.append(row)
        print(json.dumps(row), flush=True)
    keys = [k for k in rows[0] if k != "seed"]
    summary = {k: float(np.mean([r[k][0] for r in rows])) for k in keys}
    walker = [r["rule_parity/price_fast"][0] - r["rule_parity/price_parity"][0] for r in rows]
    walker += [r["rule_fast/price_fast"][0] - r["rule_fast/price_parity"][0] for r in rows]
    rule = [r["rule_fast/price_parity"][0] - r["rule_parity/price_parity"][0] for r in rows]
    se = rows[0]["rule_parity/price_parity"][1]
    print(json.dumps({"means": summary, "walker_diff_mean": float(np.mean(walker)),
                      "walker_diff_se": float(np.sqrt(2) * se / np.sqrt(len(walker))),
                      "rule_diff_mean": float(np.mean(rule)), "rule_diff_sd": float(np.std(rule, ddof=1)),
                      "pricing_se": se}))


if __name__ == "__main__":
    main()
