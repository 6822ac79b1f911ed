"""Threshold-list sizes of the C4 (and C3) rule: distinct thresholds per (date, feature) (diagnostic, GPU)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import bench
import paper_0805_1827_b200 as E
for name in sys.argv[1:] or ["c4", "c3"]:
    cfg = bench.CONFIGS[name]
    p, s = bench.build_objects(cfg, E)
    rule, _ = E.build_cmc_rule(p, s, E.CmcBuildConfig(cfg["n_train"], cfg["n_label"], cfg["rounds"]), seed=1827,
                               sampler=cfg["sampler"], mode=cfg["mode"])
    d = p.d
    rows = []
    for m in sorted(rule.ensembles):
        ens = rule.ensembles[m]
        per = {}
        for st in ens.rounds:
            per.setdefault(st.feature, set()).add(st.threshold)
        asset = [len(v) for f, v in per.items() if f < d]
        rows.append((m, len(ens.rounds), len(per), max(asset) if asset else 0, len(per.get(d, ()))))
    print(name, "date, stumps, features used, max distinct thresholds on an asset feature, on the derived feature")
    for r in rows:
        print("  ", r)
