"""Walker launches of a CMC config for ncu: build the real rule, then one label launch (date 1)
and one pricing launch (2^22 paths).  ncu -k regex:walk_units -s 8 -c 2 profiles the last two
(C5; use -s <n_dates - 1> for other configs).

usage: python tools/prof_c5.py [parity|fast] [reps] [config]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import bench
import paper_0805_1827_b200 as E
from paper_0805_1827_b200 import backend as G
from paper_0805_1827_b200.boundary_cmc import bridge_scalars
from paper_0805_1827_b200.packs import pack_market
mode = sys.argv[1] if len(sys.argv) > 1 else "parity"
cfg = bench.CONFIGS[sys.argv[3] if len(sys.argv) > 3 else "c5"]
p, s = bench.build_objects(cfg, E)
rule, _ = E.build_cmc_rule(p, s, E.CmcBuildConfig(cfg["n_train"], cfg["n_label"], cfg["rounds"]), seed=1827,
                           sampler=cfg["sampler"], mode=mode)
mp = pack_market(p, s)
rp = rule.pack()
from paper_0805_1827_b200 import _native as N
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
best = [1e9, 1e9]
for _ in range(reps):
    N.profile_reset()
    N.profile_enable(True)
    G.cmc_calc(mp, rp, 1, 1827, 0, cfg["n_train"], cfg["n_label"], bridge_scalars(p, s, 1), cfg["sampler"],
               mode=mode)
    pr = N.profile_read()
    s_lab, ms_lab = pr["walk"][2], pr["walk"][0]
    G.price_blocks(mp, rp, 1 << 22, 1827, mode=mode)
    pr = N.profile_read()
    N.profile_enable(False)
    s_all, ms_all = pr["walk"][2], pr["walk"][0]
    best = [min(best[0], ms_lab), min(best[1], ms_all - ms_lab)]
print(f"{mode}: walker labels(date1) {best[0]:.2f} ms  pricing(2^22) {best[1]:.2f} ms  (best of {reps})  "
      f"path-steps: labels {s_lab} pricing {s_all - s_lab}")
