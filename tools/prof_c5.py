"""C5 walker launches for ncu: build the real C5 rule, then one label launch (date 1) and one
pricing launch (2^22 paths).  ncu -k regex:walk_units -s 8 -c 2 profiles the last two."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import bench
import paper_0805_1827_b200 as E
from paper_0805_1827_b200 import backend as G
from paper_0805_1827_b200.boundary_cmc import bridge_scalars
from paper_0805_1827_b200.packs import pack_market
mode = sys.argv[1] if len(sys.argv) > 1 else "parity"
cfg = bench.CONFIGS["c5"]
p, s = bench.build_objects(cfg, E)
rule, _ = E.build_cmc_rule(p, s, E.CmcBuildConfig(cfg["n_train"], cfg["n_label"], cfg["rounds"]), seed=1827, mode=mode)
mp = pack_market(p, s)
rp = rule.pack()
from paper_0805_1827_b200 import _native as N
N.profile_reset()
t0 = time.perf_counter()
G.cmc_calc(mp, rp, 1, 1827, 0, cfg["n_train"], cfg["n_label"], bridge_scalars(p, s, 1), mode=mode)
t1 = time.perf_counter()
s_lab = N.profile_read()["walk"][2]
G.price_blocks(mp, rp, 1 << 22, 1827, mode=mode)
t2 = time.perf_counter()
s_all = N.profile_read()["walk"][2]
print(f"labels(date1) {1e3*(t1-t0):.2f} ms  pricing(2^22) {1e3*(t2-t1):.2f} ms  path-steps: labels {s_lab} pricing {s_all - s_lab}")
