import sys, time, cProfile, pstats, json
sys.path.insert(0, '.')
import bench, numpy as np
import paper_0805_1827_b200 as E
from paper_0805_1827_b200 import _native as N
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c5']
params, spec = bench.build_objects(cfg, E)
bench.engine_step(cfg, E, params, spec, cfg['mode'])
t0 = time.perf_counter()
pr = cProfile.Profile(); pr.enable()
est, rep, _ = bench.engine_step(cfg, E, params, spec, cfg['mode'])
pr.disable()
print('total', time.perf_counter() - t0)
print(json.dumps(rep.to_json_dict()['phases']), est.timings)
for d in rep.per_date: print(d)
pstats.Stats(pr).sort_stats('cumulative').print_stats(25)
