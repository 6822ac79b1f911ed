import cProfile, pstats, sys, time
sys_path_fix = __import__("sys").path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
sys.argv = ["bench.py"]
import bench, torch
import paper_0805_1827_b200 as E
cfg = bench.CONFIGS["c1"]
params, spec = bench.build_objects(cfg, E)
for _ in range(3): bench.engine_step(cfg, E, params, spec, cfg["mode"])
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(5): bench.engine_step(cfg, E, params, spec, cfg["mode"])
torch.cuda.synchronize(); print("ms/step", (time.perf_counter()-t)/5*1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(5): bench.engine_step(cfg, E, params, spec, cfg["mode"])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
