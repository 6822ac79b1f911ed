"""Host-side profile of one bench config's engine step (GPU box only).

    python tools/prof_host.py [c1|c2|c3|c4|c5]

Prints the wall time per price, then a cProfile of five prices sorted by
internal time (a native call's time lands in its ctypes caller).
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
sys.argv = ["bench.py"]
import bench  # noqa: E402
import torch  # noqa: E402

import paper_0805_1827_b200 as E  # noqa: E402

cfg = bench.CONFIGS[name]
params, spec = bench.build_objects(cfg, E)
for _ in range(3):
    bench.engine_step(cfg, E, params, spec, cfg["mode"])
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    bench.engine_step(cfg, E, params, spec, cfg["mode"])
torch.cuda.synchronize()
print(f"{name}: {(time.perf_counter() - t) / 5 * 1e3:.3f} ms per price")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    bench.engine_step(cfg, E, params, spec, cfg["mode"])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
