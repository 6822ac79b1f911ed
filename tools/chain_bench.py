"""Time the sequential vs warp-tile cumsum chains (brm_selftest_math kinds 8/9) on one warp."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_0805_1827_b200 import _native as N
rng = np.random.default_rng(1)
n = 10000
cases = {"uniform": np.full(n, 1.0 / n), "random": rng.random(n) / (n / 2),
         "lognormal": np.exp(rng.normal(scale=1.5, size=n)) / n / 3}
for name, a in cases.items():
    da = torch.tensor(a, device="cuda")
    out = torch.empty_like(da)
    res = {}
    for kind in (8, 9):
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            N.check(N.lib.brm_selftest_math(0, kind, N.ptr(da), None, n, N.ptr(out)))
            torch.cuda.synchronize()
            res[kind] = (time.perf_counter() - t0) * 1e6
        res[str(kind)] = out.cpu().numpy().copy()
    same = np.array_equal(res["8"].view(np.int64), res["9"].view(np.int64))
    print(f"{name:10s} n={n}: sequential {res[8]:.1f} us  warp {res[9]:.1f} us  identical={same}")
