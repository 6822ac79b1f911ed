"""Micro-rates of the walker components on one GPU (CUDA-event timed by the library profiler)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from tests import _cases as CS
from paper_0805_1827_b200 import backend as G, _native as N
from paper_0805_1827_b200.packs import RulePack

def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    N.profile_reset(); N.profile_enable(True)
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); wall = (time.perf_counter() - t0) / reps
    N.profile_enable(False)
    pr = N.profile_read()
    return wall, {k: (v[0] / reps, v[2] / reps) for k, v in pr.items() if v[1]}

out = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
k, s = G.derive_words(1, 2, 3, 4)
w, pr = timed(lambda: N.check(N.lib.brm_normals(0, int(k), int(s), 0, out.numel(), N.ptr(out))))
print(f"normals fill: {out.numel() / pr['rng'][0] / 1e6:.1f} G normals/s (kernel {pr['rng'][0]:.2f} ms)")
for d in (1, 5, 10):
    p, sp = CS.maxcall(d)
    mp = CS.packs(p, sp)
    for mode in ("parity", "fast"):
        rp = RulePack.european(True)
        n = 1 << 22
        w, pr = timed(lambda: G.price_blocks(mp, rp, n, 7, mode=mode))
        ms, steps = pr["walk"]
        print(f"d={d:2d} {mode:6s} european: {steps * d / ms / 1e6:8.1f} G asset-steps/s  ({ms:.2f} ms, {steps/n:.2f} steps/path)")
    rp = CS.random_stumps(d, 9, 100, seed=3, lo=100, hi=200)
    for mode in ("parity", "fast"):
        w, pr = timed(lambda: G.price_blocks(mp, rp, 1 << 22, 7, mode=mode))
        ms, steps = pr["walk"]
        print(f"d={d:2d} {mode:6s} cmc100  : {steps * d / ms / 1e6:8.1f} G asset-steps/s  ({ms:.2f} ms, {steps/(1<<22):.2f} steps/path)")
