"""One C5-shaped label launch (d=10, 100 stumps/date) and one pricing launch, parity or fast."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from tests import _cases as CS
from paper_0805_1827_b200 import backend as G
from paper_0805_1827_b200 import _native as N
mode = sys.argv[1] if len(sys.argv) > 1 else "parity"
n_train = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
p, s = CS.maxcall(10)
mp = CS.packs(p, s)
rp = CS.random_stumps(10, 9, 100, seed=4, lo=90, hi=160)
br = np.concatenate([p.log_drift * 3.0, p.sigma * np.sqrt(3.0), np.log(p.s0), p.sigma * 1.0, [1 / 9]])
for rep in range(2):
    N.profile_reset(); N.profile_enable(True)
    t0 = time.perf_counter()
    f, b = G.cmc_calc(mp, rp, 1, 1827, 0, n_train, 2000, br, mode=mode)
    t1 = time.perf_counter()
    st = G.price_blocks(mp, rp, 1 << 22, 1827, mode=mode)
    t2 = time.perf_counter()
    N.profile_enable(False)
    pr = N.profile_read()
print(f"labels {1e3*(t1-t0):.1f} ms, pricing 2^22 {1e3*(t2-t1):.1f} ms")
ms, nl, steps = pr["walk"]
print(f"walk kernels {ms:.1f} ms, {nl} launches, {steps} path-steps -> {steps*10/ms/1e6:.3g} G asset-steps/s")
