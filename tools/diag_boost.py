import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_0805_1827_b200 import backend as G
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(0)
n, F = 10000, 11
X = 100 * np.exp(0.3 * rng.normal(size=(n, F)))
X[:, -1] = X[:, :-1].max(axis=1)
for frac in (0.01, 0.1, 0.3, 0.5):
    beta = np.where(rng.random(n) < frac, 1.0, -1.0) * (1 + (X[:, -1] > 130))
    G.fit_ensemble_arrays(X, beta, rounds)
    t0 = time.perf_counter()
    f, *_ = G.fit_ensemble_arrays(X, beta, rounds)
    print(f"frac {frac}: {len(f)} rounds in {1e3*(time.perf_counter()-t0):.1f} ms")
