"""Time the device AdaBoost on a C5-shaped training set (diagnostic, GPU).

    BRM_BOOST_TIMING=1 python tools/boost_timing.py [n] [F] [rounds] [mode]

Prints the per-phase clock totals of CTA 0 (stderr, from the library) and the
CUDA-event time per fit.
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_0805_1827_b200 as E  # noqa: E402
from paper_0805_1827_b200 import backend as G  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 11
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 100
    mode = sys.argv[4] if len(sys.argv) > 4 else "parity"
    rng = np.random.default_rng(3)
    X = 100 * np.exp(0.25 * rng.normal(size=(n, F)))
    X[:, -1] = X[:, :-1].max(axis=1)
    beta = (X[:, -1] - 130) + 0.3 * (X[:, 0] - 100) + 8 * rng.normal(size=n)
    xs = torch.from_numpy(X).cuda()
    bs = torch.from_numpy(beta).cuda()
    for _ in range(2):
        G.fit_ensemble_arrays(xs, bs, rounds, mode=mode)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f, t, p, a, _, ic = G.fit_ensemble_arrays(xs, bs, rounds, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"n={n} F={F} rounds={rounds} mode={mode}: {np.median(ts):.3f} ms per fit "
          f"({1e3 * np.median(ts) / max(len(f), 1):.1f} us per round, {len(f)} stumps)")


if __name__ == "__main__":
    main()
