"""Fast-mode walker for a column-constant Cholesky factor (equicorrelated assets, C4):
fast_step_colconst (brm_model.cuh) forms each row's product from a running prefix -- the
fma sequence of the triangular row loop, so the launch returns the same bits."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_AB = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from tests import _cases as CS
from paper_0805_1827_b200 import backend as G
p, s = CS.basketput(40, 20)
mp = CS.packs(p, s)
rp = CS.random_stumps(40, 20, 30, seed=7, lo=80, hi=110, call_like=False)
out = {{}}
for m_start in (0, 7):
    k, st = G.derive_words(1827, 2, 9, m_start)
    v, m = G.path_values(mp, rp, mp.s0, m_start, 30000, k, st, 0, mode="fast")
    out[f"v{{m_start}}"], out[f"m{{m_start}}"] = v, m
    out[f"s{{m_start}}"] = np.array(G.stopped_sums(mp, rp, mp.s0, m_start, 30000, k, st, 0, mode="fast"))
np.savez({out!r}, **out)
"""


def test_colconst_walker_equals_triangular_product(tmp_path):
    """BRM_WALK_COLCONST=0 keeps walk_units<40, fast, WALK_CMC_LOWER>: per-path values, stop dates
    and the folded sums are bit-identical to the default (prefix) instance."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        out = str(tmp_path / f"cc{flag}.npz")
        env = dict(os.environ, BRM_WALK_COLCONST=flag)
        subprocess.run([sys.executable, "-c", _AB.format(root=root, out=out)], check=True, env=env, cwd=root)
        outs.append(np.load(out))
    for key in outs[0].files:
        assert np.array_equal(outs[0][key], outs[1][key]), key
    assert np.count_nonzero(outs[0]["m0"]) > 1000  # the rule and the payoff are exercised


def test_block_correlated_factor_takes_the_triangular_product():
    """A factor that is NOT constant below the diagonal (two correlation blocks) must not take the
    prefix step: the fast price stays within 4 combined SE of the fp64 parity walker, and the
    host-side test the library applies (fp32 entries of a column all equal) is false for it."""
    from oracle import oracle as O
    from paper_0805_1827_b200 import backend as G
    from paper_0805_1827_b200.market import BermudanSpec, MarketParams, PayoffKind
    from tests import _cases as CS
    d = 40
    rho = np.full((d, d), 0.3)
    rho[:20, :20] = 0.5
    np.fill_diagonal(rho, 1.0)
    sig = np.random.default_rng(1827).uniform(0.2, 0.4, d)
    p = MarketParams(d=d, s0=100.0, r=0.05, sigma=sig, rho=rho)
    s = BermudanSpec(100.0, 1.0, 20, PayoffKind.BASKET_PUT)
    L32 = p.corr_factor.astype(np.float32)
    assert not all(L32[i, a] == L32[a + 1, a] for a in range(d - 2) for i in range(a + 2, d))
    mp = CS.packs(p, s)
    rp = CS.random_stumps(d, 20, 30, seed=7, lo=80, hi=110, call_like=False)
    n = 1 << 17
    g = G.price_blocks(mp, rp, n, 1827, mode="fast")
    o = G.price_blocks(mp, rp, n, 1828, mode="parity")
    mg, vg, _ = O.pool_moments(g[:, 0], g[:, 1], g[:, 2])
    mo, vo, _ = O.pool_moments(o[:, 0], o[:, 1], o[:, 2])
    se = np.sqrt(vg / n + vo / n)
    assert abs(mg - mo) < 4 * se, (mg, mo, se)
