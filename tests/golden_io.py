"""Load tests/golden/golden.npz (made by tests/golden/make_golden.py from the reference)."""
from __future__ import annotations

import json
from pathlib import Path
from types import SimpleNamespace

import numpy as np

PATH = Path(__file__).resolve().parent / "golden" / "golden.npz"
_G = None


def G():
    global _G
    if _G is None:
        _G = dict(np.load(PATH))
    return _G


def packs(prefix):
    g = G()
    d, nd, k, pk = g[f"{prefix}.mp.scalars"]
    mp = SimpleNamespace(d=int(d), n_dates=int(nd), strike=float(k), payoff_kind=int(pk),
                         **{f: g[f"{prefix}.mp.{f}"] for f in ("step_mu", "step_vol", "chol", "disc_steps", "s0")})
    kind, call_like, imm = g[f"{prefix}.rp.scalars"]
    rp = SimpleNamespace(kind=int(kind), call_like=int(call_like), imm_date=int(imm), iz_space=0,
                         **{f: g[f"{prefix}.rp.{f}"] for f in ("iz_coeffs", "iz_lo", "iz_hi", "cmc_starts",
                                                                "cmc_counts", "cmc_feat", "cmc_thr", "cmc_pol",
                                                                "cmc_alpha", "cmc_intercept")})
    return mp, rp


def text(name) -> str:
    return G()[name].tobytes().decode()


def doc(name) -> dict:
    return json.loads(text(name))


PATH_CASES = ("path.maxcall5_eu", "path.maxcall5_cmc", "path.maxcall3_iz", "path.put1_iz")
