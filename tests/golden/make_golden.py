"""Generate golden vectors from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists and
oracle/build_ref.sh has installed it into oracle/_ref):

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz (small) and golden_meta.json (library versions:
the fixtures pin results at the numpy / glibc boundary of this image).  The
fixtures are committed; tests read them on any machine.
"""

from __future__ import annotations

import json
import platform
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import reference as R  # noqa: E402

B = R.bermuda()
from bermuda._kernels import get_backend  # noqa: E402
from bermuda._kernels.packs import RulePack, pack_market, quad_basis  # noqa: E402

cy = get_backend("cython")
out: dict[str, np.ndarray] = {}


def put(name, value):
    out[name] = np.asarray(value)


def pack_arrays(prefix, mp, rp):
    for f in ("step_mu", "step_vol", "chol", "disc_steps", "s0"):
        put(f"{prefix}.mp.{f}", getattr(mp, f))
    put(f"{prefix}.mp.scalars", [mp.d, mp.n_dates, mp.strike, mp.payoff_kind])
    for f in ("iz_coeffs", "iz_lo", "iz_hi", "cmc_starts", "cmc_counts", "cmc_feat", "cmc_thr", "cmc_pol",
              "cmc_alpha", "cmc_intercept"):
        put(f"{prefix}.rp.{f}", getattr(rp, f))
    put(f"{prefix}.rp.scalars", [rp.kind, rp.call_like, rp.imm_date])


# ---- RNG -----------------------------------------------------------------
keys = [(0, 0, 0, 0), (11, 3, 5, 0), (1827, 2, 9999, 8), (2**63 + 5, 1, 77, 4)]
put("rng.fields", np.array(keys, dtype=np.uint64))
words = [B.StreamKey(s, B.Phase(p), i, d).words() for s, p, i, d in keys]
put("rng.words", np.array(words, dtype=np.uint64))
for j, (k, s) in enumerate(words):
    put(f"rng.raw.{j}", cy.raw_uint64(k, s, 3 + j, 257))
    put(f"rng.normals.{j}", cy.normals(k, s, 1000 * j + 1, 4099))

# ---- per-path values through the reference walker (n_paths=1 trick) ------
def per_path(prefix, params, spec, rp, m_start, n, key, draw_base=0):
    mp = pack_market(params, spec)
    pack_arrays(prefix, mp, rp)
    k, s = key
    per = (spec.n_dates - m_start) * params.d
    vals = [cy.stopped_sums(mp, rp, mp.s0, m_start, 1, k, s, draw_base + p * per)[0] for p in range(n)]
    put(f"{prefix}.m_start", m_start)
    put(f"{prefix}.key", np.array([k, s], dtype=np.uint64))
    put(f"{prefix}.draw_base", draw_base)
    put(f"{prefix}.values", vals)
    put(f"{prefix}.sums", cy.stopped_sums(mp, rp, mp.s0, m_start, n, k, s, draw_base))


mc5 = (B.MarketParams(d=5, s0=100.0, r=0.05, sigma=0.2, delta=0.1), B.BermudanSpec(100.0, 3.0, 9))
per_path("path.maxcall5_eu", *mc5, RulePack.european(True), 0, 200, B.StreamKey(7, B.Phase.PRICING, 3).words(), 5)
cmc_rule, _ = B.build_cmc_rule(*mc5, B.CmcBuildConfig(300, 40, 12), seed=3)
per_path("path.maxcall5_cmc", *mc5, cmc_rule.pack(), 0, 300, B.StreamKey(7, B.Phase.PRICING, 4).words())
put("cmc_rule.json", np.frombuffer(cmc_rule.to_json().encode(), dtype=np.uint8))
mc3 = (B.MarketParams(d=3, s0=100.0, r=0.05, sigma=0.2, delta=0.1), B.BermudanSpec(100.0, 3.0, 9))
iz_b, iz_rep = B.build_iz_boundary(*mc3, 16, 150, max_iter=30, seed=4)
per_path("path.maxcall3_iz", *mc3, iz_b.pack(), 2, 300, B.StreamKey(9, B.Phase.PRICING, 1).words())
put("iz_boundary.json", np.frombuffer(iz_b.to_json().encode(), dtype=np.uint8))
put1 = (B.MarketParams(d=1, s0=40.0, r=0.06, sigma=0.2), B.BermudanSpec(40.0, 1.0, 10, B.PayoffKind.PUT_1D))
b1, rep1 = B.build_iz_boundary(*put1, 1, 500, seed=1827)
per_path("path.put1_iz", *put1, b1.pack(), 0, 300, B.StreamKey(1827, B.Phase.PRICING, 0).words())
put("put1.iteration_counts", rep1.iteration_counts)
put("put1.coeffs", b1.coeffs)

# ---- labels, probe solves ------------------------------------------------
mp5 = pack_market(*mc5)
later = cmc_rule.restricted_after(3).pack()
pts = B.sample_training_points(*mc5, 3, 64, 2)
lk = np.array([B.StreamKey(2, B.Phase.CMC_CALC, i, 3).words() for i in range(64)], dtype=np.uint64)
put("labels.points", pts)
put("labels.keys", lk)
put("labels.beta", cy.cmc_labels(mp5, later, pts, 3, 200, lk[:, 0], lk[:, 1], 10))
mp3 = pack_market(*mc3)
seeds = np.array([[90.0, 110.0], [120.0, 80.0], [150.0, 160.0]])
solves = [cy.iz_solve(mp3, iz_b.pack(), seeds[j], j % 3, 4, 300, 0.01, 60, 5,
                      *B.StreamKey(4, B.Phase.IZ_CALC, j, 4).words()) for j in range(3)]
put("iz_solve.seeds", seeds)
put("iz_solve.result", np.array([[lv, it, cv] for lv, it, cv in solves], dtype=np.float64))

# ---- sampler -------------------------------------------------------------
from bermuda.boundary_cmc import _draw_point  # noqa: E402

sk = [B.StreamKey(1827, B.Phase.CMC_CALC, i, 4).words() for i in range(16)]
put("sampler.points", np.array([_draw_point(*mc5, 4, k, s) for k, s in sk]))

# ---- boosting ------------------------------------------------------------
rng = np.random.default_rng(1)
X = 100 * np.exp(0.2 * rng.normal(size=(400, 6)))
X[:, 5] = X[:, :5].max(axis=1)
beta = (X[:, 0] - 100) + 0.5 * (X[:, 5] - 115) + 4 * rng.normal(size=400)
ens = B.fit_ensemble(B.TrainingSet(X, beta), 25)
put("boost.X", X)
put("boost.beta", beta)
put("boost.stumps", np.array([[s.feature, s.threshold, s.polarity, s.alpha] for s in ens.rounds]))
w = rng.uniform(0.1, 1.0, 400)
w /= w.sum()
ys = np.where(beta > 0, 1.0, -1.0)
st, err = B.fit_stump(X, ys, w)
put("fit_stump.w", w)
put("fit_stump.result", [st.feature, st.threshold, st.polarity, err])

# ---- host-side conventions ------------------------------------------------
z = rng.uniform(50, 250, size=(7, 3))
put("quad_basis.z", z)
put("quad_basis.design", quad_basis(z))
g = B.generate_glp(64, 4, B.default_box(100.0, 4))
put("glp.64x4", g.points)
put("regress.levels", 120 + g.points.sum(axis=1) * 0.05 + rng.normal(size=64))
put("regress.coeffs", B.regress_boundary(g, out["regress.levels"]))
put("partition.17x5", [r for r in B.partition(17, 5).ranges])
est = B.price(*mc5, B.CmcScoreRule(cmc_rule), 10000, 5)
put("price.cmc", [est.price, est.variance, est.ci95, est.n_paths])
put("crr.put1", B.crr_price(*put1, B.TreeSpec.bermudan(5000, 10)).price)

np.savez_compressed(HERE / "golden.npz", **out)
meta = {"numpy": np.__version__, "python": platform.python_version(), "glibc": platform.libc_ver()[1],
        "machine": platform.machine(), "reference": "bermuda " + B.__version__ + " (oracle/_ref, cython backend)"}
(HERE / "golden_meta.json").write_text(json.dumps(meta, indent=1) + "\n")
print(f"wrote {len(out)} arrays to {HERE / 'golden.npz'}")
