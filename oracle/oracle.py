"""CPU oracle: ctypes wrapper of bermuda_oracle.c plus numpy restatements.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference legs import this module; the engine in
paper_0805_1827_b200/ never does.  The walker restatement is pinned against the
built reference (oracle/_ref) by tests/test_oracle_pin.py and the committed
fixtures in tests/golden/.

Contents
  walker  : raw_uint64, normals, path_values, stopped_sums, iz_solve,
            iz_bisect, cmc_labels, sample_points, decisions  (C, -ffp-contract=off)
  boosting: fit_stump / fit_ensemble restated from boosting.py:126-206
  misc    : pool_moments (pricer.py:136-151), price (pricer.py:154-202 as one
            loop), regress (boundary_iz.py:250-276), pairwise_sum (numpy order)
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "lib" / "liboracle.so"

_dp, _ip, _up = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_uint64)


class OrcCtx(C.Structure):
    _fields_ = [("d", C.c_int), ("n_dates", C.c_int), ("payoff_kind", C.c_int), ("strike", C.c_double),
                ("step_mu", _dp), ("step_vol", _dp), ("chol", _dp), ("disc_steps", _dp),
                ("rule_kind", C.c_int), ("call_like", C.c_int), ("imm_date", C.c_int), ("nbasis", C.c_int),
                ("iz_space", C.c_int),
                ("iz_coeffs", _dp), ("iz_lo", _dp), ("iz_hi", _dp),
                ("cmc_starts", _ip), ("cmc_counts", _ip), ("cmc_feat", _ip),
                ("cmc_thr", _dp), ("cmc_pol", _dp), ("cmc_alpha", _dp), ("cmc_intercept", _dp),
                ("normals", _dp), ("normals_base", C.c_uint64), ("normals_count", C.c_uint64)]


def build() -> Path:
    """Compile liboracle.so (gcc, -ffp-contract=off) if stale."""
    src = HERE / "bermuda_oracle.c"
    if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def _load():
    build()
    lib = C.CDLL(str(LIB_PATH))
    P = C.POINTER(OrcCtx)
    sig = {
        "orc_derive_words": [C.c_uint64] * 4 + [_up, _up],
        "orc_raw_fill": [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, _up],
        "orc_normals_fill": [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, _dp],
        "orc_path_values": [P, _dp, C.c_int, C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64, _dp, _ip],
        "orc_stopped_sums": [P, _dp, C.c_int, C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64, _dp, _dp],
        "orc_iz_solve": [P, _dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                         _dp, _ip, _ip],
        "orc_iz_bisect": [P, _dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                          C.c_uint64, C.c_uint64, _dp, _ip, _ip],
        "orc_cmc_labels": [P, _dp, C.c_int64, C.c_int, C.c_int, _up, _up, C.c_uint64, _dp],
        "orc_sample_points": [P, C.c_int, C.c_int, C.c_int64, _up, _up, _dp, _dp, _dp, _dp, _dp, C.c_double, _dp],
        "orc_decision": [P, C.c_int, _dp],
        "orc_payoff_value": [P, _dp, _dp],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    return lib


_lib = _load()


def _dptr(a):
    return a.ctypes.data_as(_dp) if a is not None and a.size else None


class Ctx:
    """Oracle context over a (MarketPack, RulePack) pair (duck-typed)."""

    def __init__(self, mp, rp, normals=None, normals_base: int = 0):
        f = lambda x: np.ascontiguousarray(x, dtype=np.float64)
        i = lambda x: np.ascontiguousarray(x, dtype=np.int32)
        self.keep = [f(mp.step_mu), f(mp.step_vol), f(mp.chol), f(mp.disc_steps),
                     f(rp.iz_coeffs), f(rp.iz_lo), f(rp.iz_hi),
                     i(rp.cmc_starts), i(rp.cmc_counts), i(rp.cmc_feat),
                     f(rp.cmc_thr), f(rp.cmc_pol), f(rp.cmc_alpha), f(rp.cmc_intercept)]
        nrm = f(normals).ravel() if normals is not None else None
        self.keep.append(nrm)
        k = self.keep
        coeffs = k[4]
        nb = coeffs.shape[-1] if coeffs.ndim == 3 else 1
        ip = lambda a: a.ctypes.data_as(_ip) if a.size else None
        self.c = OrcCtx(int(mp.d), int(mp.n_dates), int(mp.payoff_kind), float(mp.strike),
                        _dptr(k[0]), _dptr(k[1]), _dptr(k[2]), _dptr(k[3]),
                        int(rp.kind), int(rp.call_like), int(rp.imm_date), int(nb), int(getattr(rp, "iz_space", 0)),
                        _dptr(k[4]), _dptr(k[5]), _dptr(k[6]), ip(k[7]), ip(k[8]), ip(k[9]),
                        _dptr(k[10]), _dptr(k[11]), _dptr(k[12]), _dptr(k[13]),
                        _dptr(nrm), int(normals_base), 0 if nrm is None else nrm.size)
        self.d = int(mp.d)
        self.mp, self.rp = mp, rp

    @property
    def ref(self):
        return C.byref(self.c)


def derive_words(seed, phase, item, date):
    k, s = C.c_uint64(), C.c_uint64()
    _lib.orc_derive_words(int(seed) & (2**64 - 1), int(phase), int(item), int(date), C.byref(k), C.byref(s))
    return np.uint64(k.value), np.uint64(s.value)


def raw_uint64(key, stream, start, count):
    out = np.empty(count, dtype=np.uint64)
    _lib.orc_raw_fill(int(key), int(stream), int(start), count, out.ctypes.data_as(_up))
    return out


def normals(key, stream, start, count):
    out = np.empty(count)
    _lib.orc_normals_fill(int(key), int(stream), int(start), count, out.ctypes.data_as(_dp))
    return out


def path_values(ctx: Ctx, start, m_start, n_paths, key, stream, draw_base=0):
    st = np.ascontiguousarray(start, dtype=np.float64)
    vals = np.empty(n_paths)
    stops = np.empty(n_paths, dtype=np.int32)
    rc = _lib.orc_path_values(ctx.ref, _dptr(st), m_start, n_paths, int(key), int(stream), int(draw_base),
                              vals.ctypes.data_as(_dp), stops.ctypes.data_as(_ip))
    if rc:
        raise ValueError("start date has no remaining exercise dates")
    return vals, stops


def stopped_sums(ctx: Ctx, start, m_start, n_paths, key, stream, draw_base=0):
    st = np.ascontiguousarray(start, dtype=np.float64)
    s, q = C.c_double(), C.c_double()
    rc = _lib.orc_stopped_sums(ctx.ref, _dptr(st), m_start, n_paths, int(key), int(stream), int(draw_base),
                               C.byref(s), C.byref(q))
    if rc:
        raise ValueError("start date has no remaining exercise dates")
    return s.value, q.value


def iz_solve(ctx: Ctx, seed_point, asset, m, n_inner, eps, max_iter, avg_window, key, stream):
    sp = np.ascontiguousarray(seed_point, dtype=np.float64).ravel()
    sp = sp if sp.size else np.zeros(1)
    lv, it, cv = C.c_double(), C.c_int32(), C.c_int32()
    rc = _lib.orc_iz_solve(ctx.ref, _dptr(sp), asset, m, n_inner, eps, max_iter, avg_window, int(key), int(stream),
                           C.byref(lv), C.byref(it), C.byref(cv))
    if rc:
        raise ValueError("start date has no remaining exercise dates")
    return lv.value, it.value, bool(cv.value)


def iz_bisect(ctx: Ctx, seed_point, asset, m, n_inner, lo, hi, tol, max_iter, key, stream):
    sp = np.ascontiguousarray(seed_point, dtype=np.float64).ravel()
    sp = sp if sp.size else np.zeros(1)
    lv, it, cv = C.c_double(), C.c_int32(), C.c_int32()
    rc = _lib.orc_iz_bisect(ctx.ref, _dptr(sp), asset, m, n_inner, lo, hi, tol, max_iter, int(key), int(stream),
                            C.byref(lv), C.byref(it), C.byref(cv))
    if rc:
        raise ValueError("start date has no remaining exercise dates")
    return lv.value, it.value, bool(cv.value)


def cmc_labels(ctx: Ctx, points, m, n_label, keys, streams, draw_base):
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, ctx.d)
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    s = np.ascontiguousarray(streams, dtype=np.uint64)
    out = np.empty(pts.shape[0])
    rc = _lib.orc_cmc_labels(ctx.ref, _dptr(pts), pts.shape[0], m, n_label, k.ctypes.data_as(_up),
                             s.ctypes.data_as(_up), int(draw_base), out.ctypes.data_as(_dp))
    if rc:
        raise ValueError("start date has no remaining exercise dates")
    return out


def bridge_scalars(params, spec, m):
    """Host scalars of the reference sampler, formed exactly as market.py does."""
    import math
    T = spec.maturity
    drift_T = params.log_drift * T
    sig_sqrt_T = params.sigma * math.sqrt(T)
    log_s0 = np.log(params.s0)
    t = m * spec.dt
    lam = (t - 0.0) / (T - 0.0)
    sd = math.sqrt((t - 0.0) * (T - t) / (T - 0.0)) if m < spec.n_dates else 0.0
    bsd = params.sigma * sd
    return np.concatenate([drift_T, sig_sqrt_T, log_s0, bsd, [lam]])


def sample_points(ctx: Ctx, params, spec, m, seed, n, item_lo=0, mode=0):
    keys = np.empty(n, dtype=np.uint64)
    streams = np.empty(n, dtype=np.uint64)
    for i in range(n):
        keys[i], streams[i] = derive_words(seed, 2, item_lo + i, m)
    b = bridge_scalars(params, spec, m)
    d = ctx.d
    out = np.empty((n, d))
    s0 = np.ascontiguousarray(params.s0, dtype=np.float64)
    _lib.orc_sample_points(ctx.ref, mode, m, n, keys.ctypes.data_as(_up), streams.ctypes.data_as(_up), _dptr(s0),
                           _dptr(b[:d].copy()), _dptr(b[d:2 * d].copy()), _dptr(b[2 * d:3 * d].copy()),
                           _dptr(b[3 * d:4 * d].copy()), float(b[4 * d]), out.ctypes.data_as(_dp))
    return out, keys, streams


def decision(ctx: Ctx, m, state):
    st = np.ascontiguousarray(state, dtype=np.float64)
    return bool(_lib.orc_decision(ctx.ref, m, _dptr(st)))


def payoff(ctx: Ctx, state):
    st = np.ascontiguousarray(state, dtype=np.float64)
    out = C.c_double()
    _lib.orc_payoff_value(ctx.ref, _dptr(st), C.byref(out))
    return out.value


# ------------------------------------------------------------- pricing ----
PATH_BLOCK = 4096


def pool_moments(counts, sums, sumsqs):
    """Sequential fold in block order (pricer.py:136-151)."""
    n = int(np.sum(counts))
    s = ss = 0.0
    for si, qi in zip(sums, sumsqs):
        s += float(si)
        ss += float(qi)
    mean = s / n
    var = (ss - s * s / n) / (n - 1) if n > 1 else 0.0
    return mean, max(var, 0.0), n


def price_blocks(ctx: Ctx, n_paths, seed, block_lo=0, block_hi=None):
    n_blocks = (n_paths + PATH_BLOCK - 1) // PATH_BLOCK
    block_hi = n_blocks if block_hi is None else block_hi
    out = np.empty((block_hi - block_lo, 3))
    for row, b in enumerate(range(block_lo, block_hi)):
        cnt = min(PATH_BLOCK, n_paths - b * PATH_BLOCK)
        k, s = derive_words(seed, 3, b, 0)
        out[row] = (cnt, *stopped_sums(ctx, ctx.mp.s0, 0, cnt, k, s, 0))
    return out


# ------------------------------------------------------------ boosting ----
def pairwise_sum(a) -> float:
    """numpy's pairwise summation order for a contiguous float64 vector."""
    a = np.asarray(a, dtype=np.float64)

    def rec(lo, n):
        if n < 8:
            r = 0.0
            for i in range(lo, lo + n):
                r += float(a[i])
            return r
        if n <= 128:
            r = [float(x) for x in a[lo:lo + 8]]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += float(a[lo + i + j])
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += float(a[lo + i])
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return rec(0, a.size)


def fit_stump(xs, ys, w):
    """Exhaustive weighted stump search with the reference tie rules (boosting.py:126-171).

    Returns (feature, threshold, polarity, err)."""
    n, F = xs.shape
    total = w.sum()
    best = None
    best_err = np.inf
    for f in range(F):
        order = np.argsort(xs[:, f], kind="stable")
        xf = xs[order, f]
        brk = np.flatnonzero(xf[1:] > xf[:-1])
        if brk.size == 0:
            continue
        pos = ys[order] > 0.0
        pc = np.cumsum(np.where(pos, w[order], 0.0))
        nc = np.cumsum(np.where(pos, 0.0, w[order]))
        ep = pc[brk] + (nc[-1] - nc[brk])
        em = total - ep
        inter = np.empty(2 * brk.size)
        inter[0::2], inter[1::2] = ep, em
        k = int(np.argmin(inter))
        if inter[k] < best_err:
            best_err = inter[k]
            best = (f, float(0.5 * (xf[brk[k >> 1]] + xf[brk[k >> 1] + 1])), 1.0 if k % 2 == 0 else -1.0)
    if best is None:
        pol = 1.0 if float(np.sum(w * ys)) >= 0.0 else -1.0
        return 0, float("-inf"), pol, float(np.sum(w[ys != pol]))
    return (*best, float(best_err))


def fit_ensemble(xs, betas, rounds):
    """Discrete AdaBoost (boosting.py:174-206): returns (feat, thr, pol, alpha, intercept)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    ys = np.where(np.asarray(betas) > 0.0, 1.0, -1.0)
    n = xs.shape[0]
    if np.unique(ys).size == 1:
        return [], [], [], [], float(ys[0])
    w = np.full(n, 1.0 / n)
    out = ([], [], [], [])
    for _ in range(rounds):
        f, thr, pol, err = fit_stump(xs, ys, w)
        if err >= 0.5:
            break
        alpha = float(0.5 * np.log((1.0 - err) / max(err, 1e-10)))
        for lst, v in zip(out, (f, thr, pol, alpha)):
            lst.append(v)
        if err <= 0.0:
            break
        pred = np.where(xs[:, f] > thr, pol, -pol)
        w = w * np.exp(-alpha * ys * pred)
        w /= w.sum()
    if not out[0]:
        return [], [], [], [], 1.0 if float(np.sum(ys)) >= 0.0 else -1.0
    return (*out, 0.0)


def regress(design, levels):
    """np.linalg.lstsq with the cross-term-free fallback (boundary_iz.py:250-276)."""
    design = np.asarray(design, dtype=np.float64)
    n, nb = design.shape
    coeffs, _, rank, _ = np.linalg.lstsq(design, levels, rcond=None)
    if rank < nb:
        k = int(round((-3 + np.sqrt(9 + 8 * (nb - 1))) / 2))
        keep = [0] + list(range(1, k + 1))
        pos = 1 + k
        for a in range(k):
            keep.append(pos)
            pos += k - a
        sub = np.linalg.lstsq(design[:, keep], levels, rcond=None)[0]
        coeffs = np.zeros(nb)
        coeffs[keep] = sub
    return coeffs


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------- lattice ----
def crr_bermudan(s0, strike, r, delta, sigma, maturity, n_dates, steps, put=True):
    """CRR lattice Bermudan price, exercise at n_dates equally spaced dates
    (restates the reference's crr_price, oracle.py:98-143, for d = 1)."""
    import math
    dt = maturity / steps
    u = math.exp(sigma * math.sqrt(dt))
    dn = 1.0 / u
    p = (math.exp((r - delta) * dt) - dn) / (u - dn)
    if not 0.0 < p < 1.0:
        raise ValueError("risk-neutral probability outside (0, 1)")
    disc = math.exp(-r * dt)
    stride = steps // n_dates
    ex = {stride * m for m in range(1, n_dates + 1)}

    def intrinsic(s):
        return np.maximum(strike - s, 0.0) if put else np.maximum(s - strike, 0.0)

    vals = intrinsic(s0 * u ** (2.0 * np.arange(steps + 1) - steps))
    for i in range(steps - 1, -1, -1):
        vals = disc * (p * vals[1:i + 2] + (1.0 - p) * vals[:i + 1])
        if i in ex:
            vals = np.maximum(vals, intrinsic(s0 * u ** (2.0 * np.arange(i + 1) - i)))
    return float(vals[0])
