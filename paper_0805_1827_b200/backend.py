"""Kernel-backend module with the reference's duck-typed surface.

Drop-in for ``bermuda._kernels.core_backend`` / ``numpy_backend``
(core_backend.py:12-58, numpy_backend.py:19-190): the same function names,
argument order and return types, computed by the sm_100a kernels of
libbermuda_b200.so.  Batched entry points (``price_blocks``,
``iz_solve_batch``, ``cmc_labels_keyed``, ``sample_points``) are what the
phase builders of this package use; the single-item functions exist so the
reference's own builders can run on this backend unchanged.

Every function takes an optional ``mode`` ("parity" or "fast", default from
BERMUDA_B200_MODE) and ``device``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .context import get_context

name = "cuda"

__all__ = ["name", "raw_uint64", "normals", "stopped_sums", "path_values", "iz_solve", "iz_solve_batch",
           "cmc_labels", "cmc_labels_keyed", "price_blocks", "sample_points", "decisions", "derive_words"]


def _dev(device):
    from .context import default_device
    return default_device() if device is None else int(device)


def derive_words(master_seed: int, phase: int, task_id: int, date_index: int):
    """(key64, stream64) of StreamKey(master_seed, phase, task_id, date_index) (rng.py:79-89)."""
    k, s = C.c_uint64(), C.c_uint64()
    N.check(N.lib.brm_derive_words(int(master_seed) & (2**64 - 1), int(phase), int(task_id) & (2**64 - 1),
                                   int(date_index) & (2**64 - 1), C.byref(k), C.byref(s)))
    return np.uint64(k.value), np.uint64(s.value)


def raw_uint64(key64, stream64, start: int, count: int, device=None) -> np.ndarray:
    out = np.empty(max(int(count), 0), dtype=np.uint64)
    if out.size:
        N.check(N.lib.brm_raw_uint64(_dev(device), int(key64), int(stream64), int(start), out.size, N.ptr(out)))
    return out


def normals(key64, stream64, start: int, count: int, device=None) -> np.ndarray:
    out = np.empty(max(int(count), 0), dtype=np.float64)
    if out.size:
        N.check(N.lib.brm_normals(_dev(device), int(key64), int(stream64), int(start), out.size, N.ptr(out)))
    return out


def stopped_sums(mp, rp, start_values, m_start: int, n_paths: int, key64, stream64, draw_base: int = 0,
                 mode=None, device=None) -> tuple[float, float]:
    """(sum, sum of squares) of discounted stopped payoffs (_core.pyx:402-430)."""
    ctx = get_context(mp, rp, device, mode)
    st = N.f64(start_values)
    s, q = C.c_double(), C.c_double()
    N.check(N.lib.brm_stopped_sums(ctx.handle, N.ptr(st), int(m_start), int(n_paths), int(key64), int(stream64),
                                   int(draw_base), C.byref(s), C.byref(q)))
    return float(s.value), float(q.value)


def path_values(mp, rp, start_values, m_start: int, n_paths: int, key64, stream64, draw_base: int = 0,
                mode=None, device=None, normals_in=None, normals_base: int = 0):
    """Per-path discounted values and stop dates (0 = never exercised).

    ``normals_in`` switches the context to host-supplied normals for this
    call (north star fixed-input parity): draw i reads normals_in[i - base].
    """
    ctx = get_context(mp, rp, device, mode)
    st = N.f64(start_values)
    vals = np.empty(int(n_paths))
    stops = np.empty(int(n_paths), dtype=np.int32)
    if normals_in is not None:
        ctx.supply_normals(normals_in, normals_base)
    try:
        N.check(N.lib.brm_path_values(ctx.handle, N.ptr(st), int(m_start), int(n_paths), int(key64),
                                      int(stream64), int(draw_base), N.ptr(vals), N.ptr(stops)))
    finally:
        if normals_in is not None:
            ctx.supply_normals(None)
    return vals, stops


def decisions(mp, rp, states, m: int, mode=None, device=None, ctx=None) -> np.ndarray:
    """Exercise decisions of the rule for states[n, d] at date m (pricer.py:104-133)."""
    ctx = get_context(mp, rp, device, mode) if ctx is None else ctx
    st = N.f64(states).reshape(-1, int(mp.d))
    out = np.empty(st.shape[0], dtype=np.int32)
    N.check(N.lib.brm_decisions(ctx.handle, N.ptr(st), st.shape[0], int(m), N.ptr(out)))
    return out.astype(bool)


def iz_solve_batch(mp, rp, seeds, assets, m: int, n_inner: int, *, solver: str = "fixed_point",
                   epsilon: float = 0.01, max_iter: int = 100, avg_window: int = 5,
                   lo: float = 0.0, hi: float = 0.0, tol: float = 1e-4, keys=None, streams=None,
                   seed: int = 0, item_lo: int = 0, mode=None, device=None, ctx=None, out=None):
    """Solve n probes at date m; returns (levels, iterations, converged).

    ``ctx`` overrides the context of (mp, rp); ``seeds`` / ``assets`` may be
    device tensors and ``out`` a (levels f64, iterations i32, converged i32)
    triple of device tensors, which are then filled without a host round trip."""
    ctx = get_context(mp, rp, device, mode) if ctx is None else ctx
    d = int(mp.d)
    if isinstance(assets, np.ndarray) or not hasattr(assets, "data_ptr"):
        assets = np.ascontiguousarray(assets, dtype=np.int32)
        n = assets.size
    else:
        n = int(assets.shape[0])
    if d > 1:
        seeds = N.f64(seeds).reshape(n, d - 1) if not hasattr(seeds, "data_ptr") else seeds
    else:
        seeds = np.zeros((n, 0))
    if out is not None:
        levels, its, conv = out
    else:
        levels = np.empty(n)
        its = np.empty(n, dtype=np.int32)
        conv = np.empty(n, dtype=np.int32)
    kp = sp = None
    if keys is not None:
        kp = np.ascontiguousarray(keys, dtype=np.uint64)
        sp = np.ascontiguousarray(streams, dtype=np.uint64)
    solver_id = {"fixed_point": 0, "bisection": 1}[solver]
    N.check(N.lib.brm_iz_solve(ctx.handle, solver_id, N.ptr(seeds) if d > 1 else None, N.ptr(assets), n, int(m),
                               int(n_inner), float(epsilon), int(max_iter), int(avg_window), float(lo), float(hi),
                               float(tol), N.ptr(kp), N.ptr(sp), int(seed) & (2**64 - 1), int(item_lo),
                               N.ptr(levels), N.ptr(its), N.ptr(conv)))
    if out is not None:
        return levels, its, conv
    return levels, its, conv.astype(bool)


def iz_solve(mp, rp, seed_point, asset_index: int, m: int, n_inner: int, epsilon: float, max_iter: int,
             avg_window: int, key64, stream64, mode=None, device=None):
    """Fixed-point probe solve (_core.pyx:433-512): (level, iterations, converged)."""
    lv, it, cv = iz_solve_batch(mp, rp, np.asarray(seed_point, dtype=np.float64).reshape(1, -1), [asset_index], m,
                                n_inner, epsilon=epsilon, max_iter=max_iter, avg_window=avg_window,
                                keys=[int(key64)], streams=[int(stream64)], mode=mode, device=device)
    return float(lv[0]), int(it[0]), bool(cv[0])


def cmc_labels(mp, rp, points, m: int, n_label: int, keys, streams, draw_base: int, mode=None, device=None):
    """beta_i = payoff(x_i) - continuation (_core.pyx:515-550) on streams (keys[i], streams[i])."""
    ctx = get_context(mp, rp, device, mode)
    pts = N.f64(points).reshape(-1, int(mp.d))
    n = pts.shape[0]
    out = np.empty(n)
    kp = np.ascontiguousarray(keys, dtype=np.uint64)
    sp = np.ascontiguousarray(streams, dtype=np.uint64)
    N.check(N.lib.brm_cmc_labels(ctx.handle, N.ptr(pts), n, int(m), int(n_label), N.ptr(kp), N.ptr(sp), 0, 0,
                                 int(draw_base), N.ptr(out)))
    return out


def cmc_labels_keyed(mp, rp, points, m: int, n_label: int, seed: int, item_lo: int, draw_base: int,
                     out=None, mode=None, device=None):
    """Labels with streams StreamKey(seed, CMC_CALC, item_lo + i, m) derived on the device.

    ``points`` and ``out`` may be device tensors (no host round trip)."""
    ctx = get_context(mp, rp, device, mode)
    n = points.shape[0]
    if out is None:
        out = np.empty(n)
    pts = points if not isinstance(points, np.ndarray) else N.f64(points).reshape(n, int(mp.d))
    N.check(N.lib.brm_cmc_labels(ctx.handle, N.ptr(pts), n, int(m), int(n_label), None, None,
                                 int(seed) & (2**64 - 1), int(item_lo), int(draw_base), N.ptr(out)))
    return out


def sample_points(mp, rp, m: int, seed: int, item_lo: int, n: int, bridge=None, sampler: str = "bridge",
                  out=None, mode=None, device=None):
    """Training points on StreamKey(seed, CMC_CALC, item, m) (boundary_cmc.py:164-189)."""
    ctx = get_context(mp, rp, device, mode)
    if out is None:
        out = np.empty((int(n), int(mp.d)))
    mode_id = {"bridge": 0, "forward": 1}[sampler]
    b = N.f64(bridge) if bridge is not None else None
    N.check(N.lib.brm_sample_points(ctx.handle, mode_id, int(m), int(seed) & (2**64 - 1), int(item_lo), int(n),
                                    N.ptr(b), N.ptr(out)))
    return out


def price_blocks(mp, rp, n_paths: int, seed: int, block_lo: int = 0, block_hi: int | None = None, out=None,
                 mode=None, device=None):
    """Per-block (count, sum, sumsq) of PATH_BLOCK=4096-path blocks (pricer.py:154-164)."""
    ctx = get_context(mp, rp, device, mode)
    n_blocks = (int(n_paths) + 4095) // 4096
    block_hi = n_blocks if block_hi is None else int(block_hi)
    if out is None:
        out = np.empty((block_hi - int(block_lo), 3))
    N.check(N.lib.brm_price_blocks(ctx.handle, int(n_paths), int(seed) & (2**64 - 1), int(block_lo), block_hi,
                                   N.ptr(out)))
    return out


def fit_ensemble_arrays(xs, betas, rounds: int, mode=None, device=None, weights=None, single: bool = False,
                        stream=None):
    """Device AdaBoost (boosting.py:174-206) -> (feat, thr, pol, alpha, err, intercept) arrays.

    ``single`` runs one fit_stump search (boosting.py:126-171) with ``weights``."""
    from .context import resolve_mode
    xs = xs if not isinstance(xs, np.ndarray) else N.f64(xs)
    betas = betas if not isinstance(betas, np.ndarray) else N.f64(betas)
    w = None if weights is None else (weights if not isinstance(weights, np.ndarray) else N.f64(weights))
    n, F = int(xs.shape[0]), int(xs.shape[1])
    r = 1 if single else int(rounds)
    feat = np.empty(r, dtype=np.int32)
    thr, pol, alpha, err = np.empty(r), np.empty(r), np.empty(r), np.empty(r)
    count, icept = C.c_int32(), C.c_double()
    N.check(N.lib.brm_fit_ensemble(_dev(device), resolve_mode(mode), N.FIT_SINGLE_STUMP if single else 0,
                                   N.stream_handle(stream), N.ptr(xs), N.ptr(betas), N.ptr(w), n, F, r,
                                   N.ptr(feat), N.ptr(thr), N.ptr(pol), N.ptr(alpha), N.ptr(err),
                                   C.addressof(count), C.addressof(icept), None))
    c = count.value
    return feat[:c], thr[:c], pol[:c], alpha[:c], err[:c], float(icept.value)


def fit_ensemble_device(xs, betas, rounds: int, out, mode=None, device=None, stream=None) -> None:
    """Device AdaBoost with device-resident results and no host synchronisation
    (BRM_FIT_DEVICE_RESULT): ``out`` holds device tensors feat[int32, rounds],
    thr/pol/alpha/err[f64, rounds], count[int32, 1], intercept[f64, 1] and
    optionally n_pos[int32, 1] (positive labels)."""
    from .context import resolve_mode
    n, F = int(xs.shape[0]), int(xs.shape[1])
    N.check(N.lib.brm_fit_ensemble(_dev(device), resolve_mode(mode), N.FIT_DEVICE_RESULT, N.stream_handle(stream),
                                   N.ptr(xs), N.ptr(betas), None, n, F, int(rounds), N.ptr(out["feat"]),
                                   N.ptr(out["thr"]), N.ptr(out["pol"]), N.ptr(out["alpha"]), N.ptr(out["err"]),
                                   N.ptr(out["count"]), N.ptr(out["intercept"]), N.ptr(out.get("n_pos"))))


def lstsq(design, levels, k_coords: int, device=None, stream=None):
    """Device least squares with the cross-term-free fallback (boundary_iz.py:250-276)."""
    design = N.f64(design)
    levels = N.f64(levels)
    n, nb = design.shape
    out = np.empty(nb)
    deficient = C.c_int32()
    N.check(N.lib.brm_lstsq(_dev(device), N.stream_handle(stream), N.ptr(design), N.ptr(levels), n, nb,
                            int(k_coords), N.ptr(out), C.byref(deficient)))
    return out, bool(deficient.value)


def cmc_calc(mp, rp, m: int, seed: int, item_lo: int, n: int, n_label: int, bridge=None, sampler: str = "bridge",
             out_features=None, out_beta=None, mode=None, device=None, ctx=None):
    """Sample, featurise and label training points [item_lo, item_lo+n) of date m on the device
    (under ``ctx``'s rule when given, else the context of (mp, rp))."""
    ctx = get_context(mp, rp, device, mode) if ctx is None else ctx
    d = int(mp.d)
    F = d + 1 if d > 1 else 1
    if out_features is None:
        out_features = np.empty((int(n), F))
    if out_beta is None:
        out_beta = np.empty(int(n))
    b = N.f64(bridge) if bridge is not None else None
    N.check(N.lib.brm_cmc_calc(ctx.handle, {"bridge": 0, "forward": 1}[sampler], int(m), int(seed) & (2**64 - 1),
                               int(item_lo), int(n), int(n_label), N.ptr(b), N.ptr(out_features), N.ptr(out_beta)))
    return out_features, out_beta
