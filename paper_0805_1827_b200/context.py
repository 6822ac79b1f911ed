"""Device-resident contexts for (MarketPack, RulePack) pairs.

Replaces the reference's ``_ctx`` cache (core_backend.py:23-33), which pins
numpy buffers for the Cython walker: here a context is a device image of the
two packs in HBM, created once per pack pair (cached by pack identity, like
the reference) and per (device, precision mode).  Packs may be this
package's or the reference's own objects (duck-typed on the field names).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

from . import _native as N

__all__ = ["Context", "get_context", "default_mode", "default_device", "MODES"]

MODES = {"parity": N.MODE_PARITY, "fast": N.MODE_FAST}


def default_mode() -> int:
    """BERMUDA_B200_MODE=parity|fast (parity by default)."""
    name = os.environ.get("BERMUDA_B200_MODE", "parity").lower()
    if name not in MODES:
        raise ValueError(f"unknown BERMUDA_B200_MODE {name!r} (expected 'parity' or 'fast')")
    return MODES[name]


def resolve_mode(mode) -> int:
    if mode is None:
        return default_mode()
    if isinstance(mode, str):
        if mode not in MODES:
            raise ValueError(f"unknown mode {mode!r} (expected 'parity' or 'fast')")
        return MODES[mode]
    return int(mode)


def default_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # torch is plumbing only; the engine does not need it
        pass
    return 0


class Context:
    """One brm_ctx: market + rule image on one device in one precision mode."""

    def __init__(self, mp, rp, device: int | None = None, mode=None, capacity: int | None = None):
        self.device = default_device() if device is None else int(device)
        self.mode = resolve_mode(mode)
        self.d = int(mp.d)
        self.n_dates = int(mp.n_dates)
        self.strike = float(mp.strike)
        self.payoff_kind = int(mp.payoff_kind)
        self.call_like = int(rp.call_like)
        keep = []

        def arr(x, dt=np.float64):
            a = np.ascontiguousarray(x, dtype=dt)
            keep.append(a)
            return a.ctypes.data if a.size else None

        md = N.MarketDesc(self.d, self.n_dates, self.payoff_kind, self.strike,
                          arr(mp.step_mu), arr(mp.step_vol), arr(mp.chol), arr(mp.disc_steps), arr(mp.s0))
        coeffs = np.ascontiguousarray(rp.iz_coeffs, dtype=np.float64)
        nbasis = int(coeffs.shape[-1]) if coeffs.ndim == 3 else 1
        feat = np.ascontiguousarray(rp.cmc_feat, dtype=np.int32)
        rd = N.RuleDesc(int(rp.kind), self.call_like, int(rp.imm_date), nbasis,
                        int(getattr(rp, "iz_space", 0)),
                        arr(coeffs), arr(rp.iz_lo), arr(rp.iz_hi), int(feat.size),
                        arr(rp.cmc_starts, np.int32), arr(rp.cmc_counts, np.int32), arr(feat, np.int32),
                        arr(rp.cmc_thr), arr(rp.cmc_pol), arr(rp.cmc_alpha), arr(rp.cmc_intercept))
        handle = C.c_void_p()
        if capacity is not None:
            # slotted CMC image, every date empty; dates are filled on the device
            N.check(N.lib.brm_ctx_create_cmc(C.byref(md), self.call_like, int(capacity), self.device, self.mode,
                                             C.byref(handle)))
        else:
            N.check(N.lib.brm_ctx_create(C.byref(md), C.byref(rd), self.device, self.mode, C.byref(handle)))
        self.handle = handle
        self._finalizer = weakref.finalize(self, N.lib.brm_ctx_destroy, handle)
        self._normals = None

    @classmethod
    def cmc_slots(cls, mp, call_like: bool, capacity: int, device: int | None = None, mode=None) -> "Context":
        """Device-resident CMC rule image (brm_ctx_create_cmc): room for
        ``capacity`` stumps per date, filled by :meth:`set_ensemble`."""
        from .packs import RulePack
        return cls(mp, RulePack.european(call_like), device, mode, capacity=capacity)

    def set_presort(self, on: bool) -> None:
        """brm_cmc_calc sorts the sampled points' feature columns on a side stream beside the label
        walk, for the fit_ensemble_device call on the same feature tensor that follows."""
        N.check(N.lib.brm_ctx_set_presort(self.handle, 1 if on else 0))

    def set_ensemble(self, m: int, feat, thr, pol, alpha, count, intercept) -> None:
        """Write date m's ensemble (device tensors sized [capacity], count and
        intercept as 1-element tensors) into the image, on the context's stream."""
        N.check(N.lib.brm_ctx_set_ensemble(self.handle, int(m), N.ptr(feat), N.ptr(thr), N.ptr(pol), N.ptr(alpha),
                                           N.ptr(count), N.ptr(intercept)))

    def iz_fit(self, m: int, design, J: int, nb: int, k_coords: int, levels, n_fits: int, log_space: bool,
               out_coeffs=None, out_rank=None) -> None:
        """Fit date m's boundary surface(s) on the device into this image
        (brm_iz_fit): no host round trip when the arrays are device tensors."""
        N.check(N.lib.brm_iz_fit(self.handle, int(m), N.ptr(design), int(J), int(nb), int(k_coords), N.ptr(levels),
                                 int(n_fits), 1 if log_space else 0, N.ptr(out_coeffs), N.ptr(out_rank)))

    def close(self) -> None:
        self._finalizer()

    def set_stream(self, stream) -> None:
        """Launch on a caller stream (a torch.cuda.Stream, raw handle, or None)."""
        N.check(N.lib.brm_ctx_set_stream(self.handle, N.stream_handle(stream)))

    def supply_normals(self, normals, base: int = 0) -> None:
        """Fixed-input mode: draw i of every stream reads normals[i - base]."""
        if normals is None:
            N.check(N.lib.brm_ctx_supply_normals(self.handle, None, 0, 0))
            self._normals = None
            return
        a = N.f64(normals).ravel()
        N.check(N.lib.brm_ctx_supply_normals(self.handle, N.ptr(a), int(base), int(a.size)))
        self._normals = a


_cache_lock = threading.Lock()
_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def get_context(mp, rp, device: int | None = None, mode=None) -> Context:
    """Context for a pack pair, cached by pack identity like the reference."""
    device = default_device() if device is None else int(device)
    mode = resolve_mode(mode)
    with _cache_lock:
        by_rule = _cache.setdefault(mp, weakref.WeakKeyDictionary())
        by_key = by_rule.setdefault(rp, {})
        ctx = by_key.get((device, mode))
        if ctx is None:
            ctx = Context(mp, rp, device, mode)
            by_key[(device, mode)] = ctx
        return ctx
