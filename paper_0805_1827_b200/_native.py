"""ctypes binding of libbermuda_b200.so (include/bermuda_b200.h).

The library is the only compute path of this package: importing this module
loads it and raises if it is missing, and every call checks the returned
status and raises the exception the reference raises in the same situation
(``ValueError`` for bad arguments, ``MemoryError`` for allocation failures).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_LIB_PATH = Path(os.environ.get("BRM_LIB_PATH") or Path(__file__).resolve().parent / "lib" / "libbermuda_b200.so")

BRM_OK, BRM_EINVAL, BRM_ENOMEM, BRM_ECUDA, BRM_ENODEV = range(5)
MODE_PARITY, MODE_FAST = 0, 1
FIT_SINGLE_STUMP = 1
FIT_DEVICE_RESULT = 2
ABI_VERSION = 3

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_up = C.POINTER(C.c_uint64)


class MarketDesc(C.Structure):
    _fields_ = [("d", C.c_int32), ("n_dates", C.c_int32), ("payoff_kind", C.c_int32), ("strike", C.c_double),
                ("step_mu", C.c_void_p), ("step_vol", C.c_void_p), ("chol", C.c_void_p),
                ("disc_steps", C.c_void_p), ("s0", C.c_void_p)]


class RuleDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("call_like", C.c_int32), ("imm_date", C.c_int32),
                ("nbasis", C.c_int32), ("iz_space", C.c_int32),
                ("iz_coeffs", C.c_void_p), ("iz_lo", C.c_void_p), ("iz_hi", C.c_void_p),
                ("n_stumps", C.c_int32),
                ("cmc_starts", C.c_void_p), ("cmc_counts", C.c_void_p), ("cmc_feat", C.c_void_p),
                ("cmc_thr", C.c_void_p), ("cmc_pol", C.c_void_p), ("cmc_alpha", C.c_void_p),
                ("cmc_intercept", C.c_void_p)]


# (name, restype-is-status, argtypes) -- one row per symbol of bermuda_b200.h
_SIGNATURES = {
    "brm_abi_version": (C.c_int, []),
    "brm_last_error": (C.c_char_p, []),
    "brm_device_count": (C.c_int, [_ip]),
    "brm_ctx_create": (C.c_int, [C.POINTER(MarketDesc), C.POINTER(RuleDesc), C.c_int32, C.c_int32,
                                 C.POINTER(C.c_void_p)]),
    "brm_ctx_destroy": (C.c_int, [C.c_void_p]),
    "brm_ctx_create_cmc": (C.c_int, [C.POINTER(MarketDesc), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(C.c_void_p)]),
    "brm_ctx_set_ensemble": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p]),
    "brm_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "brm_ctx_supply_normals": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64]),
    "brm_derive_words": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, _up, _up]),
    "brm_raw_uint64": (C.c_int, [C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]),
    "brm_normals": (C.c_int, [C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]),
    "brm_selftest_math": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "brm_stopped_sums": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_uint64,
                                   C.c_uint64, C.c_void_p, C.c_void_p]),
    "brm_path_values": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_uint64,
                                  C.c_uint64, C.c_void_p, C.c_void_p]),
    "brm_decisions": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    "brm_price_blocks": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, C.c_void_p]),
    "brm_cmc_labels": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                 C.c_void_p, C.c_uint64, C.c_int64, C.c_uint64, C.c_void_p]),
    "brm_sample_points": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, C.c_int64, C.c_int64,
                                    C.c_void_p, C.c_void_p]),
    "brm_iz_solve": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                               C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                               C.c_void_p, C.c_void_p, C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p,
                               C.c_void_p]),
    "brm_cmc_calc": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_int32,
                               C.c_void_p, C.c_void_p, C.c_void_p]),
    "brm_fit_presort": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32]),
    "brm_ctx_set_presort": (C.c_int, [C.c_void_p, C.c_int32]),
    "brm_fit_ensemble": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "brm_profile_enable": (C.c_int, [C.c_int32]),
    "brm_profile_reset": (C.c_int, []),
    "brm_profile_read": (C.c_int, [C.c_int32, _dp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "brm_transfer_read": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "brm_lstsq": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                            C.c_void_p, _ip]),
    "brm_iz_fit": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                             C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
}


def _load() -> C.CDLL:
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -m paper_0805_1827_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.brm_abi_version() != ABI_VERSION:
        raise ImportError("libbermuda_b200.so ABI version mismatch")
    return lib


lib = _load()
SYMBOLS = tuple(_SIGNATURES)


class EngineError(RuntimeError):
    """CUDA-side failure (launch error, no device)."""


def check(status: int) -> None:
    if status == BRM_OK:
        return
    msg = (lib.brm_last_error() or b"").decode(errors="replace")
    if status == BRM_EINVAL:
        raise ValueError(msg)
    if status == BRM_ENOMEM:
        raise MemoryError(msg)
    raise EngineError(f"libbermuda_b200: {msg}")


def ptr(a) -> C.c_void_p | None:
    """Address of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: torch's default stream has handle 0


def stream_handle(stream) -> C.c_void_p | None:
    """cudaStream_t of a torch.cuda.Stream / raw handle.  None -> library default;
    a stream whose handle is 0 (torch's default stream) -> cudaStreamLegacy."""
    if stream is None:
        return None
    raw = getattr(stream, "cuda_stream", stream)
    return C.c_void_p(raw if raw else CUDA_STREAM_LEGACY)


def device_count() -> int:
    n = C.c_int32(0)
    st = lib.brm_device_count(C.byref(n))
    return int(n.value) if st == BRM_OK else 0


PROF_KINDS = ("walk", "iz", "boost", "sample", "finish", "lstsq", "rng", "decisions", "aux")


def profile_read() -> dict:
    """{family: (device ms, launches, executed path-steps)} since the last reset."""
    out = {}
    for i, name in enumerate(PROF_KINDS):
        ms, nl, ns = C.c_double(), C.c_uint64(), C.c_uint64()
        check(lib.brm_profile_read(i, C.byref(ms), C.byref(nl), C.byref(ns)))
        out[name] = (ms.value, int(nl.value), int(ns.value))
    return out


def transfer_read() -> tuple[int, int]:
    """(host->device, device->host) bytes staged by the library since the last reset."""
    a, b = C.c_uint64(), C.c_uint64()
    check(lib.brm_transfer_read(C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)


def profile_enable(on: bool = True) -> None:
    check(lib.brm_profile_enable(1 if on else 0))


def profile_reset() -> None:
    check(lib.brm_profile_reset())
