"""The C ABI library loads and exports every symbol include/bermuda_b200.h declares (CPU only)."""
import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "bermuda_b200.h"
LIB = ROOT / "paper_0805_1827_b200" / "lib" / "libbermuda_b200.so"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(brm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_backend_surface():
    names = declared_functions()
    # one entry point per reference kernel-backend function (core_backend.py:12-58)
    for needed in ("brm_raw_uint64", "brm_normals", "brm_stopped_sums", "brm_iz_solve", "brm_cmc_labels"):
        assert needed in names
    # phase-level entry points
    for needed in ("brm_price_blocks", "brm_cmc_calc", "brm_fit_ensemble", "brm_lstsq", "brm_sample_points"):
        assert needed in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(LIB))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_0805_1827_b200 import _native as N
    assert set(declared_functions()) == set(N.SYMBOLS)
    assert N.lib.brm_abi_version() == N.ABI_VERSION == 3


def test_errors_map_to_reference_exceptions_without_a_gpu():
    from paper_0805_1827_b200 import _native as N
    import pytest
    # invalid arguments are rejected before any device work (ValueError like _core.pyx:406-407)
    assert N.lib.brm_ctx_create(None, None, 0, 0, None) == N.BRM_EINVAL
    with pytest.raises(ValueError):
        N.check(N.BRM_EINVAL)
    with pytest.raises(MemoryError):
        N.check(N.BRM_ENOMEM)
