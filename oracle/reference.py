"""Import the unmodified reference package built into oracle/_ref (test infrastructure only).

oracle/build_ref.sh installs /root/reference/pkg there (Cython backend
included) in the build container; the directory travels with the repo
snapshot to the GPU box.  Importing this module raises ImportError when the
build is absent, so tests that need the live reference skip cleanly.
"""
from __future__ import annotations

import importlib
import sys
from pathlib import Path

REF_DIR = Path(__file__).resolve().parent / "_ref"

if not (REF_DIR / "bermuda" / "__init__.py").exists():
    raise ImportError(f"reference build missing at {REF_DIR} (run oracle/build_ref.sh)")


def bermuda():
    """The reference package module (``bermuda``) from oracle/_ref."""
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    mod = importlib.import_module("bermuda")
    from bermuda._kernels import available_backends
    if "cython" not in available_backends():
        raise ImportError("reference built without its Cython walker")
    return mod
