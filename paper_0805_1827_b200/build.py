"""Build libbermuda_b200.so in-tree with nvcc for sm_100a.

``python -m paper_0805_1827_b200.build [--ptxas-v]`` compiles every
``csrc/*.cu`` (in parallel) and links ``lib/libbermuda_b200.so``.  The
library is rebuilt only when a source or header is newer than it.
"""

from __future__ import annotations

import concurrent.futures
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIBDIR = PKG / "lib"
# BRM_LIB_OUT / BRM_NVCC_DEFS: build a variant library elsewhere (A/B timing of
# compile-time kernel options, loaded with BRM_LIB_PATH)
LIB = Path(os.environ["BRM_LIB_OUT"]) if os.environ.get("BRM_LIB_OUT") else LIBDIR / "libbermuda_b200.so"
OBJDIR = LIB.parent / "obj"
EXTRA_DEFS = os.environ.get("BRM_NVCC_DEFS", "").split()

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-I", str(INCLUDE), "-I", str(CSRC)]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA 12.9 toolkit is required to build libbermuda_b200.so")


def _stale() -> bool:
    if not LIB.exists():
        return True
    built = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]
    return any(p.stat().st_mtime > built for p in deps)


def _compile(src: Path, ptxas_v: bool) -> tuple[Path, str]:
    obj = OBJDIR / (src.stem + ".o")
    cmd = [_nvcc(), *ARCH, *FLAGS, *EXTRA_DEFS, "-c", str(src), "-o", str(obj)]
    if ptxas_v:
        cmd += ["-Xptxas", "-v"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
    return obj, res.stderr


def build(force: bool = False, ptxas_v: bool = False, verbose: bool = False) -> Path:
    """Compile and link the engine; returns the library path."""
    if not force and not ptxas_v and not _stale():
        return LIB
    OBJDIR.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    with concurrent.futures.ThreadPoolExecutor(max_workers=len(sources)) as ex:
        results = list(ex.map(lambda s: _compile(s, ptxas_v), sources))
    if verbose or ptxas_v:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), *ARCH, "-shared", "-o", str(tmp), *[str(o) for o, _ in results],
           "-Xcompiler", "-fPIC", "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, ptxas_v="--ptxas-v" in sys.argv, verbose=True)
    print(LIB)
