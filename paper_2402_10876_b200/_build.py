"""In-tree build of the sm_100a extension ``_lib/libtwgemm.so``.

One explicit nvcc invocation (``-gencode arch=compute_100a,code=sm_100a``;
plain ``-arch=sm_100a`` makes ptxas target sm_100 and reject tcgen05).  The
library is plain C ABI (include/tw_gemm.h), so it carries no torch types and
is loaded with ctypes.  Rebuilds only when a source is newer than the .so.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libtwgemm.so"
SOURCES = ["tw_gemm.cu", "tw_aux.cu", "tw_capi.cu"]
HEADERS = ["sm100_ptx.cuh", "tw_kernels.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared", "-cudart", "static",
    "--expt-relaxed-constexpr",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise FileNotFoundError("nvcc not found (set NVCC or put it on PATH)")


def _stale() -> bool:
    if not LIB.exists():
        return True
    built = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "tw_gemm.h", Path(__file__)]
    return any(d.stat().st_mtime > built for d in deps if d.exists())


def build_native(force: bool = False, verbose: bool = False) -> Path:
    """Compile libtwgemm.so in-tree (no-op when up to date)."""
    if not force and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    extra = os.environ.get("TW_NVCC_EXTRA", "").split()
    cmd = [nvcc_path(), *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"),
           *[str(CSRC / s) for s in SOURCES], "-o", str(tmp)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import sys
    print(build_native(force="--force" in sys.argv, verbose="-v" in sys.argv))
