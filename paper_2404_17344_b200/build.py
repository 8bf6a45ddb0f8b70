"""Build libaddkern_b200.so in-tree with nvcc for sm_100a.

The library is a plain C-ABI shared object (include/addkern_b200.h): no torch
types cross the boundary, Python binds it with ctypes (_native.py).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libaddkern_b200.so"
SOURCES = ["ak_lib.cu", "ak_probe.cu", "ak_dense.cu", "ak_cg.cu"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


#: checked variant (-DAK_CHECKED: device invariant traps, guard bands + NaN poisoning of
#: the library's buffers, verified after every entry point) -- test infrastructure,
#: loaded only by tests/test_gpu_checked.py through AK_LIB_PATH
CHECKED_LIB = PKG / "libaddkern_b200_checked.so"


def _stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "addkern_b200.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=()) -> Path:
    """Compile the library (out/defines: variant builds for tuning experiments)."""
    target = Path(out) if out else LIB
    if out is None and not force and not _stale():
        return LIB
    cuda_home = Path(_nvcc()).resolve().parent.parent
    cmd = [
        _nvcc(), "-O3", "-std=c++17", "-lineinfo",
        "-gencode", "arch=compute_100a,code=sm_100a",
        "--shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=default",
        "-Xptxas", "-v" if verbose else "-O3",
        "-I", str(ROOT / "include"),
        *[str(CSRC / s) for s in SOURCES],
        "-L", str(cuda_home / "lib64"), "-lcufft",
        "-Xlinker", f"-rpath,{cuda_home / 'lib64'}",
        *[f"-D{d}" for d in defines],
        "-o", str(target) + ".tmp",
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode})")
    os.replace(str(target) + ".tmp", target)
    return target


def build_checked(force: bool = False) -> Path:
    """The checked variant (see CHECKED_LIB)."""
    if not force and not _stale(CHECKED_LIB):
        return CHECKED_LIB
    return build(force=True, out=CHECKED_LIB, defines=("AK_CHECKED",))


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
