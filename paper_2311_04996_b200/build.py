"""Build ``libctcwfst_b200.so`` in-tree with nvcc for sm_100a.

    python -m paper_2311_04996_b200.build

One nvcc invocation over csrc/*.cu -> a position-independent shared object
(static cudart) loaded through ctypes by ``_lib.py``. ``-lineinfo`` keeps the
ncu source view mapped to csrc/.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
SRC = sorted((PKG / "csrc").glob("*.cu")) + sorted((PKG / "csrc").glob("*.cpp"))
HDRS = sorted((PKG / "csrc").glob("*.h")) + sorted((PKG.parent / "include").glob("*.h"))
OUT = PKG / "libctcwfst_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SRC + HDRS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return OUT
    cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
           "-o", str(OUT), *os.environ.get("CTW_NVCC_FLAGS", "").split(), *map(str, SRC)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv))
