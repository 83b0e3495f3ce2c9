"""Build recipe for ``oracle/_ref``: the UNMODIFIED reference package
(``/root/reference/pkg/src/ctcwfst``) compiled into CPython extension modules.

TEST / BASELINE INFRASTRUCTURE ONLY. Nothing under ``oracle/`` is on the
product path: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may load it.

Why compile instead of import: ``/root/reference`` does not exist on the GPU
box, and reference sources may not be copied into this repository. Cython
compiles every reference module where it lies (the ``.py`` modules as plain
Python-semantics extension modules, ``_kernel.pyx`` exactly as the
reference's own ``pkg/setup.py:12-22`` does: ``-O3``, no fast-math). Only the
binaries land in ``oracle/_ref/ctcwfst/`` (git-ignored, shipped to the GPU box
with the snapshot); the generated C goes to a scratch dir under /tmp.

Usage: ``python oracle/build_ref.py`` (no-op when /root/reference is absent
and the binaries already exist).
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from pathlib import Path

REF_PKG = Path("/root/reference/pkg/src/ctcwfst")
OUT = Path(__file__).resolve().parent / "_ref" / "ctcwfst"
SCRATCH = Path("/tmp/ctw_ref_build")


def _ext_suffix() -> str:
    return sysconfig.get_config_var("EXT_SUFFIX")


def built() -> bool:
    return (OUT / f"_kernel{_ext_suffix()}").exists() and (OUT / f"decoder{_ext_suffix()}").exists()


def build(verbose: bool = False) -> bool:
    """Compile every reference module; returns False when the reference tree
    is not present (e.g. on the GPU box) so callers can skip."""
    if not REF_PKG.is_dir():
        return built()
    import numpy as np

    OUT.mkdir(parents=True, exist_ok=True)
    SCRATCH.mkdir(parents=True, exist_ok=True)
    inc = [sysconfig.get_paths()["include"], np.get_include()]
    suffix = _ext_suffix()
    sources = sorted(REF_PKG.glob("*.py")) + [REF_PKG / "_kernel.pyx"]

    def one(src: Path) -> None:
        mod = src.stem
        so = OUT / f"{mod}{suffix}"
        if so.exists() and so.stat().st_mtime >= src.stat().st_mtime:
            return
        c_file = SCRATCH / f"{mod}.c"
        # .py modules keep plain Python semantics: annotations are NOT turned
        # into C type checks (annotation_typing=False). The .pyx kernel keeps
        # its own cdef typing, as in the reference's setup.py.
        directives = [] if src.suffix == ".pyx" else ["-X", "annotation_typing=False", "-X", "binding=True"]
        cmd = [
            sys.executable, "-m", "cython", "-3", *directives, "--module-name", f"ctcwfst.{mod}",
            "-o", str(c_file), str(src),
        ]
        subprocess.run(cmd, check=True, capture_output=not verbose)
        cc = ["gcc", "-O3" if src.suffix == ".pyx" else "-O1", "-shared", "-fPIC",
              "-fno-strict-aliasing", *[f"-I{p}" for p in inc], str(c_file), "-o", str(so)]
        subprocess.run(cc, check=True, capture_output=not verbose)

    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as pool:
        list(pool.map(one, sources))
    # package marker so `import ctcwfst` resolves to the compiled __init__
    return built()


if __name__ == "__main__":
    ok = build(verbose="-v" in sys.argv)
    print("oracle/_ref built" if ok else "oracle/_ref unavailable")
    sys.exit(0 if ok else 1)
