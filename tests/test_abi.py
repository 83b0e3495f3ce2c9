"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every function include/ctcwfst_b200.h declares; host-side types mirror the
reference's contract."""

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared():
    txt = (ROOT / "include" / "ctcwfst_b200.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ctw_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2311_04996_b200 import _lib

    lib = C.CDLL(str(_lib.lib_path()))
    names = declared()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTED_SYMBOLS) <= set(names)


def test_abi_version_and_status_codes():
    from paper_2311_04996_b200 import _lib, kernels

    L = _lib.load(require_gpu=False)
    assert L.ctw_abi_version() == 1
    assert (kernels.OK, kernels.ERR_EPS_ITERS, kernels.ERR_NO_SURVIVORS) == (0, 1, 2)
    h = (ROOT / "include" / "ctcwfst_b200.h").read_text()
    assert "#define CTW_ABI_VERSION 1" in h


def test_struct_layouts_match_header():
    from paper_2311_04996_b200 import _lib

    assert C.sizeof(_lib.CtwConfig) == 40
    assert C.sizeof(_lib.CtwExport) == 8 * 16


def test_product_path_has_no_cpu_fallback(monkeypatch, tmp_path):
    """Without the native library the package must fail loudly."""
    from paper_2311_04996_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setenv("CTW_B200_LIB", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()


def test_product_does_not_import_oracle():
    pkg = ROOT / "paper_2311_04996_b200"
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src, flags=re.M), p
        assert "/root/reference" not in src, p
