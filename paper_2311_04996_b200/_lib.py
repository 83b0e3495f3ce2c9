"""ctypes binding of ``libctcwfst_b200.so`` (the C-ABI in include/ctcwfst_b200.h).

The shared library is built in-tree by ``build.py`` (nvcc, sm_100a). There is
no CPU fallback: if the library or a CUDA device is missing, every decode
entry point raises ``RuntimeError`` naming the cause.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libctcwfst_b200.so"

OK, ERR_EPS_ITERS, ERR_NO_SURVIVORS, ERR_OOM = 0, 1, 2, 3

P = C.c_void_p
I32, I64, F64 = C.c_int32, C.c_int64, C.c_double


class CtwConfig(C.Structure):
    _fields_ = [("beam", F64), ("max_active", I64), ("acoustic_scale", F64),
                ("relax_eps", F64), ("max_ne_iters", I64)]


class CtwExport(C.Structure):
    _fields_ = [
        ("n_frames", I64), ("n_records", I64), ("n_olab", I64),
        ("counts", C.POINTER(I64)), ("rec_prev", C.POINTER(I64)), ("rec_state", C.POINTER(I32)),
        ("rec_cost", C.POINTER(F64)), ("rec_olab_off", C.POINTER(I64)),
        ("rec_olab_pool", C.POINTER(I32)),
        ("n_tok", I64), ("tok_state", C.POINTER(I32)), ("tok_cost", C.POINTER(F64)),
        ("tok_bp", C.POINTER(I64)), ("tok_chain_off", C.POINTER(I64)),
        ("tok_chain_pool", C.POINTER(I32)), ("n_chain", I64),
    ]


class CtwLattice(C.Structure):
    """ctw_lattice (include/ctcwfst_b200.h)."""
    _fields_ = [
        ("status", I32), ("final_mode", I32), ("frame_count", I32), ("best", F64), ("lattice_beam", F64),
        ("n_seeds", I64), ("seed_state", C.POINTER(I32)), ("seed_cost", C.POINTER(F64)),
        ("seed_lab_off", C.POINTER(I64)), ("seed_lab", C.POINTER(I32)),
        ("n_arcs", I64), ("arc_src", C.POINTER(I32)), ("arc_dst", C.POINTER(I32)),
        ("arc_frame", C.POINTER(I32)), ("arc_src_state", C.POINTER(I32)), ("arc_dst_state", C.POINTER(I32)),
        ("arc_w", C.POINTER(F64)),
        ("arc_dst_final", C.POINTER(F64)), ("arc_lab_off", C.POINTER(I64)), ("arc_lab", C.POINTER(I32)),
        ("closure_items", I64), ("closure_pruned", I64),
    ]


_SIGS = {
    "ctw_abi_version": (I32, []),
    "ctw_last_error": (C.c_char_p, []),
    "ctw_device_count": (I32, []),
    "ctw_graph_create": (I32, [P] * 7 + [I64, I64, I64, I32, C.POINTER(P)]),
    "ctw_graph_load": (I32, [C.c_char_p, I32, C.POINTER(P)]),
    "ctw_graph_destroy": (None, [P]),
    "ctw_graph_info": (I32, [P] + [C.POINTER(I64)] * 5),
    "ctw_lanes_create": (I32, [P, I32, C.POINTER(CtwConfig), P, C.POINTER(P)]),
    "ctw_lanes_destroy": (None, [P]),
    "ctw_lanes_reserve": (I32, [P, I32]),
    "ctw_lane_reset": (I32, [P, P, I32, P, P, P]),
    "ctw_lane_set_boost": (I32, [P, I32, P, I64]),
    "ctw_lane_set_fsa": (I32, [P, I32, I32, P, P]),
    "ctw_advance": (I32, [P, P, I32, P, I32, I32, P, P, I32, P, P]),
    "ctw_best_path": (I32, [P, P, I32, P, I64, P, P, P, P]),
    "ctw_advance_best": (I32, [P, P, I32, P, I32, I32, P, P, I32, P, P, P, I64, P, P, P, P]),
    "ctw_lane_compact": (I32, [P, P, I32, P]),
    "ctw_lanes_presize": (I32, [P, P, I32]),
    "ctw_lane_info": (I32, [P, I32, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]),
    "ctw_lane_capacity": (I32, [P, I32, P]),
    "ctw_lane_export": (I32, [P, I32, I64, I64, P, I64, C.POINTER(CtwExport)]),
    "ctw_export_free": (None, [C.POINTER(CtwExport)]),
    "ctw_lanes_stats": (I32, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(F64), C.POINTER(I64),
                              C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]),
    "ctw_lanes_reset_stats": (I32, [P]),
    "ctw_lanes_profile": (I32, [P, P]),
    "ctw_lanes_host_timing": (I32, [P, P]),
    "ctw_lanes_set_search": (I32, [P, I32]),
    "ctw_lanes_search_info": (I32, [P, P]),
    "ctw_lanes_graph_info": (I32, [P, P]),
    "ctw_lanes_stream": (P, [P]),
    "ctw_lane_lattice": (I32, [P, P, I32, P, I32, I32, P, I32, F64, P]),
    "ctw_lattice_free": (None, [C.POINTER(CtwLattice)]),
    "ctw_lattice_nbest": (I32, [C.POINTER(CtwLattice), I32, I64, P, I64, P, P, C.POINTER(I32), C.POINTER(I64)]),
    "ctw_lattice_nbest_phrases": (I32, [C.POINTER(CtwLattice), I32, P, P, P, P, P, I32, I64, P, I64, P, P,
                                        C.POINTER(I32), C.POINTER(I64)]),
    "ctw_advance_chunk_compat": (I32, [P] * 6 + [I64, I64] + [P] * 5 + [I64, P, I64, I64, F64, F64,
                                      I64, F64, I64, P, I64, I64, I32, C.POINTER(I64),
                                      C.POINTER(CtwExport)]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def lib_path() -> Path:
    return Path(os.environ.get("CTW_B200_LIB", LIB_PATH))


def load(require_gpu: bool = True):
    """Load the native library (once). Raises RuntimeError when it is missing
    or, with ``require_gpu``, when no CUDA device is visible."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not path.exists():
            raise RuntimeError(
                f"native library {path} is missing: run `python __graft_entry__.py build` "
                "(nvcc sm_100a); there is no CPU fallback")
        L = C.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.ctw_abi_version() != 1:
            raise RuntimeError("libctcwfst_b200 ABI mismatch")
        _lib = L
    if require_gpu and _lib.ctw_device_count() < 1:
        raise RuntimeError("no CUDA device visible: the B200 decoder has no CPU fallback")
    return _lib


def last_error() -> str:
    return (load(False).ctw_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str) -> int:
    if rc < 0:
        raise RuntimeError(f"{what} failed ({rc}): {last_error()}")
    return rc


def ptr(a) -> int | None:
    """Address of a numpy array's data (c_void_p arguments take the int:
    ~10x cheaper than ctypes.data_as on the per-chunk streaming path)."""
    if a is None:
        return None
    return a.ctypes.data


def take_export(e: CtwExport, free: bool = True) -> dict:
    """Copy an export struct into numpy arrays (and free the C arrays)."""

    def arr(p, n, dt):
        if n <= 0:
            return np.zeros(0, dtype=dt)
        return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)

    nr, nt = e.n_records, e.n_tok
    out = {
        "counts": arr(e.counts, e.n_frames, np.int64),
        "rec_prev": arr(e.rec_prev, nr, np.int64),
        "rec_state": arr(e.rec_state, nr, np.int32),
        "rec_cost": arr(e.rec_cost, nr, np.float64),
        "rec_olab_off": arr(e.rec_olab_off, nr + 1, np.int64) if e.rec_olab_off else np.zeros(1, np.int64),
        "rec_olab_pool": arr(e.rec_olab_pool, e.n_olab, np.int32),
        "tok_state": arr(e.tok_state, nt, np.int32),
        "tok_cost": arr(e.tok_cost, nt, np.float64),
        "tok_bp": arr(e.tok_bp, nt, np.int64),
        "tok_chain_off": arr(e.tok_chain_off, nt + 1, np.int64) if e.tok_chain_off else np.zeros(1, np.int64),
        "tok_chain_pool": arr(e.tok_chain_pool, e.n_chain, np.int32),
    }
    if free:
        load(False).ctw_export_free(C.byref(e))
    return out
