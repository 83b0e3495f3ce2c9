"""The reference's kernel plug-in seam, served by the GPU.

``advance_chunk`` has the exact positional contract of the reference frame
kernel (pkg/src/ctcwfst/_pykernel.py:28-48, _kernel.pyx:115-135): graph CSR
arrays, the active token set with backpointers and pending olabel chains, a
(frames, V) float64 log-likelihood matrix, the five decoder scalars, an
optional boost vector and the first record index; it returns
``(status, err_frame, counts, rec_prev, rec_state, rec_cost, rec_olab_off,
rec_olab_pool)``. It runs the sm_100a kernels through
``ctw_advance_chunk_compat`` so the reference's own tests can inject it:
``DecodeState(graph, config, kernel=kernels.advance_chunk)``.

There is no CPU fallback (the reference's ``python_advance_chunk`` and
``CTCWFST_PURE_PYTHON`` switch, kernels.py:14-31, do not exist here): without
the native library or a GPU every call raises RuntimeError.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

OK = _lib.OK
ERR_EPS_ITERS = _lib.ERR_EPS_ITERS
ERR_NO_SURVIVORS = _lib.ERR_NO_SURVIVORS

KERNEL_NAME = "cuda-sm_100a"


def compiled_available() -> bool:
    """True when the native library loads and a CUDA device is visible."""
    try:
        _lib.load()
    except (RuntimeError, OSError):
        return False
    return True


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def advance_chunk(off, eps_end, ilabel, olabel, weight, nextstate, act_state, act_cost, act_bp,
                  act_chain_off, act_chain_pool, loglik, acoustic_scale, beam, max_active, relax_eps,
                  max_ne_iters, boost, base, device: int = 0):
    L = _lib.load()
    g = [_c(off, np.int64), _c(eps_end, np.int64), _c(ilabel, np.int32), _c(olabel, np.int32),
         _c(weight, np.float64), _c(nextstate, np.int32)]
    act = [_c(act_state, np.int32), _c(act_cost, np.float64), _c(act_bp, np.int64),
           _c(act_chain_off, np.int64), _c(act_chain_pool, np.int32)]
    ll = _c(loglik, np.float64)
    if ll.ndim != 2:
        raise ValueError("loglik must be a (frames, tokens) matrix")
    bst = None if boost is None else _c(boost, np.float64)
    err = C.c_int64(-1)
    e = _lib.CtwExport()
    rc = L.ctw_advance_chunk_compat(
        *[_lib.ptr(a) for a in g], len(g[0]) - 1, len(g[2]), *[_lib.ptr(a) for a in act], len(act[0]),
        _lib.ptr(ll), ll.shape[0], ll.shape[1], float(acoustic_scale), float(beam), int(max_active),
        float(relax_eps), int(max_ne_iters), _lib.ptr(bst), 0 if bst is None else len(bst), int(base),
        int(device), C.byref(err), C.byref(e))
    if rc == _lib.ERR_OOM:
        raise MemoryError()
    _lib.check(rc, "advance_chunk")
    out = _lib.take_export(e)
    return (int(rc), int(err.value), out["counts"], out["rec_prev"], out["rec_state"], out["rec_cost"],
            out["rec_olab_off"], out["rec_olab_pool"])
