"""Python face of the CPU oracle (``oracle/ctw_oracle.c``).

TEST / BASELINE INFRASTRUCTURE ONLY -- never imported by the product package.
Allowed importers: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs.

It restates, on top of the C frame kernel, the channel bookkeeping of the
reference (``/root/reference/pkg/src/ctcwfst/decoder.py``):

* ``advance_chunk``  -- same 19-argument / 8-tuple contract as
  ``_pykernel.py:28-248`` (so it can be injected as ``kernel=``).
* ``OracleChannel``  -- ``DecodeState`` semantics: seeding (decoder.py:173-229),
  chunk commit / atomic failure (decoder.py:264-341), ``best_path``
  (decoder.py:377-415) and ``history_records`` (decoder.py:251-260).
* ``decode_batch``   -- decoder.py:436-463 (thread pool; the C kernel releases
  the GIL because ctypes drops it around foreign calls).

Parity status: pinned. tests/test_oracle.py checks it against
``tests/golden/*.npz`` (generated from the reference by
``tests/golden/make_golden.py``) and against the compiled reference in
``oracle/_ref`` when that is built.
"""

from __future__ import annotations

import bisect
import ctypes as C
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

OK, ERR_EPS_ITERS, ERR_NO_SURVIVORS, ERR_OOM = 0, 1, 2, 3
_MAX_ACTIVE_CAP = 2**60


def build_lib(force: bool = False) -> Path:
    src = HERE / "ctw_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
             str(src), "-o", str(LIB_PATH), "-lm"],
            check=True,
        )
    return LIB_PATH


class _Result(C.Structure):
    _fields_ = [
        ("status", C.c_int64), ("err_frame", C.c_int64), ("n_frames", C.c_int64),
        ("n_records", C.c_int64), ("n_olab", C.c_int64),
        ("counts", C.POINTER(C.c_int64)), ("rec_prev", C.POINTER(C.c_int64)),
        ("rec_state", C.POINTER(C.c_int32)), ("rec_cost", C.POINTER(C.c_double)),
        ("rec_olab_off", C.POINTER(C.c_int64)), ("rec_olab_pool", C.POINTER(C.c_int32)),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build_lib()
        L = C.CDLL(str(LIB_PATH))
        P = C.c_void_p
        L.ctwo_advance_chunk.restype = C.c_int64
        L.ctwo_advance_chunk.argtypes = [P] * 6 + [C.c_int64] + [P] * 5 + [C.c_int64, P, C.c_int64,
                                          C.c_int64, C.c_double, C.c_double, C.c_int64, C.c_double,
                                          C.c_int64, P, C.c_int64, C.POINTER(_Result)]
        L.ctwo_seed.restype = C.c_int64
        L.ctwo_seed.argtypes = [P] * 5 + [C.c_int64, C.c_int64, C.c_double, C.c_int64, P,
                                          C.POINTER(_Result)]
        L.ctwo_result_free.argtypes = [C.POINTER(_Result)]
        L.ctwo_best.restype = C.c_int64
        L.ctwo_best.argtypes = [P, P, C.c_int64, P, C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _take(r: _Result):
    nf, nr, no = r.n_frames, r.n_records, r.n_olab

    def arr(ptr, n, dt):
        if n == 0:
            return np.zeros(0, dtype=dt)
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)

    out = (
        int(r.status), int(r.err_frame),
        arr(r.counts, nf, np.int64), arr(r.rec_prev, nr, np.int64),
        arr(r.rec_state, nr, np.int32), arr(r.rec_cost, nr, np.float64),
        arr(r.rec_olab_off, nr + 1, np.int64), arr(r.rec_olab_pool, no, np.int32),
    )
    lib().ctwo_result_free(C.byref(r))
    return out


def advance_chunk(off, eps_end, ilabel, olabel, weight, nextstate, act_state, act_cost, act_bp,
                  act_chain_off, act_chain_pool, loglik, acoustic_scale, beam, max_active,
                  relax_eps, max_ne_iters, boost, base):
    """Drop-in for ``_pykernel.advance_chunk`` (same arguments, same 8-tuple)."""
    arrs = [_c(off, np.int64), _c(eps_end, np.int64), _c(ilabel, np.int32), _c(olabel, np.int32),
            _c(weight, np.float64), _c(nextstate, np.int32), _c(act_state, np.int32),
            _c(act_cost, np.float64), _c(act_bp, np.int64), _c(act_chain_off, np.int64),
            _c(act_chain_pool, np.int32)]
    ll = _c(loglik, np.float64)
    bst = None if boost is None else _c(boost, np.float64)
    r = _Result()
    status = lib().ctwo_advance_chunk(
        *[_p(a) for a in arrs[:6]], len(arrs[0]) - 1, *[_p(a) for a in arrs[6:]], len(arrs[6]),
        _p(ll), ll.shape[0], ll.shape[1] if ll.ndim == 2 else 0, float(acoustic_scale), float(beam),
        int(min(max_active, _MAX_ACTIVE_CAP)), float(relax_eps), int(max_ne_iters), _p(bst),
        int(base), C.byref(r))
    out = _take(r)
    if status == ERR_OOM:
        raise MemoryError()
    return out


class OracleError(Exception):
    """Raised where the reference raises DecodeError."""


class OracleChannel:
    """DecodeState restatement over the C kernel (decoder.py:150-341)."""

    def __init__(self, fg, beam=17.0, max_active=10_000, acoustic_scale=1.0, relax_eps=1e-9,
                 max_ne_iters=None, boost=None):
        self.fg = fg
        self.beam, self.max_active, self.scale, self.relax = beam, max_active, acoustic_scale, relax_eps
        self.max_ne_iters = max_ne_iters if max_ne_iters is not None else 2 * fg.num_states
        self.boost = None if boost is None else _c(boost, np.float64)
        self.frame_count = 0
        self.num_tokens = None
        self.frames = []  # (prev, state, cost, olab_off, olab_pool)
        self.frame_base = []
        self.next_record = 0
        self._seed()

    @classmethod
    def from_config(cls, fg, config, boost=None):
        return cls(fg, config.beam, config.max_active, config.acoustic_scale,
                   config.nonemitting_relax_epsilon, config.max_nonemitting_iters, boost)

    def _seed(self):
        fg = self.fg
        g = [_c(fg.off, np.int64), _c(fg.eps_end, np.int64), _c(fg.olabel, np.int32),
             _c(fg.weight, np.float64), _c(fg.nextstate, np.int32)]
        r = _Result()
        st = lib().ctwo_seed(*[_p(a) for a in g], fg.num_states, fg.start, self.relax,
                             self.max_ne_iters, _p(self.boost), C.byref(r))
        _, _, _, _, state, cost, ooff, opool = _take(r)
        if st == ERR_EPS_ITERS:
            raise OracleError("epsilon iteration cap exceeded while seeding the channel")
        self.act_state, self.act_cost = state, cost
        self.act_bp = np.full(len(state), -1, dtype=np.int64)
        self.act_chain_off, self.act_chain_pool = ooff, opool

    def advance_frames(self, loglik):
        fg = self.fg
        loglik = np.ascontiguousarray(loglik, dtype=np.float64)
        if loglik.shape[0] == 0:
            return
        width = loglik.shape[1]
        if self.num_tokens is None:
            if width < fg.max_ilabel:
                raise OracleError(f"frame has {width} tokens but the graph expects at least {fg.max_ilabel}")
            self.num_tokens = width
        elif width != self.num_tokens:
            raise OracleError(f"frame has {width} tokens, channel was created with {self.num_tokens}")
        status, err, counts, prev, state, cost, ooff, opool = advance_chunk(
            fg.off, fg.eps_end, fg.ilabel, fg.olabel, fg.weight, fg.nextstate, self.act_state,
            self.act_cost, self.act_bp, self.act_chain_off, self.act_chain_pool, loglik, self.scale,
            self.beam, self.max_active, self.relax, self.max_ne_iters, self.boost, self.next_record)
        if status == ERR_EPS_ITERS:
            raise OracleError(f"nonemitting iteration cap exceeded at frame {self.frame_count + err} (epsilon cycle?)")
        if status == ERR_NO_SURVIVORS:
            raise OracleError(f"no tokens survive frame {self.frame_count + err}")
        first = 0
        for n in counts.tolist():
            self.frames.append((prev[first:first + n], state[first:first + n], cost[first:first + n],
                                ooff[first:first + n + 1] - ooff[first], opool[ooff[first]:ooff[first + n]]))
            self.frame_base.append(self.next_record)
            self.next_record += n
            first += n
        self.frame_count += len(counts)
        last = self.frames[-1]
        self.act_state, self.act_cost = last[1], last[2]
        self.act_bp = np.arange(self.frame_base[-1], self.frame_base[-1] + len(last[1]), dtype=np.int64)
        self.act_chain_off = np.zeros(len(last[1]) + 1, dtype=np.int64)
        self.act_chain_pool = np.zeros(0, dtype=np.int32)

    def history_records(self):
        out = []
        for prev, state, cost, ooff, opool in self.frames:
            out.append([(int(prev[i]), tuple(int(o) for o in opool[ooff[i]:ooff[i + 1]]),
                         int(state[i]), float(cost[i])) for i in range(len(state))])
        return out

    def best_path(self):
        """-> (words tuple, total_cost, frame_count); decoder.py:377-415."""
        if self.frame_count == 0:
            raise OracleError("no frames decoded")
        final = _c(self.fg.final, np.float64)
        tot = C.c_double()
        st, co = _c(self.act_state, np.int32), _c(self.act_cost, np.float64)
        i = lib().ctwo_best(_p(st), _p(co), len(st), _p(final), C.byref(tot))
        if i < 0:
            raise OracleError("no surviving hypotheses")
        segs = []
        rec = int(self.act_bp[i])
        while rec >= 0:
            fr = bisect.bisect_right(self.frame_base, rec) - 1
            prev, _, _, ooff, opool = self.frames[fr]
            j = rec - self.frame_base[fr]
            segs.append(opool[ooff[j]:ooff[j + 1]])
            rec = int(prev[j])
        words = []
        for s in reversed(segs):
            words.extend(int(o) for o in s)
        return tuple(words), float(tot.value), self.frame_count


def decode_utterance(fg, config, loglik, boost=None):
    ch = OracleChannel.from_config(fg, config, boost)
    ch.advance_frames(loglik)
    return ch.best_path()


def decode_batch(fg, config, utterances, workers=1, boost=None):
    """decoder.py:436-463: per-index results, exceptions reported in place."""
    def run(i):
        try:
            return decode_utterance(fg, config, utterances[i], boost)
        except Exception as e:  # noqa: BLE001
            return e

    if workers <= 1 or len(utterances) <= 1:
        return [run(i) for i in range(len(utterances))]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(run, range(len(utterances))))
