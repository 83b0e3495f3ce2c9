"""Lattices and n-best lists (the reference has none,
SPEC.md:312).

A lattice is built on the device after a lane has decoded a whole utterance
(``csrc/ctw_lattice.cu``, definition in DESIGN.md "Lattice"): its nodes are
the seed tokens and the per-frame survivors the decoder recorded (the
reference's history records, bit-identical to the reference); between two
consecutive layers there is one arc per (source token, emitting arc,
surviving destination) with the minimum epsilon continuation's cost and
output labels; arcs whose best complete path is more than ``lattice_beam``
above the best path are pruned. ``Lattice.nbest(n)`` returns the n lowest-cost
distinct word sequences (A* over the kept arcs with exact remaining costs).

    lats = decode_lattices(graph, config, utterances, lattice_beam=6.0)
    for lat in lats:
        print(lat.best_path.words, [h.words for h in lat.nbest(5)])
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from .decoder import DecodeFailure, Hypothesis, decode_batch


class _CArrays:
    """Owner of one ctw_lattice's C arrays (freed with the last reference)."""

    __slots__ = ("c", "__weakref__")

    def __init__(self, c: _lib.CtwLattice):
        self.c = c

    def __del__(self):
        try:
            _lib.load().ctw_lattice_free(C.byref(self.c))
        except Exception:  # interpreter shutdown
            pass


class Lattice:
    """Pruned lattice of one utterance (host copy of ``ctw_lattice``).

    Node ids: seeds ``0 .. n_seeds-1`` (the start state's epsilon closure),
    then ``n_seeds + record index``. Arc arrays are sorted by (frame, src,
    dst, weight)."""

    def __init__(self, c: _lib.CtwLattice, best_path: Hypothesis):
        # the arrays below are zero-copy views of the C arrays; one owner
        # object frees them (ctw_lattice_free) once the lattice and every
        # array taken from it are gone
        owner = _CArrays(c)
        self._owner = owner
        self._c = owner.c
        self.best_path = best_path
        self.status = int(c.status)
        self.final_mode = bool(c.final_mode)
        self.frame_count = int(c.frame_count)
        self.best_cost = float(c.best)
        self.lattice_beam = float(c.lattice_beam)
        self.closure_items = int(c.closure_items)
        self.closure_pruned = int(c.closure_pruned)
        ns, na = int(c.n_seeds), int(c.n_arcs)

        def arr(p, n, dt):  # n elements at a C pointer, kept alive by the owner
            if not n:
                return np.zeros(0, dt)
            nb = n * np.dtype(dt).itemsize
            buf = (C.c_char * nb).from_address(C.cast(p, C.c_void_p).value)
            buf._owner = owner
            return np.frombuffer(buf, dt)

        self.seed_state = arr(c.seed_state, ns, np.int32)
        self.seed_cost = arr(c.seed_cost, ns, np.float64)
        soff = arr(c.seed_lab_off, ns + 1, np.int64)
        slab = arr(c.seed_lab, int(soff[-1]) if ns else 0, np.int32)
        self.seed_labels = [tuple(int(x) for x in slab[soff[k]:soff[k + 1]]) for k in range(ns)]
        self.src = arr(c.arc_src, na, np.int32)
        self.dst = arr(c.arc_dst, na, np.int32)
        self.frame = arr(c.arc_frame, na, np.int32)
        self.dst_state = arr(c.arc_dst_state, na, np.int32)
        self.src_state = arr(c.arc_src_state, na, np.int32)
        self.weight = arr(c.arc_w, na, np.float64)
        self.dst_final = arr(c.arc_dst_final, na, np.float64)
        self.label_off = arr(c.arc_lab_off, na + 1, np.int64) if na else np.zeros(1, np.int64)
        self.label_pool = arr(c.arc_lab, int(self.label_off[-1]), np.int32)
        self._labels = None

    @property
    def labels(self) -> list:
        """Output labels of every arc (tuples; built on first use)."""
        if self._labels is None:
            off, pool = self.label_off.tolist(), self.label_pool.tolist()
            self._labels = [tuple(pool[off[k]:off[k + 1]]) for k in range(len(off) - 1)]
        return self._labels

    @property
    def num_arcs(self) -> int:
        return len(self.src)

    def nbest(self, n: int, max_pops: int = 2_000_000, phrases: "PhraseBoost | None" = None) -> list[Hypothesis]:
        """The n lowest-cost distinct word sequences, best first; with
        ``phrases``, costs include the phrase automaton's (multi-word
        boosting by lattice rescoring)."""
        if n <= 0:
            return []
        L = _lib.load()
        cap = 1024
        while True:
            words = np.zeros(cap, np.int32)
            off = np.zeros(n + 1, np.int64)
            costs = np.zeros(n, np.float64)
            found = C.c_int32()
            pops = C.c_int64()
            if phrases is None:
                rc = L.ctw_lattice_nbest(C.byref(self._c), n, max_pops, _lib.ptr(words), cap, _lib.ptr(off),
                                         _lib.ptr(costs), C.byref(found), C.byref(pops))
            else:
                f = phrases
                rc = L.ctw_lattice_nbest_phrases(C.byref(self._c), f.num_states, _lib.ptr(f.goto_off),
                                                 _lib.ptr(f.goto_word), _lib.ptr(f.goto_next), _lib.ptr(f.fail),
                                                 _lib.ptr(f.out_cost), n, max_pops, _lib.ptr(words), cap,
                                                 _lib.ptr(off), _lib.ptr(costs), C.byref(found), C.byref(pops))
            if rc == -2:
                cap = int(off[int(found.value)]) + 16
                continue
            _lib.check(rc, "lattice n-best")
            self.last_pops = int(pops.value)
            return [Hypothesis(tuple(int(x) for x in words[off[k]:off[k + 1]]), float(costs[k]), self.frame_count)
                    for k in range(int(found.value))]


class PhraseBoost:
    """Multi-word (phrase) boosting as a deterministic Aho-Corasick automaton
    over word ids. ``phrases`` maps a word-id tuple to a magnitude; like the
    reference's word tables (boosting.py:33-55) a boost of m is the cost -m,
    paid once per occurrence of the phrase in a hypothesis (overlapping and
    nested occurrences all count). A one-word phrase is the reference's word
    boost; longer phrases are beyond the reference.
    Applied by ``Lattice.nbest(n, phrases=...)`` (lattice rescoring)."""

    def __init__(self, phrases: dict):
        children = [{}]
        own = [0.0]
        for ph, mag in phrases.items():
            ph = tuple(int(w) for w in ph)
            if not ph or any(w <= 0 for w in ph):
                raise ValueError("phrases are non-empty tuples of word ids > 0")
            s = 0
            for w in ph:
                nxt = children[s].get(w)
                if nxt is None:
                    nxt = len(children)
                    children[s][w] = nxt
                    children.append({})
                    own.append(0.0)
                s = nxt
            own[s] += -float(mag)
        n = len(children)
        fail = [0] * n
        out = list(own)
        order = []
        queue = list(children[0].values())
        order.extend(queue)
        while queue:  # breadth first: failure links and accumulated outputs
            nq = []
            for s in queue:
                for w, t in children[s].items():
                    f = fail[s]
                    while f and w not in children[f]:
                        f = fail[f]
                    fail[t] = children[f][w] if (w in children[f] and children[f][w] != t) else 0
                    nq.append(t)
            for t in nq:
                out[t] = own[t] + out[fail[t]]
            queue = nq
        self.num_states = n
        offs, ws, ns = [0], [], []
        for s in range(n):
            for w in sorted(children[s]):
                ws.append(w)
                ns.append(children[s][w])
            offs.append(len(ws))
        self.goto_off = np.asarray(offs, np.int32)
        self.goto_word = np.asarray(ws or [0], np.int32)
        self.goto_next = np.asarray(ns or [0], np.int32)
        self.fail = np.asarray(fail, np.int32)
        self.out_cost = np.asarray(out, np.float64)
        self._children = children
        self.phrases = {tuple(int(w) for w in p): float(m) for p, m in phrases.items()}

    @property
    def single_words(self) -> bool:
        """Only one-word phrases: equivalent to the reference's one-state
        word boost, so the decoder uses the dense word table for it."""
        return all(len(p) == 1 for p in self.phrases)

    def word_costs(self, width: int) -> np.ndarray:
        """Dense per-word cost vector (boosting.py:58-67 layout)."""
        v = np.zeros(width, np.float64)
        for ph, mag in self.phrases.items():
            if ph[0] < width:
                v[ph[0]] += -float(mag)
        return v

    def to_fst(self, max_olabel: int):
        """The explicit acceptor (every word label from every state), for
        composition-based checks: arcs w:w with the entry cost of delta(b, w);
        every state final with weight 0."""
        from .synth import Fst

        nxt = self.dense_next(max_olabel + 1)
        src, lab, w, ns = [], [], [], []
        for b in range(self.num_states):
            for x in range(1, max_olabel + 1):
                t = int(nxt[b, x])
                src.append(b)
                lab.append(x)
                w.append(float(self.out_cost[t]))
                ns.append(t)
        return Fst(self.num_states, 0, src, lab, lab, w, ns, np.zeros(self.num_states))

    def dense_next(self, width: int) -> np.ndarray:
        """Transition table next[b, w] for word labels 0..width-1 (label 0
        keeps the state): the full automaton delta, breadth first (a state
        copies its failure state's row, then overrides its own gotos)."""
        n = self.num_states
        if n > 65535:
            raise ValueError("phrase automaton too large (> 65535 states)")
        nxt = np.zeros((n, width), np.uint16)
        order = [0]
        head = 0
        while head < len(order):
            s = order[head]
            head += 1
            if s:
                nxt[s] = nxt[int(self.fail[s])]
            for w, t in self._children[s].items():
                if w < width:
                    nxt[s, w] = t
                order.append(t)
        nxt[:, 0] = np.arange(n, dtype=np.uint16)
        return nxt

    def cost(self, words) -> float:
        """Boost cost of a word sequence under the automaton."""
        s, c = 0, 0.0
        for w in words:
            while s and w not in self._children[s]:
                s = int(self.fail[s])
            s = self._children[s].get(w, 0)
            c += float(self.out_cost[s])
        return c


def decode_lattices(graph, config, utterances: Sequence, lattice_beam: float = 6.0, boost=None, *,
                    device: int | None = None, max_lanes: int | None = None, search: str = "exact") -> list:
    """decode_batch plus a pruned lattice per utterance: a list of Lattice
    (``.best_path`` is decode_batch's Hypothesis) or DecodeFailure, in input
    order."""
    if not (lattice_beam >= 0):
        raise ValueError("lattice_beam must be >= 0")
    return decode_batch(graph, config, utterances, boost=boost, device=device, max_lanes=max_lanes,
                        lattice_beam=float(lattice_beam), search=search)


def build_lattices(pool, states, mats, on_dev, packed, hyps, lattice_beam: float) -> list:
    """ctw_lane_lattice over lanes that decoded their whole utterance."""
    from .decoder import _pack_rows

    n = len(states)
    ids = np.asarray([s._lane for s in states], np.int32)
    frames = np.asarray([m.shape[0] for m in mats], np.int32)
    width = int(mats[0].shape[1])
    buf, offs, base, dcode, loc = _pack_rows(mats, on_dev, packed, frames, width)
    outs = (_lib.CtwLattice * n)()
    keep = buf
    _lib.check(_lib.load().ctw_lane_lattice(pool.handle, _lib.ptr(ids), n, C.c_void_p(base), dcode, loc,
                                            _lib.ptr(offs), width, float(lattice_beam), C.cast(outs, C.c_void_p)),
               "lattice")
    del keep
    res = []
    for k in range(n):
        c = _lib.CtwLattice()
        C.memmove(C.byref(c), C.byref(outs[k]), C.sizeof(_lib.CtwLattice))
        lat = Lattice(c, hyps[k])
        if lat.status == 3:
            # even the large-capacity re-run could not hold an epsilon
            # closure: no silently truncated lattice (reported per index)
            from .errors import DecodeError

            lat = DecodeError("lattice: an epsilon closure exceeded the per-item capacity "
                              "(the lattice would be incomplete)")
        res.append(lat)
    return res


def nbest_lattices(lattices: Sequence, n: int, max_pops: int = 2_000_000, phrases: "PhraseBoost | None" = None,
                   workers: int | None = None) -> list:
    """``Lattice.nbest`` over many lattices on a host thread pool (the C
    search runs with the GIL released): a list of n-best lists in input
    order; a DecodeFailure entry stays a DecodeFailure."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    def one(lat):
        return lat.nbest(n, max_pops=max_pops, phrases=phrases) if isinstance(lat, Lattice) else lat

    lattices = list(lattices)
    workers = workers or min(len(lattices), os.cpu_count() or 1)
    if workers <= 1 or len(lattices) <= 1:
        return [one(x) for x in lattices]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(one, lattices))


__all__ = ["Lattice", "PhraseBoost", "decode_lattices", "nbest_lattices", "DecodeFailure"]
