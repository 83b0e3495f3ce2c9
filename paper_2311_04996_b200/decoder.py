"""Batched frame-synchronous WFST beam search on B200 -- the decode engine.

Drop-in for the reference engine (pkg/src/ctcwfst/decoder.py): same public
names, argument meaning, results and error behaviour, but every channel is a
*lane* resident in HBM and all lanes of a call advance in one sm_100a kernel
launch (paper_2311_04996_b200/csrc/ctw_kernels.cu) through the C-ABI in
include/ctcwfst_b200.h.

Reference map (decoder.py unless noted):
  DecoderConfig :34-48   Token :51-54   Hypothesis :57-61   DecodeFailure :64-67
  FlatGraph :70-127 / flatten :130-138 -> graph upload (ctw_graph_create)
  DecodeState :150-341 -> one lane; seeding :173-229 (ctw_lane_reset),
      set_boost :231-238, history_records :251-260 (ctw_lane_export),
      advance_frames :264-341 (ctw_advance; chunk-atomic, errors name the frame)
  create_channel :344-350   advance :353-358   prune :361-374 (host rule)
  best_path :377-415 (ctw_best_path)   decode_utterance :422-433
  decode_batch :436-463 -> ONE batched launch over all utterances (lanes)
  instead of a host thread pool.

Passing ``kernel=`` to DecodeState keeps the reference's plug-in seam
(decoder.py:154, :163): the channel is then kept on the host exactly as the
reference does and the callable does the frames -- e.g.
``kernels.advance_chunk`` (the GPU under the 19-argument contract).
"""

from __future__ import annotations

import bisect
import ctypes as C
import math
import threading
import warnings
import weakref
from dataclasses import dataclass
from typing import NamedTuple, Sequence

import numpy as np

from . import _lib
from .errors import DecodeError
from .wfst import EPSILON, Wfst

INF = math.inf
_MAX_ACTIVE_CAP = 2**60  # decoder.py:31


@dataclass(frozen=True)
class DecoderConfig:
    beam: float = 17.0
    max_active: int = 10_000
    acoustic_scale: float = 1.0
    nonemitting_relax_epsilon: float = 1e-9
    max_nonemitting_iters: int | None = None  # None: 2 x graph states

    def __post_init__(self):
        if not self.beam > 0:
            raise ValueError(f"beam must be positive, got {self.beam}")
        if self.max_active < 1:
            raise ValueError(f"max_active must be >= 1, got {self.max_active}")
        if not self.acoustic_scale > 0:
            raise ValueError(f"acoustic_scale must be positive, got {self.acoustic_scale}")


class Token(NamedTuple):
    state: int
    cost: float
    backpointer: int  # global record index, -1 at the root


@dataclass(frozen=True)
class Hypothesis:
    words: tuple[int, ...]
    total_cost: float
    frame_count: int


@dataclass(frozen=True)
class DecodeFailure:
    index: int
    error: Exception


# --------------------------------------------------------------- graph -----


class FlatGraph:
    """CSR arc arrays of a decoding graph (decoder.py:70-127 layout): per
    state the arcs are stably sorted by input label, so epsilon arcs are
    [off[s], eps_end[s]) and emitting arcs [eps_end[s], off[s+1]). The arrays
    are uploaded to HBM once per device on first use."""

    __slots__ = ("num_states", "start", "off", "eps_end", "ilabel", "olabel", "weight",
                 "nextstate", "final", "max_ilabel", "max_olabel", "_dev", "__weakref__")

    def __init__(self, g=None):
        self._dev = {}
        if g is None:
            return
        if g.is_empty:
            raise DecodeError("empty graph")
        n = g.num_states
        src, il, ol, w, ns = [], [], [], [], []
        for s in g.states():
            for a in g.arcs(s):
                src.append(s)
                il.append(a.ilabel)
                ol.append(a.olabel)
                w.append(a.weight)
                ns.append(a.nextstate)
        final = np.full(n, INF)
        for s, fw in g.finals.items():
            final[s] = fw
        self._set(n, g.start, np.asarray(src, np.int64), np.asarray(il, np.int32),
                  np.asarray(ol, np.int32), np.asarray(w, np.float64), np.asarray(ns, np.int32), final)

    @classmethod
    def from_arrays(cls, num_states, start, src, ilabel, olabel, weight, nextstate, final):
        """Build from per-arc arrays (any arc order; the source-state order and
        the per-state stable ilabel order are established here). Use this for
        graphs too large for Python ``Wfst`` objects."""
        fg = cls()
        if num_states <= 0:
            raise DecodeError("empty graph")
        fg._set(int(num_states), int(start), np.asarray(src, np.int64), np.asarray(ilabel, np.int32),
                np.asarray(olabel, np.int32), np.asarray(weight, np.float64),
                np.asarray(nextstate, np.int32), np.asarray(final, np.float64))
        return fg

    @classmethod
    def from_csr(cls, obj):
        """Adopt any FlatGraph-shaped object (e.g. the reference's)."""
        fg = cls()
        fg.num_states = int(obj.num_states)
        fg.start = int(obj.start)
        fg.off = np.ascontiguousarray(obj.off, np.int64)
        fg.eps_end = np.ascontiguousarray(obj.eps_end, np.int64)
        fg.ilabel = np.ascontiguousarray(obj.ilabel, np.int32)
        fg.olabel = np.ascontiguousarray(obj.olabel, np.int32)
        fg.weight = np.ascontiguousarray(obj.weight, np.float64)
        fg.nextstate = np.ascontiguousarray(obj.nextstate, np.int32)
        fg.final = np.ascontiguousarray(obj.final, np.float64)
        fg.max_ilabel = int(obj.max_ilabel)
        fg.max_olabel = int(obj.max_olabel)
        return fg

    def _set(self, n, start, src, il, ol, w, ns, final):
        order = np.lexsort((il, src))  # by state, then stable by ilabel
        src = src[order]
        self.num_states = n
        self.start = start
        self.ilabel = np.ascontiguousarray(il[order])
        self.olabel = np.ascontiguousarray(ol[order])
        self.weight = np.ascontiguousarray(w[order])
        self.nextstate = np.ascontiguousarray(ns[order])
        counts = np.bincount(src, minlength=n) if len(src) else np.zeros(n, np.int64)
        self.off = np.zeros(n + 1, np.int64)
        np.cumsum(counts, out=self.off[1:])
        eps_counts = np.bincount(src[self.ilabel == EPSILON], minlength=n) if len(src) else np.zeros(n, np.int64)
        self.eps_end = self.off[:-1] + eps_counts
        self.final = np.ascontiguousarray(final, np.float64)
        self.max_ilabel = int(self.ilabel.max()) if len(il) else 0
        self.max_olabel = int(self.olabel.max()) if len(ol) else 0

    @property
    def num_arcs(self) -> int:
        return int(self.off[-1])

    def device_graph(self, device: int | None = None) -> "DeviceGraph":
        dev = _resolve_device(device)
        dg = self._dev.get(dev)
        if dg is None:
            dg = DeviceGraph(self, dev)
            self._dev[dev] = dg
        return dg


_flatten_lock = threading.Lock()
_adopted: dict = {}


def flatten(g) -> FlatGraph:
    """Flatten once per graph instance (cached on ``g._flat``); accepts our
    Wfst, the reference's Wfst/FlatGraph, or a FlatGraph."""
    if isinstance(g, FlatGraph):
        return g
    if hasattr(g, "off") and hasattr(g, "eps_end"):
        with _flatten_lock:  # foreign FlatGraph-shaped object: adopt once
            hit = _adopted.get(id(g))
            if hit is None or hit[0] is not g:
                hit = (g, FlatGraph.from_csr(g))
                _adopted[id(g)] = hit
                while len(_adopted) > 8:
                    _adopted.pop(next(iter(_adopted)))
            return hit[1]
    with _flatten_lock:
        cached = getattr(g, "_flat", None)
        if not isinstance(cached, FlatGraph):
            cached = FlatGraph(g)
            try:
                g._flat = cached
            except AttributeError:
                pass
        return cached


def _resolve_device(device) -> int:
    if device is not None:
        return int(device)
    try:
        import torch

        if torch.cuda.is_available():
            return int(torch.cuda.current_device())
    except Exception:  # noqa: BLE001
        pass
    return 0


class DeviceGraph:
    """A FlatGraph resident in HBM of one device (ctw_graph)."""

    def __init__(self, fg: FlatGraph, device: int):
        L = _lib.load()
        h = C.c_void_p()
        _lib.check(L.ctw_graph_create(_lib.ptr(fg.off), _lib.ptr(fg.eps_end), _lib.ptr(fg.ilabel),
                                      _lib.ptr(fg.olabel), _lib.ptr(fg.weight), _lib.ptr(fg.nextstate),
                                      _lib.ptr(fg.final), fg.num_states, fg.num_arcs, fg.start,
                                      device, C.byref(h)), "graph upload")
        self.handle = h
        self.device = device
        self.fg_ref = weakref.ref(fg)
        self.pools: dict = {}
        self._lock = threading.Lock()
        self._fin = weakref.finalize(self, L.ctw_graph_destroy, h)

    def pool(self, config: DecoderConfig, num_states: int, search: str = "exact") -> "LanePool":
        ne = config.max_nonemitting_iters if config.max_nonemitting_iters is not None else 2 * num_states
        key = (config.beam, min(config.max_active, _MAX_ACTIVE_CAP), config.acoustic_scale,
               config.nonemitting_relax_epsilon, ne)
        mode = _search_mode(search)
        if ne < min(1 << 16, num_states + 1) and (key, mode) not in self.pools:
            # ctw_api.cu prune_flag: a cap that could bind keeps the full
            # Gauss-Seidel pass accounting (no early beam pruning, no fast mode)
            warnings.warn(f"max_nonemitting_iters={ne} can bind before the epsilon closure converges "
                          f"(< min(65536, num_states + 1)): early beam pruning and the fast search mode "
                          f"are disabled for this configuration (exact but slower)", RuntimeWarning, stacklevel=3)
        with self._lock:
            p = self.pools.get((key, mode))
            if p is None:
                p = LanePool(self, key, mode)
                self.pools[(key, mode)] = p
            return p


SEARCH_MODES = ("exact", "fast")


def _search_mode(search) -> str:
    """Search mode of a lane pool (include/ctcwfst_b200.h ctw_lanes_set_search):
    "exact" reproduces the reference kernel record for record (histories,
    prev pointers); "fast" is the words-exact throughput mode (identical
    best-path words, costs within the reference's relax_eps stop rule)."""
    if search is None:
        return "exact"
    if search not in SEARCH_MODES:
        raise ValueError(f"search must be one of {SEARCH_MODES}, got {search!r}")
    return search


class LanePool:
    """A ctw_lanes set (one decoder configuration on one device graph) with a
    free list; DecodeState objects borrow lanes from it."""

    def __init__(self, dg: DeviceGraph, key, search: str = "exact"):
        L = _lib.load()
        self.dg = dg
        self.cfg = _lib.CtwConfig(key[0], key[1], key[2], key[3], key[4])
        h = C.c_void_p()
        _lib.check(L.ctw_lanes_create(dg.handle, 0, C.byref(self.cfg), None, C.byref(h)), "lane set creation")
        self.handle = h
        self.search = search
        _lib.check(L.ctw_lanes_set_search(h, SEARCH_MODES.index(search)), "search mode")
        self.size = 0
        self.free: list[int] = []
        self.lock = threading.Lock()
        self._fin = weakref.finalize(self, L.ctw_lanes_destroy, h)

    def acquire(self, n: int) -> list[int]:
        with self.lock:
            if len(self.free) < n:
                want = self.size + (n - len(self.free))
                got = _lib.check(_lib.load().ctw_lanes_reserve(self.handle, want), "lane reservation")
                self.free.extend(range(self.size, got))
                self.size = got
            ids = self.free[-n:] if n else []
            del self.free[len(self.free) - n:]
            return ids

    def release(self, ids) -> None:
        with self.lock:
            self.free.extend(ids)

    def reset(self, ids, boosts) -> np.ndarray:
        """Fresh channels on lanes `ids`. A boost is a dense per-word cost
        vector (the reference's tables) or a PhraseBoost (phrase automaton
        composed inside the search)."""
        n = len(ids)
        idarr = np.asarray(ids, np.int32)
        st = np.zeros(n, np.int32)
        L = _lib.load()
        width = self.dg.fg_ref().max_olabel + 1 if self.dg.fg_ref() is not None else None
        dense = []
        for lane, b in zip(ids, boosts):
            if b is not None and hasattr(b, "dense_next") and b.single_words and width is not None:
                b = b.word_costs(width)  # one-word phrases: the reference's one-state boost
            if b is not None and hasattr(b, "dense_next"):
                nxt = b.dense_next(width)
                cost = np.ascontiguousarray(b.out_cost, np.float64)
                _lib.check(L.ctw_lane_set_fsa(self.handle, int(lane), int(b.num_states), _lib.ptr(nxt),
                                              _lib.ptr(cost)), "phrase automaton")
                dense.append(None)
            else:
                _lib.check(L.ctw_lane_set_fsa(self.handle, int(lane), 0, None, None), "phrase automaton")
                dense.append(b)
        boosts = dense
        keep = [None if b is None else np.ascontiguousarray(b, np.float64) for b in boosts]
        ptrs = (C.c_void_p * n)(*[None if b is None else b.ctypes.data for b in keep])
        lens = np.asarray([0 if b is None else len(b) for b in keep], np.int64)
        _lib.check(_lib.load().ctw_lane_reset(self.handle, _lib.ptr(idarr), n, ptrs, _lib.ptr(lens),
                                              _lib.ptr(st)), "lane reset")
        return st

    def stats(self) -> dict:
        v = [C.c_int64(), C.c_int64(), C.c_double(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()]
        _lib.load().ctw_lanes_stats(self.handle, *[C.byref(x) for x in v])
        return {"launches": v[0].value, "decode_launches": v[1].value, "decode_ms": v[2].value,
                "arcs": v[3].value, "src_tokens": v[4].value, "frames": v[5].value, "max_slots": v[6].value}

    def profile(self) -> dict:
        """Per-stage SM cycles of the frame kernel (ctw_lanes_profile)."""
        v = np.zeros(16, np.int64)
        _lib.load().ctw_lanes_profile(self.handle, _lib.ptr(v))
        names = ("emit", "eps", "beam_count", "select", "records", "reset", "eps_passes", "select_frames",
                 "slots", "eps_items", "eps_arcs", "in_beam", "tie_frames", "ties", "eps_disc_arcs", "r15")
        return dict(zip(names, (int(x) for x in v)))

    def host_timing(self) -> dict:
        """Host-side breakdown of the advance calls (ctw_lanes_host_timing)."""
        v = np.zeros(10, np.float64)
        _lib.load().ctw_lanes_host_timing(self.handle, _lib.ptr(v))
        return {"stage_s": float(v[0]), "presize_s": float(v[1]), "wait_s": float(v[2]), "post_s": float(v[3]),
                "reruns": int(v[4]), "calls": int(v[5]),
                "grow_lanes": {"table": int(v[6]), "history": int(v[7]), "pool": int(v[8]), "sources": int(v[9])}}

    def capacity(self, lane: int) -> dict:
        """Device buffer capacities of one lane (ctw_lane_capacity)."""
        v = np.zeros(6, np.int64)
        _lib.check(_lib.load().ctw_lane_capacity(self.handle, int(lane), _lib.ptr(v)), "lane capacity")
        return {"table_log2": int(v[0]), "sources": int(v[1]), "records": int(v[2]), "frames": int(v[3]),
                "olabel_pool": int(v[4]), "bytes": int(v[5])}

    def reset_stats(self) -> None:
        _lib.load().ctw_lanes_reset_stats(self.handle)

    def search_info(self) -> dict:
        """Requested search mode and how many decode launches ran fast."""
        v = np.zeros(3, np.int64)
        _lib.load().ctw_lanes_search_info(self.handle, _lib.ptr(v))
        return {"search": SEARCH_MODES[int(v[0])], "fast_launches": int(v[1]), "decode_launches": int(v[2])}

    def graph_info(self) -> dict:
        """Streaming steps launched as one CUDA graph (ctw_lanes_graph_info)."""
        v = np.zeros(3, np.int64)
        _lib.load().ctw_lanes_graph_info(self.handle, _lib.ptr(v))
        return {"graph_launches": int(v[0]), "graphs_captured": int(v[1]), "graphs_off": bool(v[2])}


# ---------------------------------------------------- loglik marshalling ---


def _to_lane_device(x, device: int):
    """A CUDA tensor on another GPU than the lane set's is copied to the lane
    set's device (the kernels dereference raw device pointers)."""
    if getattr(x, "is_cuda", False) and x.device.index != device:
        return x.to(f"cuda:{device}")
    return x


def _as_frames(x, device: int | None = None):
    """(array, on_device) for a (frames, tokens) matrix given as numpy, torch
    (CPU or CUDA) or any DLPack producer; CUDA tensors end up on `device`."""
    if isinstance(x, np.ndarray):
        return x, False
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None:
        if not isinstance(x, torch.Tensor) and hasattr(x, "__dlpack__"):
            x = torch.from_dlpack(x)
        if isinstance(x, torch.Tensor):
            if x.is_cuda:
                if x.dtype not in (torch.float32, torch.float64):
                    x = x.double()
                if device is not None:
                    x = _to_lane_device(x, device)
                return x.contiguous(), True
            x = x.numpy()
    return np.asarray(x), False


def _host_matrix(x):
    a = np.asarray(x)
    if a.dtype != np.float32:
        a = np.ascontiguousarray(a, dtype=np.float64)
    else:
        a = np.ascontiguousarray(a)
    return a


# ---------------------------------------------------------- DecodeState ----


class DecodeState:
    """All mutable state of one decoding channel (decoder.py:150-341).

    Default: the channel is a lane in HBM. With ``kernel=`` the reference's
    host bookkeeping is used around that kernel callable (plug-in seam)."""

    def __init__(self, graph, config: DecoderConfig, kernel=None, device: int | None = None,
                 search: str = "exact"):
        self.graph = flatten(graph)
        self.config = config
        self.frame_count = 0
        self.num_tokens: int | None = None
        self._boost: np.ndarray | None = None
        self._kernel = kernel
        self._max_ne_iters = (config.max_nonemitting_iters if config.max_nonemitting_iters is not None
                              else 2 * self.graph.num_states)
        if kernel is None:
            dg = self.graph.device_graph(device)
            self._pool = dg.pool(config, self.graph.num_states, search)
            self._lane = self._pool.acquire(1)[0]
            self._fin = weakref.finalize(self, self._pool.release, [self._lane])
            self._cache = None
        else:
            self._pool = None
            self.frames: list = []
            self.frame_base: list[int] = []
            self.next_record = 0
        self._seed_initial_tokens()

    # -- seeding ---------------------------------------------------------------

    def _seed_initial_tokens(self):
        if self._pool is not None:
            st = self._pool.reset([self._lane], [self._boost])
            self._cache = None
            if st[0] != _lib.OK:
                raise DecodeError("epsilon iteration cap exceeded while seeding the channel")
            return
        self._host_seed()

    def _host_seed(self):
        """decoder.py:173-229 restated for the host (plug-in) mode."""
        fg = self.graph
        states, costs, chains = [fg.start], [0.0], [()]
        slot_of = {fg.start: 0}
        iters = 0
        while True:
            iters += 1
            if iters > self._max_ne_iters:
                raise DecodeError("epsilon iteration cap exceeded while seeding the channel")
            best_gain = 0.0
            j = 0
            while j < len(states):
                s, c, ch = states[j], costs[j], chains[j]
                for a in range(int(fg.off[s]), int(fg.eps_end[s])):
                    nc = c + fg.weight[a]
                    ol = int(fg.olabel[a])
                    if self._boost is not None and ol != 0:
                        nc = nc + self._boost[ol]
                    if not nc < INF:
                        continue
                    d = int(fg.nextstate[a])
                    nch = ch + (ol,) if ol != 0 else ch
                    k = slot_of.get(d)
                    if k is None:
                        slot_of[d] = len(states)
                        states.append(d)
                        costs.append(nc)
                        chains.append(nch)
                        best_gain = INF
                    elif nc < costs[k]:
                        best_gain = max(best_gain, costs[k] - nc)
                        costs[k] = nc
                        chains[k] = nch
                j += 1
            if best_gain <= self.config.nonemitting_relax_epsilon:
                break
        order = sorted(range(len(states)), key=states.__getitem__)
        self._h_state = np.asarray([states[j] for j in order], np.int32)
        self._h_cost = np.asarray([costs[j] for j in order], np.float64)
        self._h_bp = np.full(len(order), -1, np.int64)
        pool: list[int] = []
        offs = [0]
        for j in order:
            pool.extend(chains[j])
            offs.append(len(pool))
        self._h_chain_off = np.asarray(offs, np.int64)
        self._h_chain_pool = np.asarray(pool, np.int32)

    # -- boost -------------------------------------------------------------------

    @property
    def boost(self) -> np.ndarray | None:
        return self._boost

    @boost.setter
    def boost(self, value):
        """Direct assignment (no re-seed), read at the next advance like the
        reference (decoder.py:287-305; exercised by test_decoder.py:343)."""
        self._boost = None if value is None else np.ascontiguousarray(value, np.float64)
        if self._pool is not None:
            b = self._boost
            _lib.check(_lib.load().ctw_lane_set_boost(self._pool.handle, self._lane, _lib.ptr(b),
                                                      0 if b is None else len(b)), "set boost")

    def set_boost(self, boost):
        """Bind a dense per-word boost cost vector (or a PhraseBoost) before
        the first frame and re-run the initial closure (decoder.py:231-238)."""
        if self.frame_count != 0:
            raise DecodeError("boost table must be attached before any frame is decoded")
        if boost is not None and hasattr(boost, "dense_next"):  # PhraseBoost: composed inside the search
            if self._pool is None:
                raise DecodeError("phrase boosting needs the native lane path (no kernel= plug-in)")
            self._boost = boost
        else:
            self._boost = None if boost is None else np.ascontiguousarray(boost, np.float64)
        self._seed_initial_tokens()

    def compact_history(self) -> int:
        """Partial-history garbage collection (ctw_lane_compact): drop the
        records no active token can reach; best_path and later partial
        hypotheses are unchanged, history_records() then lists the kept
        records only. Returns the records kept."""
        if self._pool is None:
            raise DecodeError("history compaction needs the native lane path")
        kept = np.zeros(1, np.int64)
        ids = np.asarray([self._lane], np.int32)
        _lib.check(_lib.load().ctw_lane_compact(self._pool.handle, _lib.ptr(ids), 1, _lib.ptr(kept)),
                   "history compaction")
        self._cache = None
        return int(kept[0])

    # -- introspection -------------------------------------------------------------

    def _export(self) -> dict:
        if self._cache is None:
            e = _lib.CtwExport()
            _lib.check(_lib.load().ctw_lane_export(self._pool.handle, self._lane, 0, 0, None, 0, C.byref(e)),
                       "history export")
            self._cache = _lib.take_export(e)
        return self._cache

    @property
    def act_state(self) -> np.ndarray:
        return self._h_state if self._pool is None else self._export()["tok_state"]

    @property
    def act_cost(self) -> np.ndarray:
        return self._h_cost if self._pool is None else self._export()["tok_cost"]

    @property
    def act_bp(self) -> np.ndarray:
        return self._h_bp if self._pool is None else self._export()["tok_bp"]

    @property
    def act_chain_off(self) -> np.ndarray:
        return self._h_chain_off if self._pool is None else self._export()["tok_chain_off"]

    @property
    def act_chain_pool(self) -> np.ndarray:
        return self._h_chain_pool if self._pool is None else self._export()["tok_chain_pool"]

    def active_tokens(self) -> list[Token]:
        return [Token(int(s), float(c), int(b)) for s, c, b in zip(self.act_state, self.act_cost, self.act_bp)]

    def active_states(self) -> set[int]:
        return {int(s) for s in self.act_state}

    def history_records(self) -> list[list[tuple[int, tuple[int, ...], int, float]]]:
        """Per-frame (prev, olabels, state, cost) records, reference layout."""
        if self._pool is None:
            return [_rows(*fr) for fr in self.frames]
        e = self._export()
        out, first = [], 0
        off, pool = e["rec_olab_off"], e["rec_olab_pool"]
        for n in e["counts"].tolist():
            out.append([(int(e["rec_prev"][i]), tuple(int(o) for o in pool[off[i]:off[i + 1]]),
                         int(e["rec_state"][i]), float(e["rec_cost"][i])) for i in range(first, first + n)])
            first += n
        return out

    # -- advancing ---------------------------------------------------------------

    def _check_width(self, width: int) -> None:
        fg = self.graph
        if self.num_tokens is None:
            if width < fg.max_ilabel:
                raise DecodeError(f"frame has {width} tokens but the graph expects at least {fg.max_ilabel}")
        elif width != self.num_tokens:
            raise DecodeError(f"frame has {width} tokens, channel was created with {self.num_tokens}")

    def advance_frames(self, loglik):
        """Advance over a chunk of frames; commits entirely or, on error,
        leaves the channel unchanged (decoder.py:264-341)."""
        if self._pool is None:
            return self._host_advance(np.ascontiguousarray(loglik, dtype=np.float64))
        x, on_dev = _as_frames(loglik, self._pool.dg.device if self._pool is not None else None)
        if x.ndim != 2:
            raise DecodeError("log-likelihoods must be a (frames, tokens) matrix")
        if x.shape[0] == 0:
            return
        self._check_width(int(x.shape[1]))
        if self.num_tokens is None:
            self.num_tokens = int(x.shape[1])
        _advance_lanes(self._pool, [self], [x], on_dev)

    def _host_advance(self, loglik: np.ndarray):
        if loglik.ndim != 2:
            raise DecodeError("log-likelihoods must be a (frames, tokens) matrix")
        if loglik.shape[0] == 0:
            return
        self._check_width(loglik.shape[1])
        if self.num_tokens is None:
            self.num_tokens = loglik.shape[1]
        fg = self.graph
        status, err, counts, prev, state, cost, ooff, opool = self._kernel(
            fg.off, fg.eps_end, fg.ilabel, fg.olabel, fg.weight, fg.nextstate, self._h_state, self._h_cost,
            self._h_bp, self._h_chain_off, self._h_chain_pool, loglik, self.config.acoustic_scale,
            self.config.beam, min(self.config.max_active, _MAX_ACTIVE_CAP),
            self.config.nonemitting_relax_epsilon, self._max_ne_iters, self._boost, self.next_record)
        _raise_status(status, self.frame_count + int(err))
        first = 0
        for n in (int(c) for c in counts):
            self.frames.append((prev[first:first + n], state[first:first + n], cost[first:first + n],
                                ooff[first:first + n + 1] - ooff[first], opool[ooff[first]:ooff[first + n]]))
            self.frame_base.append(self.next_record)
            self.next_record += n
            first += n
        self.frame_count += len(counts)
        _, st, co, _, _ = self.frames[-1]
        self._h_state, self._h_cost = st, co
        self._h_bp = np.arange(self.frame_base[-1], self.frame_base[-1] + len(st), dtype=np.int64)
        self._h_chain_off = np.zeros(len(st) + 1, np.int64)
        self._h_chain_pool = np.zeros(0, np.int32)


def _rows(prev, state, cost, ooff, opool):
    return [(int(prev[i]), tuple(int(o) for o in opool[ooff[i]:ooff[i + 1]]), int(state[i]), float(cost[i]))
            for i in range(len(state))]


def _raise_status(status: int, frame: int) -> None:
    if status == _lib.ERR_EPS_ITERS:
        raise DecodeError(f"nonemitting iteration cap exceeded at frame {frame} (epsilon cycle?)")
    if status == _lib.ERR_NO_SURVIVORS:
        raise DecodeError(f"no tokens survive frame {frame}")
    if status == _lib.ERR_OOM:
        raise MemoryError()


def _advance_lanes(pool: LanePool, states: Sequence[DecodeState], mats, on_dev: bool,
                   raise_first: bool = True, packed=None, with_best: bool = False):
    """One ctw_advance over several channels of the same lane pool. Returns a
    list of per-channel exceptions (None = committed). ``packed`` =
    (buffer, element offsets) passes an already-packed (n, F, V) block
    without re-copying it. ``with_best``: ctw_advance_best -- the partial
    best paths come back from the same call; returns (errors, hypotheses)."""
    n = len(states)
    frame_list = [m.shape[0] for m in mats]
    width = int(mats[0].shape[1])
    L = _lib.load()
    if with_best:
        cap = int(sum(s.frame_count for s in states) + sum(frame_list) + 8 * n) + 16
        ids = np.asarray([s._lane for s in states], np.int32)
        frames = np.asarray(frame_list, np.int32)
        status, err, bst = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.int32)
        woff, fc, cost = np.empty(n + 1, np.int64), np.empty(n, np.int64), np.empty(n, np.float64)
        words = np.empty(cap, np.int32)
        buf, offs, base, dcode, loc = _pack_rows(mats, on_dev, packed, frames, width)
        keep = buf
        p = _lib.ptr
        rc = L.ctw_advance_best(pool.handle, p(ids), n, base, dcode, loc, p(offs), p(frames), width, p(status),
                                p(err), p(words), cap, p(woff), p(cost), p(fc), p(bst))
        if rc != -2:
            _lib.check(rc, "advance")
    else:
        ids = np.asarray([s._lane for s in states], np.int32)
        frames = np.asarray(frame_list, np.int32)
        status = np.zeros(n, np.int32)
        err = np.zeros(n, np.int32)
        buf, offs, base, dcode, loc = _pack_rows(mats, on_dev, packed, frames, width)
        keep = buf
        _lib.check(L.ctw_advance(pool.handle, _lib.ptr(ids), n, C.c_void_p(base), dcode, loc,
                                 _lib.ptr(offs), _lib.ptr(frames), width, _lib.ptr(status),
                                 _lib.ptr(err)), "advance")
    del keep
    errors = []
    st_l, er_l = status.tolist(), err.tolist()
    for i, s in enumerate(states):
        s._cache = None
        if st_l[i] == _lib.OK:
            s.frame_count += frame_list[i]
            errors.append(None)
        else:
            try:
                _raise_status(st_l[i], s.frame_count + er_l[i])
            except (DecodeError, MemoryError) as e:
                errors.append(e)
    if raise_first:
        for e in errors:
            if e is not None:
                raise e
    if not with_best:
        return errors
    if rc == -2:  # (the word window was too small: the chunk is committed, ask again)
        return errors, _best_lanes(pool, states)
    return errors, _hyps_from(n, words, woff, cost, fc, bst)


def _hyps_from(n, words, woff, cost, fc, st) -> list:
    out = []
    # (one conversion to Python objects per array, then plain list slicing)
    wl, ol, cl, fl, sl = words[:int(woff[n])].tolist(), woff.tolist(), cost.tolist(), fc.tolist(), st.tolist()
    for i in range(n):
        if sl[i] == 2:
            out.append(DecodeError("no frames decoded"))
        elif sl[i] == 1:
            out.append(DecodeError("no surviving hypotheses"))
        else:
            out.append(Hypothesis(words=tuple(wl[ol[i]:ol[i + 1]]), total_cost=cl[i], frame_count=fl[i]))
    return out


def _pack_rows(mats, on_dev, packed, frames, width):
    """(buffer, element offsets, base pointer, dtype code, location) of the
    log-likelihood rows of several channels: one contiguous host or device
    buffer (an already-packed (n, F, V) block is used as is)."""
    n = len(mats)
    if packed is not None:
        buf, offs = packed
        offs = np.asarray(offs, np.int64)
    elif on_dev:
        import torch

        dt = torch.float64 if any(m.dtype == torch.float64 for m in mats) else torch.float32
        buf = mats[0].to(dt).contiguous() if n == 1 else torch.cat([m.to(dt).reshape(-1) for m in mats])
        offs = None
    else:
        dt = np.float64 if any(m.dtype != np.float32 for m in mats) else np.float32
        buf = np.ascontiguousarray(mats[0], dt) if n == 1 else np.concatenate(
            [np.ascontiguousarray(m, dt).reshape(-1) for m in mats])
        offs = None
    if offs is None:
        offs = np.zeros(n, np.int64)
        if n > 1:
            np.cumsum(frames[:-1].astype(np.int64) * width, out=offs[1:])
    if on_dev:
        import torch

        torch.cuda.current_stream(buf.device).synchronize()
        base, dcode, loc = buf.data_ptr(), (1 if buf.dtype == torch.float64 else 0), 1
    else:
        base, dcode, loc = buf.ctypes.data, (1 if buf.dtype == np.float64 else 0), 0
    return buf, offs, base, dcode, loc


def _best_lanes(pool: LanePool, states: Sequence[DecodeState]) -> list:
    """Batched best_path (one launch); returns Hypothesis or DecodeError per channel."""
    n = len(states)
    ids = np.asarray([s._lane for s in states], np.int32)
    cap = int(sum(s.frame_count + 8 for s in states)) + 16
    L = _lib.load()
    while True:
        words = np.zeros(cap, np.int32)
        woff = np.zeros(n + 1, np.int64)
        cost = np.zeros(n, np.float64)
        fc = np.zeros(n, np.int64)
        st = np.zeros(n, np.int32)
        rc = L.ctw_best_path(pool.handle, _lib.ptr(ids), n, _lib.ptr(words), cap, _lib.ptr(woff),
                             _lib.ptr(cost), _lib.ptr(fc), _lib.ptr(st))
        if rc == -2:
            cap = int(woff[n]) + 16
            continue
        _lib.check(rc, "best path")
        break
    return _hyps_from(n, words, woff, cost, fc, st)


# ------------------------------------------------------------- functions ---


def create_channel(graph, config: DecoderConfig | None = None) -> DecodeState:
    """Fresh channel: start token with its epsilon closure, zero frames."""
    return DecodeState(flatten(graph), config if config is not None else DecoderConfig())


def advance(ch: DecodeState, frame):
    """Process one frame of log-likelihoods (one value per acoustic token)."""
    row = np.ascontiguousarray(frame, dtype=np.float64)
    if row.ndim != 1:
        raise DecodeError("advance takes a single frame vector; see advance_frames")
    ch.advance_frames(row[None, :])


def prune(tokens: Sequence[Token], beam: float, max_active: int) -> list[Token]:
    """Reference pruning rule (decoder.py:361-374): keep cost <= min + beam,
    then the max_active smallest by (cost, state), returned in state order.
    The device kernel implements the same selection (radix select)."""
    if not tokens:
        raise ValueError("prune needs a non-empty token set")
    cutoff = min(t.cost for t in tokens) + beam
    kept = [t for t in tokens if t.cost <= cutoff]
    if len(kept) > max_active:
        kept = sorted(kept, key=lambda t: (t.cost, t.state))[:max_active]
    return sorted(kept, key=lambda t: t.state)


def best_path(ch: DecodeState) -> Hypothesis:
    """Least-cost hypothesis, preferring final states (decoder.py:377-415);
    the channel is left untouched."""
    if ch.frame_count == 0:
        raise DecodeError("no frames decoded")
    if ch._pool is not None:
        r = _best_lanes(ch._pool, [ch])[0]
        if isinstance(r, Exception):
            raise r
        return r
    fg = ch.graph
    best_i, best, any_final = -1, INF, False
    for i, (s, c) in enumerate(zip(ch._h_state, ch._h_cost)):
        fw = fg.final[s]
        if fw != INF and (not any_final or c + fw < best):
            any_final, best, best_i = True, c + fw, i
    if not any_final:
        for i, c in enumerate(ch._h_cost):
            if c < best:
                best, best_i = c, i
    if best_i < 0:
        raise DecodeError("no surviving hypotheses")
    segs = []
    rec = int(ch._h_bp[best_i])
    while rec >= 0:
        f = bisect.bisect_right(ch.frame_base, rec) - 1
        prev, _, _, ooff, opool = ch.frames[f]
        i = rec - ch.frame_base[f]
        segs.append(opool[ooff[i]:ooff[i + 1]])
        rec = int(prev[i])
    words = tuple(int(o) for seg in reversed(segs) for o in seg)
    return Hypothesis(words=words, total_cost=float(best), frame_count=ch.frame_count)


def decode_utterance(graph, config: DecoderConfig, loglik, boost: np.ndarray | None = None) -> Hypothesis:
    """Offline decode of one utterance (whole log-likelihood matrix)."""
    ch = create_channel(graph, config)
    if boost is not None:
        ch.set_boost(boost)
    ch.advance_frames(loglik)
    return best_path(ch)


def decode_batch(graph, config: DecoderConfig, utterances: Sequence, workers: int = 1, boost=None,
                 *, device: int | None = None, max_lanes: int | None = None, lattice_beam: float | None = None,
                 search: str = "exact") -> list:
    """Decode utterances independently; results keep the input order,
    failures are reported per index (decoder.py:436-463).

    All utterances of a group of ``max_lanes`` (default: all) are decoded as
    lanes of ONE kernel launch; ``workers`` is accepted for signature
    compatibility (parallelism is the lane batch). ``boost`` is one dense
    vector for every utterance, or a sequence with one vector/None per
    utterance (per-utterance boosting). ``search="fast"`` selects the
    words-exact throughput mode (identical words; see ``SEARCH_MODES``)."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    fg = flatten(graph)
    n = len(utterances)
    per_utt = boost is not None and not isinstance(boost, np.ndarray) and isinstance(boost, (list, tuple))
    if per_utt and len(boost) != n:
        raise ValueError("per-utterance boost list must match the number of utterances")
    results: list = [None] * n
    pool = fg.device_graph(device).pool(config, fg.num_states, search)
    group = _auto_group(pool, config, utterances, n) if max_lanes is None else max(1, int(max_lanes))
    for g0 in range(0, n, group):
        _decode_split(fg, config, pool, utterances, list(range(g0, min(n, g0 + group))), boost, per_utt, results,
                      lattice_beam)
    return results


def _auto_group(pool: "LanePool", config: DecoderConfig, utterances, n: int) -> int:
    """Lanes per launch when the caller does not say: everything that fits in
    the device's free memory (history reserved at min(max_active, 65536)
    records x 20 B per frame, as ctw_advance pre-sizes it, plus ~8 MB of
    table-sized buffers per lane), at least 64."""
    if n <= 64:
        return n
    try:
        import torch

        free, _ = torch.cuda.mem_get_info(pool.dg.device)
        frames = int(utterances.shape[1]) if getattr(utterances, "ndim", 0) == 3 else \
            max(int(np.shape(u)[0]) for u in utterances)
    except Exception:  # noqa: BLE001 - no estimate: one group, OOM splits below
        return n
    per_lane = 20 * min(config.max_active, 65536) * max(1, frames) + (8 << 20)
    return max(64, min(n, len(pool.free) + int(0.8 * free) // per_lane))


def _decode_split(fg, config, pool, utterances, idx, boost, per_utt, results, lattice_beam):
    """_decode_group, halving the group when the device runs out of memory;
    a single utterance that does not fit fails with MemoryError at its index
    (the reference's C_ERR_OOM, _kernel.pyx:491-492)."""
    try:
        _decode_group(fg, config, pool, utterances, idx, boost, per_utt, results, lattice_beam)
    except RuntimeError as e:
        if "out of memory" not in str(e):
            raise
        if len(idx) == 1:
            results[idx[0]] = DecodeFailure(idx[0], MemoryError(str(e)))
            return
        h = len(idx) // 2
        _decode_split(fg, config, pool, utterances, idx[:h], boost, per_utt, results, lattice_beam)
        _decode_split(fg, config, pool, utterances, idx[h:], boost, per_utt, results, lattice_beam)


def _packed_source(utterances, device: int | None = None):
    """(buffer, on_device, frames, width) when the batch is one contiguous
    (n, F, V) numpy array or CUDA tensor -- decoded without per-utterance
    copies; else None."""
    if isinstance(utterances, np.ndarray) and utterances.ndim == 3:
        a = utterances if utterances.dtype in (np.float32, np.float64) else utterances.astype(np.float64)
        return np.ascontiguousarray(a), False
    try:
        import torch
    except ImportError:  # pragma: no cover
        return None
    if isinstance(utterances, torch.Tensor) and utterances.ndim == 3:
        t = utterances if utterances.dtype in (torch.float32, torch.float64) else utterances.double()
        if t.is_cuda:
            if device is not None:
                t = _to_lane_device(t, device)
            return t.contiguous(), True
        return np.ascontiguousarray(t.numpy()), False
    return None


def _decode_group(fg, config, pool: LanePool, utterances, idx, boost, per_utt, results, lattice_beam=None):
    lanes = pool.acquire(len(idx))
    packed_src = _packed_source(utterances, pool.dg.device)
    try:
        boosts = [(boost[i] if per_utt else boost) for i in idx]
        st = pool.reset(lanes, boosts)
        chans, mats, order, dev_flags = [], [], [], []
        for k, i in enumerate(idx):
            ch = DecodeState.__new__(DecodeState)
            ch.graph, ch.config, ch.frame_count, ch.num_tokens = fg, config, 0, None
            ch._boost, ch._kernel, ch._pool, ch._lane, ch._cache = boosts[k], None, pool, lanes[k], None
            if st[k] != _lib.OK:
                results[i] = DecodeFailure(i, DecodeError("epsilon iteration cap exceeded while seeding the channel"))
                continue
            try:
                x, on_dev = ((packed_src[0][i], packed_src[1]) if packed_src is not None
                             else _as_frames(utterances[i], pool.dg.device))
                if x.ndim != 2:
                    raise DecodeError("log-likelihoods must be a (frames, tokens) matrix")
                if x.shape[0] == 0:
                    raise DecodeError("no frames decoded")
                ch._check_width(int(x.shape[1]))
            except Exception as e:  # noqa: BLE001 - reported per index
                results[i] = DecodeFailure(i, e)
                continue
            chans.append(ch)
            mats.append(x)
            order.append(i)
            dev_flags.append(on_dev)
        # one launch per (width, location) class -- normally exactly one
        classes: dict = {}
        for k in range(len(chans)):
            classes.setdefault((int(mats[k].shape[1]), dev_flags[k]), []).append(k)
        for (_, on_dev), ks in classes.items():
            packed = None
            if packed_src is not None:
                buf = packed_src[0]
                per = int(buf.shape[1]) * int(buf.shape[2])
                packed = (buf, [order[k] * per for k in ks])
            errs = _advance_lanes(pool, [chans[k] for k in ks], [mats[k] for k in ks], on_dev,
                                  raise_first=False, packed=packed)
            ok = [k for k, e in zip(ks, errs) if e is None]
            for k, e in zip(ks, errs):
                if e is not None:
                    results[order[k]] = DecodeFailure(order[k], e)
            if ok:
                hyps = _best_lanes(pool, [chans[k] for k in ok])
                for k, h in zip(ok, hyps):
                    results[order[k]] = DecodeFailure(order[k], h) if isinstance(h, Exception) else h
                if lattice_beam is not None:
                    from .lattice import build_lattices

                    lk = [k for k, h in zip(ok, hyps) if not isinstance(h, Exception)]
                    if lk:
                        pk = None
                        if packed is not None:
                            pos = {k: j for j, k in enumerate(ks)}
                            pk = (packed[0], [packed[1][pos[k]] for k in lk])
                        lats = build_lattices(pool, [chans[k] for k in lk], [mats[k] for k in lk], on_dev, pk,
                                              [results[order[k]] for k in lk], lattice_beam)
                        for k, lat in zip(lk, lats):
                            results[order[k]] = DecodeFailure(order[k], lat) if isinstance(lat, Exception) else lat
    finally:
        pool.release(lanes)
