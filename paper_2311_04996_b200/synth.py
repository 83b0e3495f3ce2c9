"""Synthetic CTC decoding systems: T o L o G graphs and planted log-probs.

The benchmark workloads of BASELINE.json need
TLG graphs up to millions of arcs on a box without the reference tree, built in
seconds: the reference's pure-Python builders take ~35 s per 2.5M arcs. This
module restates the reference's graph semantics on numpy arrays and composes
them with the native builder (csrc/ctw_graphbuild.cpp):

  T  compact CTC topology          topology.py:94-112
  L  left-pushed lexicon + closure lexicon.py:59-87
  G  ARPA backoff acceptor         arpa.py:140-205  (random, NON-uniform n-gram
     probabilities with explicit n-grams clamped to beat their backoff route,
     as in the reference's test generator tests/conftest.py:66-107 -- uniform
     weights make tied hypotheses common)
  TLG = arc_sort(connect(compose(T, compose(L, G))))   graph.py:9-17

Log-probs: CTC-style planted paths (a random word sequence rendered as unit
repeats + blanks, tests/conftest.py:135-163 / benchmark.py:54-81), either as
the reference's gap/noise matrices or as log-softmax of noisy logits
(Conformer-shaped, blank-dominant).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .decoder import FlatGraph

LN10 = math.log(10.0)
INF = math.inf


# ------------------------------------------------------------- FST arrays --


class Fst:
    """CSR FST in numpy arrays (arcs grouped by source state)."""

    def __init__(self, num_states, start, src, il, ol, w, ns, final):
        src = np.asarray(src, np.int64)
        order = np.argsort(src, kind="stable")
        self.num_states = int(num_states)
        self.start = int(start)
        self.ilabel = np.ascontiguousarray(np.asarray(il, np.int32)[order])
        self.olabel = np.ascontiguousarray(np.asarray(ol, np.int32)[order])
        self.weight = np.ascontiguousarray(np.asarray(w, np.float64)[order])
        self.nextstate = np.ascontiguousarray(np.asarray(ns, np.int32)[order])
        self.off = np.zeros(self.num_states + 1, np.int64)
        if len(src):
            np.cumsum(np.bincount(src, minlength=self.num_states), out=self.off[1:])
        self.final = np.ascontiguousarray(np.asarray(final, np.float64))

    @property
    def num_arcs(self) -> int:
        return int(self.off[-1])

    def to_flat(self) -> FlatGraph:
        src = np.repeat(np.arange(self.num_states, dtype=np.int64), np.diff(self.off))
        return FlatGraph.from_arrays(self.num_states, self.start, src, self.ilabel, self.olabel, self.weight,
                                     self.nextstate, self.final)

    def to_wfst(self):
        from .wfst import Arc, Wfst

        g = Wfst(self.num_states, self.start)
        for s in range(self.num_states):
            for k in range(self.off[s], self.off[s + 1]):
                g.add_arc(s, Arc(int(self.ilabel[k]), int(self.olabel[k]), float(self.weight[k]),
                                 int(self.nextstate[k])))
            if self.final[s] != INF:
                g.set_final(s, float(self.final[s]))
        return g

    @classmethod
    def from_wfst(cls, g) -> "Fst":
        src, il, ol, w, ns = [], [], [], [], []
        for s in g.states():
            for a in g.arcs(s):
                src.append(s)
                il.append(a.ilabel)
                ol.append(a.olabel)
                w.append(a.weight)
                ns.append(a.nextstate)
        fin = np.full(g.num_states, INF)
        for s, v in g.finals.items():
            fin[s] = v
        return cls(g.num_states, g.start, src, il, ol, w, ns, fin)


class _CFst(C.Structure):
    _fields_ = [("num_states", C.c_int64), ("num_arcs", C.c_int64), ("start", C.c_int64),
                ("off", C.POINTER(C.c_int64)), ("ilabel", C.POINTER(C.c_int32)),
                ("olabel", C.POINTER(C.c_int32)), ("weight", C.POINTER(C.c_double)),
                ("nextstate", C.POINTER(C.c_int32)), ("final_w", C.POINTER(C.c_double))]


def _graphlib():
    L = _lib.load(require_gpu=False)
    if not getattr(L, "_ctw_fst_ready", False):
        for name in ("ctw_fst_compose",):
            getattr(L, name).argtypes = [C.POINTER(_CFst), C.POINTER(_CFst), C.POINTER(_CFst)]
            getattr(L, name).restype = C.c_int
        for name in ("ctw_fst_connect", "ctw_fst_arcsort_ilabel"):
            getattr(L, name).argtypes = [C.POINTER(_CFst), C.POINTER(_CFst)]
            getattr(L, name).restype = C.c_int
        L.ctw_fst_free.argtypes = [C.POINTER(_CFst)]
        L._ctw_fst_ready = True
    return L


def _to_c(f: Fst) -> _CFst:
    c = _CFst()
    c.num_states, c.num_arcs, c.start = f.num_states, f.num_arcs, f.start
    c.off = f.off.ctypes.data_as(C.POINTER(C.c_int64))
    c.ilabel = f.ilabel.ctypes.data_as(C.POINTER(C.c_int32))
    c.olabel = f.olabel.ctypes.data_as(C.POINTER(C.c_int32))
    c.weight = f.weight.ctypes.data_as(C.POINTER(C.c_double))
    c.nextstate = f.nextstate.ctypes.data_as(C.POINTER(C.c_int32))
    c.final_w = f.final.ctypes.data_as(C.POINTER(C.c_double))
    return c


def _from_c(c: _CFst) -> Fst:
    n, a = c.num_states, c.num_arcs

    def arr(p, k, dt):
        return np.ctypeslib.as_array(p, shape=(k,)).astype(dt, copy=True) if k > 0 else np.zeros(0, dt)

    off = arr(c.off, n + 1, np.int64)
    f = Fst.__new__(Fst)
    f.num_states, f.start = int(n), int(c.start)
    f.off = off if n >= 0 else np.zeros(1, np.int64)
    f.ilabel, f.olabel = arr(c.ilabel, a, np.int32), arr(c.olabel, a, np.int32)
    f.weight, f.nextstate = arr(c.weight, a, np.float64), arr(c.nextstate, a, np.int32)
    f.final = arr(c.final_w, n, np.float64)
    _graphlib().ctw_fst_free(C.byref(c))
    return f


def compose(a: Fst, b: Fst) -> Fst:
    out = _CFst()
    ca, cb = _to_c(a), _to_c(b)
    _graphlib().ctw_fst_compose(C.byref(ca), C.byref(cb), C.byref(out))
    return _from_c(out)


def connect(g: Fst) -> Fst:
    out = _CFst()
    cg = _to_c(g)
    _graphlib().ctw_fst_connect(C.byref(cg), C.byref(out))
    return _from_c(out)


def arc_sort(g: Fst) -> Fst:
    out = _CFst()
    cg = _to_c(g)
    _graphlib().ctw_fst_arcsort_ilabel(C.byref(cg), C.byref(out))
    return _from_c(out)


def build_tlg(t: Fst, l: Fst, g: Fst) -> Fst:
    """graph.py:9-17 semantics: arc_sort(connect(compose(T, compose(L, G))))."""
    tlg = connect(compose(t, compose(l, g)))
    if tlg.num_states == 0:
        raise ValueError("empty decoding graph (label alphabets do not chain)")
    return arc_sort(tlg)


# ---------------------------------------------------------- T, L, G build --


def ctc_topo_compact(num_units: int, blank_id: int) -> Fst:
    """topology.py:94-112: start 0 with a blank:eps loop and u:u arcs into
    per-unit states; each unit state loops on u:eps and returns by eps:eps."""
    nb = [u for u in range(num_units) if u != blank_id]
    n = 1 + len(nb)
    src, il, ol, w, ns = [0], [blank_id + 1], [0], [0.0], [0]
    for q, u in enumerate(nb, start=1):
        src.append(0), il.append(u + 1), ol.append(u + 1), w.append(0.0), ns.append(q)
    for q, u in enumerate(nb, start=1):
        src += [q, q]
        il += [u + 1, 0]
        ol += [0, 0]
        w += [0.0, 0.0]
        ns += [q, 0]
    return Fst(n, 0, src, il, ol, w, ns, np.zeros(n))


def lexicon_fst(prons: list[tuple[int, ...]], word_ids: list[int], costs=None) -> Fst:
    """lexicon.py:59-87: every pronunciation leaves the shared start with its
    word id on the first unit arc and loops back by an eps:eps arc."""
    src, il, ol, w, ns = [], [], [], [], []
    n = 1
    for e, (pron, wid) in enumerate(zip(prons, word_ids)):
        prev = 0
        for i, u in enumerate(pron):
            nxt = n
            n += 1
            src.append(prev), il.append(u + 1), ns.append(nxt)
            ol.append(wid if i == 0 else 0)
            w.append(float(costs[e]) if (costs is not None and i == 0) else 0.0)
            prev = nxt
        src.append(prev), il.append(0), ol.append(0), w.append(0.0), ns.append(0)
    fin = np.full(n, INF)
    fin[0] = 0.0
    return Fst(n, 0, src, il, ol, w, ns, fin)


BOS, EOS = -1, -2  # sentence markers inside n-gram tuples


@dataclass
class NgramModel:
    """log10 probabilities / backoffs keyed by word-id tuples (BOS/EOS markers)."""

    max_order: int
    orders: dict = field(default_factory=dict)  # k -> {gram: (logp, backoff or None)}

    def backoff(self, ctx) -> float:
        e = self.orders.get(len(ctx), {}).get(ctx)
        return 0.0 if e is None or e[1] is None else e[1]

    def to_arpa(self, name) -> str:
        """ARPA text (words named by ``name(id)``) for cross-checks with the
        reference parser."""
        sym = {BOS: "<s>", EOS: "</s>"}
        lines = ["\\data\\"] + [f"ngram {k}={len(self.orders[k])}" for k in sorted(self.orders)]
        for k in sorted(self.orders):
            lines += ["", f"\\{k}-grams:"]
            for gram, (lp, bo) in self.orders[k].items():
                words = " ".join(sym.get(x) or name(x) for x in gram)
                lines.append(f"{lp!r}\t{words}" + ("" if bo is None else f"\t{bo!r}"))
        lines += ["", "\\end\\", ""]
        return "\n".join(lines)


def _backoff_route(m: NgramModel, ctx: tuple, w: int, lp1: dict, bows: dict) -> float:
    """log10 p(w | ctx) by the standard backoff recursion over the n-grams
    generated so far (explicit entry, else backoff(ctx) + p(w | ctx[1:]))."""
    if not ctx:
        return lp1[w]
    e = m.orders.get(len(ctx) + 1, {}).get(ctx + (w,))
    if e is not None:
        return e[0]
    ce = m.orders.get(len(ctx), {}).get(ctx)
    bo = (ce[1] if ce is not None and ce[1] is not None else 0.0) if len(ctx) > 1 else bows.get(ctx[0], 0.0)
    return bo + _backoff_route(m, ctx[1:], w, lp1, bows)


def random_ngram(rng, vocab: int, order: int, followers: float = 0.6, tri_contexts: float = 0.3,
                 tri_followers: int = 8) -> NgramModel:
    """Random non-uniform backoff LM over word ids 1..vocab (conftest.py:66-107
    generalised to trigrams). Explicit n-grams are clamped to be at least as
    likely as their backoff route (+0.05 log10), so min-cost graph paths
    follow the deterministic backoff recursion.

    followers: expected bigram followers per context as a fraction of vocab
    (<= 1) or an absolute count (> 1)."""
    words = list(range(1, vocab + 1))
    probs = rng.dirichlet(np.ones(vocab + 1))
    lp1 = {w: math.log10(max(p, 1e-6)) for w, p in zip(words, probs[:-1])}
    lp1[EOS] = math.log10(max(probs[-1], 1e-6))
    m = NgramModel(max_order=max(1, order))
    if order == 1:
        m.orders[1] = {(BOS,): (-99.0, None), (EOS,): (lp1[EOS], None)}
        m.orders[1].update({(w,): (lp1[w], None) for w in words})
        return m
    contexts = [BOS] + words
    bows = {h: math.log10(rng.uniform(0.2, 0.8)) for h in contexts}
    m.orders[1] = {(BOS,): (-99.0, bows[BOS]), (EOS,): (lp1[EOS], None)}
    m.orders[1].update({(w,): (lp1[w], bows[w]) for w in words})
    cand = np.asarray(words + [EOS], np.int64)
    k_mean = followers * (vocab + 1) if followers <= 1 else followers
    big = {}
    for h in contexts:
        k = int(min(len(cand), max(1, rng.poisson(k_mean))))
        fol = rng.choice(cand, size=k, replace=False)
        mass = rng.uniform(0.4, 0.9)
        q = rng.dirichlet(np.ones(k))
        for w, qq in zip(fol.tolist(), q):
            lp2 = max(math.log10(max(mass * qq, 1e-6)), bows[h] + lp1[w] + 0.05)
            big[(h, w)] = [lp2, None]
    m.orders[2] = big
    # orders 3..order: a fraction of the (k-1)-gram histories become contexts
    # (with a backoff weight) and get Poisson(ho_followers) explicit k-grams,
    # clamped above their backoff route like the bigrams
    for k in range(3, order + 1):
        lower = m.orders[k - 1]
        hist = [g for g in lower if g[-1] != EOS]
        frac = tri_contexts if k == 3 else tri_contexts * 0.5
        foll = tri_followers if k == 3 else max(1, tri_followers // 2)
        n_ctx = int(frac * len(hist))
        pick = rng.choice(len(hist), size=n_ctx, replace=False) if n_ctx else []
        cur = {}
        for i in sorted(pick):
            h = hist[i]
            bo = math.log10(rng.uniform(0.2, 0.8))
            lower[h][1] = bo
            kk = int(min(len(cand), max(1, rng.poisson(foll))))
            fol = rng.choice(cand, size=kk, replace=False)
            mass = rng.uniform(0.4, 0.9)
            q = rng.dirichlet(np.ones(kk))
            for w, qq in zip(fol.tolist(), q):
                route = _backoff_route(m, h[1:], w, lp1, bows)
                lp = max(math.log10(max(mass * qq, 1e-6)), bo + route + 0.05)
                cur[h + (w,)] = [lp, None]
        m.orders[k] = cur
    for kk in list(m.orders):
        if kk >= 2:
            m.orders[kk] = {g: (v[0], v[1]) for g, v in m.orders[kk].items()}
    m.max_order = max(2, order)
    return m


def grammar_fst(m: NgramModel) -> Fst:
    """arpa.py:140-205 semantics: one state per n-gram context, word arcs
    weighted -ln(10)*log10 p, eps backoff arcs, </s> as final weights."""
    state_of = {(): 0}
    for k in range(1, m.max_order):
        for gram in m.orders.get(k, {}):
            if gram[-1] != EOS and gram not in state_of:
                state_of[gram] = len(state_of)
    n = len(state_of)

    def dest(gram):
        h = gram[max(0, len(gram) - (m.max_order - 1)):]
        while h and h not in state_of:
            h = h[1:]
        return state_of[h]

    src, il, ol, w, ns = [], [], [], [], []
    fin = np.full(n, INF)
    for k in sorted(m.orders):
        for gram, (lp, _) in m.orders[k].items():
            wd, ctx = gram[-1], gram[:-1]
            s = state_of.get(ctx)
            if s is None:
                continue
            wt = -LN10 * lp
            if wd == EOS:
                if wt < fin[s]:
                    fin[s] = wt
            elif wd != BOS:
                src.append(s), il.append(wd), ol.append(wd), w.append(wt), ns.append(dest(gram))
    for ctx, s in state_of.items():
        if ctx:
            h = ctx[1:]
            while h and h not in state_of:
                h = h[1:]
            src.append(s), il.append(0), ol.append(0), w.append(-LN10 * m.backoff(ctx)), ns.append(state_of[h])
    if not np.isfinite(fin).any():
        fin[:] = 0.0
    return Fst(n, state_of.get((BOS,), 0), src, il, ol, w, ns, fin)


# ---------------------------------------------------------------- systems --


@dataclass
class SystemSpec:
    num_units: int = 30          # acoustic tokens incl. blank (V)
    num_words: int = 50
    order: int = 2
    seed: int = 0
    min_pron: int = 2
    max_pron: int = 7
    blank_id: int = 0
    followers: float = 0.6       # bigram followers per context (fraction or count)
    tri_contexts: float = 0.3
    tri_followers: int = 8


@dataclass
class System:
    spec: SystemSpec
    prons: list
    model: NgramModel
    t: Fst
    l: Fst
    g: Fst
    tlg: Fst
    graph: FlatGraph

    @property
    def num_units(self) -> int:
        return self.spec.num_units


def _draw_prons(spec: SystemSpec, rng) -> list:
    nb = [u for u in range(spec.num_units) if u != spec.blank_id]
    prons: set = set()
    tries = 0
    while len(prons) < spec.num_words:
        ln = int(rng.integers(spec.min_pron, spec.max_pron + 1))
        prons.add(tuple(int(nb[i]) for i in rng.integers(0, len(nb), size=ln)))
        tries += 1
        if tries > 100 * spec.num_words:
            raise ValueError("cannot draw enough distinct pronunciations")
    return sorted(prons)


def system_with_graph(spec: SystemSpec, graph: FlatGraph) -> System:
    """The System of `spec` around an already built graph (e.g. a .ctwg
    written by another process): pronunciations redrawn (what the log-prob
    generators need), grammar / lexicon FSTs not rebuilt."""
    return System(spec, _draw_prons(spec, np.random.default_rng(spec.seed)), None, None, None, None, None, graph)


def build_system(spec: SystemSpec) -> System:
    rng = np.random.default_rng(spec.seed)
    prons_l = _draw_prons(spec, rng)
    model = random_ngram(rng, spec.num_words, spec.order, spec.followers, spec.tri_contexts, spec.tri_followers)
    t = ctc_topo_compact(spec.num_units, spec.blank_id)
    l = lexicon_fst(prons_l, list(range(1, spec.num_words + 1)))
    g = grammar_fst(model)
    tlg = build_tlg(t, l, g)
    return System(spec, prons_l, model, t, l, g, tlg, tlg.to_flat())


def render_path(rng, sys_: System, frames: int) -> list[int]:
    """Random word sequence rendered as CTC units: each unit repeated 1-2
    frames then a blank; only whole words; padded with blanks."""
    blank = sys_.spec.blank_id
    path: list[int] = []
    while True:
        pron = sys_.prons[int(rng.integers(0, len(sys_.prons)))]
        r = []
        for u in pron:
            r.extend([u] * int(rng.integers(1, 3)))
            r.append(blank)
        if len(path) + len(r) > frames:
            break
        path.extend(r)
    path.extend([blank] * (frames - len(path)))
    return path


def planted_utterances(sys_: System, n: int, frames: int, seed: int = 0, gap: float = 12.0,
                       noise: float = 0.5, dtype=np.float64) -> list[np.ndarray]:
    """conftest.py:135-163 style: planted token ~N(-0.05, 0.02), others
    ~N(-gap, noise)."""
    rng = np.random.default_rng(seed)
    out = []
    V = sys_.num_units
    for _ in range(n):
        path = render_path(rng, sys_, frames)
        mat = rng.normal(-gap, noise, size=(frames, V))
        mat[np.arange(frames), path] = rng.normal(-0.05, 0.02, size=frames)
        out.append(mat.astype(dtype))
    return out


def conformer_logprobs(sys_: System, n: int, frames: int, seed: int = 0, delta: float = 6.0,
                       sigma: float = 1.5, dtype=np.float32) -> np.ndarray:
    """(n, frames, V) log-softmax of N(0, sigma) logits with +delta on a
    planted CTC path (blank-dominant, Conformer-CTC shaped). Utterance i
    depends only on (seed, i), not on n."""
    V = sys_.num_units
    out = np.empty((n, frames, V), dtype=dtype)
    for i in range(n):
        rng = np.random.default_rng([seed, i])
        logits = rng.normal(0.0, sigma, size=(frames, V))
        path = render_path(rng, sys_, frames)
        logits[np.arange(frames), path] += delta
        m = logits.max(axis=-1, keepdims=True)
        out[i] = logits - m - np.log(np.exp(logits - m).sum(axis=-1, keepdims=True))
    return out
