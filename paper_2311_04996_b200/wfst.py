"""Graph load: WFST container, AT&T text I/O and symbol tables.

This is the "graph load" entry of the decode API. It mirrors the reference's
public surface (pkg/src/ctcwfst/wfst.py: ``Arc`` :39-43, ``SymbolTable``
:46-95, ``read_symbols`` :98-124, ``Wfst`` :131-210, ``read_fst_text``
:213-268, ``write_fst_text`` :271-291, ``arc_sort`` :294-304) so graphs built
or loaded for the reference load unchanged here. Offline construction
algorithms (compose/connect) are out of scope for the decode path; the
benchmark graphs are synthesised natively by ``synth.py``.

Weights are tropical costs (lower is better); +inf final weight = non-final.
"""

from __future__ import annotations

import math
from typing import Iterator, NamedTuple

from .errors import FstParseError, SymbolTableError

EPSILON = 0
NO_STATE = -1
INF = math.inf


class Arc(NamedTuple):
    ilabel: int
    olabel: int
    weight: float
    nextstate: int


class SymbolTable:
    """Bijective symbol <-> id map; id 0 is the epsilon symbol."""

    def __init__(self, epsilon_symbol: str = "<eps>"):
        self._by_sym: dict[str, int] = {epsilon_symbol: EPSILON}
        self._by_id: dict[int, str] = {EPSILON: epsilon_symbol}

    def add(self, symbol: str, sym_id: int | None = None) -> int:
        have = self._by_sym.get(symbol)
        if have is not None:
            if sym_id is not None and sym_id != have:
                raise SymbolTableError(f"symbol {symbol!r} already mapped to id {have}")
            return have
        if sym_id is None:
            sym_id = max(self._by_id) + 1
        elif sym_id < 0:
            raise SymbolTableError(f"negative symbol id {sym_id}")
        elif sym_id in self._by_id:
            raise SymbolTableError(f"id {sym_id} already mapped to {self._by_id[sym_id]!r}")
        self._by_sym[symbol] = sym_id
        self._by_id[sym_id] = symbol
        return sym_id

    def id(self, symbol: str) -> int:
        if symbol not in self._by_sym:
            raise SymbolTableError(f"unknown symbol {symbol!r}")
        return self._by_sym[symbol]

    def symbol(self, sym_id: int) -> str:
        if sym_id not in self._by_id:
            raise SymbolTableError(f"unknown symbol id {sym_id}")
        return self._by_id[sym_id]

    def __contains__(self, symbol: str) -> bool:
        return symbol in self._by_sym

    def __len__(self) -> int:
        return len(self._by_sym)

    def items(self) -> Iterator[tuple[str, int]]:
        return iter(sorted(self._by_sym.items(), key=lambda kv: kv[1]))

    def max_id(self) -> int:
        return max(self._by_id)


def read_symbols(text: str) -> SymbolTable:
    """``symbol id`` per line; the first entry must map epsilon to 0."""
    table: SymbolTable | None = None
    for lineno, raw in enumerate(text.splitlines(), start=1):
        fields = raw.split()
        if not fields:
            continue
        if len(fields) != 2:
            raise FstParseError(f"expected 'symbol id', got {raw!r}", lineno)
        try:
            sym_id = int(fields[1])
        except ValueError:
            raise FstParseError(f"bad symbol id {fields[1]!r}", lineno) from None
        if table is None:
            if sym_id != 0:
                raise FstParseError("first entry must map the epsilon symbol to 0", lineno)
            table = SymbolTable(epsilon_symbol=fields[0])
            continue
        try:
            table.add(fields[0], sym_id)
        except SymbolTableError as e:
            raise FstParseError(str(e), lineno) from None
    if table is None:
        raise FstParseError("empty symbol table")
    return table


def write_symbols(table: SymbolTable) -> str:
    return "".join(f"{s} {i}\n" for s, i in table.items())


class Wfst:
    """States 0..n-1 with per-state arc lists and a final-cost map."""

    __slots__ = ("start", "_arcs", "finals", "_flat")

    def __init__(self, num_states: int = 0, start: int = NO_STATE):
        self.start = start
        self._arcs: list[list[Arc]] = [[] for _ in range(num_states)]
        self.finals: dict[int, float] = {}
        self._flat = None  # decoder-side cache (FlatGraph), see decoder.flatten

    @classmethod
    def empty(cls) -> "Wfst":
        return cls(0, NO_STATE)

    @property
    def num_states(self) -> int:
        return len(self._arcs)

    @property
    def is_empty(self) -> bool:
        return not self._arcs

    def _valid(self, s: int) -> None:
        if not 0 <= s < len(self._arcs):
            raise ValueError(f"state {s} out of range (num_states={len(self._arcs)})")

    def add_state(self) -> int:
        self._arcs.append([])
        return len(self._arcs) - 1

    def add_states(self, n: int) -> None:
        for _ in range(n):
            self._arcs.append([])

    def set_start(self, state: int) -> None:
        self._valid(state)
        self.start = state

    def add_arc(self, state: int, arc: Arc) -> None:
        self._valid(state)
        self._valid(arc.nextstate)
        self._arcs[state].append(arc)

    def set_final(self, state: int, weight: float = 0.0) -> None:
        self._valid(state)
        if weight == INF:
            self.finals.pop(state, None)
        else:
            self.finals[state] = weight

    def final(self, state: int) -> float:
        return self.finals.get(state, INF)

    def is_final(self, state: int) -> bool:
        return state in self.finals

    def arcs(self, state: int) -> list[Arc]:
        return self._arcs[state]

    def states(self) -> range:
        return range(len(self._arcs))

    def num_arcs(self) -> int:
        return sum(map(len, self._arcs))

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, Wfst):
            return NotImplemented
        return (self.start, self._arcs, self.finals) == (other.start, other._arcs, other.finals)

    def __repr__(self) -> str:
        return (f"Wfst(states={self.num_states}, arcs={self.num_arcs()}, start={self.start}, "
                f"finals={len(self.finals)})")


def _int_field(tok: str, what: str, lineno: int) -> int:
    try:
        v = int(tok)
    except ValueError:
        raise FstParseError(f"bad {what} {tok!r}", lineno) from None
    if v < 0:
        raise FstParseError(f"negative {what} {v}", lineno)
    return v


def _weight_field(tok: str, lineno: int) -> float:
    try:
        return float(tok)
    except ValueError:
        raise FstParseError(f"bad weight {tok!r}", lineno) from None


def read_fst_text(text: str) -> Wfst:
    """AT&T text: ``src dst ilabel olabel [weight]`` arc lines and
    ``state [weight]`` final lines; the first line's state is the start;
    missing weights are 0."""
    arcs: list[tuple[int, Arc]] = []
    finals: dict[int, float] = {}
    start = NO_STATE
    top = -1
    for lineno, raw in enumerate(text.splitlines(), start=1):
        f = raw.split()
        n = len(f)
        if n == 0:
            continue
        if n == 1 or n == 2:
            s = _int_field(f[0], "state", lineno)
            finals[s] = _weight_field(f[1], lineno) if n == 2 else 0.0
            top = max(top, s)
            if start == NO_STATE:
                start = s
        elif n == 4 or n == 5:
            src = _int_field(f[0], "state", lineno)
            dst = _int_field(f[1], "state", lineno)
            il = _int_field(f[2], "input label", lineno)
            ol = _int_field(f[3], "output label", lineno)
            w = _weight_field(f[4], lineno) if n == 5 else 0.0
            arcs.append((src, Arc(il, ol, w, dst)))
            top = max(top, src, dst)
            if start == NO_STATE:
                start = src
        else:
            raise FstParseError(f"expected 2, 4, or 5 fields, got {n}", lineno)
    if start == NO_STATE:
        raise FstParseError("no states found")
    g = Wfst(top + 1, start)
    for src, arc in arcs:
        g.add_arc(src, arc)
    for s, w in finals.items():
        g.set_final(s, w)
    return g


def _fmt_weight(w: float) -> str:
    if math.isfinite(w) and w == math.floor(w) and abs(w) < 1e16:
        return str(int(w))
    return repr(w)


def write_fst_text(g: Wfst) -> str:
    """Inverse of ``read_fst_text`` (start state first, weights always written)."""
    if g.is_empty:
        return ""
    lines: list[str] = []
    order = [g.start] + [s for s in g.states() if s != g.start]
    for s in order:
        for a in g.arcs(s):
            lines.append(f"{s} {a.nextstate} {a.ilabel} {a.olabel} {_fmt_weight(a.weight)}\n")
        if g.is_final(s):
            lines.append(f"{s} {_fmt_weight(g.final(s))}\n")
    return "".join(lines)


def arc_sort(g: Wfst, key: str = "ilabel") -> Wfst:
    """Copy with each state's arcs stably sorted by ``ilabel`` or ``olabel``."""
    if key not in ("ilabel", "olabel"):
        raise ValueError(f"sort key must be 'ilabel' or 'olabel', got {key!r}")
    field = 0 if key == "ilabel" else 1
    out = Wfst(g.num_states, g.start)
    for s in g.states():
        for a in sorted(g.arcs(s), key=lambda arc: arc[field]):
            out.add_arc(s, a)
    out.finals = dict(g.finals)
    return out
