"""Binary CSR graph files (the graph load path at scale).

The reference loads graphs from AT&T text (``wfst.read_fst_text``,
wfst.py:213-268, ~9 s per 2.5 M arcs) and flattens them in Python
(``flatten``, decoder.py:130-138). A ``.ctwg`` file stores the flattened
arrays (decoder.py:70-127 layout) directly, so loading is a memory map and
``ctw_graph_load`` (C-ABI) can put a graph in HBM without any Python:

    offset 0   char[8]  "CTWGRAPH"
               u32 version (1), u32 flags (0)
               i64 num_states, num_arcs, start, max_ilabel, max_olabel
    offset 64  i64 off[S+1] | i64 eps_end[S] | i32 ilabel[A] | i32 olabel[A]
               | f64 weight[A] | i32 nextstate[A] | f64 final[S]
               (each array starts on an 8-byte boundary; little endian)
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .decoder import FlatGraph, flatten
from .errors import GraphError

MAGIC = b"CTWGRAPH"
VERSION = 1
HEADER = 64

_LAYOUT = (("off", np.int64, "S1"), ("eps_end", np.int64, "S"), ("ilabel", np.int32, "A"),
           ("olabel", np.int32, "A"), ("weight", np.float64, "A"), ("nextstate", np.int32, "A"),
           ("final", np.float64, "S"))


def _sizes(S: int, A: int):
    n = {"S1": S + 1, "S": S, "A": A}
    off = HEADER
    out = []
    for name, dt, k in _LAYOUT:
        cnt = n[k]
        out.append((name, dt, off, cnt))
        off += cnt * np.dtype(dt).itemsize
        off = (off + 7) & ~7
    return out, off


def save_graph(graph, path) -> Path:
    """Write any graph ``flatten`` accepts as a .ctwg file."""
    fg = flatten(graph)
    path = Path(path)
    S, A = int(fg.num_states), int(fg.num_arcs)
    layout, total = _sizes(S, A)
    hdr = np.zeros(HEADER, np.uint8)
    hdr[:8] = np.frombuffer(MAGIC, np.uint8)
    hdr[8:16] = np.frombuffer(np.array([VERSION, 0], np.uint32).tobytes(), np.uint8)
    hdr[16:56] = np.frombuffer(np.array([S, A, fg.start, fg.max_ilabel, fg.max_olabel], np.int64).tobytes(), np.uint8)
    with open(path, "wb") as f:
        f.write(hdr.tobytes())
        pos = HEADER
        for name, dt, off, cnt in layout:
            if off > pos:
                f.write(b"\0" * (off - pos))
            a = np.ascontiguousarray(getattr(fg, name), dt)
            if len(a) != cnt:
                raise GraphError(f"{name} has {len(a)} entries, expected {cnt}")
            f.write(a.tobytes())
            pos = off + a.nbytes
        if total > pos:
            f.write(b"\0" * (total - pos))
    return path


def load_graph(path, mmap: bool = True) -> FlatGraph:
    """Read a .ctwg file into a FlatGraph (arrays memory-mapped by default)."""
    path = Path(path)
    head = np.fromfile(path, np.uint8, count=HEADER)
    if len(head) < HEADER or head[:8].tobytes() != MAGIC:
        raise GraphError(f"{path}: not a CTWGRAPH file")
    ver = int(np.frombuffer(head[8:12].tobytes(), np.uint32)[0])
    if ver != VERSION:
        raise GraphError(f"{path}: unsupported version {ver}")
    S, A, start, mil, mol = (int(x) for x in np.frombuffer(head[16:56].tobytes(), np.int64))
    layout, total = _sizes(S, A)
    if path.stat().st_size < total:
        raise GraphError(f"{path}: truncated ({path.stat().st_size} < {total} bytes)")
    fg = FlatGraph()
    fg.num_states, fg.start, fg.max_ilabel, fg.max_olabel = S, start, mil, mol
    for name, dt, off, cnt in layout:
        if mmap:
            a = np.memmap(path, dtype=dt, mode="r", offset=off, shape=(cnt,))
        else:
            with open(path, "rb") as f:
                f.seek(off)
                a = np.fromfile(f, dtype=dt, count=cnt)
        setattr(fg, name, a)
    if S <= 0 or not (0 <= start < S) or int(fg.off[-1]) != A:
        raise GraphError(f"{path}: inconsistent header / CSR")
    return fg
