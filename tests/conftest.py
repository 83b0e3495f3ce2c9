"""Shared test setup.

Markers: ``gpu`` = needs a CUDA device (run on the B200 box with -m gpu).
Everything else runs on CPU. ``oracle/`` (the CPU restatement + the compiled
reference in oracle/_ref) is test infrastructure and is imported only here
and in the tests.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_names():
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load_golden(name):
    d = dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
    for k in ("num_states", "start", "max_active", "max_ne_iters", "ok_chunks", "frame_count"):
        d[k] = int(d[k])
    for k in ("beam", "acoustic_scale", "relax_eps", "best_cost"):
        d[k] = float(d[k])
    d["has_boost"] = bool(d["has_boost"])
    d["boost_poke"] = bool(d["boost_poke"])
    d["error"] = str(d["error"])
    return d


class GoldenGraph:
    """FlatGraph-shaped view of a fixture (what both decoders accept)."""

    def __init__(self, d):
        self.num_states = d["num_states"]
        self.start = d["start"]
        for k in ("off", "eps_end", "ilabel", "olabel", "weight", "nextstate", "final"):
            setattr(self, k, d[k])
        self.max_ilabel = int(d["ilabel"].max()) if len(d["ilabel"]) else 0
        self.max_olabel = int(d["olabel"].max()) if len(d["olabel"]) else 0


def golden_chunks(d):
    cuts = np.cumsum(d["chunk_sizes"])[:-1]
    return np.split(d["frames"], cuts) if len(d["chunk_sizes"]) else []


def expected_history(d):
    out, i, j = [], 0, 0
    for n in d["counts"].tolist():
        rows = []
        for _ in range(n):
            k = int(d["rec_olab_len"][i])
            rows.append((int(d["rec_prev"][i]), tuple(int(x) for x in d["rec_olab"][j:j + k]),
                         int(d["rec_state"][i]), float(d["rec_cost"][i])))
            i += 1
            j += k
        out.append(rows)
    return out


def ref_available() -> bool:
    sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
    try:
        import ctcwfst  # noqa: F401
    except ImportError:
        return False
    return True


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.build_lib()
    return oracle


def history_signature(hist):
    """Tie-insensitive view of a history: per frame, the sorted records as
    (state, cost, olabels, transcript-so-far) where the transcript follows
    the prev chain to the root. Two decoders that pick different but
    exactly-tied predecessors (same cost) yield the same signature as long as
    the tied paths carry the same words."""
    words = {}
    out = []
    base = 0
    for frame in hist:
        rows = []
        for k, (prev, ols, state, cost) in enumerate(frame):
            w = (words[prev] if prev >= 0 else ()) + tuple(ols)
            words[base + k] = w
            rows.append((state, cost, tuple(ols), w))
        base += len(frame)
        out.append(sorted(rows))
    return out


def assert_history_equivalent(got, want, exact_prev=True):
    if exact_prev:
        assert got == want
        return
    assert [len(f) for f in got] == [len(f) for f in want]
    assert history_signature(got) == history_signature(want)
