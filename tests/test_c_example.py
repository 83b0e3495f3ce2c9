"""The C-ABI without Python: examples/c_decode.c compiles against
include/ctcwfst_b200.h and links libctcwfst_b200.so (CPU); on a GPU its
transcripts and costs equal decode_batch's for the same graph file and
log-likelihoods."""

import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2311_04996_b200"


def _build(tmp_path) -> Path:
    exe = tmp_path / "c_decode"
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", str(ROOT / "include"), str(ROOT / "examples" / "c_decode.c"),
                    "-L", str(PKG), "-lctcwfst_b200", f"-Wl,-rpath,{PKG}", "-o", str(exe)], check=True)
    return exe


def test_c_example_builds_and_links(tmp_path):
    exe = _build(tmp_path)
    assert exe.exists()


@pytest.mark.gpu
def test_c_example_matches_python(tmp_path):
    from paper_2311_04996_b200 import DecoderConfig, decode_batch, save_graph, synth

    s = synth.build_system(synth.SystemSpec(num_units=12, num_words=40, order=3, seed=4, min_pron=1, max_pron=4))
    n, F = 5, 60
    ll = np.stack(synth.planted_utterances(s, n, F, seed=3, gap=4.0, noise=1.0)).astype(np.float32)
    g = save_graph(s.graph, tmp_path / "g.ctwg")
    (tmp_path / "ll.f32").write_bytes(ll.tobytes())
    exe = _build(tmp_path)
    out = subprocess.run([str(exe), str(g), str(tmp_path / "ll.f32"), str(n), str(F), str(ll.shape[2])],
                         check=True, capture_output=True, text=True).stdout.split("\n")
    want = decode_batch(s.graph, DecoderConfig(), list(ll))
    for line, h in zip(out, want):
        parts = line.split()
        assert float(parts[1]) == h.total_cost
        assert tuple(int(x) for x in parts[2:]) == h.words
