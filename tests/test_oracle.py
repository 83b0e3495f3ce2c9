"""The CPU oracle (oracle/ctw_oracle.c) pinned against the reference.

1. Golden vectors generated from the reference itself (tests/golden/).
2. When oracle/_ref (the compiled, unmodified reference) is built: random
   systems decoded by both, history / best path compared bit-for-bit.
"""

import numpy as np
import pytest

from conftest import GoldenGraph, expected_history, golden_chunks, golden_names, load_golden, ref_available


def _cfg(d):
    from oracle import OracleChannel

    return dict(beam=d["beam"], max_active=d["max_active"], acoustic_scale=d["acoustic_scale"],
                relax_eps=d["relax_eps"], max_ne_iters=None if d["max_ne_iters"] < 0 else d["max_ne_iters"])


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_golden(oracle_mod, name):
    d = load_golden(name)
    fg = GoldenGraph(d)
    boost = d["boost"] if d["has_boost"] else None
    ch = oracle_mod.OracleChannel(fg, boost=None if d["boost_poke"] else boost, **_cfg(d))
    if d["boost_poke"]:
        ch.boost = boost
    assert ch.act_state.tolist() == d["seed_state"].tolist()
    assert ch.act_cost.tolist() == d["seed_cost"].tolist()
    err = ""
    for c in golden_chunks(d):
        try:
            ch.advance_frames(c)
        except oracle_mod.OracleError as e:
            err = str(e)
            break
    assert err == d["error"]
    assert ch.history_records() == expected_history(d)
    assert ch.act_state.tolist() == d["tok_state"].tolist()
    assert ch.act_cost.tolist() == d["tok_cost"].tolist()
    assert ch.act_bp.tolist() == d["tok_bp"].tolist()
    if d["frame_count"]:
        words, cost, fc = ch.best_path()
        assert list(words) == d["best_words"].tolist()
        assert cost == d["best_cost"]
        assert fc == d["frame_count"]


def test_oracle_kernel_contract_shapes(oracle_mod):
    d = load_golden("kat_expansion")
    g = GoldenGraph(d)
    out = oracle_mod.advance_chunk(g.off, g.eps_end, g.ilabel, g.olabel, g.weight, g.nextstate,
                                   np.array([0, 3], np.int32), np.array([0.0, 0.0]), np.array([-1, -1], np.int64),
                                   np.zeros(3, np.int64), np.zeros(0, np.int32), d["frames"], 1.0, 1e9, 10**9,
                                   1e-9, 8, None, 0)
    status, err, counts, prev, state, cost, ooff, opool = out
    assert status == 0 and err == -1
    assert counts.tolist() == [1] and state.tolist() == [1]
    assert cost[0] == pytest.approx(0.5, abs=1e-12)
    assert ooff.tolist() == [0, 1] and opool.tolist() == [1]


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(10))
def test_oracle_matches_compiled_reference(oracle_mod, seed):
    import ctcwfst
    from ctcwfst.decoder import DecoderConfig, DecodeState, best_path, flatten
    from paper_2311_04996_b200 import synth

    spec = synth.SystemSpec(num_units=6 + seed, num_words=8 + 3 * seed, order=1 + seed % 3, seed=seed,
                            min_pron=1, max_pron=4)
    s = synth.build_system(spec)
    fg_ref = flatten(s.tlg.to_wfst_ref(ctcwfst) if hasattr(s.tlg, "to_wfst_ref") else _to_ref(ctcwfst, s.tlg))
    rng = np.random.default_rng(seed)
    frames = rng.normal(-3.0, 2.5, size=(40, spec.num_units)) if seed % 2 else \
        synth.planted_utterances(s, 1, 40, seed=seed)[0]
    cfg = DecoderConfig(beam=[6.0, 10.0, 17.0][seed % 3], max_active=[20, 200, 10_000][seed % 3])
    ch = DecodeState(fg_ref, cfg)
    oc = oracle_mod.OracleChannel.from_config(fg_ref, cfg)
    for i in range(0, 40, 9):
        ch.advance_frames(frames[i:i + 9])
        oc.advance_frames(frames[i:i + 9])
    assert oc.history_records() == ch.history_records()
    h = best_path(ch)
    assert oc.best_path() == (h.words, h.total_cost, h.frame_count)


def _to_ref(ctcwfst, f):
    from ctcwfst.wfst import Arc, Wfst

    g = Wfst(num_states=f.num_states, start=f.start)
    for s in range(f.num_states):
        for k in range(f.off[s], f.off[s + 1]):
            g.add_arc(s, Arc(int(f.ilabel[k]), int(f.olabel[k]), float(f.weight[k]), int(f.nextstate[k])))
        if np.isfinite(f.final[s]):
            g.set_final(s, float(f.final[s]))
    return g
