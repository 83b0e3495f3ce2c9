"""Debug: trace the reference Gauss-Seidel frame step and compare its tie
winners with the (pd, gpos, arc) emulation used by the GPU kernel."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle"), str(ROOT / "tests")]
import oracle as O
from paper_2311_04996_b200 import DecoderConfig, synth
from conftest import history_signature

INF = float("inf")


def gs_frame(fg, src, row, scale, boost=None, relax=1e-9):
    """Reference frame step (emit + GS eps), returning slot list with events."""
    off, ee, il, ol, w, ns = fg.off, fg.eps_end, fg.ilabel, fg.olabel, fg.weight, fg.nextstate
    slot_of, st, cost, win = {}, [], [], []   # win = (kind, pass, pos_src, arc)
    first = {}
    for i, (s, c) in enumerate(src):
        for a in range(ee[s], off[s + 1]):
            nc = c + (-scale * row[il[a] - 1]) + w[a]
            if not nc < INF:
                continue
            d = int(ns[a])
            if d not in slot_of:
                slot_of[d] = len(st); st.append(d); cost.append(nc); win.append(("emit", 0, i, a))
            elif nc < cost[slot_of[d]]:
                cost[slot_of[d]] = nc; win[slot_of[d]] = ("emit", 0, i, a)
    n_emit = len(st)
    p = 0
    ties = []
    while True:
        p += 1
        mi = 0.0
        j = 0
        while j < len(st):
            s, c = st[j], cost[j]
            for a in range(off[s], ee[s]):
                nc = c + w[a]
                if not nc < INF:
                    continue
                d = int(ns[a])
                if d not in slot_of:
                    slot_of[d] = len(st); st.append(d); cost.append(nc); win.append(("eps", p, j, a)); mi = INF
                else:
                    k = slot_of[d]
                    if nc < cost[k]:
                        mi = max(mi, cost[k] - nc); cost[k] = nc; win[k] = ("eps", p, j, a)
                    elif nc == cost[k] and win[k] != ("eps", p, j, a):
                        ties.append((k, ("eps", p, j, a), win[k]))
            j += 1
        if mi <= relax:
            break
    return st, cost, win, n_emit, p, ties


def main(seed):
    spec = dict(num_units=4 + 3 * seed, num_words=10 + 7 * seed, order=1 + seed % 3, seed=seed, min_pron=1, max_pron=5)
    s = synth.build_system(synth.SystemSpec(**spec))
    fg = s.graph
    g = np.load(ROOT / "gpurun_out" / f"rand_hist_{seed}.npz")
    frames = g["frames"]
    cfg = DecoderConfig(beam=[4.0, 9.0, 17.0, 1e9][seed % 4], max_active=[7, 60, 10_000, 300][seed % 4])
    oc = O.OracleChannel.from_config(fg, cfg)
    step = [60, 1, 7, 13][seed % 4]
    for i in range(0, 60, step):
        oc.advance_frames(frames[i:i + step])
    want = oc.history_records()
    got, i = [], 0
    for n in g["counts"]:
        got.append([(int(g["rec_prev"][k]), tuple(int(x) for x in g["rec_olab_pool"][g["rec_olab_off"][k]:g["rec_olab_off"][k + 1]]),
                     int(g["rec_state"][k]), float(g["rec_cost"][k])) for k in range(i, i + n)])
        i += n
    f = next(k for k in range(len(want)) if want[k] != got[k])
    print("first differing frame", f, "signature equal:", history_signature(got) == history_signature(want))
    diffs = [(a, b) for a, b in zip(want[f], got[f]) if a != b]
    print(len(diffs), "records differ; first:", diffs[:3])
    # trace frame f from the reference's frame f-1 survivors
    src = [(r[2], r[3]) for r in want[f - 1]]
    st, cost, win, n_emit, passes, ties = gs_frame(fg, src, frames[f], 1.0)
    print("slots", len(st), "emit", n_emit, "passes", passes, "ties", len(ties))
    bad_states = {a[2] for a, b in diffs}
    for k, cand, w0 in ties:
        if st[k] in bad_states:
            print("tie at slot", k, "state", st[k], "winner", w0, "loser", cand)


if __name__ == "__main__":
    main(int(sys.argv[1]))


def chain(seed, state_target):
    spec = dict(num_units=4 + 3 * seed, num_words=10 + 7 * seed, order=1 + seed % 3, seed=seed, min_pron=1, max_pron=5)
    s = synth.build_system(synth.SystemSpec(**spec))
    fg = s.graph
    g = np.load(ROOT / "gpurun_out" / f"rand_hist_{seed}.npz")
    frames = g["frames"]
    cfg = DecoderConfig(beam=[4.0, 9.0, 17.0, 1e9][seed % 4], max_active=[7, 60, 10_000, 300][seed % 4])
    oc = O.OracleChannel.from_config(fg, cfg)
    step = [60, 1, 7, 13][seed % 4]
    for i in range(0, 60, step):
        oc.advance_frames(frames[i:i + step])
    want = oc.history_records()
    f = 57
    src = [(r[2], r[3]) for r in want[f - 1]]
    st, cost, win, n_emit, passes, ties = gs_frame(fg, src, frames[f], 1.0)
    slot_of = {x: k for k, x in enumerate(st)}
    k = slot_of[state_target]
    while True:
        w = win[k]
        print("slot", k, "state", st[k], "cost", repr(cost[k]), "win", w, "ties:", [t[1] for t in ties if t[0] == k and t[1][1:] != w[1:]][:6])
        if w[0] == "emit":
            print("   source", w[2], src[w[2]])
            break
        k = w[2]
