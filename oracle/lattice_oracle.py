"""CPU restatement of the lattice definition and an
enumeration n-best -- the oracle for csrc/ctw_lattice.cu.

TEST INFRASTRUCTURE ONLY (like oracle.py): imported by tests/ alone.

Parity status: the reference has no lattice, so this oracle
is anchored on (a) the reference's own records (the nodes come from
OracleChannel, pinned to the reference's goldens by tests/test_oracle.py),
(b) the reference's arc arithmetic (_kernel.pyx:249-253, :307-310) and
best_path rule (decoder.py:384-400): the lattice's best complete path must
equal best_path (tests/test_lattice.py), and (c) brute-force enumeration of
every complete path for the n-best list.
"""

from __future__ import annotations

import math

import numpy as np

INF = math.inf


def _closure(fg, s_state, f_ll, scale, boost):
    """All (emitting arc e, reached state y, min cost, labels) for one source
    state: e then epsilon arcs, label-correcting (exact min over paths)."""
    out = []
    for e in range(int(fg.eps_end[s_state]), int(fg.off[s_state + 1])):
        il, ol = int(fg.ilabel[e]), int(fg.olabel[e])
        c0 = (-scale * float(f_ll[il - 1])) + float(fg.weight[e])
        if boost is not None and ol != 0:
            c0 = c0 + float(boost[ol])
        if not c0 < INF:
            continue
        best = {int(fg.nextstate[e]): (c0, (ol,) if ol else ())}
        queue = [int(fg.nextstate[e])]
        while queue:
            u = queue.pop(0)
            cu, lu = best[u]
            for a in range(int(fg.off[u]), int(fg.eps_end[u])):
                y = int(fg.nextstate[a])
                oy = int(fg.olabel[a])
                cy = cu + float(fg.weight[a])
                if boost is not None and oy != 0:
                    cy = cy + float(boost[oy])
                if not cy < INF:
                    continue
                if y not in best or cy < best[y][0]:
                    best[y] = (cy, lu + ((oy,) if oy else ()))
                    queue.append(y)
        for y, (c, labs) in best.items():
            out.append((e, y, c, labs))
    return out


def lattice(fg, scale, loglik, seeds, frames, beam, boost=None):
    """seeds: [(state, cost, labels)]; frames: per frame [(state, cost)] (the
    decoder's survivors). Returns dict(best, final_mode, arcs=[(frame,
    src_node, dst_node, dst_state, w, labels, score)], beta, alpha, n_seeds)
    where score = alpha(src) + w + beta(dst); arcs are ALL candidates (the
    caller applies the beam) ."""
    T = len(frames)
    S0 = len(seeds)
    node_base = [S0]
    for fr in frames[:-1]:
        node_base.append(node_base[-1] + len(fr))
    alpha = [c for _, c, _ in seeds] + [c for fr in frames for _, c in fr]
    final = np.asarray(fg.final, dtype=np.float64)
    last = frames[-1]
    fm = any(final[s] < INF for s, _ in last)
    beta = [INF] * len(alpha)
    best = INF
    for k, (s, c) in enumerate(last):
        fw = float(final[s]) if fm else 0.0
        if fm and not fw < INF:
            continue
        beta[node_base[T - 1] + k] = fw
        best = min(best, c + fw)
    arcs = []
    for f in range(T - 1, -1, -1):
        dmap = {s: node_base[f] + k for k, (s, _) in enumerate(frames[f])}
        src = [(k, s) for k, (s, _, _) in enumerate(seeds)] if f == 0 else \
            [(node_base[f - 1] + k, s) for k, (s, _) in enumerate(frames[f - 1])]
        for node, s_state in src:
            for e, y, w, labs in _closure(fg, s_state, loglik[f], scale, boost):
                d = dmap.get(y)
                if d is None or not beta[d] < INF:
                    continue
                tail = w + beta[d]
                beta[node] = min(beta[node], tail)
                arcs.append((f, node, d, y, w, labs, alpha[node] + tail))
    return dict(best=best, final_mode=fm, arcs=arcs, beta=beta, alpha=alpha, n_seeds=S0)


def kept(lat, beam, slack=0.0):
    cut = lat["best"] + beam + slack
    return [a for a in lat["arcs"] if a[6] <= cut]


def phrase_cost(words, phrases):
    """Brute force: every occurrence of every phrase (overlapping, nested)
    pays -magnitude."""
    c = 0.0
    for ph, mag in phrases.items():
        k = len(ph)
        for i in range(len(words) - k + 1):
            if tuple(words[i:i + k]) == tuple(ph):
                c += -float(mag)
    return c


def nbest(lat, arcs, seeds, n, final, bound=None, max_paths=500_000, phrases=None):
    """Brute force: every complete path through `arcs` (seed -> last layer)
    with total cost <= bound (default best + lattice beam of the arcs'
    scores, i.e. all paths that can matter), total = seed cost + sum w +
    final; distinct word sequences, best first."""
    T = max((a[0] for a in arcs), default=-1) + 1
    out_arcs = {}
    for a in arcs:
        out_arcs.setdefault(a[1], []).append(a)
    lat_state = {a[2]: a[3] for a in arcs}
    fm = lat["final_mode"]

    def fin(node):
        return (float(final[lat_state[node]]) if fm else 0.0) if node in lat_state else INF

    # exact remaining cost over the given arcs, for the enumeration bound
    rem = {}
    for a in sorted(arcs, key=lambda a: -a[0]):
        if a[0] == T - 1:
            rem.setdefault(a[2], fin(a[2]))
        c = a[4] + rem.get(a[2], INF)
        if c < rem.get(a[1], INF):
            rem[a[1]] = c
    if bound is None:
        bound = max((a[6] for a in arcs), default=INF)
    paths = []

    def dfs(node, cost, words, layer):
        if len(paths) > max_paths:
            raise RuntimeError("enumeration too large")
        if cost + rem.get(node, INF) > bound + 1e-9:
            return
        if layer == T:
            fw = fin(node)
            if fw < INF:
                paths.append((cost + fw + (phrase_cost(words, phrases) if phrases else 0.0), words))
            return
        for a in out_arcs.get(node, []):
            dfs(a[2], cost + a[4], words + a[5], layer + 1)

    for k, (s, c, labs) in enumerate(seeds):
        dfs(k, c, tuple(labs), 0)
    paths.sort(key=lambda p: p[0])
    seen, res = set(), []
    for c, w in paths:
        if w in seen:
            continue
        seen.add(w)
        res.append((w, c))
        if len(res) == n:
            break
    return res
