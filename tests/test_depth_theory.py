"""The Eq. 4 levels are a function of the final distances alone.

If S_r is the set settled before round r and Δ_r the round's threshold, then
S_{r+1} = {v : d(v) < Δ_r}, and Δ_r = min over slots u->v with
d(u) < Δ_{r-1} <= d(v) of d(u) + w(u,v) + minw(v) (engine.cpp:149-181).  A
large-diameter pipeline can therefore compute exact distances with any SSSP
schedule and then recover depth_per_source (and the levels) with one monotone
sweep over the distance-sorted vertices, using a bucket array of
max-successor-distance per key.  These CPU tests pin both restatements
against the oracle's Eq. 4 round process on graphs with ties, disconnected
parts and skew.
"""
import numpy as np
import pytest

import fixtures as F


def _rows(g):
    off = np.asarray(g.offsets, np.int64)
    return off, np.asarray(g.adjacency, np.int64), np.asarray(g.weights, np.float64)


def levels_direct(g, s, d):
    """Δ_r by its definition (O(n) per round): the levels as sorted id lists."""
    off, adj, w = _rows(g)
    minw = np.asarray(g.min_incident_weight, np.float64)
    tau = 1.0                        # S_0 = {d < 1} = {s} (weights >= 1)
    levels = [[s]]
    while True:
        best = np.inf
        for u in np.flatnonzero(d < tau):
            for e in range(off[u], off[u + 1]):
                v = adj[e]
                if d[v] >= tau:
                    best = min(best, d[u] + w[e] + minw[v])
        if best == np.inf:
            return levels
        levels.append(sorted(np.flatnonzero((d >= tau) & (d < best)).tolist()))
        tau = best


def levels_sweep(g, s, d):
    """The same levels by one sweep: vertices in distance order; bucket[k] holds
    the largest d(v) over inserted slots u->v with key k = d(u) + w + minw(v);
    key k is live at threshold tau iff bucket[k] >= tau (v still unsettled).
    Every key exceeds the current tau, and it exceeds it by at most
    max w + max minw."""
    off, adj, w = _rows(g)
    minw = np.asarray(g.min_incident_weight, np.float64)
    reach = np.flatnonzero(np.isfinite(d))
    order = reach[np.argsort(d[reach], kind="stable")]
    bucket = {}

    def insert(u):
        for e in range(off[u], off[u + 1]):
            v = adj[e]
            if d[v] > d[u]:
                k = d[u] + w[e] + minw[v]
                bucket[k] = max(bucket.get(k, -1.0), d[v])

    span = (w.max() if len(w) else 0) + (minw[np.isfinite(minw)].max() if np.isfinite(minw).any() else 0)
    tau, i, levels = 1.0, 1, [[s]]
    insert(s)
    while True:
        nxt = next((k for k in np.arange(tau + 1, tau + span + 1) if bucket.get(k, -1.0) >= tau), None)
        if nxt is None:
            return levels
        j = i
        while j < len(order) and d[order[j]] < nxt:
            j += 1
        lvl = order[i:j]
        for u in lvl:
            insert(u)
        levels.append(sorted(lvl.tolist()))
        i, tau = j, float(nxt)


def _graphs(W):
    yield F.tie_square_graph()
    yield F.path_graph(6)
    yield F.race_graph(16)
    yield F.graph_of([(0, 1, 1), (1, 2, 1), (10, 11, 1), (11, 12, 1)])
    for seed in range(6):
        yield W.build_csr(F.random_edges(60, 120, 6, seed))
    yield W.build_csr(W.assign_weights(W.gen_grid(9, 11), 1, 5, 2))
    yield W.build_csr(W.assign_weights(W.gen_grid(7, 7), 1, 1, 2))        # unit weights: BFS levels
    yield W.build_csr(W.assign_weights(W.gen_kronecker(7, 8.0, 3), 1, 30, 3))
    yield W.build_csr(W.assign_weights(W.gen_ba(120, 3, 4), 1, 9, 4))


def test_levels_are_a_function_of_distances(W, oracle):
    checked = 0
    for g in _graphs(W):
        for s in sorted({0, g.n // 2, g.n - 1}):
            o = oracle.eq4_source(g, s)
            d = o["dist"]
            ends, order = o["ends"], o["order"]
            want = [sorted(order[ends[i]:ends[i + 1]].tolist()) for i in range(len(ends) - 1)]
            assert len(want) == o["depth"]
            assert levels_direct(g, s, d) == want
            assert levels_sweep(g, s, d) == want
            checked += 1
    assert checked >= 40


def test_no_dag_edge_inside_a_level(W, oracle):
    """Within an Eq. 4 level no vertex precedes another on a shortest path, so
    sigma and delta may process a level's vertices in any order."""
    for g in _graphs(W):
        off, adj, w = _rows(g)
        o = oracle.eq4_source(g, 0)
        d, ends, order = o["dist"], o["ends"], o["order"]
        level = np.full(g.n, -1)
        for i in range(len(ends) - 1):
            level[order[ends[i]:ends[i + 1]]] = i
        for u in range(g.n):
            if level[u] < 0:
                continue
            for e in range(off[u], off[u + 1]):
                v = adj[e]
                if d[u] + w[e] == d[v]:
                    assert level[v] > level[u]
