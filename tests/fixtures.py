"""Graph fixtures of the reference's test_util.hpp (:17-89), rebuilt in
Python.  random_edges uses numpy's generator, not mt19937 -- the graphs are
seeded and deterministic but not the reference's; parity is always checked
against the oracle on the same graph."""
import numpy as np

import paper_1701_05975_b200 as W


def graph_of(entries):
    return W.build_csr(W.EdgeList.of(entries))


def path_graph(k, w=1.0):
    return graph_of([(i, i + 1, w) for i in range(k - 1)])


def star_graph(n, w=1.0):
    return graph_of([(0, i, w) for i in range(1, n)])


def cycle_graph(k, w=1.0):
    return graph_of([(i, (i + 1) % k, w) for i in range(k)])


def complete_graph(n, w=1.0):
    return graph_of([(i, j, w) for i in range(n) for j in range(i + 1, n)])


def tie_square_graph():
    """test_util.hpp:57-62: (0,1,1) (0,2,2) (1,2,1) (2,3,1)."""
    return graph_of([(0, 1, 1.0), (0, 2, 2.0), (1, 2, 1.0), (2, 3, 1.0)])


def race_graph(k=64):
    """test_engine.cpp:304-326: k middle vertices all reach target k+1 at d=2."""
    return graph_of([(0, i, 1.0) for i in range(1, k + 1)] + [(i, k + 1, 1.0) for i in range(1, k + 1)])


def random_edges(n, extra, wmax, seed):
    """Random spanning tree + `extra` random edges, integer weights (test_util.hpp:64-84)."""
    rng = np.random.default_rng(seed)
    es = []
    for v in range(1, n):
        es.append((int(rng.integers(0, v)), v, float(rng.integers(1, wmax + 1))))
    for _ in range(extra):
        a, b = int(rng.integers(0, n)), int(rng.integers(0, n))
        if a != b:
            es.append((a, b, float(rng.integers(1, wmax + 1))))
    return W.EdgeList.of(es)


def random_tree(n, wmax, seed):
    return random_edges(n, 0, wmax, seed)


def weighted(el, lo, hi, seed):
    return W.assign_weights(el, lo, hi, seed)
