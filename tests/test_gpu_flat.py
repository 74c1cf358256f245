"""GPU parity of the distance-first kernel for flat graphs (bc_flat.cuh,
set_param("flat", 1)): near-far SSSP with window-sorted output, sigma / delta
pulled in distance order, and the Eq. 4 depth recovered from the distances by
the threshold sweep.  Same bars as test_gpu_parity.py: BC 1e-9 relative,
depth_per_source exact.  Every run asserts the flat kernel did the work
(flat_fallback_sources == 0: no source is handed to another kernel)."""
import numpy as np
import pytest

import fixtures as F
from test_gpu_parity import check_graph

pytestmark = pytest.mark.gpu


def flat_graph(W, g, delta=0):
    gg = W.GpuGraph(g)
    gg.set_param("flat", 1)
    if delta:
        gg.set_param("flat_delta", delta)
    return gg


def _cases(W):
    yield "tie_square", F.tie_square_graph()
    yield "path", F.path_graph(9)
    yield "cycle", F.cycle_graph(7)
    yield "star", F.star_graph(8)
    yield "islands", F.graph_of([(0, 1, 1), (1, 2, 1), (10, 11, 1), (11, 12, 1)])
    yield "grid_ties", W.build_csr(W.assign_weights(W.gen_grid(17, 23), 1, 3, 5))
    yield "grid_unit", W.build_csr(W.assign_weights(W.gen_grid(20, 20), 1, 1, 5))
    yield "grid_wide", W.build_csr(W.assign_weights(W.gen_grid(40, 31), 1, 1000, 7))
    yield "tree", W.build_csr(F.random_tree(300, 9, 4))


@pytest.mark.parametrize("delta", [0, 1, 37])
def test_flat_matches_oracle(W, oracle, delta):
    for name, g in _cases(W):
        gg = flat_graph(W, g, delta)
        try:
            src = None if g.n <= 64 else W.sample_sources(g.n, 48, 3)
            check_graph(W, oracle, g, sources=src, edge=True, gg=gg)
            assert gg.last_kernel().startswith("bc_flat_kernel"), name
            assert gg.last_run_stats()["flat_fallback_sources"] == 0, name
        finally:
            gg.close()


def test_flat_halved_duplicates_and_all_sources(W, oracle):
    g = W.build_csr(W.assign_weights(W.gen_grid(12, 15), 1, 50, 2))
    gg = flat_graph(W, g)
    try:
        check_graph(W, oracle, g, edge=True, gg=gg)
        src = np.array([5, 5, 0, 179, 5])
        check_graph(W, oracle, g, sources=src, edge=True, halved=True, gg=gg)
    finally:
        gg.close()


def test_flat_long_distances(W, oracle):
    """Distances far beyond n (the round-1 kernel's counting-sort range, which
    handed such sources to one-warp teams): the window sort only needs the
    window width."""
    for g in (F.path_graph(40, w=1000.0), W.build_csr(W.assign_weights(W.gen_grid(40, 31), 1, 1000, 7))):
        gg = flat_graph(W, g)
        try:
            check_graph(W, oracle, g, edge=True, gg=gg)
            assert gg.last_kernel().startswith("bc_flat_kernel")
            assert gg.last_run_stats()["flat_fallback_sources"] == 0
        finally:
            gg.close()


def test_flat_auto_grid512_vs_eq4_oracle(W, oracle):
    """A 512x512 grid with the BASELINE weights 1-1000 (n = 2^18: the flat
    kernel is picked automatically): node / edge BC and depth_per_source
    against the oracle's Eq. 4 process."""
    g = W.build_csr(W.assign_weights(W.gen_grid(512, 512), 1, 1000, 1))
    src = W.sample_sources(g.n, 6, 1)
    gg = W.GpuGraph(g)
    try:
        check_graph(W, oracle, g, sources=src, edge=True, gg=gg)
        assert gg.last_kernel().startswith("bc_flat_kernel")
        assert gg.last_run_stats()["flat_fallback_sources"] == 0
    finally:
        gg.close()


def test_flat_falls_back_when_ineligible(W, oracle):
    """Degree above the sweep's 8 slots per vertex: the normal shapes run."""
    g = F.star_graph(30)
    gg = flat_graph(W, g)
    try:
        check_graph(W, oracle, g, edge=True, gg=gg)
        assert not gg.last_kernel().startswith("bc_flat_kernel")
    finally:
        gg.close()


def test_flat_grid_sampled_vs_reference(W, ref):
    el = W.assign_weights(W.gen_grid(96, 96), 1, 1000, 1)
    g = W.build_csr(el)
    rg = ref.build_csr(el.u, el.v, el.w)
    try:
        src = W.sample_sources(g.n, 64, 1)
        want = ref.bc_parallel(rg, "we", 8, sources=src)
        gg = flat_graph(W, g)
        try:
            r = gg.bc(W.EngineOptions(sources=src))
        finally:
            gg.close()
        rel = np.abs(r.node_bc - want["node_bc"]) / np.maximum(1e-12, np.abs(want["node_bc"]))
        assert (rel <= 1e-9).all()
        assert np.array_equal(r.depth_per_source, want["depth"])
    finally:
        ref.free_csr(rg)


def test_flat_graph_strict_merge_and_dumps_use_teams(W, ref, oracle):
    """A strict merge (bitwise reference order) and the single-source dumps run
    on one-warp teams even where the flat kernel is selected."""
    el = W.assign_weights(W.gen_grid(20, 26), 1, 9, 4)
    g = W.build_csr(el)
    rg = ref.build_csr(el.u, el.v, el.w)
    gg = flat_graph(W, g)
    try:
        src = W.sample_sources(g.n, 40, 2)
        want = ref.bc_parallel(rg, "we-warp4", 3, sources=src, edge_bc=True, strict_merge=True)
        r = gg.bc(W.EngineOptions(strategy=W.parse_strategy("we-warp4"), compute_edge_bc=True, strict_merge=True,
                                  sources=src))
        assert np.array_equal(r.node_bc.view(np.uint64), want["node_bc"].view(np.uint64))
        assert np.array_equal(r.edge_bc.view(np.uint64), want["edge_bc"].view(np.uint64))
        d = gg.dump_source(7)
        o = oracle.eq4_source(g, 7)
        assert np.array_equal(d["dist"], o["dist"]) and np.array_equal(d["sigma"], o["sigma"])
        assert d["depth"] == o["depth"]
        r2 = gg.bc(W.EngineOptions(sources=src))
        assert gg.last_kernel().startswith("bc_flat_kernel")
        assert np.abs(r2.node_bc - r.node_bc).max() <= 1e-9 * max(1.0, np.abs(r.node_bc).max())
    finally:
        gg.close()
        ref.free_csr(rg)


def test_flat_refuses_asymmetric_rows(W):
    """A caller CSR whose rows are not mirror images (not from build_csr) never
    reaches the flat kernel: its dataflows count DAG edges from both ends."""
    u32 = lambda *a: np.array(a, np.uint32)
    f64 = lambda *a: np.array(a, np.float64)
    # rows 0->1 (w1), 1->0 (w1), 1->2 (w2), 2->1 (w3: the twin disagrees)
    g = W.CsrGraph(n=3, m=2, offsets=u32(0, 1, 3, 4), adjacency=u32(1, 0, 2, 1), weights=f64(1, 1, 2, 3),
                   edge_id=u32(0, 0, 1, 1), min_incident_weight=f64(1, 1, 3), original_id=np.arange(3, dtype=np.uint64),
                   edge_u=u32(0, 1), edge_v=u32(1, 2))
    gg = flat_graph(W, g)
    try:
        gg.bc(W.EngineOptions())
        assert not gg.last_kernel().startswith("bc_flat_kernel")
    finally:
        gg.close()
    ok = W.build_csr(W.assign_weights(W.gen_grid(5, 5), 1, 9, 1))
    gg = flat_graph(W, ok)
    try:
        gg.bc(W.EngineOptions())
        assert gg.last_kernel().startswith("bc_flat_kernel")
    finally:
        gg.close()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_flat_random_sparse_graphs(W, oracle, seed):
    """The flat kernel on random sparse graphs (not lattices): degree <= 8,
    several components, weight ranges from ties-heavy to wide, both CTA
    shapes; node / edge BC and depth against the oracle's Eq. 4."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(300, 900))
    el = W.gen_er(n, float(rng.uniform(1.5, 3.5)), seed)
    keep = np.ones(len(el), bool)
    deg = np.zeros(n + 1, np.int64)
    for i, (a, b) in enumerate(zip(el.u.tolist(), el.v.tolist())):  # cap the degree at 8
        if deg[a] >= 8 or deg[b] >= 8:
            keep[i] = False
        else:
            deg[a] += 1
            deg[b] += 1
    el = W.EdgeList(el.u[keep], el.v[keep], el.w[keep])
    for lo, hi in ((1, 2), (1, 300)):
        g = W.build_csr(W.assign_weights(el, lo, hi, seed))
        for threads in (1024, 256):
            gg = flat_graph(W, g)
            try:
                gg.set_param("flat_threads", threads)
                check_graph(W, oracle, g, sources=W.sample_sources(g.n, 60, seed), edge=True, gg=gg)
                assert gg.last_kernel().startswith("bc_flat_kernel")
                assert gg.last_run_stats()["flat_fallback_sources"] == 0
            finally:
                gg.close()



@pytest.mark.parametrize("sq", [0, 32])
def test_flat_near_queue_spill(W, oracle, sq):
    """Near queues entirely in global memory (flat_sq 0) and a 32-entry
    shared-memory part that most phases overflow into q0 / q1."""
    for name, g in _cases(W):
        gg = flat_graph(W, g)
        try:
            gg.set_param("flat_sq", sq)
            src = None if g.n <= 64 else W.sample_sources(g.n, 32, 5)
            check_graph(W, oracle, g, sources=src, edge=True, gg=gg)
            assert gg.last_kernel().startswith("bc_flat_kernel"), name
        finally:
            gg.close()
