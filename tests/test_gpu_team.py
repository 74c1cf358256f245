"""GPU parity of the team kernel (bc_team.cuh): one source per cluster of C
CTAs, for every cluster size the launcher supports, against the CPU oracle.

Same bars as test_gpu_parity.py: dist and sigma bit-exact, per-source delta
1e-12 relative, BC 1e-9 relative, depth_per_source exact.  The cases target
what the team decomposition changes: edge ranges split across CTAs (hub rows
shared by several CTAs -> sigma/delta by global atomics), ping-pong queues,
the DSMEM phase ring, and the row-scan fallback.
"""
import numpy as np
import pytest

import fixtures as F
from test_gpu_parity import assert_close, check_graph

pytestmark = pytest.mark.gpu

# cluster size; "w" = one-warp teams (32-thread CTA per source)
CLUSTERS = (1, 2, 4, 8, 16, "w")


def team_graph(W, g, c):
    gg = W.GpuGraph(g)
    if c == "w":
        gg.set_param("cluster", 1)
        gg.set_param("threads", 32)
    else:
        gg.set_param("cluster", c)
    return gg


@pytest.mark.parametrize("c", CLUSTERS)
def test_team_known_answers(W, oracle, c):
    for g in (F.path_graph(3), F.tie_square_graph(), F.star_graph(9), F.cycle_graph(4), F.complete_graph(7),
              F.graph_of([(0, 1, 1), (1, 2, 1), (10, 11, 1), (11, 12, 1)])):
        gg = team_graph(W, g, c)
        check_graph(W, oracle, g, gg=gg)
        gg.close()
    g = F.tie_square_graph()
    gg = team_graph(W, g, c)
    d = gg.dump_source(0)
    gg.close()
    assert d["dist"].tolist() == [0.0, 1.0, 2.0, 3.0]
    assert d["sigma"][3] == 2.0
    assert d["delta"][1:].tolist() == [1.0, 1.0, 0.0]


@pytest.mark.parametrize("c", CLUSTERS)
def test_team_race_and_dump(W, oracle, c):
    g = F.race_graph(64)
    gg = team_graph(W, g, c)
    for _ in range(5):
        d = gg.dump_source(0)
        assert d["sigma"][65] == 64.0 and d["dist"][65] == 2.0 and d["depth"] == 3
    gg.close()
    for seed in (3, 14):
        g = W.build_csr(F.random_edges(120, 400, 10, seed))
        gg = team_graph(W, g, c)
        for s in (0, 5, 119):
            d = gg.dump_source(s)
            o = oracle.eq4_source(g, s)
            assert np.array_equal(d["dist"], o["dist"]), f"dist s={s}"
            assert np.array_equal(d["sigma"], o["sigma"]), f"sigma s={s}"
            assert_close(d["delta"], o["delta"], 1e-12, f"delta s={s}")
            assert d["depth"] == o["depth"]
        gg.close()


@pytest.mark.parametrize("c", CLUSTERS)
def test_team_random_equivalence(W, oracle, c):
    rng = np.random.default_rng(1234 + (c if isinstance(c, int) else ord(c)))
    for i in range(12):
        seed = int(rng.integers(1, 2**62))
        if i % 2 == 0:
            n = int(rng.integers(5, 300))
            el = W.gen_er(n, float(rng.uniform(1.0, min(24.0, n - 1.0))), seed)
        else:
            el = W.gen_kronecker(int(rng.integers(3, 10)), float(rng.uniform(1.0, 24.0)), seed)
        g = W.build_csr(W.assign_weights(el, 1, int(rng.integers(1, 60)), seed))
        if g.n < 2:
            continue
        gg = team_graph(W, g, c)
        check_graph(W, oracle, g, gg=gg, sources=[0, 0, g.n - 1] if i % 3 == 0 else None)
        gg.close()


@pytest.mark.parametrize("c", CLUSTERS)
def test_team_hub_rows_and_sampled(W, oracle, c):
    # skewed: hub rows of thousands of slots are split across the CTAs
    el = W.assign_weights(W.gen_kronecker(13, 32.0, 9), 1, 255, 9)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 48, 2)
    gg = team_graph(W, g, c)
    check_graph(W, oracle, g, gg=gg, sources=src, edge=True)
    gg.close()


@pytest.mark.parametrize("c", (1, 8, "w"))
def test_team_dag_overflow_fallback(W, oracle, c):
    a = 60
    g = F.graph_of([(i, a + j, 1.0) for i in range(a) for j in range(a)])
    gg = team_graph(W, g, c)
    check_graph(W, oracle, g, gg=gg)
    assert gg.last_run_stats()["dag_overflow_sources"] > 0
    gg.close()


@pytest.mark.parametrize("c", (2, 16, "w"))
def test_team_unpacked_slots(W, oracle, c):
    el = W.gen_er(3000, 6.0, 7)
    el.w = (np.random.default_rng(7).integers(1, 1_100_000, len(el))).astype(np.float64)
    g = W.build_csr(el)
    gg = team_graph(W, g, c)
    assert not gg.info()["packed_slots"]
    check_graph(W, oracle, g, sources=list(range(0, 3000, 151)), gg=gg)
    gg.close()


@pytest.mark.parametrize("c", (1, 8, "w"))
def test_team_grid_large_diameter(W, oracle, c):
    el = W.assign_weights(W.gen_grid(64, 64), 1, 1000, 1)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 12, 1)
    gg = team_graph(W, g, c)
    check_graph(W, oracle, g, gg=gg, sources=src, edge=True)
    gg.close()


def test_one_warp_team_grid_levels_and_dag(W, oracle):
    """Large-diameter grid on one-warp teams: level sets and the recorded DAG
    per level equal the oracle's Eq. 4 structure."""
    el = W.assign_weights(W.gen_grid(48, 40), 1, 1000, 2)
    g = W.build_csr(el)
    gg = team_graph(W, g, "w")
    off, adj, wt = g.offsets, g.adjacency, g.weights
    for s in (0, 777, g.n - 1):
        o = oracle.eq4_source(g, s)
        ol = [np.sort(o["order"][o["ends"][i]:o["ends"][i + 1]]) for i in range(len(o["ends"]) - 1)]
        lv = gg.levels(s)
        assert len(lv) == len(ol) and all(np.array_equal(a, b) for a, b in zip(lv, ol))
        segs, ov = gg.dag(s)
        assert not ov
        dist = o["dist"]
        for L, lvl in enumerate(ol):
            want = sorted((int(adj[e]), int(x)) for x in lvl for e in range(off[x], off[x + 1])
                          if dist[adj[e]] + wt[e] == dist[x])
            got = sorted(zip(segs[L][0].tolist(), segs[L][1].tolist()))
            assert got == want, f"s={s} level {L}"
    gg.close()


def test_one_warp_team_large_distances(W, oracle):
    """Distances past 2^31 (u32 distances, n * max_w < 2^32) on one-warp teams."""
    g = F.graph_of([(i, i + 1, 30_000_000.0) for i in range(99)])  # path: d reaches 2.97e9
    gg = team_graph(W, g, "w")
    check_graph(W, oracle, g, gg=gg, sources=[0, 5, 99], edge=True)
    gg.close()


@pytest.mark.parametrize("c", (4, 8))
def test_team_fill_clusters(W, oracle, c):
    """C >= 4 clusters plus the concurrent 2-CTA fill launch on the SMs they
    strand (both share the source counter): parity on a sampled R-MAT, and
    the launch count shows the fill ran."""
    el = W.assign_weights(W.gen_kronecker(14, 32.0, 5), 1, 255, 5)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 200, 4)
    gg = W.GpuGraph(g)
    try:
        gg.set_param("cluster", c)
        gg.set_param("fill", 1)
        check_graph(W, oracle, g, gg=gg, sources=src, edge=True)
        assert gg.last_run_stats()["launches"] == 3
    finally:
        gg.close()


def test_rmat20_auto_shape_uses_fill():
    """The auto launch shape of R-MAT-20: 4-CTA clusters plus
    2-CTA fill teams (the in-flight distances stay within the L2 budget)."""
    import paper_1701_05975_b200 as W
    g = W.build_csr(W.assign_weights(W.gen_kronecker(20, 32.0, 1), 1, 255, 1))
    gg = W.GpuGraph(g)
    try:
        gg.bc(W.EngineOptions(sources=W.sample_sources(g.n, 300, 1)))
        assert gg.last_kernel() == "bc_team_kernel<1024,4>" and gg.last_run_stats()["launches"] == 3
    finally:
        gg.close()

