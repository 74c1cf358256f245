"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (north_star): distances bit-exact, sigma bit-exact (all
values here are < 2^53), per-source delta within 1e-12 relative, BC within
1e-9 relative (fp64, summation order differs), depth_per_source equal to the
reference's Eq. 4 round counts.  Cases follow the reference's own tests:
test_brandes.cpp, test_engine.cpp, acceptance.cpp.
"""
import numpy as np
import pytest

from conftest import approx_rel
import fixtures as F

pytestmark = pytest.mark.gpu


def assert_close(got, want, rtol, what=""):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, what
    ok = approx_rel(got, want, rtol)
    if not ok.all():
        i = int(np.argmin(ok))
        raise AssertionError(f"{what}: index {i} got {got[i]!r} want {want[i]!r} ({(~ok).sum()} bad)")


def check_graph(W, oracle, g, sources=None, edge=True, halved=False, gg=None):
    own = gg is None
    gg = gg or W.GpuGraph(g)
    try:
        opt = W.EngineOptions(compute_edge_bc=edge, sources=sources,
                              normalization=W.Normalization.Halved if halved else W.Normalization.Raw)
        r = gg.bc(opt)
    finally:
        if own:
            gg.close()
    node, eb, depth = oracle.bc_eq4(g, sources=sources, halved=halved, edge_bc=edge)
    assert_close(r.node_bc, node, 1e-9, "node_bc")
    if edge:
        assert_close(r.edge_bc, eb, 1e-9, "edge_bc")
    assert np.array_equal(r.depth_per_source, depth), "depth_per_source"
    return r


def check_sources_dump(W, oracle, g, sources):
    gg = W.GpuGraph(g)
    try:
        for s in sources:
            d = gg.dump_source(int(s))
            o = oracle.eq4_source(g, int(s))
            assert np.array_equal(d["dist"], o["dist"]), f"dist s={s}"
            assert np.array_equal(d["sigma"], o["sigma"]), f"sigma s={s}"
            assert_close(d["delta"], o["delta"], 1e-12, f"delta s={s}")
            assert d["depth"] == o["depth"], f"depth s={s}"
    finally:
        gg.close()


# ---------------------------------------------------------------- known answers

def test_path_of_three(W):
    g = F.path_graph(3)
    r = W.bc_parallel(g)
    assert r.node_bc.tolist() == [0.0, 2.0, 0.0]                   # test_brandes.cpp:24-31
    assert r.depth_per_source.tolist() == [3, 2, 3]               # test_engine.cpp:376-380
    h = W.bc_parallel(g, W.EngineOptions(normalization=W.Normalization.Halved))
    assert h.node_bc.tolist() == [0.0, 1.0, 0.0]
    e = W.bc_parallel(g, W.EngineOptions(compute_edge_bc=True))
    assert e.edge_bc.tolist() == [4.0, 4.0]                        # test_brandes.cpp:39-44
    s = W.bc_parallel(g, W.EngineOptions(sources=[0]))
    assert s.node_bc.tolist() == [0.0, 1.0, 0.0]                   # test_engine.cpp:196-202
    assert s.depth_per_source[0] == 3


def test_tie_square_enumerated(W):
    g = F.tie_square_graph()
    r = W.bc_parallel(g, W.EngineOptions(compute_edge_bc=True))
    assert_close(r.node_bc, [0.0, 2.0, 4.0, 0.0], 1e-12, "node")  # test_brandes.cpp:48-56
    assert_close(r.edge_bc, [4.0, 2.0, 6.0, 6.0], 1e-12, "edge")
    gg = W.GpuGraph(g)
    d = gg.dump_source(0)
    gg.close()
    assert d["dist"].tolist() == [0.0, 1.0, 2.0, 3.0]              # test_engine.cpp:137-140
    assert d["sigma"][3] == 2.0                                    # strict rule keeps the tie
    assert d["delta"][1:].tolist() == [1.0, 1.0, 0.0]              # test_engine.cpp:183-193


def test_closed_forms(W):                                          # acceptance.cpp:200-231
    for k in (2, 3, 6, 17):
        want = [2.0 * i * (k - 1 - i) for i in range(k)]
        assert_close(W.bc_parallel(F.path_graph(k)).node_bc, want, 0.0, f"path {k}")
    for n in (4, 9):
        want = [float((n - 1) * (n - 2))] + [0.0] * (n - 1)
        assert_close(W.bc_parallel(F.star_graph(n)).node_bc, want, 0.0, f"star {n}")
    assert_close(W.bc_parallel(F.cycle_graph(4)).node_bc, [1.0] * 4, 1e-12, "C4")
    for n in (4, 7):
        assert_close(W.bc_parallel(F.complete_graph(n)).node_bc, [0.0] * n, 0.0, f"K{n}")


def test_shared_target_race(W):                                    # acceptance.cpp:233-266
    g = F.race_graph(64)
    assert g.original_id[65] == 65
    gg = W.GpuGraph(g)
    for _ in range(20):
        d = gg.dump_source(0)
        assert d["sigma"][65] == 64.0 and d["dist"][65] == 2.0 and d["depth"] == 3
    gg.close()


def test_diamond_sigma(W):                                         # test_engine.cpp:156-162
    g = F.graph_of([(0, 1, 1), (0, 2, 1), (1, 3, 1), (2, 3, 1)])
    gg = W.GpuGraph(g)
    assert gg.dump_source(0)["sigma"][3] == 2.0
    gg.close()


def test_tree_descendants(W, oracle):                              # test_engine.cpp:238-248
    g = W.build_csr(F.random_tree(60, 7, 42))
    for s in (0, 7, 31):
        r = W.bc_parallel(g, W.EngineOptions(sources=[s]))
        want = oracle.eq4_source(g, s)["node_acc"]
        assert_close(r.node_bc, want, 1e-9, f"tree s={s}")


def test_disconnected_and_isolated(W, oracle):
    g = F.graph_of([(0, 1, 1), (1, 2, 1), (10, 11, 1), (11, 12, 1)])  # test_brandes.cpp:101-106
    assert_close(W.bc_parallel(g).node_bc, [0, 2, 0, 0, 2, 0], 0.0, "two paths")
    check_graph(W, oracle, g)


def test_duplicates_subsets_and_errors(W, oracle):
    g = W.build_csr(F.random_edges(50, 100, 10, 21))
    check_graph(W, oracle, g, sources=[3, 3, 7, 0, 49, 3])       # duplicates count twice
    check_graph(W, oracle, g, sources=[5], halved=True)
    r = W.bc_parallel(g, W.EngineOptions(sources=[]))             # test_engine.cpp:395-402
    assert not r.node_bc.any() and len(r.node_bc) == g.n
    with pytest.raises(ValueError):
        W.bc_parallel(g, W.EngineOptions(sources=[g.n]))          # test_engine.cpp:382-393
    with pytest.raises(ValueError):
        W.bc_parallel(g, W.EngineOptions(strategy=W.Strategy(W.FrontierMode.Queue, 5)))
    with pytest.raises(ValueError):
        W.bc_parallel(g, W.EngineOptions(workers=0))
    empty = W.build_csr(W.EdgeList())
    assert len(W.bc_parallel(empty).node_bc) == 0


# ---------------------------------------------------------------- per-source state

def test_dump_matches_oracle_random(W, oracle):                    # test_engine.cpp:266-302
    for seed in (3, 14, 15):
        g = W.build_csr(F.random_edges(80, 160, 10, seed))
        check_sources_dump(W, oracle, g, [5, 0, 79])


def test_dump_matches_reference_engine(W, ref):
    """Bit-level: GPU dist/sigma == the compiled reference's solve_source."""
    el = F.weighted(W.gen_er(300, 8.0, 55), 1, 10, 55)
    g = W.build_csr(el)
    rg = ref.build_csr(el.u, el.v, el.w)
    gg = W.GpuGraph(g)
    try:
        for s in (0, 17, 299):
            d = gg.dump_source(s)
            o = ref.solve_source(rg, s, "we")
            assert np.array_equal(d["dist"], o["dist"])
            assert np.array_equal(d["sigma"], o["sigma"])
            assert_close(d["delta"], o["delta"], 1e-12, "delta")
            assert d["depth"] == o["depth"]
    finally:
        gg.close()
        ref.free_csr(rg)


# ---------------------------------------------------------------- property sweeps

def test_random_er_kronecker_equivalence(W, oracle):               # acceptance.cpp:97-155
    rng = np.random.default_rng(20240901)
    checked = 0
    for i in range(40):
        seed = int(rng.integers(1, 2**62))
        if i % 2 == 0:
            n = int(rng.integers(5, 201))
            el = W.gen_er(n, float(rng.uniform(1.0, min(16.0, n - 1.0))), seed)
        else:
            el = W.gen_kronecker(int(rng.integers(3, 8)), float(rng.uniform(1.0, 16.0)), seed)
        g = W.build_csr(W.assign_weights(el, 1, 10, seed))
        if g.n < 2:
            continue
        checked += 1
        check_graph(W, oracle, g)
    assert checked > 30


def test_dag_overflow_fallback(W, oracle):
    """K_{60,60} with unit weights: ~n^2/4 DAG edges overflow the per-source
    DAG buffer, forcing the row-scan delta fallback."""
    a = 60
    g = F.graph_of([(i, a + j, 1.0) for i in range(a) for j in range(a)])
    gg = W.GpuGraph(g)
    r = check_graph(W, oracle, g, gg=gg)
    assert gg.last_run_stats()["dag_overflow_sources"] > 0
    gg.close()
    assert r is not None


def test_unpacked_slots(W, oracle):
    """n * max_weight forces 64-bit (neighbour, weight) slots."""
    el = W.gen_er(3000, 6.0, 7)
    el.w = (np.random.default_rng(7).integers(1, 1_100_000, len(el))).astype(np.float64)
    g = W.build_csr(el)
    gg = W.GpuGraph(g)
    assert not gg.info()["packed_slots"]
    check_graph(W, oracle, g, sources=list(range(0, 3000, 97)), gg=gg)
    gg.close()


def test_schedule_knobs_do_not_change_results(W, oracle):
    el = F.weighted(W.gen_kronecker(10, 12.0, 5), 1, 40, 5)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 64, 1)
    node, _, depth = oracle.bc_eq4(g, sources=src)
    for threads, near in ((128, 1), (256, 0), (512, 1000), (128, 3)):
        gg = W.GpuGraph(g)
        gg.set_tuning(threads, 0, near)
        r = gg.bc(W.EngineOptions(sources=src))
        gg.close()
        assert_close(r.node_bc, node, 1e-9, f"threads={threads} near={near}")
        assert np.array_equal(r.depth_per_source, depth)


def test_er4096_all_sources_vs_reference(W, ref):
    """BASELINE config 1 (ER n=4096 deg 8 w 1-64, all sources) against the
    compiled reference's bc_parallel: BC 1e-9, depth_per_source exact."""
    el = W.assign_weights(W.gen_er(4096, 8.0, 1), 1, 64, 1)
    g = W.build_csr(el)
    rg = ref.build_csr(el.u, el.v, el.w)
    want = ref.bc_parallel(rg, "we", 8)
    ref.free_csr(rg)
    r = W.bc_parallel(g)
    assert_close(r.node_bc, want["node_bc"], 1e-9, "node_bc")
    assert np.array_equal(r.depth_per_source, want["depth"])


@pytest.mark.slow
def test_rmat16_sampled_vs_oracle(W, oracle):
    el = W.assign_weights(W.gen_kronecker(16, 32.0, 1), 1, 255, 1)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 64, 1)
    check_graph(W, oracle, g, sources=src, edge=True)


@pytest.mark.slow
def test_grid_sampled_vs_oracle(W, oracle):
    el = W.assign_weights(W.gen_grid(128, 128), 1, 1000, 1)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 16, 1)
    check_graph(W, oracle, g, sources=src, edge=False)


@pytest.mark.slow
def test_ba_sampled_vs_oracle(W, oracle):
    el = W.assign_weights(W.gen_ba(8192, 10, 1), 1, 100, 1)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 64, 1)
    check_graph(W, oracle, g, sources=src, edge=True)


def test_dyadic_fractional_weights(W, oracle):
    """Weights i / 2^k (0.5, 2.5, 1.25, ...; the SPEC's own `0 1 2.5` example)
    run as integers scaled by 2^K: fp64 distances are exact multiples of
    2^-K, so dist, sigma, depth and BC equal the reference's."""
    rng = np.random.default_rng(5)
    el = W.gen_er(300, 6.0, 5)
    el.w = rng.choice([0.5, 1.25, 2.5, 3.0, 0.75, 7.125], len(el)).astype(np.float64)
    g = W.build_csr(el)
    check_graph(W, oracle, g, edge=True)
    src = W.sample_sources(g.n, 12, 2)
    check_sources_dump(W, oracle, g, src)
    for shape in ({"cluster": 1}, {"cluster": 2}, {"cluster": 1, "threads": 32}, {"flat": 1}):
        gg = W.GpuGraph(g)
        try:
            for k, v in shape.items():
                gg.set_param(k, v)
            check_graph(W, oracle, g, sources=src, edge=True, gg=gg)
        finally:
            gg.close()
    grid = W.build_csr(W.EdgeList(*[np.asarray(a) for a in (W.gen_grid(20, 20).u, W.gen_grid(20, 20).v)],
                                  rng.choice([0.5, 1.5, 2.25], 2 * 20 * 19).astype(np.float64)))
    gg = W.GpuGraph(grid)
    try:
        gg.set_param("flat", 1)
        check_graph(W, oracle, grid, edge=True, gg=gg)
        assert gg.last_kernel().startswith("bc_flat_kernel")
    finally:
        gg.close()


def test_non_dyadic_weights_are_refused(W):
    el = W.gen_er(50, 4.0, 3)
    el.w = np.full(len(el), 0.1)
    with pytest.raises(RuntimeError, match="dyadic"):
        W.GpuGraph(W.build_csr(el))
