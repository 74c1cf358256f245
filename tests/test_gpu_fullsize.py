"""Parity at the BASELINE.json sizes themselves (sampled sources, so the CPU
oracle finishes in seconds).  R-MAT-20, BA-65536 and the 2048x2048 grid
against the oracle's exact Eq. 4 process (BC, edge BC and depth_per_source;
the oracle's pending-list Eq. 4 takes ~4 s per grid source), the grid also
against binary-heap Brandes and the size-independent additivity of BC over
source sets; R-MAT-24 (BASELINE config 5) on a 4-source sample.
"""
import numpy as np
import pytest

from test_gpu_parity import assert_close

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _graph(W, kind):
    if kind == "rmat20":
        return W.build_csr(W.assign_weights(W.gen_kronecker(20, 32.0, 1), 1, 255, 1))
    if kind == "ba65536":
        return W.build_csr(W.assign_weights(W.gen_ba(65536, 10, 1), 1, 100, 1))
    if kind == "rmat24":
        return W.build_csr(W.assign_weights(W.gen_kronecker(24, 32.0, 1), 1, 255, 1))
    return W.build_csr(W.assign_weights(W.gen_grid(2048, 2048), 1, 1000, 1))


@pytest.mark.parametrize("kind,k", [("rmat20", 6), ("ba65536", 24), ("rmat24", 4)])
def test_fullsize_vs_eq4_oracle(W, oracle, kind, k):
    g = _graph(W, kind)
    src = W.sample_sources(g.n, k, 1)
    gg = W.GpuGraph(g)
    r = gg.bc(W.EngineOptions(sources=src, compute_edge_bc=True))
    gg.close()
    node, edge, depth = oracle.bc_eq4(g, sources=src, edge_bc=True)
    assert_close(r.node_bc, node, 1e-9, f"{kind} node_bc")
    assert_close(r.edge_bc, edge, 1e-9, f"{kind} edge_bc")
    assert np.array_equal(r.depth_per_source, depth), f"{kind} depth"


def test_fullsize_grid_vs_heap_brandes_and_additivity(W, oracle):
    g = _graph(W, "grid2048")
    src = W.sample_sources(g.n, 2, 1)
    gg = W.GpuGraph(g)
    both = gg.bc(W.EngineOptions(sources=src, compute_edge_bc=True))
    assert gg.last_kernel().startswith("bc_flat_kernel") and gg.last_run_stats()["flat_fallback_sources"] == 0
    parts = [gg.bc(W.EngineOptions(sources=[s])) for s in src]
    gg.close()
    node, edge, depth = oracle.bc_eq4(g, sources=src, edge_bc=True)
    assert_close(both.node_bc, node, 1e-9, "grid node_bc vs Eq. 4 oracle")
    assert_close(both.edge_bc, edge, 1e-9, "grid edge_bc vs Eq. 4 oracle")
    assert np.array_equal(both.depth_per_source, depth), "grid depth vs Eq. 4 oracle"
    assert_close(both.node_bc, oracle.brandes(g, sources=src), 1e-9, "grid node_bc vs brandes")
    assert_close(both.node_bc, parts[0].node_bc + parts[1].node_bc, 1e-9, "additivity over sources")
    assert all(both.depth_per_source[s] == p.depth_per_source[s] for s, p in zip(src, parts))
    assert all(both.depth_per_source[s] > 1000 for s in src)  # ~1e5 Eq. 4 rounds on this grid
