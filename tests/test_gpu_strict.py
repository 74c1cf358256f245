"""Strict merge (EngineOptions::strict_merge, engine.cpp:389-413) on the GPU:
node and edge BC must be BITWISE the compiled reference's bc_parallel output
for the same lane width.  The reference commits sources in list order and sums
each delta over its row in slot order as `lane_width` interleaved partials
(engine.cpp:183-212); WBC_STRICT_MERGE reproduces both orders.  With one
worker the reference's default (non-strict) path has the same order too.
"""
import numpy as np
import pytest

import fixtures as F

pytestmark = pytest.mark.gpu

STRATS = ("we", "warp4", "we-warp8", "warp16", "we-warp32")


def _graphs(W):
    yield "er", F.weighted(W.gen_er(600, 6.0, 21), 1, 20, 21)
    yield "rmat", W.assign_weights(W.gen_kronecker(11, 16.0, 4), 1, 255, 4)
    yield "ba", W.assign_weights(W.gen_ba(900, 5, 2), 1, 9, 2)   # small weights: many ties
    yield "grid", W.assign_weights(W.gen_grid(24, 30), 1, 4, 3)
    yield "unit", W.assign_weights(W.gen_er(300, 10.0, 8), 1, 1, 8)  # sigma ties everywhere


def _same(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _run(W, g, strat, sources, halved=False, shape=None):
    gg = W.GpuGraph(g)
    try:
        if shape == "w":
            gg.set_param("cluster", 1)
            gg.set_param("threads", 32)
        elif shape is not None:
            gg.set_param("cluster", shape)
        opt = W.EngineOptions(strategy=W.parse_strategy(strat), compute_edge_bc=True, strict_merge=True,
                              sources=sources,
                              normalization=W.Normalization.Halved if halved else W.Normalization.Raw)
        return gg.bc(opt)
    finally:
        gg.close()


@pytest.mark.parametrize("strat", STRATS)
def test_strict_bitwise_vs_reference(W, ref, strat):
    for name, el in _graphs(W):
        g = W.build_csr(el)
        rg = ref.build_csr(el.u, el.v, el.w)
        try:
            src = W.sample_sources(g.n, 70, 5)
            src = np.concatenate([src, src[:3]])          # duplicates count twice (engine.cpp:349-361)
            want = ref.bc_parallel(rg, strat, 3, sources=src, edge_bc=True, strict_merge=True)
            r = _run(W, g, strat, src)
            assert _same(r.node_bc, want["node_bc"]), f"{name} {strat}: node_bc not bitwise"
            assert _same(r.edge_bc, want["edge_bc"]), f"{name} {strat}: edge_bc not bitwise"
            assert np.array_equal(r.depth_per_source, want["depth"]), f"{name} {strat}: depth"
        finally:
            ref.free_csr(rg)


@pytest.mark.parametrize("shape", [1, 2, 4, "w"])
def test_strict_every_team_shape(W, ref, shape):
    el = W.assign_weights(W.gen_kronecker(12, 16.0, 9), 1, 255, 9)
    g = W.build_csr(el)
    rg = ref.build_csr(el.u, el.v, el.w)
    try:
        src = W.sample_sources(g.n, 50, 2)
        want = ref.bc_parallel(rg, "we-warp4", 2, sources=src, edge_bc=True, strict_merge=True, halved=True)
        r = _run(W, g, "we-warp4", src, halved=True, shape=shape)
        assert _same(r.node_bc, want["node_bc"]) and _same(r.edge_bc, want["edge_bc"])
    finally:
        ref.free_csr(rg)


def test_strict_all_sources_equals_single_worker_default(W, ref):
    """All sources, lane width 1: the reference's one-worker default path
    sums in the same order as its strict path, so both are bitwise ours."""
    el = F.weighted(W.gen_er(700, 5.0, 13), 1, 30, 13)
    g = W.build_csr(el)
    rg = ref.build_csr(el.u, el.v, el.w)
    try:
        want = ref.bc_parallel(rg, "np", 1, edge_bc=True)
        r = W.bc_parallel(g, W.EngineOptions(strategy=W.parse_strategy("np"), compute_edge_bc=True,
                                             strict_merge=True))
        assert _same(r.node_bc, want["node_bc"]) and _same(r.edge_bc, want["edge_bc"])
        assert np.array_equal(r.depth_per_source, want["depth"])
    finally:
        ref.free_csr(rg)


def test_strict_is_run_to_run_identical_and_close_to_default(W):
    el = W.assign_weights(W.gen_kronecker(12, 16.0, 2), 1, 255, 2)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 300, 1)
    a = _run(W, g, "we", src)
    b = _run(W, g, "we", src, shape=2)
    assert _same(a.node_bc, b.node_bc) and _same(a.edge_bc, b.edge_bc)
    gg = W.GpuGraph(g)
    try:
        d = gg.bc(W.EngineOptions(compute_edge_bc=True, sources=src))
    finally:
        gg.close()
    F_ok = np.abs(d.node_bc - a.node_bc) <= 1e-9 * np.maximum(1e-12, np.abs(a.node_bc))
    assert F_ok.all()


def test_strict_multi_handle(W, ref):
    el = F.weighted(W.gen_er(400, 6.0, 17), 1, 15, 17)
    g = W.build_csr(el)
    rg = ref.build_csr(el.u, el.v, el.w)
    try:
        src = W.sample_sources(g.n, 90, 4)
        want = ref.bc_parallel(rg, "warp8", 4, sources=src, edge_bc=True, strict_merge=True)
        mg = W.MultiGpuGraph(g, [0, 0])
        try:
            r = mg.bc(W.EngineOptions(strategy=W.parse_strategy("warp8"), compute_edge_bc=True, strict_merge=True,
                                      sources=src))
        finally:
            mg.close()
        assert _same(r.node_bc, want["node_bc"]) and _same(r.edge_bc, want["edge_bc"])
    finally:
        ref.free_csr(rg)


def test_strict_rejects_bad_lane_width(W):
    """The ABI validates the lane width like validate_strategy (engine.cpp:110-114)."""
    import ctypes as C
    g = F.path_graph(4)
    gg = W.GpuGraph(g)
    try:
        lib = W._lib.load()
        node = np.zeros(g.n)
        for lw, ok in ((3, False), (64, False), (16, True), (0, True)):
            flags = W._lib.WBC_STRICT_MERGE | (lw << 8)
            rc = lib.wbc_gpu_bc(gg.handle, None, 0, flags, node.ctypes.data_as(C.c_void_p), None, None, None)
            assert (rc == 0) == ok, (lw, rc)
            if not ok:
                assert rc == W._lib.WBC_E_INVALID and "lane width" in W._lib.last_error()
    finally:
        gg.close()
