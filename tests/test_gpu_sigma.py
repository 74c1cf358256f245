"""sigma is an integer-valued fp64 count (engine.cpp:73-77): exact in any
summation order only while it stays below 2^53.  A unit-weight k x k grid has
C(2k-2, k-1) shortest corner-to-corner paths: k = 30 gives 3.0e16 >= 2^53,
k = 20 gives 3.5e10.  Every kernel family must flag the first and not the
second (wbc_gpu_last_run_info [5], BcResult.sigma_exact)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = {"auto": {}, "one_warp": {"cluster": 1, "threads": 32}, "team1": {"cluster": 1},
          "team2": {"cluster": 2}, "flat": {"flat": 1}}


def _grid(W, k):
    return W.build_csr(W.assign_weights(W.gen_grid(k, k), 1, 1, 1))


def test_oracle_agrees_on_the_case(oracle, W):
    g = _grid(W, 30)
    o = oracle.eq4_source(g, 0)
    assert o["sigma"].max() >= 2.0 ** 53
    assert oracle.eq4_source(_grid(W, 20), 0)["sigma"].max() < 2.0 ** 53


@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_sigma_overflow_flagged(W, shape):
    for k, big in ((30, True), (20, False)):
        g = _grid(W, k)
        gg = W.GpuGraph(g)
        try:
            for name, val in SHAPES[shape].items():
                gg.set_param(name, val)
            r = gg.bc(W.EngineOptions(sources=[0, 5]))
            assert gg.last_run_stats()["sigma_overflow"] is big, (shape, k)
            assert r.sigma_exact is (not big)
            if shape == "flat":
                assert gg.last_kernel().startswith("bc_flat_kernel")
        finally:
            gg.close()
