"""Engine option surface of engine.hpp (strategies, validation), CPU-only."""
import pytest

import paper_1701_05975_b200 as W
import fixtures as F


def test_strategy_names_and_parsing():                                      # test_engine.cpp:41-52
    S, Q = W.FrontierMode.ScanAll, W.FrontierMode.Queue
    assert W.strategy_name(W.Strategy(S, 1)) == "np"
    assert W.strategy_name(W.Strategy(Q, 1)) == "we"
    assert W.strategy_name(W.Strategy(S, 8)) == "warp8"
    assert W.strategy_name(W.Strategy(Q, 32)) == "we-warp32"
    assert W.parse_strategy("np").frontier_mode == S
    assert W.parse_strategy("we-warp4").lane_width == 4
    assert W.parse_strategy("warp").lane_width == 32
    assert W.parse_strategy("we-warp").frontier_mode == Q
    for bad in ("bogus", "warp5", "we-warpx"):
        with pytest.raises(ValueError):
            W.parse_strategy(bad)


def test_validation_precedes_gpu_work():                                    # test_engine.cpp:382-393
    g = F.path_graph(3)
    with pytest.raises(ValueError):
        W.bc_parallel(g, W.EngineOptions(strategy=W.Strategy(W.FrontierMode.Queue, 5)))
    with pytest.raises(ValueError):
        W.bc_parallel(g, W.EngineOptions(workers=0))
    with pytest.raises(ValueError):
        W.bc_parallel(g, W.EngineOptions(sources=[7]))
    with pytest.raises(ValueError):
        W.bc_parallel(g, W.EngineOptions(settle_rule=W.SettleRule.LessEqual))


def test_empty_inputs_need_no_gpu():                                        # test_engine.cpp:395-402
    assert len(W.bc_parallel(W.build_csr(W.EdgeList())).node_bc) == 0
    r = W.bc_parallel(F.path_graph(3), W.EngineOptions(sources=[]))
    assert r.node_bc.tolist() == [0.0, 0.0, 0.0] and r.depth_per_source.tolist() == [0, 0, 0]
