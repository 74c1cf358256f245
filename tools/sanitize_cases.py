"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck).  Each case is checked against the oracle too.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1701_05975_b200 as W  # noqa: E402
from oracle import Oracle  # noqa: E402

O = Oracle()
tol = lambda a, b: np.abs(a - b) <= np.maximum(1e-12, 1e-9 * np.maximum(np.abs(a), np.abs(b)))  # noqa: E731
kron = W.build_csr(W.assign_weights(W.gen_kronecker(11, 16.0, 3), 1, 255, 3))
grid = W.build_csr(W.assign_weights(W.gen_grid(24, 24), 1, 1000, 3))
bip = W.build_csr(W.EdgeList.of([(i, 60 + j, 1.0) for i in range(60) for j in range(60)]))  # DAG > buffer: row-scan fallback
cases = [("per-CTA kernel (tiny graph)", kron, {}),
         ("team C=1", kron, {"cluster": 1}),
         ("team C=2", kron, {"cluster": 2}),
         ("team C=4", kron, {"cluster": 4}),
         ("one-warp team", grid, {"cluster": 1, "threads": 32}),
         ("team C=4 + 2-CTA fill", kron, {"cluster": 4, "fill": 1}),
         ("flat kernel, 1024 threads", grid, {"flat": 1, "slots": 3}),
         ("flat kernel, 256 threads", grid, {"flat": 1, "flat_threads": 256, "slots": 2}),
         ("flat kernel, near queues spilling", grid, {"flat": 1, "flat_sq": 32, "slots": 3}),
         ("flat kernel, long distances", W.build_csr(W.assign_weights(W.gen_grid(6, 6), 200, 1000, 3)), {"flat": 1}),
         ("flat kernel, unit weights", W.build_csr(W.assign_weights(W.gen_grid(12, 10), 1, 1, 3)), {"flat": 1}),
         ("strict merge (team C=2)", kron, {"cluster": 2, "_strict": 8}),
         ("team C=1, DAG overflow", bip, {"cluster": 1}),
         ("team C=4, DAG overflow", bip, {"cluster": 4})]
for name, g, params in cases:
    src = W.sample_sources(g.n, 12 if params.get("flat") else 6, 1)  # flat: more sources than CTAs cycle the sweep buffers
    gg = W.GpuGraph(g, 0)
    strict = params.pop("_strict", 0)
    for k, v in params.items():
        gg.set_param(k, v)
    opt = W.EngineOptions(sources=src, compute_edge_bc=True)
    if strict:
        opt.strict_merge, opt.strategy = True, W.Strategy(W.FrontierMode.Queue, strict)
    r = gg.bc(opt)
    kern = gg.last_kernel()
    gg.close()
    node, edge, depth = O.bc_eq4(g, sources=src, edge_bc=True)
    ok = tol(r.node_bc, node).all() and tol(r.edge_bc, edge).all() and np.array_equal(r.depth_per_source, depth)
    print(f"{name:28s} {kern:26s} {'ok' if ok else 'MISMATCH'}", flush=True)
    assert ok
