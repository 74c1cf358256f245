"""One-off parity check at R-MAT scale 24 (not in the test suite: the graph
build alone takes ~80 s): 2 sampled sources on the GPU against the oracle's
binary-heap Brandes, node BC within 1e-9."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1701_05975_b200 as W
from oracle import Oracle
t = time.time()
g = W.build_csr(W.assign_weights(W.gen_kronecker(24, 32.0, 1), 1, 255, 1))
print(f"build {time.time()-t:.1f}s n={g.n} m={g.m}", flush=True)
src = W.sample_sources(g.n, 2, 1)
gg = W.GpuGraph(g, 0)
r = gg.bc(W.EngineOptions(sources=src))
print(f"gpu {r.elapsed:.2f}s kernel {gg.last_kernel()} depth {r.depth_per_source[src].tolist()}", flush=True)
t = time.time()
want = Oracle().brandes(g, sources=src)
err = np.abs(r.node_bc - want) / np.maximum(1e-12, np.maximum(np.abs(r.node_bc), np.abs(want)))
print(f"oracle brandes {time.time()-t:.1f}s; max rel err {err.max():.3e}; bad {(err > 1e-9).sum()} of {g.n}; sum {want.sum():.6e}")
assert (err <= 1e-9).all()
print("R-MAT-24 parity OK")
