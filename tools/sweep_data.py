"""Dev: sweep inputs (sorted distances, entries) of one grid-2048 source for
tools/sweep_bench.cu, with the expected depth from the oracle's Eq. 4."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import scipy.sparse.csgraph as cg
import paper_1701_05975_b200 as W
from oracle import Oracle

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep"
side = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
os.makedirs(out, exist_ok=True)
g = W.build_csr(W.assign_weights(W.gen_grid(side, side), 1, 1000, 1))
s = int(W.sample_sources(g.n, 1, 1)[0])
rows = np.repeat(np.arange(g.n), np.diff(g.offsets.astype(np.int64)))
A = sp.csr_matrix((g.weights, g.adjacency, g.offsets.astype(np.int64)), shape=(g.n, g.n))
d = cg.dijkstra(A, indices=s).astype(np.int64)
order = np.argsort(d, kind="stable")
pos = np.empty(g.n, np.int64); pos[order] = np.arange(g.n)
minw = g.min_incident_weight.astype(np.int64)
ent = np.zeros((g.n, 4), np.uint32)
du, dv, w = d[rows], d[g.adjacency], g.weights.astype(np.int64)
keep = dv > du
key = (w + minw[g.adjacency]) | ((dv - du) << 16)
slot = np.arange(len(rows)) - g.offsets[rows]
ent[pos[rows[keep]], slot[keep]] = key[keep]
np.ascontiguousarray(d[order].astype(np.uint32)).tofile(f"{out}/ord_d.bin")
ent.tofile(f"{out}/ent.bin")
_, _, depth = Oracle().bc_eq4(g, sources=[s])
B = 32
while B < int(g.weights.max()) + int(minw.max()) + 2:
    B <<= 1
open(f"{out}/meta.txt", "w").write(f"{g.n} {B} {int(depth[s])}\n")
print("source", s, "depth", int(depth[s]), "B", B)
