"""Dev probe: one graph, several launch shapes (set_param sets) in turn.
    python tools/probe_shapes.py --graph rmat24 --k 296 --reps 2 "cluster=16" "cluster=12" "cluster=9,fill=0"
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_05975_b200 as W

ap = argparse.ArgumentParser()
ap.add_argument("--graph", default="rmat20")
ap.add_argument("--k", type=int, default=256)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("shapes", nargs="+")
a = ap.parse_args()
t = time.time()
if a.graph == "ba":
    g = W.build_csr(W.assign_weights(W.gen_ba(65536, 10, 1), 1, 100, 1))
elif a.graph.startswith("grid"):
    s_ = int(a.graph[4:])
    g = W.build_csr(W.assign_weights(W.gen_grid(s_, s_), 1, 1000, 1))
else:
    g = W.build_csr(W.assign_weights(W.gen_kronecker(int(a.graph[4:]), 32.0, 1), 1, 255, 1))
print(f"graph {a.graph} n={g.n} m={g.m} built in {time.time()-t:.1f}s", flush=True)
src = W.sample_sources(g.n, a.k, 1)
for rnd in range(2):
    for sh in a.shapes:
        gg = W.GpuGraph(g, 0)
        for kv in sh.split(","):
            if kv == "default":
                continue
            k_, v_ = kv.split("=")
            gg.set_param(k_, int(v_))
        best = 0.0
        for rep in range(a.reps):
            r = gg.bc(W.EngineOptions(sources=src))
            best = max(best, g.m * len(src) / r.elapsed / 1e9)
        print(f"[{rnd}] {sh:24s} best {best:.2f} GTEPS  {gg.last_kernel()}  {gg.last_run_stats()}", flush=True)
        gg.close()
