"""Dev probe: build one graph, then time several launch shapes on it (not the bench)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_05975_b200 as W

ap = argparse.ArgumentParser()
ap.add_argument("--graph", default="rmat24")
ap.add_argument("--k", type=int, default=296)
ap.add_argument("--clusters", default="2,4,8")
ap.add_argument("--nears", default="0")
ap.add_argument("--l2hots", default="-1")
ap.add_argument("--mids", default="")
a = ap.parse_args()
t = time.time()
if a.graph.startswith("grid"):
    s_ = int(a.graph[4:])
    el = W.gen_grid(s_, s_); t1 = time.time()
    el = W.assign_weights(el, 1, 1000, 1); t2 = time.time()
elif a.graph == "ba":
    el = W.gen_ba(65536, 10, 1); t1 = time.time()
    el = W.assign_weights(el, 1, 100, 1); t2 = time.time()
else:
    sc = int(a.graph[4:])
    el = W.gen_kronecker(sc, 32.0, 1); t1 = time.time()
    el = W.assign_weights(el, 1, 255, 1); t2 = time.time()
g = W.build_csr(el); t3 = time.time()
del el
print(f"graph {a.graph} n={g.n} m={g.m}: gen {t1-t:.1f}s weights {t2-t1:.1f}s csr {t3-t2:.1f}s", flush=True)
t = time.time(); gg = W.GpuGraph(g, 0); print(f"upload {time.time()-t:.1f}s {gg.info()}", flush=True)
src = W.sample_sources(g.n, a.k, 1)
import itertools
default_near = gg.info()["near_width"]
for c, nw, lh, md in itertools.product(a.clusters.split(","), a.nears.split(","), a.l2hots.split(","),
                                     a.mids.split(",") if a.mids else ["-"]):
    if md != "-":
        gg.set_param("mid", int(md))
    gg.set_param("cluster", int(c))
    if int(nw) > 0:
        gg.set_param("near_width", int(nw))
    gg.set_param("l2hot", int(lh))
    for rep in range(2):
        r = gg.bc(W.EngineOptions(sources=src))
    st = gg.last_run_stats()
    print(f"cluster={c} near={gg.info()['near_width']} l2hot={lh} mid={md}: {r.elapsed*1e3:.1f} ms for {len(src)} sources -> {g.m*len(src)/r.elapsed/1e9:.2f} GTEPS; "
          f"{gg.last_kernel()} slots {st['slots']} depth mean {r.depth_per_source[src].mean():.1f}", flush=True)
