"""Dev probe: quick GPU timing of the BC path on a named config (not the bench)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1701_05975_b200 as W

ap = argparse.ArgumentParser()
ap.add_argument("--graph", default="rmat20")
ap.add_argument("--k", type=int, default=256)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--slots", type=int, default=0)
ap.add_argument("--near", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--hot", type=int, default=-1)
ap.add_argument("--prof", action="store_true")
ap.add_argument("--strict", default="", help="strategy token: run with strict_merge (e.g. we, we-warp8)")
ap.add_argument("--edge", action="store_true")
ap.add_argument("--param", action="append", default=[], help="name=value")
a = ap.parse_args()
t = time.time()
if a.graph.startswith("rmat"):
    el = W.assign_weights(W.gen_kronecker(int(a.graph[4:]), 32.0, 1), 1, 255, 1)
elif a.graph == "er":
    el = W.assign_weights(W.gen_er(4096, 8.0, 1), 1, 64, 1)
elif a.graph == "ba":
    el = W.assign_weights(W.gen_ba(65536, 10, 1), 1, 100, 1)
elif a.graph.startswith("mortongrid"):  # the same grid (same weights), vertex ids in Morton order
    s = int(a.graph[10:]); el = W.assign_weights(W.gen_grid(s, s), 1, 1000, 1)
    def morton(i):
        r, c = np.asarray(i) // s, np.asarray(i) % s
        z = np.zeros_like(r)
        for b in range(16):
            z |= ((c >> b) & 1) << (2 * b) | ((r >> b) & 1) << (2 * b + 1)
        return z
    mu, mv = morton(el.u.astype(np.int64)), morton(el.v.astype(np.int64))
    o = np.argsort(np.minimum(mu, mv) * 4 + (mu > mv), kind="stable")  # first appearance follows Morton order
    el = W.EdgeList(mu[o].astype(np.uint64), mv[o].astype(np.uint64), el.w[o])
elif a.graph.startswith("grid"):
    s = int(a.graph[4:]); el = W.assign_weights(W.gen_grid(s, s), 1, 1000, 1)
g = W.build_csr(el)
print(f"graph {a.graph} n={g.n} m={g.m} built in {time.time()-t:.1f}s", flush=True)
gg = W.GpuGraph(g, 0)
gg.set_tuning(a.threads, a.slots, a.near, a.hot)
if a.prof: gg.set_profiling(True)
for kv in a.param:
    k_, v_ = kv.split('='); gg.set_param(k_, int(v_))
print(gg.info(), flush=True)
src = W.sample_sources(g.n, a.k, 1)
for rep in range(a.reps):
    opt = W.EngineOptions(sources=src, compute_edge_bc=a.edge)
    if a.strict:
        opt.strict_merge, opt.strategy = True, W.parse_strategy(a.strict)
    r = gg.bc(opt)
    st = gg.last_run_stats()
    print(f"rep {rep}: {r.elapsed*1e3:.1f} ms for {len(src)} sources -> {g.m*len(src)/r.elapsed/1e9:.2f} GTEPS; "
          f"{r.elapsed/len(src)*1e3:.3f} ms/src; stats {st}; depth mean {r.depth_per_source[src].mean():.1f}", flush=True)
    if a.prof:
        pc = gg.profile_counters(); k = len(src)
        print("  per source: " + ", ".join(f"{kk}={v/k:.4g}" for kk, v in pc.items()) + f"  (2m={2*g.m})", flush=True)
        cyc = {kk: v for kk, v in pc.items() if kk.startswith("cyc_")}
        print("  aborts:", {kk: v for kk, v in pc.items() if kk.startswith("abort_")}, flush=True)
        tot = sum(cyc.values()) or 1
        print("  phase share: " + ", ".join(f"{kk[4:]}={100*v/tot:.1f}%" for kk, v in cyc.items()) +
              f"; per-CTA ms/source at 1.9GHz = {tot/k/1.9e6:.2f}", flush=True)
