"""Debug: per-source dumps of the team kernel vs the oracle on a kron-13 graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1701_05975_b200 as W
from oracle import Oracle
c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 13
O = Oracle()
el = W.assign_weights(W.gen_kronecker(scale, 32.0, 9), 1, 255, 9)
g = W.build_csr(el)
print("n", g.n, "m", g.m)
gg = W.GpuGraph(g); gg.set_param("cluster", c)
src = W.sample_sources(g.n, int(os.environ.get("NSRC", "8")), 2)
nbad_total = 0
for s in list(src) * int(os.environ.get("REPS", "1")):
    d = gg.dump_source(int(s)); o = O.eq4_source(g, int(s))
    bad_d = np.flatnonzero(d["dist"] != o["dist"]); bad_s = np.flatnonzero(d["sigma"] != o["sigma"])
    rel = np.abs(d["delta"] - o["delta"]) / np.maximum(1e-12, np.abs(o["delta"]))
    bad_x = np.flatnonzero(rel > 1e-12)
    nbad_total += len(bad_x) > 0
    if os.environ.get("QUIET"): continue
    print(f"s={s} depth {d['depth']} vs {o['depth']} bad dist {len(bad_d)} sigma {len(bad_s)} delta {len(bad_x)}",
          "| sigma ex", [(int(i), d['sigma'][i], o['sigma'][i]) for i in bad_s[:3]],
          "| delta ex", [(int(i), d['delta'][i], o['delta'][i], o['dist'][i]) for i in bad_x[:3]])

print("BAD SOURCES", nbad_total)
if os.environ.get("QUIET"): sys.exit(0)
print("--- level structure check")
for s in src:
    lv = gg.levels(int(s)); o = O.eq4_source(g, int(s))
    ol = [np.sort(o["order"][o["ends"][i]:o["ends"][i + 1]]) for i in range(len(o["ends"]) - 1)]
    diff = [i for i in range(min(len(lv), len(ol))) if len(lv[i]) != len(ol[i]) or not np.array_equal(lv[i], ol[i])]
    tot = sum(len(x) for x in lv)
    print(f"s={s} levels {len(lv)} vs {len(ol)}; settled {tot} vs {sum(len(x) for x in ol)}; unique {len(np.unique(np.concatenate(lv)))}; first diff {diff[:3]}",
          [ (len(lv[i]), len(ol[i])) for i in diff[:3]])

print("--- DAG check")
off, adj, wt = g.offsets, g.adjacency, g.weights
for s in src:
    o = O.eq4_source(g, int(s)); dist = o["dist"]
    ol = [o["order"][o["ends"][i]:o["ends"][i + 1]] for i in range(len(o["ends"]) - 1)]
    segs, ov = gg.dag(int(s))
    nbad = 0; msg = []
    for L, lvl in enumerate(ol):
        want = set()
        for x in lvl:
            for e in range(off[x], off[x + 1]):
                u = adj[e]
                if dist[u] + wt[e] == dist[x]:
                    want.add((int(u), int(x), int(e)))
        wp = sorted((a, b) for a, b, _ in want)
        gp = sorted(zip(segs[L][0].tolist(), segs[L][1].tolist())) if L < len(segs) else []
        if wp != gp:
            nbad += 1
            if len(msg) < 2:
                ws_, gs_ = set(wp), set(gp)
                msg.append((L, len(lvl), len(wp), len(gp), list(ws_ - gs_)[:3], list(gs_ - ws_)[:3], len(gp) - len(set(gp))))
    print(f"s={s} overflow={ov} bad levels {nbad}", msg)
