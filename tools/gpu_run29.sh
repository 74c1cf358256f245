timeout 900 python -m pytest tests/test_gpu_team.py -q -x 2>&1 | tail -2
timeout 2400 python - <<'PY' 2>&1 | tail -8
import sys, time
sys.path.insert(0, ".")
import paper_1701_05975_b200 as W
t = time.time()
g = W.build_csr(W.assign_weights(W.gen_kronecker(24, 32.0, 1), 1, 255, 1))
print(f"build {time.time()-t:.1f}s", flush=True)
gg = W.GpuGraph(g, 0)
src = W.sample_sources(g.n, 592, 1)
for c, fill in ((16, 0), (16, 1), (8, 0), (8, 1)):
    gg.set_param("cluster", c); gg.set_param("fill", fill)
    for _ in range(2):
        r = gg.bc(W.EngineOptions(sources=src))
    print(f"C={c} fill={fill}: {g.m*len(src)/r.elapsed/1e9:.2f} GTEPS stats {gg.last_run_stats()} sum {r.node_bc.sum():.6e}", flush=True)
PY
