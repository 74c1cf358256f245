"""The N>1 bench path on real kernels: source sharding across ranks plus the
one BC all-reduce.  This pool has one GPU, so two ranks share
it and reduce over gloo (NCCL refuses two ranks on one device); the
partitioning and reduction code is the same as the NCCL run's."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, approx_rel

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(cmd, tmp_path):
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_two_ranks_match_one(tmp_path):
    common = ["--workload", "rmat16", "--steps", "1", "--warmup", "3", "--no-cpu-baseline"]
    one = _run([sys.executable, "bench.py"] + common + ["--dump-bc", str(tmp_path / "one.npy")], tmp_path)
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
                "--dist-backend", "gloo"] + common + ["--dump-bc", str(tmp_path / "two.npy")], tmp_path)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["config"]["sources_per_step"] == one["config"]["sources_per_step"]
    a, b = np.load(tmp_path / "one.npy"), np.load(tmp_path / "two.npy")
    assert a.shape == b.shape and approx_rel(a, b, 1e-9).all()     # only the fp64 summation order differs


# ---------------------------------------------------------------- in-process multi-GPU handle

def _random_graph(W, n, avg, seed, lo=1, hi=20):
    return W.build_csr(W.assign_weights(W.gen_er(n, avg, seed), lo, hi, seed))


@pytest.mark.parametrize("devices,nccl", [([0, 0], None), ([0, 0, 0], False), ([0], True)])
def test_multi_handle_matches_oracle(W, oracle, devices, nccl):
    """wbc_gpu_multi_*: sources strided over the listed devices, partials combined
    by device copies (a device repeats) or NCCL (forced on one device)."""
    if nccl:
        import torch  # noqa: F401  -- loads the process's libnccl.so.2 the handle binds to
    g = _random_graph(W, 700, 6.0, 11)
    mg = W.MultiGpuGraph(g, devices, nccl=nccl)
    try:
        info = mg.info()
        assert info["num_devices"] == len(devices) and info["uses_nccl"] == bool(nccl)
        for sources, halved in ((None, False), (W.sample_sources(g.n, 37, 5), True), ([3], False), ([], False)):
            opt = W.EngineOptions(compute_edge_bc=True, sources=sources,
                                  normalization=W.Normalization.Halved if halved else W.Normalization.Raw)
            r = mg.bc(opt)
            if sources is not None and len(sources) == 0:
                assert not r.node_bc.any() and not r.edge_bc.any() and not r.depth_per_source.any()
                continue
            node, eb, depth = oracle.bc_eq4(g, sources=sources, halved=halved, edge_bc=True)
            assert approx_rel(r.node_bc, node, 1e-9).all()
            assert approx_rel(r.edge_bc, eb, 1e-9).all()
            assert np.array_equal(r.depth_per_source, depth)
    finally:
        mg.close()


def test_multi_handle_errors(W):
    g = _random_graph(W, 50, 4.0, 2)
    mg = W.MultiGpuGraph(g, [0, 0])
    try:
        with pytest.raises(ValueError):
            mg.bc(W.EngineOptions(sources=[50]))
    finally:
        mg.close()
    with pytest.raises(Exception):
        W.MultiGpuGraph(g, [4096])


def test_bc_parallel_shards_over_env_devices(W, oracle, monkeypatch):
    g = _random_graph(W, 400, 5.0, 3)
    monkeypatch.setenv("WBC_GPU_DEVICES", "0,0")
    assert W.resolve_devices() == [0, 0]
    r = W.bc_parallel(g, W.EngineOptions(compute_edge_bc=True))
    node, eb, depth = oracle.bc_eq4(g, edge_bc=True)
    assert approx_rel(r.node_bc, node, 1e-9).all() and approx_rel(r.edge_bc, eb, 1e-9).all()
    assert np.array_equal(r.depth_per_source, depth)
