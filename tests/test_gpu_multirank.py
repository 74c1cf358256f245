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


def test_bc_distributed_device_path_one_rank_nccl(W, oracle):
    """distributed.bc_distributed's device path (wbc_gpu_bc_device into one
    fp64 buffer, one NCCL all-reduce) in a one-rank NCCL group: node / edge BC
    and depth against the oracle, duplicates and Halved included."""
    import torch
    import torch.distributed as dist

    from paper_1701_05975_b200.distributed import bc_distributed

    g = _random_graph(W, 600, 6.0, 9)
    src = np.array([5, 9, 5, 100, 599], np.uint32)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        for halved in (False, True):
            opt = W.EngineOptions(compute_edge_bc=True, sources=src,
                                  normalization=W.Normalization.Halved if halved else W.Normalization.Raw)
            r = bc_distributed(g, opt)
            node, eb, depth = oracle.bc_eq4(g, sources=src, halved=halved, edge_bc=True)
            assert approx_rel(r.node_bc, node, 1e-9).all() and approx_rel(r.edge_bc, eb, 1e-9).all()
            assert np.array_equal(r.depth_per_source, depth)
    finally:
        dist.destroy_process_group()


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif("_gpus() < 2", reason="needs two GPUs (distinct-device NCCL)")
def test_multi_handle_distinct_devices_nccl(W, oracle):
    """wbc_gpu_multi_* over two distinct devices: real NCCL over NVLink."""
    import torch  # noqa: F401
    g = _random_graph(W, 900, 6.0, 21)
    mg = W.MultiGpuGraph(g, [0, 1], nccl=True)
    try:
        assert mg.info() == {"num_devices": 2, "uses_nccl": True}
        src = W.sample_sources(g.n, 77, 3)
        r = mg.bc(W.EngineOptions(compute_edge_bc=True, sources=src))
        node, eb, depth = oracle.bc_eq4(g, sources=src, edge_bc=True)
        assert approx_rel(r.node_bc, node, 1e-9).all() and approx_rel(r.edge_bc, eb, 1e-9).all()
        assert np.array_equal(r.depth_per_source, depth)
    finally:
        mg.close()


@pytest.mark.skipif("_gpus() < 2", reason="needs two GPUs (one NCCL rank per GPU)")
def test_bench_self_spawns_two_ranks(tmp_path):
    """`python bench.py --gpus 2` (no launcher) runs two NCCL ranks and reduces
    to the one-rank BC."""
    common = ["--workload", "rmat16", "--steps", "1", "--warmup", "3", "--no-cpu-baseline"]
    one = _run([sys.executable, "bench.py"] + common + ["--dump-bc", str(tmp_path / "one.npy")], tmp_path)
    two = _run([sys.executable, "bench.py", "--gpus", "2"] + common + ["--dump-bc", str(tmp_path / "two.npy")], tmp_path)
    assert two["n_gpus"] == 2 and two["config"]["nccl"]["nranks"] == 2
    a, b = np.load(tmp_path / "one.npy"), np.load(tmp_path / "two.npy")
    assert approx_rel(a, b, 1e-9).all()


def test_bench_self_spawn_refuses_missing_gpus():
    """--gpus N beyond the visible devices fails loudly (NCCL needs one GPU per rank)."""
    n = _gpus() + 1
    p = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--workload", "rmat16", "--steps", "1",
                        "--warmup", "3", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert p.returncode != 0 and f"needs {n} visible GPUs" in p.stderr


def test_bench_self_spawn_gloo_two_ranks_one_gpu(tmp_path):
    """The self-spawn path itself on the one-GPU pool: --gpus 2 with gloo (ranks share the GPU)."""
    common = ["--workload", "rmat16", "--steps", "1", "--warmup", "3", "--no-cpu-baseline"]
    two = _run([sys.executable, "bench.py", "--gpus", "2", "--dist-backend", "gloo"] + common, tmp_path)
    assert two["n_gpus"] == 2
