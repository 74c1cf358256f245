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
