"""bench.py keeps the driver's JSON contract: one line, the BASELINE metric,
the reference arm's shape on CPU, and (on a GPU) roofline / cpu_baseline /
e2e / clocks / gpu_launches on the GPU arm."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]


def _bench(args, timeout=900):
    p = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


@pytest.fixture(scope="module")
def have_ref():
    from oracle import REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")


def test_reference_arm_line(have_ref):
    d = _bench(["--impl", "reference", "--workload", "er4096", "--steps", "1", "--warmup", "0"])
    assert d["impl"] == "reference" and d["metric"] == METRIC and d["unit"] == "GTEPS"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["steps"] == 1 and d["warmup"] == 0 and d["config"]["workload"] == "er4096"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _bench(["--workload", "rmat16", "--steps", "3", "--warmup", "3"])
    assert d["metric"] == METRIC and d["unit"] == "GTEPS" and d["n_gpus"] == 1
    assert d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["data"] == "synthetic"
    assert d["config"]["workload"] == "rmat16" and "model" not in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3 and r["kernel"].startswith("bc_")
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3 and "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    cb = d["cpu_baseline"]
    assert cb["unit"] == "GTEPS" and cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
