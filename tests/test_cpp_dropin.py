"""Compiles tests/cpp/test_dropin.cpp against include/wbc/*.hpp (the
reference-compatible C++ API) and libwbc_b200.so, then runs it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1701_05975_b200", "lib")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "test_dropin")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp",
           "test_dropin.cpp"), "-L", LIBDIR, "-lwbc_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    subprocess.run(cmd, check=True)
    return out


def test_cpp_dropin_cpu(binary):
    r = subprocess.run([binary, "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_gpu(binary):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_gpu_sharded(binary):
    """The same C++ checks with bc_parallel sharding its sources over two
    replicas (one physical GPU listed twice -> device-copy reduction)."""
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True, env=dict(os.environ, WBC_GPU_DEVICES="0,0"))
    assert r.returncode == 0, r.stdout + r.stderr
