"""The C-ABI library loads on a GPU-less host and exports every symbol that
include/wbc_gpu.h declares, plus the C++ drop-in entry points of
include/wbc/*.hpp.  No compute call is made here."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wbc_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wbc_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("wbc_gpu_graph_create", "wbc_gpu_bc", "wbc_gpu_sssp_dump", "wbc_gpu_sssp_levels", "wbc_gpu_sssp_dag", "wbc_gpu_last_kernel", "wbc_gpu_graph_destroy",
                 "wbc_gpu_last_error", "wbc_gpu_bc_device"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1701_05975_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(declared_functions()) <= bound, set(declared_functions()) - bound


def test_cpp_dropin_symbols_exported():
    from paper_1701_05975_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", "-C", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for sig in ("wbc::bc_parallel(wbc::CsrGraph const&, wbc::EngineOptions const&)",
                "wbc::build_csr(wbc::EdgeList const&)",
                "wbc::parse_edge_list(std::istream&, double)",
                "wbc::parse_strategy(std::",
                "wbc::gen_kronecker(int, double, unsigned long, wbc::KroneckerInitiator const&)",
                "wbc::sample_sources(unsigned int, unsigned int, unsigned long)"):
        assert sig in out, sig


def test_no_oracle_in_product():
    """The product never links or imports the oracle (test infrastructure)."""
    from paper_1701_05975_b200 import _lib
    deps = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "wbc_ref" not in deps
    pkg = os.path.join(ROOT, "paper_1701_05975_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")):
                src = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "wbc_oracle" not in src and "libwbc_ref" not in src, f


def test_c_abi_error_paths_without_gpu():
    """Argument validation happens before any device work."""
    from paper_1701_05975_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.wbc_gpu_graph_create(0, 0, None, None, None, None, None, 0, None) == _lib.WBC_E_INVALID
    import numpy as np
    off = np.array([0, 1, 2], np.uint32)
    adj = np.array([1, 0], np.uint32)
    w = np.array([0.1, 0.1])                      # not a dyadic fraction i / 2^k -> unsupported
    mw = np.array([0.1, 0.1])
    rc = lib.wbc_gpu_graph_create(2, 1, off.ctypes.data, adj.ctypes.data, w.ctypes.data, mw.ctypes.data, None,
                                  -1, ctypes.byref(h))
    assert rc == _lib.WBC_E_UNSUPPORTED
    assert "dyadic" in _lib.last_error()
    for bad_w in (0.0, -1.0, float("inf")):       # weights must be positive and finite
        w2 = np.array([bad_w, bad_w])
        rc = lib.wbc_gpu_graph_create(2, 1, off.ctypes.data, adj.ctypes.data, w2.ctypes.data, w2.ctypes.data,
                                      None, -1, ctypes.byref(h))
        assert rc == _lib.WBC_E_UNSUPPORTED
    w = np.array([1.5, 1.5])
    bad = np.array([0, 1, 3], np.uint32)          # offsets[n] != 2m
    rc = lib.wbc_gpu_graph_create(2, 1, bad.ctypes.data, adj.ctypes.data, w.ctypes.data, mw.ctypes.data, None,
                                  -1, ctypes.byref(h))
    assert rc == _lib.WBC_E_INVALID


def test_flag_and_status_constants_match_the_header():
    """The Python mirror's flag / status values are the header's #defines."""
    from paper_1701_05975_b200 import _lib
    text = open(HEADER).read()
    defs = {k: int(v) for k, v in re.findall(r"#define\s+(WBC_[A-Z0-9_]+)\s+\(?(-?\d+)u?\)?", text)}
    for name in ("WBC_OK", "WBC_E_INVALID", "WBC_E_UNSUPPORTED", "WBC_E_CUDA", "WBC_E_NOMEM", "WBC_HALVED",
                 "WBC_EDGE_BC", "WBC_STRICT_MERGE", "WBC_MULTI_NO_NCCL", "WBC_MULTI_FORCE_NCCL"):
        assert name in defs, name
        assert getattr(_lib, name) == defs[name], name
    assert "WBC_DETERMINISTIC WBC_STRICT_MERGE" in text
