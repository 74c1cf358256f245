"""ctypes binding of lib/libwbc_b200.so (include/wbc_gpu.h).

The shared library is built in-tree by ``make -C paper_1701_05975_b200`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
every call raises ``RuntimeError`` naming the build command.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# WBC_LIB overrides the library path (A/B experiments between builds)
LIB_PATH = os.environ.get("WBC_LIB") or os.path.join(HERE, "lib", "libwbc_b200.so")

WBC_OK = 0
WBC_E_INVALID = -1
WBC_E_UNSUPPORTED = -2
WBC_E_CUDA = -3
WBC_E_NOMEM = -4
WBC_E_NOT_BUILT = -5
WBC_E_PARSE = -6
WBC_HALVED = 1
WBC_EDGE_BC = 2
WBC_STRICT_MERGE = 4
WBC_MULTI_NO_NCCL = 1
WBC_MULTI_FORCE_NCCL = 2

vp = C.c_void_p
u32, u64, i32, i64, f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_int64, C.c_double

# (name, restype, argtypes) -- every symbol include/wbc_gpu.h declares.
SIGNATURES = [
    ("wbc_gpu_graph_create", i32, [u32, u32, vp, vp, vp, vp, vp, i32, C.POINTER(vp)]),
    ("wbc_gpu_graph_destroy", None, [vp]),
    ("wbc_gpu_bc", i32, [vp, vp, u64, u32, vp, vp, vp, C.POINTER(f64)]),
    ("wbc_gpu_bc_device", i32, [vp, vp, u64, u32, vp, vp, vp, vp]),
    ("wbc_gpu_sssp_dump", i32, [vp, u32, vp, vp, vp, C.POINTER(u32)]),
    ("wbc_gpu_last_kernel", i32, [vp, C.c_char_p, C.c_size_t]),
    ("wbc_gpu_sssp_dag", i32, [vp, u32, vp, vp, vp, C.POINTER(u32), C.POINTER(u32)]),
    ("wbc_gpu_sssp_levels", i32, [vp, u32, vp, C.POINTER(u32), vp, C.POINTER(u32)]),
    ("wbc_gpu_graph_info", i32, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32), C.POINTER(i32),
                                 C.POINTER(u32), C.POINTER(u64)]),
    ("wbc_gpu_set_tuning", i32, [vp, i32, i32, u32, i64]),
    ("wbc_gpu_set_param", i32, [vp, C.c_char_p, i64]),
    ("wbc_gpu_set_profiling", i32, [vp, i32]),
    ("wbc_gpu_profile_counters", i32, [vp, vp]),
    ("wbc_gpu_last_run_stats", i32, [vp, vp]),
    ("wbc_gpu_last_run_info", i32, [vp, vp, u32]),
    ("wbc_gpu_last_error", C.c_char_p, []),
    ("wbc_gpu_device_count", i32, [C.POINTER(i32)]),
    ("wbc_gpu_multi_create", i32, [u32, u32, vp, vp, vp, vp, vp, vp, i32, i32, C.POINTER(vp)]),
    ("wbc_gpu_multi_bc", i32, [vp, vp, u64, u32, vp, vp, vp, C.POINTER(f64)]),
    ("wbc_gpu_multi_info", i32, [vp, C.POINTER(i32), C.POINTER(i32)]),
    ("wbc_gpu_multi_device_graph", vp, [vp, i32]),
    ("wbc_gpu_multi_destroy", None, [vp]),
    ("wbc_host_parse_edge_list", i32, [C.c_char_p, C.c_size_t, f64, C.POINTER(vp), C.POINTER(u64)]),
    ("wbc_host_edges_new", vp, [u64, vp, vp, vp]),
    ("wbc_host_edges_len", u64, [vp]),
    ("wbc_host_edges_self_loops", u64, [vp]),
    ("wbc_host_edges_get", None, [vp, vp, vp, vp]),
    ("wbc_host_edges_free", None, [vp]),
    ("wbc_host_gen_er", i32, [u64, f64, u64, C.POINTER(vp)]),
    ("wbc_host_gen_kronecker", i32, [i32, f64, u64, C.POINTER(vp)]),
    ("wbc_host_gen_ba", i32, [u64, u32, u64, C.POINTER(vp)]),
    ("wbc_host_gen_grid", i32, [u32, u32, C.POINTER(vp)]),
    ("wbc_host_assign_weights", i32, [vp, i32, i32, u64]),
    ("wbc_host_sample_sources", i32, [u32, u32, u64, vp, C.POINTER(u32)]),
    ("wbc_host_build_csr", i32, [vp, C.POINTER(vp)]),
    ("wbc_host_csr_dims", None, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u64)]),
    ("wbc_host_csr_get", None, [vp] + [vp] * 8),
    ("wbc_host_csr_free", None, [vp]),
]

_lib = None


def load():
    """Load (once) and return the native library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
                               "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().wbc_gpu_last_error().decode(errors="replace")
