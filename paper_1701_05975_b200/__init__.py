"""B200-native weighted betweenness centrality (Brandes) -- Python mirror of
the reference's C++ API (/root/reference/proj/include/wbc/*.hpp).

Same names, argument meanings and error behaviour as the reference:

* ``parse_edge_list`` / ``build_csr`` / ``graph_stats`` / ``to_edge_list`` /
  ``write_edge_list``            -> graph.hpp:43-90
* ``gen_er`` / ``gen_kronecker`` / ``assign_weights`` / ``sample_sources``
                                 -> generate.hpp:20-35 (identical streams)
  plus ``gen_ba`` / ``gen_grid`` for the BA and grid configs.
* ``Strategy`` / ``parse_strategy`` / ``strategy_name`` / ``EngineOptions`` /
  ``bc_parallel`` / ``BcResult``  -> engine.hpp:14-130, result.hpp:9-24

``std::invalid_argument`` maps to ``ValueError``, ``wbc::ParseError`` to
``ParseError`` (a ``RuntimeError`` carrying ``.line``), other failures to
``RuntimeError``.  ``bc_parallel`` runs on the GPU through the C ABI
(include/wbc_gpu.h); there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import io
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

__all__ = [
    "ParseError", "EdgeList", "CsrGraph", "GraphStats", "parse_edge_list", "build_csr", "graph_stats",
    "to_edge_list", "write_edge_list", "gen_er", "gen_kronecker", "gen_ba", "gen_grid", "assign_weights",
    "sample_sources", "FrontierMode", "Strategy", "valid_lane_width", "strategy_name", "parse_strategy",
    "SettleRule", "Normalization", "EngineOptions", "BcResult", "GpuGraph", "MultiGpuGraph", "device_count",
    "resolve_devices", "bc_parallel", "kInf",
]

kInf = float("inf")


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class ParseError(RuntimeError):
    """Input failure carrying the 1-based line number (graph.hpp:34-41)."""

    def __init__(self, line: int, what: str):
        super().__init__(what)
        self.line = line


def _raise(rc: int):
    msg = L.last_error()
    if rc == L.WBC_E_INVALID:
        raise ValueError(msg)
    raise RuntimeError(msg)


# --------------------------------------------------------------------------- graph

@dataclass
class EdgeList:
    """Validated edge list (graph.hpp:26-31) as parallel arrays."""

    u: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    v: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    w: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    self_loops_dropped: int = 0

    def __len__(self):
        return len(self.u)

    @staticmethod
    def of(entries: Sequence[tuple]) -> "EdgeList":
        """EdgeList from (u, v, w) tuples (w optional, default 1.0)."""
        u = np.array([e[0] for e in entries], np.uint64)
        v = np.array([e[1] for e in entries], np.uint64)
        w = np.array([e[2] if len(e) > 2 else 1.0 for e in entries], np.float64)
        return EdgeList(u, v, w)


@dataclass
class CsrGraph:
    """Immutable undirected CSR (graph.hpp:56-69)."""

    n: int
    m: int
    offsets: np.ndarray
    adjacency: np.ndarray
    weights: np.ndarray
    edge_id: np.ndarray
    min_incident_weight: np.ndarray
    original_id: np.ndarray
    edge_u: np.ndarray
    edge_v: np.ndarray
    merged_duplicates: int = 0

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])


@dataclass
class GraphStats:
    n: int
    m: int
    max_degree: int
    avg_degree: float


def _take_edges(h) -> EdgeList:
    lib = L.load()
    n = lib.wbc_host_edges_len(h)
    el = EdgeList(np.zeros(n, np.uint64), np.zeros(n, np.uint64), np.zeros(n, np.float64),
                  int(lib.wbc_host_edges_self_loops(h)))
    if n:
        lib.wbc_host_edges_get(h, _p(el.u), _p(el.v), _p(el.w))
    lib.wbc_host_edges_free(h)
    return el


def _make_edges(el: EdgeList):
    u = np.ascontiguousarray(el.u, np.uint64)
    v = np.ascontiguousarray(el.v, np.uint64)
    w = np.ascontiguousarray(el.w, np.float64)
    return L.load().wbc_host_edges_new(len(u), _p(u), _p(v), _p(w))


def parse_edge_list(source, default_weight: float = 1.0) -> EdgeList:
    """Reads 'u v' / 'u v w' lines from a str, bytes or text stream (graph.hpp:43-47)."""
    if hasattr(source, "read"):
        source = source.read()
    data = source.encode() if isinstance(source, str) else bytes(source)
    h = C.c_void_p()
    line = C.c_uint64()
    rc = L.load().wbc_host_parse_edge_list(data, len(data), float(default_weight), C.byref(h), C.byref(line))
    if rc == L.WBC_E_PARSE:
        raise ParseError(int(line.value), L.last_error())
    if rc:
        _raise(rc)
    return _take_edges(h)


def build_csr(edges: EdgeList) -> CsrGraph:
    """Compaction, min-weight dedup, two slots per edge (graph.hpp:71-74)."""
    lib = L.load()
    eh = _make_edges(edges)
    h = C.c_void_p()
    rc = lib.wbc_host_build_csr(eh, C.byref(h))
    lib.wbc_host_edges_free(eh)
    if rc:
        _raise(rc)
    n, m, merged = C.c_uint32(), C.c_uint32(), C.c_uint64()
    lib.wbc_host_csr_dims(h, C.byref(n), C.byref(m), C.byref(merged))
    n, m = n.value, m.value
    g = CsrGraph(n, m, np.zeros(n + 1, np.uint32), np.zeros(2 * m, np.uint32), np.zeros(2 * m, np.float64),
                 np.zeros(2 * m, np.uint32), np.zeros(n, np.float64), np.zeros(n, np.uint64),
                 np.zeros(m, np.uint32), np.zeros(m, np.uint32), int(merged.value))
    lib.wbc_host_csr_get(h, _p(g.offsets), _p(g.adjacency), _p(g.weights), _p(g.edge_id),
                         _p(g.min_incident_weight), _p(g.original_id), _p(g.edge_u), _p(g.edge_v))
    lib.wbc_host_csr_free(h)
    return g


def graph_stats(g: CsrGraph) -> GraphStats:
    deg = np.diff(g.offsets.astype(np.int64)) if g.n else np.zeros(0, np.int64)
    return GraphStats(g.n, g.m, int(deg.max()) if g.n else 0, 2.0 * g.m / g.n if g.n else 0.0)


def to_edge_list(g: CsrGraph) -> EdgeList:
    w = np.zeros(g.m, np.float64)
    w[g.edge_id] = g.weights
    return EdgeList(g.original_id[g.edge_u], g.original_id[g.edge_v], w)


def write_edge_list(out, edges: EdgeList, header: Sequence[str] = ()) -> None:
    for h in header:
        out.write(f"# {h}\n")
    for a, b, w in zip(edges.u.tolist(), edges.v.tolist(), edges.w.tolist()):
        out.write(f"{a} {b} {_g17(w)}\n")


def _g17(x: float) -> str:
    return "%.17g" % x


# --------------------------------------------------------------------------- generators

def _gen(fn, *args) -> EdgeList:
    h = C.c_void_p()
    rc = fn(*args, C.byref(h))
    if rc:
        _raise(rc)
    return _take_edges(h)


def gen_er(n: int, avg_degree: float, seed: int) -> EdgeList:
    """G(n, m) with m = round(n*avg_degree/2) (generate.hpp:20-23)."""
    return _gen(L.load().wbc_host_gen_er, n, float(avg_degree), seed)


def gen_kronecker(scale: int, avg_degree: float, seed: int) -> EdgeList:
    """R-MAT descent 0.57/0.19/0.19/0.05 (generate.hpp:10-27)."""
    return _gen(L.load().wbc_host_gen_kronecker, scale, float(avg_degree), seed)


def gen_ba(n: int, m: int, seed: int) -> EdgeList:
    """Barabasi-Albert preferential attachment (new; include/wbc/generate.hpp)."""
    return _gen(L.load().wbc_host_gen_ba, n, m, seed)


def gen_grid(rows: int, cols: int) -> EdgeList:
    """Row-major 4-neighbour lattice (new; include/wbc/generate.hpp)."""
    return _gen(L.load().wbc_host_gen_grid, rows, cols)


def assign_weights(edges: EdgeList, lo: int, hi: int, seed: int) -> EdgeList:
    """Uniform integer weights in [lo, hi] (generate.hpp:29-31)."""
    lib = L.load()
    h = _make_edges(edges)
    rc = lib.wbc_host_assign_weights(h, lo, hi, seed)
    if rc:
        lib.wbc_host_edges_free(h)
        _raise(rc)
    out = _take_edges(h)
    out.self_loops_dropped = edges.self_loops_dropped
    return out


def sample_sources(n: int, k: int, seed: int) -> np.ndarray:
    """k distinct ascending ids from [0, n) (generate.hpp:33-35)."""
    out = np.zeros(max(min(k, n), 1), np.uint32)
    ln = C.c_uint32()
    rc = L.load().wbc_host_sample_sources(n, k, seed, _p(out), C.byref(ln))
    if rc:
        _raise(rc)
    return out[: ln.value].copy()


# --------------------------------------------------------------------------- engine

class FrontierMode(enum.Enum):
    ScanAll = 0
    Queue = 1


@dataclass
class Strategy:
    frontier_mode: FrontierMode = FrontierMode.Queue
    lane_width: int = 1


def valid_lane_width(w: int) -> bool:
    return w in (1, 4, 8, 16, 32)


def strategy_name(s: Strategy) -> str:
    q = s.frontier_mode == FrontierMode.Queue
    if s.lane_width == 1:
        return "we" if q else "np"
    return ("we-warp" if q else "warp") + str(s.lane_width)


def parse_strategy(token: str) -> Strategy:
    """np | we | warp[W] | we-warp[W] (engine.cpp:21-40)."""
    if token == "np":
        return Strategy(FrontierMode.ScanAll, 1)
    if token == "we":
        return Strategy(FrontierMode.Queue, 1)
    if token.startswith("we-warp"):
        mode, rest = FrontierMode.Queue, token[7:]
    elif token.startswith("warp"):
        mode, rest = FrontierMode.ScanAll, token[4:]
    else:
        raise ValueError(f"unknown strategy '{token}'")
    try:
        w = int(rest) if rest else 32
    except ValueError:
        w = 0
    if not valid_lane_width(w):
        raise ValueError(f"invalid lane width in strategy '{token}' (expected 1, 4, 8, 16 or 32)")
    return Strategy(mode, w)


class SettleRule(enum.Enum):
    StrictLess = 0
    LessEqual = 1


class Normalization(enum.Enum):
    Raw = 0
    Halved = 1


@dataclass
class EngineOptions:
    strategy: Strategy = field(default_factory=Strategy)
    workers: int = 1
    compute_edge_bc: bool = False
    normalization: Normalization = Normalization.Raw
    strict_merge: bool = False
    settle_rule: SettleRule = SettleRule.StrictLess
    sources: Optional[Sequence[int]] = None


@dataclass
class BcResult:
    node_bc: np.ndarray
    edge_bc: np.ndarray
    depth_per_source: np.ndarray
    elapsed: float = 0.0
    # False when some shortest-path count reached 2^53 (sigma is exact below
    # it, engine.cpp:73-77): BC may then differ from the reference's
    sigma_exact: bool = True


def _validate(opt: EngineOptions) -> None:
    if not valid_lane_width(opt.strategy.lane_width):
        raise ValueError(f"invalid lane width {opt.strategy.lane_width} (expected 1, 4, 8, 16 or 32)")
    if opt.workers < 1:
        raise ValueError("bc_parallel: workers must be >= 1")
    if opt.settle_rule != SettleRule.StrictLess:
        raise ValueError("bc_parallel: SettleRule::LessEqual is a CPU-only negative control (not run on GPU)")


def _run_bc(fn, h, n: int, m: int, opt: Optional[EngineOptions]) -> BcResult:
    """Shared argument handling of wbc_gpu_bc / wbc_gpu_multi_bc (engine.cpp:372-457)."""
    opt = opt or EngineOptions()
    _validate(opt)
    node = np.zeros(n, np.float64)
    edge = np.zeros(m if opt.compute_edge_bc else 0, np.float64)
    depth = np.zeros(n, np.uint32)
    if opt.sources is not None:
        src = np.ascontiguousarray(np.asarray(opt.sources, dtype=np.int64))
        if len(src) and (src.min() < 0 or src.max() >= n):
            raise ValueError("bc_parallel: source id out of range")
        src = src.astype(np.uint32)
        if len(src) == 0:
            return BcResult(node, edge, depth, 0.0)
    else:
        src = None
    flags = (L.WBC_HALVED if opt.normalization == Normalization.Halved else 0) | \
            (L.WBC_EDGE_BC if opt.compute_edge_bc else 0)
    if opt.strict_merge:  # source-ordered commit, the reference's summation order (engine.cpp:389-413)
        flags |= L.WBC_STRICT_MERGE | (opt.strategy.lane_width & 0xFF) << 8
    el = C.c_double()
    rc = fn(h, _p(src), 0 if src is None else len(src), flags, _p(node),
            _p(edge) if opt.compute_edge_bc else None, _p(depth), C.byref(el))
    if rc:
        _raise(rc)
    return BcResult(node, edge, depth, el.value)


def _run_info(h) -> dict:
    """wbc_gpu_last_run_info: synchronises the graph's device, then reads the run's counters."""
    st = np.zeros(6, np.uint64)
    rc = L.load().wbc_gpu_last_run_info(h, _p(st), len(st))
    if rc:
        _raise(rc)
    return dict(slots=int(st[0]), threads=int(st[1]), dag_overflow_sources=int(st[2]), launches=int(st[3]),
                flat_fallback_sources=int(st[4]), sigma_overflow=bool(st[5]))


def _csr_arrays(g: CsrGraph):
    return [np.ascontiguousarray(g.offsets, np.uint32), np.ascontiguousarray(g.adjacency, np.uint32),
            np.ascontiguousarray(g.weights, np.float64), np.ascontiguousarray(g.min_incident_weight, np.float64),
            np.ascontiguousarray(g.edge_id, np.uint32)]


class GpuGraph:
    """A CsrGraph resident on one GPU (wbc_gpu_graph_create); reuse across runs."""

    def __init__(self, g: CsrGraph, device: int = -1):
        lib = L.load()
        self.n, self.m = int(g.n), int(g.m)
        off, adj, w, mw, eid = _csr_arrays(g)
        h = C.c_void_p()
        rc = lib.wbc_gpu_graph_create(self.n, self.m, _p(off), _p(adj), _p(w), _p(mw),
                                      _p(eid) if len(eid) == len(adj) else None, device, C.byref(h))
        if rc:
            _raise(rc)
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            L.load().wbc_gpu_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        n, m, mw, nw = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        packed, gb = C.c_int(), C.c_uint64()
        L.load().wbc_gpu_graph_info(self._h, C.byref(n), C.byref(m), C.byref(mw), C.byref(packed), C.byref(nw),
                                    C.byref(gb))
        return dict(n=n.value, m=m.value, max_weight=mw.value, packed_slots=bool(packed.value),
                    near_width=nw.value, graph_bytes=gb.value)

    def set_tuning(self, threads_per_cta: int = 0, max_slots: int = 0, near_width: int = 0,
                   hot_vertices: int = -1):
        rc = L.load().wbc_gpu_set_tuning(self._h, threads_per_cta, max_slots, near_width, hot_vertices)
        if rc:
            _raise(rc)

    def set_param(self, name: str, value: int):
        rc = L.load().wbc_gpu_set_param(self._h, name.encode(), int(value))
        if rc:
            _raise(rc)

    def set_profiling(self, on: bool = True):
        L.load().wbc_gpu_set_profiling(self._h, int(on))

    def profile_counters(self) -> dict:
        out = np.zeros(16, np.uint64)
        rc = L.load().wbc_gpu_profile_counters(self._h, _p(out))
        if rc:
            _raise(rc)
        keys = ["rounds", "relaxed_slots", "near_scanned", "far_scanned", "refills", "improvements",
                "dag_edges", "cyc_init", "cyc_relax", "cyc_threshold", "cyc_settle", "cyc_backward",
                "abort_near", "abort_front", "abort_dag", "abort_dist"]
        return {k: int(v) for k, v in zip(keys, out)}

    def last_run_stats(self) -> dict:
        """Outcome of the last run (wbc_gpu_last_run_info; synchronises the device)."""
        return _run_info(self._h)

    def last_kernel(self) -> str:
        buf = C.create_string_buffer(96)
        L.load().wbc_gpu_last_kernel(self._h, buf, len(buf))
        return buf.value.decode()

    def bc(self, opt: Optional[EngineOptions] = None) -> BcResult:
        """bc_parallel semantics on the resident graph (engine.cpp:372-457)."""
        r = _run_bc(L.load().wbc_gpu_bc, self._h, self.n, self.m, opt)
        r.sigma_exact = not _run_info(self._h)["sigma_overflow"]
        return r

    def bc_device(self, d_sources_ptr: int, k: int, d_node_ptr: int, d_depth_ptr: int = 0,
                  d_edge_ptr: int = 0, halved: bool = False, edge_bc: bool = False, stream: int = 0) -> None:
        """Device-resident run (wbc_gpu_bc_device): pointers are CUDA device addresses
        (e.g. torch ``tensor.data_ptr()``); accumulates into node/edge; async on `stream`."""
        flags = (L.WBC_HALVED if halved else 0) | (L.WBC_EDGE_BC if edge_bc else 0)
        rc = L.load().wbc_gpu_bc_device(self._h, d_sources_ptr or None, k, flags, d_node_ptr or None,
                                        d_edge_ptr or None, d_depth_ptr or None, stream or None)
        if rc:
            _raise(rc)

    def dump_source(self, s: int) -> dict:
        """Final dist / sigma / delta / depth of one source (wbc_gpu_sssp_dump)."""
        n = self.n
        dist, sigma, delta = np.zeros(n), np.zeros(n), np.zeros(n)
        depth = C.c_uint32()
        rc = L.load().wbc_gpu_sssp_dump(self._h, s, _p(dist), _p(sigma), _p(delta), C.byref(depth))
        if rc:
            _raise(rc)
        return dict(dist=dist, sigma=sigma, delta=delta, depth=depth.value)

    def dag(self, s: int):
        """Recorded DAG edges per level (wbc_gpu_sssp_dag): list of (pred, succ) arrays, overflow flag."""
        n, m = self.n, self.m
        pred = np.zeros(max(2 * m, 1), np.uint32)
        succ = np.zeros(max(2 * m, 1), np.uint32)
        ends = np.zeros(n + 2, np.uint32)
        nl, ov = C.c_uint32(), C.c_uint32()
        rc = L.load().wbc_gpu_sssp_dag(self._h, s, _p(pred), _p(succ), _p(ends), C.byref(nl), C.byref(ov))
        if rc:
            _raise(rc)
        return [(pred[ends[i]:ends[i + 1]], succ[ends[i]:ends[i + 1]]) for i in range(nl.value)], bool(ov.value)

    def levels(self, s: int) -> list:
        """Eq. 4 levels of one source as sorted id arrays (wbc_gpu_sssp_levels)."""
        n = self.n
        order = np.zeros(max(n, 1), np.uint32)
        ends = np.zeros(n + 2, np.uint32)
        olen, nl = C.c_uint32(), C.c_uint32()
        rc = L.load().wbc_gpu_sssp_levels(self._h, s, _p(order), C.byref(olen), _p(ends), C.byref(nl))
        if rc:
            _raise(rc)
        return [np.sort(order[ends[i]:ends[i + 1]]) for i in range(nl.value)]



def device_count() -> int:
    """Visible CUDA devices (wbc_gpu_device_count); 0 without a GPU."""
    c = C.c_int()
    return c.value if L.load().wbc_gpu_device_count(C.byref(c)) == 0 else 0


def resolve_devices(device: int = -1) -> list:
    """Devices bc_parallel runs on: `device` if >= 0, else WBC_GPU_DEVICES
    ("0,1,..." or "all"), else -- under a one-process-per-GPU launcher
    (WORLD_SIZE > 1 or LOCAL_RANK set) -- the current device, else every
    visible device (host_engine.cpp resolve_devices)."""
    if device >= 0:
        return [device]
    count = device_count()
    if count < 1:
        return [-1]
    env = os.environ.get("WBC_GPU_DEVICES", "")
    if env and env != "all":
        out = [int(t) for t in env.split(",") if t]
        if out:
            return out
    launched = "LOCAL_RANK" in os.environ or int(os.environ.get("WORLD_SIZE", "1") or 1) > 1
    if launched and env != "all":
        return [-1]
    return list(range(count))


class MultiGpuGraph:
    """A CsrGraph replicated on several GPUs (wbc_gpu_multi_create).  bc() shards
    the sources strided across the devices and combines the partial BC with one
    NCCL all-reduce, or device copies when NCCL is absent / a device repeats.
    Results match GpuGraph.bc to fp64 summation order."""

    def __init__(self, g: CsrGraph, devices: Sequence[int], nccl: Optional[bool] = None):
        lib = L.load()
        self.n, self.m = int(g.n), int(g.m)
        off, adj, w, mw, eid = _csr_arrays(g)
        devs = np.ascontiguousarray(np.asarray(list(devices), dtype=np.int32))
        flags = 0 if nccl is None else (L.WBC_MULTI_FORCE_NCCL if nccl else L.WBC_MULTI_NO_NCCL)
        h = C.c_void_p()
        rc = lib.wbc_gpu_multi_create(self.n, self.m, _p(off), _p(adj), _p(w), _p(mw),
                                      _p(eid) if len(eid) == len(adj) else None, _p(devs), len(devs), flags,
                                      C.byref(h))
        if rc:
            _raise(rc)
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            L.load().wbc_gpu_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        nd, nc = C.c_int(), C.c_int()
        rc = L.load().wbc_gpu_multi_info(self._h, C.byref(nd), C.byref(nc))
        if rc:
            _raise(rc)
        return dict(num_devices=nd.value, uses_nccl=bool(nc.value))

    def set_param(self, name: str, value: int):
        lib = L.load()
        for i in range(self.info()["num_devices"]):
            rc = lib.wbc_gpu_set_param(lib.wbc_gpu_multi_device_graph(self._h, i), name.encode(), int(value))
            if rc:
                _raise(rc)

    def bc(self, opt: Optional[EngineOptions] = None) -> BcResult:
        lib = L.load()
        r = _run_bc(lib.wbc_gpu_multi_bc, self._h, self.n, self.m, opt)
        r.sigma_exact = not any(_run_info(lib.wbc_gpu_multi_device_graph(self._h, i))["sigma_overflow"]
                                for i in range(self.info()["num_devices"]))
        return r

def bc_parallel(g: CsrGraph, opt: Optional[EngineOptions] = None) -> BcResult:
    """Drop-in for wbc::bc_parallel (engine.hpp:122-130) running on the GPU."""
    opt = opt or EngineOptions()
    _validate(opt)
    if opt.sources is not None:
        src = np.asarray(opt.sources, dtype=np.int64)
        if len(src) and (src.min() < 0 or src.max() >= g.n):
            raise ValueError("bc_parallel: source id out of range")
    if g.n == 0:
        return BcResult(np.zeros(0), np.zeros(0), np.zeros(0, np.uint32), 0.0)
    if opt.sources is not None and len(opt.sources) == 0:
        return BcResult(np.zeros(g.n), np.zeros(g.m if opt.compute_edge_bc else 0), np.zeros(g.n, np.uint32), 0.0)
    devs = resolve_devices()
    gg = MultiGpuGraph(g, devs) if len(devs) > 1 else GpuGraph(g, devs[0])
    try:
        return gg.bc(opt)
    finally:
        gg.close()
