"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU checkers.

* ``Oracle``  -> oracle/liboracle.so, the plain-C restatement (wbc_oracle.c)
* ``RefLib``  -> oracle/_ref/libwbc_ref.so, the UNMODIFIED reference library
  compiled from /root/reference/proj/src plus our extern "C" shim.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the reported CPU baseline.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwbc_ref.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Csr:
    """Plain CSR container with the reference's CsrGraph fields (graph.hpp:56-69)."""

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
    extra: dict = field(default_factory=dict)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """The plain-C restatement (oracle/wbc_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        for name in ("orc_build_csr", "orc_brandes", "orc_eq4_source", "orc_bc_eq4", "orc_eq4_profile"):
            getattr(self.lib, name).restype = C.c_int

    def build_csr(self, u, v, w) -> Csr:
        u = np.ascontiguousarray(u, dtype=np.uint64)
        v = np.ascontiguousarray(v, dtype=np.uint64)
        w = _f64(w)
        L = len(u)
        n_out, m_out, merged = C.c_uint32(), C.c_uint32(), C.c_uint64()
        offsets = np.zeros(2 * L + 1, np.uint32)
        adjacency = np.zeros(max(2 * L, 1), np.uint32)
        weights = np.zeros(max(2 * L, 1), np.float64)
        edge_id = np.zeros(max(2 * L, 1), np.uint32)
        minw = np.zeros(max(2 * L, 1), np.float64)
        orig = np.zeros(max(2 * L, 1), np.uint64)
        eu = np.zeros(max(L, 1), np.uint32)
        ev = np.zeros(max(L, 1), np.uint32)
        rc = self.lib.orc_build_csr(
            C.c_uint64(L), _ptr(u), _ptr(v), _ptr(w), C.byref(n_out), C.byref(m_out),
            _ptr(offsets), _ptr(adjacency), _ptr(weights), _ptr(edge_id), _ptr(minw),
            _ptr(orig), _ptr(eu), _ptr(ev), C.byref(merged))
        if rc:
            raise MemoryError("orc_build_csr failed")
        n, m = n_out.value, m_out.value
        return Csr(n, m, offsets[: n + 1].copy(), adjacency[: 2 * m].copy(), weights[: 2 * m].copy(),
                   edge_id[: 2 * m].copy(), minw[:n].copy(), orig[:n].copy(), eu[:m].copy(),
                   ev[:m].copy(), merged.value)

    @staticmethod
    def _graph(g):
        return (_u32(g.offsets), _u32(g.adjacency), _f64(g.weights), _u32(g.edge_id),
                _f64(g.min_incident_weight))

    def brandes(self, g, sources=None, halved=False, edge_bc=False):
        off, adj, w, eid, _ = self._graph(g)
        src = None if sources is None else _u32(sources)
        k = -1 if sources is None else len(src)
        node = np.zeros(g.n, np.float64)
        edge = np.zeros(g.m, np.float64) if edge_bc else None
        rc = self.lib.orc_brandes(C.c_uint32(g.n), C.c_uint32(g.m), _ptr(off), _ptr(adj), _ptr(w),
                                  _ptr(eid), _ptr(src), C.c_int64(k), C.c_int(int(halved)),
                                  _ptr(node), _ptr(edge))
        if rc:
            raise ValueError("source id out of range")
        return (node, edge) if edge_bc else node

    def eq4_source(self, g, s, less_equal=False, edge_bc=False):
        off, adj, w, eid, minw = self._graph(g)
        n = g.n
        dist = np.zeros(n, np.float64)
        sigma = np.zeros(n, np.float64)
        delta = np.zeros(n, np.float64)
        order = np.zeros(n + 1, np.uint32)
        ends = np.zeros(n + 2, np.uint32)
        olen, elen = C.c_uint32(), C.c_uint32()
        acc = np.zeros(n, np.float64)
        eacc = np.zeros(g.m, np.float64) if edge_bc else None
        rc = self.lib.orc_eq4_source(C.c_uint32(n), _ptr(off), _ptr(adj), _ptr(w), _ptr(eid), _ptr(minw),
                                     C.c_uint32(s), C.c_int(int(less_equal)), _ptr(dist), _ptr(sigma),
                                     _ptr(delta), _ptr(order), C.byref(olen), _ptr(ends), C.byref(elen),
                                     _ptr(acc), _ptr(eacc))
        if rc:
            raise ValueError("source out of range")
        out = dict(dist=dist, sigma=sigma, delta=delta, order=order[: olen.value].copy(),
                   ends=ends[: elen.value].copy(), depth=elen.value - 1, node_acc=acc)
        if edge_bc:
            out["edge_acc"] = eacc
        return out

    def bc_eq4(self, g, sources=None, halved=False, edge_bc=False):
        off, adj, w, eid, minw = self._graph(g)
        src = None if sources is None else _u32(sources)
        k = -1 if sources is None else len(src)
        node = np.zeros(g.n, np.float64)
        edge = np.zeros(g.m, np.float64) if edge_bc else None
        depth = np.zeros(g.n, np.uint32)
        rc = self.lib.orc_bc_eq4(C.c_uint32(g.n), C.c_uint32(g.m), _ptr(off), _ptr(adj), _ptr(w), _ptr(eid),
                                 _ptr(minw), _ptr(src), C.c_int64(k), C.c_int(int(halved)), _ptr(node),
                                 _ptr(edge), _ptr(depth))
        if rc:
            raise ValueError("source id out of range")
        return node, edge, depth

    def eq4_profile(self, g, s):
        off, adj, w, _, minw = self._graph(g)
        st = np.zeros(9, np.float64)
        self.lib.orc_eq4_profile(C.c_uint32(g.n), _ptr(off), _ptr(adj), _ptr(w), _ptr(minw),
                                 C.c_uint32(s), _ptr(st))
        keys = ["rounds", "pending_sum", "relaxed_slots", "improvements", "dag_edges",
                "max_pending", "max_frontier", "reached", "max_dist"]
        return dict(zip(keys, st.tolist()))


class RefError(Exception):
    pass


class RefLib:
    """The reference library itself (oracle/_ref/libwbc_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_edges_new.restype = C.c_void_p
        L.ref_edges_len.restype = C.c_uint64
        L.ref_edges_len.argtypes = [C.c_void_p]
        L.ref_edges_self_loops.restype = C.c_uint64
        L.ref_edges_self_loops.argtypes = [C.c_void_p]
        L.ref_edges_free.argtypes = [C.c_void_p]
        L.ref_edges_get.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_edges_set.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_csr_n.restype = C.c_uint32
        L.ref_csr_n.argtypes = [C.c_void_p]
        L.ref_csr_m.restype = C.c_uint32
        L.ref_csr_m.argtypes = [C.c_void_p]
        L.ref_csr_merged.restype = C.c_uint64
        L.ref_csr_merged.argtypes = [C.c_void_p]
        L.ref_csr_free.argtypes = [C.c_void_p]
        L.ref_csr_get.argtypes = [C.c_void_p] + [C.c_void_p] * 8
        L.ref_format_node_tsv.restype = C.c_uint64
        L.ref_format_node_tsv.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]
        L.ref_format_edge_tsv.restype = C.c_uint64
        L.ref_format_edge_tsv.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]

    def _check(self, rc):
        if rc:
            msg = self.lib.ref_last_error().decode()
            if rc == -1:
                raise ValueError(msg)
            raise RefError(msg)

    # -- edge lists (returned as numpy triples) --
    def _take_edges(self, h):
        L = self.lib.ref_edges_len(h)
        u = np.zeros(L, np.uint64)
        v = np.zeros(L, np.uint64)
        w = np.zeros(L, np.float64)
        if L:
            self.lib.ref_edges_get(h, _ptr(u), _ptr(v), _ptr(w))
        loops = self.lib.ref_edges_self_loops(h)
        self.lib.ref_edges_free(h)
        return u, v, w, loops

    def _make_edges(self, u, v, w):
        h = C.c_void_p(self.lib.ref_edges_new())
        u = np.ascontiguousarray(u, np.uint64)
        v = np.ascontiguousarray(v, np.uint64)
        w = _f64(w)
        self.lib.ref_edges_set(h, len(u), _ptr(u), _ptr(v), _ptr(w))
        return h

    def gen_er(self, n, avg_degree, seed):
        h = C.c_void_p()
        self._check(self.lib.ref_gen_er(C.c_uint64(n), C.c_double(avg_degree), C.c_uint64(seed), C.byref(h)))
        return self._take_edges(h)[:3]

    def gen_kronecker(self, scale, avg_degree, seed):
        h = C.c_void_p()
        self._check(self.lib.ref_gen_kronecker(C.c_int(scale), C.c_double(avg_degree), C.c_uint64(seed),
                                               C.byref(h)))
        return self._take_edges(h)[:3]

    def assign_weights(self, u, v, w, lo, hi, seed):
        h = self._make_edges(u, v, w)
        self._check(self.lib.ref_assign_weights(h, C.c_int(lo), C.c_int(hi), C.c_uint64(seed)))
        return self._take_edges(h)[:3]

    def sample_sources(self, n, k, seed):
        out = np.zeros(max(min(k, n), 1), np.uint32)
        ln = C.c_uint32()
        self._check(self.lib.ref_sample_sources(C.c_uint32(n), C.c_uint32(k), C.c_uint64(seed), _ptr(out),
                                                C.byref(ln)))
        return out[: ln.value].copy()

    def parse_edge_list(self, text: str, default_weight=1.0):
        h = C.c_void_p()
        rc = self.lib.ref_parse_edge_list(text.encode(), C.c_double(default_weight), C.byref(h))
        if rc:
            msg = self.lib.ref_last_error().decode()
            raise (ValueError if rc == -1 else RefError)(msg)
        return self._take_edges(h)

    # -- CSR --
    def build_csr_handle(self, u, v, w):
        eh = self._make_edges(u, v, w)
        h = C.c_void_p()
        self._check(self.lib.ref_csr_build(eh, C.byref(h)))
        self.lib.ref_edges_free(eh)
        return h

    def csr_arrays(self, h) -> Csr:
        n, m = self.lib.ref_csr_n(h), self.lib.ref_csr_m(h)
        off = np.zeros(n + 1, np.uint32)
        adj = np.zeros(max(2 * m, 1), np.uint32)
        w = np.zeros(max(2 * m, 1), np.float64)
        eid = np.zeros(max(2 * m, 1), np.uint32)
        minw = np.zeros(max(n, 1), np.float64)
        orig = np.zeros(max(n, 1), np.uint64)
        eu = np.zeros(max(m, 1), np.uint32)
        ev = np.zeros(max(m, 1), np.uint32)
        self.lib.ref_csr_get(h, _ptr(off), _ptr(adj), _ptr(w), _ptr(eid), _ptr(minw), _ptr(orig), _ptr(eu),
                             _ptr(ev))
        return Csr(n, m, off, adj[: 2 * m], w[: 2 * m], eid[: 2 * m], minw[:n], orig[:n], eu[:m], ev[:m],
                   self.lib.ref_csr_merged(h))

    def build_csr(self, u, v, w) -> Csr:
        h = self.build_csr_handle(u, v, w)
        g = self.csr_arrays(h)
        g.extra["handle"] = h
        return g

    def csr_from_arrays(self, g) -> Csr:
        """A reference CsrGraph holding the arrays of ``g`` (any object with the
        CsrGraph fields): the repo's build_csr output is array-identical to the
        reference's (tests/test_host_graph.py), so this skips the reference's
        single-threaded build on large graphs."""
        off, adj, eid = _u32(g.offsets), _u32(g.adjacency), _u32(g.edge_id)
        w, minw = _f64(g.weights), _f64(g.min_incident_weight)
        h = C.c_void_p()
        self.lib.ref_csr_from_arrays.argtypes = [C.c_uint32, C.c_uint32] + [C.c_void_p] * 5 + [C.c_void_p]
        self._check(self.lib.ref_csr_from_arrays(C.c_uint32(g.n), C.c_uint32(g.m), _ptr(off), _ptr(adj), _ptr(w),
                                                 _ptr(eid), _ptr(minw), C.byref(h)))
        out = Csr(g.n, g.m, off, adj, w, eid, minw, np.zeros(0, np.uint64), np.zeros(0, np.uint32),
                  np.zeros(0, np.uint32))
        out.extra["handle"] = h
        return out

    def free_csr(self, g):
        h = g.extra.pop("handle", None)
        if h is not None:
            self.lib.ref_csr_free(h)

    def brandes(self, g, sources=None, halved=False, edge_bc=False, eps=0.0):
        h = g.extra["handle"]
        src = None if sources is None else _u32(sources)
        k = -1 if sources is None else len(src)
        node = np.zeros(max(g.n, 1), np.float64)
        edge = np.zeros(max(g.m, 1), np.float64)
        el = C.c_double()
        self._check(self.lib.ref_brandes(h, _ptr(src), C.c_int64(k), C.c_int(int(edge_bc)), C.c_int(int(halved)),
                                         C.c_double(eps), _ptr(node), _ptr(edge), C.byref(el)))
        node = node[: g.n]
        return (node, edge[: g.m]) if edge_bc else node

    def brute_force(self, g):
        node = np.zeros(max(g.n, 1), np.float64)
        self._check(self.lib.ref_brute_force(g.extra["handle"], _ptr(node)))
        return node[: g.n]

    def bc_parallel(self, g, strategy="we", workers=1, sources=None, edge_bc=False, halved=False,
                    strict_merge=False, less_equal=False):
        h = g.extra["handle"]
        src = None if sources is None else _u32(sources)
        k = -1 if sources is None else len(src)
        node = np.zeros(max(g.n, 1), np.float64)
        edge = np.zeros(max(g.m, 1), np.float64)
        depth = np.zeros(max(g.n, 1), np.uint32)
        el = C.c_double()
        self._check(self.lib.ref_bc_parallel(h, strategy.encode(), C.c_int(workers), _ptr(src), C.c_int64(k),
                                             C.c_int(int(edge_bc)), C.c_int(int(halved)),
                                             C.c_int(int(strict_merge)), C.c_int(int(less_equal)), _ptr(node),
                                             _ptr(edge), _ptr(depth), C.byref(el)))
        return dict(node_bc=node[: g.n], edge_bc=edge[: g.m] if edge_bc else None, depth=depth[: g.n],
                    elapsed=el.value)

    def solve_source(self, g, s, strategy="we", less_equal=False):
        n = g.n
        dist = np.zeros(n, np.float64)
        sigma = np.zeros(n, np.float64)
        delta = np.zeros(n, np.float64)
        acc = np.zeros(n, np.float64)
        order = np.zeros(n + 1, np.uint32)
        ends = np.zeros(n + 2, np.uint32)
        depth, olen, elen = C.c_uint32(), C.c_uint32(), C.c_uint32()
        self._check(self.lib.ref_solve_source(g.extra["handle"], C.c_uint32(s), strategy.encode(),
                                              C.c_int(int(less_equal)), _ptr(dist), _ptr(sigma), _ptr(delta),
                                              C.byref(depth), _ptr(order), C.byref(olen), _ptr(ends),
                                              C.byref(elen), _ptr(acc)))
        return dict(dist=dist, sigma=sigma, delta=delta, depth=depth.value, order=order[: olen.value].copy(),
                    ends=ends[: elen.value].copy(), node_acc=acc)

    def format_edge_tsv(self, g, edge_bc):
        edge_bc = _f64(edge_bc)
        L = self.lib.ref_format_edge_tsv(g.extra["handle"], _ptr(edge_bc), None, 0)
        buf = C.create_string_buffer(int(L) + 1)
        self.lib.ref_format_edge_tsv(g.extra["handle"], _ptr(edge_bc), buf, L)
        return buf.raw[:L].decode()

    def format_node_tsv(self, g, node_bc):
        node_bc = _f64(node_bc)
        L = self.lib.ref_format_node_tsv(g.extra["handle"], _ptr(node_bc), None, 0)
        buf = C.create_string_buffer(int(L) + 1)
        self.lib.ref_format_node_tsv(g.extra["handle"], _ptr(node_bc), buf, L)
        return buf.raw[:L].decode()
