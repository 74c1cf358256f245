"""Generates tests/golden/*.npz|json from the REFERENCE itself (oracle/_ref/
libwbc_ref.so, compiled from /root/reference/proj/src by oracle/Makefile).

Run here (the build container, where /root/reference exists):
    python tests/golden/make_golden.py
The outputs are committed; nothing on the GPU box reads /root/reference.

Contents (every value produced by the reference's own code):
  * fixture graphs of test_util.hpp / test_brandes.cpp / test_engine.cpp /
    acceptance.cpp (path, star, cycle, complete, tie-square, diamond,
    64-way race, disconnected paths) and seeded reference-generator graphs;
  * for each: CSR arrays (build_csr), brandes_sequential node+edge BC,
    bc_parallel('we', 1 worker) node BC + depth_per_source, brute_force_bc
    (n <= 300), and solve_source + accumulate_dependencies state for a few
    sources;
  * generator streams (gen_er, gen_kronecker, assign_weights, sample_sources);
  * ER-4096 (BASELINE config 1) all-source BC + depth;
  * parser cases (accepted lists and ParseError line/message).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import RefLib  # noqa: E402

R = RefLib()


def chain(k, w=1.0):
    return [(i, i + 1, w) for i in range(k - 1)]


FIXTURES = {
    "path3": chain(3),
    "path6": chain(6),
    "path17": chain(17),
    "star4": [(0, i, 1.0) for i in range(1, 4)],
    "star9": [(0, i, 1.0) for i in range(1, 9)],
    "cycle4": [(i, (i + 1) % 4, 1.0) for i in range(4)],
    "complete4": [(i, j, 1.0) for i in range(4) for j in range(i + 1, 4)],
    "complete7": [(i, j, 1.0) for i in range(7) for j in range(i + 1, 7)],
    "tie_square": [(0, 1, 1.0), (0, 2, 2.0), (1, 2, 1.0), (2, 3, 1.0)],
    "diamond": [(0, 1, 1.0), (0, 2, 1.0), (1, 3, 1.0), (2, 3, 1.0)],
    "race64": [(0, i, 1.0) for i in range(1, 65)] + [(i, 65, 1.0) for i in range(1, 65)],
    "two_paths": [(0, 1, 1.0), (1, 2, 1.0), (10, 11, 1.0), (11, 12, 1.0)],
    "dup_min": [(0, 1, 3.0), (1, 0, 5.0), (1, 2, 2.0), (7, 3, 1.0), (3, 900, 2.0)],
}


def edges_of(lst):
    return (np.array([e[0] for e in lst], np.uint64), np.array([e[1] for e in lst], np.uint64),
            np.array([e[2] for e in lst], np.float64))


def record(out, name, u, v, w, dump_sources=(0,)):
    g = R.build_csr(u, v, w)
    out[f"{name}/u"], out[f"{name}/v"], out[f"{name}/w"] = u, v, w
    for f in ("offsets", "adjacency", "weights", "edge_id", "min_incident_weight", "original_id", "edge_u",
              "edge_v"):
        out[f"{name}/csr_{f}"] = getattr(g, f)
    out[f"{name}/csr_nm"] = np.array([g.n, g.m, g.merged_duplicates], np.uint64)
    if g.n:
        nb, eb = R.brandes(g, edge_bc=True)
        out[f"{name}/brandes_node"], out[f"{name}/brandes_edge"] = nb, eb
        out[f"{name}/brandes_halved"] = R.brandes(g, halved=True)
        r = R.bc_parallel(g, "we", 1)
        out[f"{name}/bcpar_node"], out[f"{name}/bcpar_depth"] = r["node_bc"], r["depth"]
        if g.n <= 300:
            out[f"{name}/brute_node"] = R.brute_force(g)
        for s in dump_sources:
            if s < g.n:
                st = R.solve_source(g, s, "we")
                for k in ("dist", "sigma", "delta", "order", "ends"):
                    out[f"{name}/src{s}_{k}"] = st[k]
                out[f"{name}/src{s}_depth"] = np.array([st["depth"]], np.uint32)
    R.free_csr(g)


def main():
    out = {}
    for name, lst in FIXTURES.items():
        record(out, name, *edges_of(lst), dump_sources=(0, 1))
    # seeded reference-generator graphs (acceptance.cpp style, weights 1-10)
    for i, (kind, a, b, seed) in enumerate([("er", 60, 6.0, 11), ("er", 150, 8.0, 12), ("kr", 5, 6.0, 13),
                                            ("kr", 7, 10.0, 14), ("er", 200, 3.0, 15), ("kr", 6, 2.0, 16)]):
        u, v, w = R.gen_er(a, b, seed) if kind == "er" else R.gen_kronecker(a, b, seed)
        u, v, w = R.assign_weights(u, v, w, 1, 10, seed)
        record(out, f"gen{i}", u, v, w, dump_sources=(0, 5, 17))
    # generator streams
    for n, d, s in ((64, 6.0, 33), (16, 4.0, 9), (1000, 20.0, 12)):
        u, v, w = R.gen_er(n, d, s)
        out[f"stream/er_{n}_{d}_{s}"] = np.stack([u, v]).astype(np.uint64)
        out[f"stream/erw_{n}_{d}_{s}"] = R.assign_weights(u, v, w, 1, 10, s)[2]
    for sc, d, s in ((6, 6.0, 34), (4, 4.0, 9), (12, 16.0, 1)):
        u, v, w = R.gen_kronecker(sc, d, s)
        out[f"stream/kr_{sc}_{d}_{s}"] = np.stack([u, v]).astype(np.uint64)
        out[f"stream/krw_{sc}_{d}_{s}"] = R.assign_weights(u, v, w, 1, 255, s)[2]
    for n, k, s in ((4093, 64, 1), (10, 20, 3), (655907, 4096, 1), (1000, 1000, 7)):
        out[f"stream/sample_{n}_{k}_{s}"] = R.sample_sources(n, k, s)
    # BASELINE config 1: ER n=4096 deg 8 w 1-64, all sources
    u, v, w = R.gen_er(4096, 8.0, 1)
    u, v, w = R.assign_weights(u, v, w, 1, 64, 1)
    g = R.build_csr(u, v, w)
    r = R.bc_parallel(g, "we", 8)
    out["er4096/node_bc"], out["er4096/depth"] = r["node_bc"], r["depth"]
    out["er4096/brandes_node"] = R.brandes(g)
    src = R.sample_sources(g.n, 32, 1)
    nb, eb = R.brandes(g, sources=src, edge_bc=True)
    out["er4096/sample32_src"], out["er4096/sample32_node"], out["er4096/sample32_edge"] = src, nb, eb
    R.free_csr(g)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)

    cases = ["0 1 2.5\n1 2 1.0", "# comment\n3 4", "0 0 1.0\n0 1 1.0", "\n  \n0\t1\t3\n\n2 3\n",
             "0 1 1.0\n0 x 1.0", "5", "1 2 3 4", "-1 2", "0 1 0\n", "0 1 -2\n", "# c\n\n0 1\nbad\n",
             "0 1 inf", "0 1 nan", "+1 2", "7 3 1e-1\r\n3 900 2\r\n", "1 2 0x1p3", "1 2 1e400",
             "18446744073709551615 0 1", "18446744073709551616 0 1", "   # indented comment\n1 2",
             "\v1 2", "1 2 3\n\n\n4 5 -0"]
    parse = []
    for c in cases:
        for dw in (1.0, 7.0):
            try:
                u, v, w, loops = R.parse_edge_list(c, dw)
                parse.append(dict(text=c, default_weight=dw, ok=True, u=[int(x) for x in u], v=[int(x) for x in v],
                                  w=[float(x) for x in w], self_loops=int(loops)))
            except Exception as ex:  # ParseError from the reference
                parse.append(dict(text=c, default_weight=dw, ok=False, error=str(ex)))
    with open(os.path.join(HERE, "parse_cases.json"), "w") as f:
        json.dump(parse, f, indent=1)
    print(f"wrote {len(out)} arrays, {len(parse)} parse cases")


if __name__ == "__main__":
    main()
