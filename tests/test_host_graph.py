"""The native host layer (CSR loader + generators in libwbc_b200.so, CPU-only
calls) against the reference's outputs in tests/golden/: bit-exact CSR
arrays, generator streams and parser behaviour (test_graph.cpp,
test_generate.cpp, acceptance.cpp criterion 8)."""
import io
import json
import os

import numpy as np
import pytest

import paper_1701_05975_b200 as W

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden.npz"))
NAMES = sorted({k.split("/")[0] for k in GOLD.files if "/csr_nm" in k})
CSR_FIELDS = ("offsets", "adjacency", "weights", "edge_id", "min_incident_weight", "original_id", "edge_u",
              "edge_v")


@pytest.mark.parametrize("name", NAMES)
def test_build_csr_matches_reference(name):
    g = W.build_csr(W.EdgeList(GOLD[f"{name}/u"], GOLD[f"{name}/v"], GOLD[f"{name}/w"]))
    n, m, merged = (int(x) for x in GOLD[f"{name}/csr_nm"])
    assert (g.n, g.m, g.merged_duplicates) == (n, m, merged)
    for f in CSR_FIELDS:
        assert np.array_equal(getattr(g, f), GOLD[f"{name}/csr_{f}"]), f


def test_csr_contract_examples():
    tri = W.build_csr(W.EdgeList.of([(0, 1, 1), (1, 2, 1), (0, 2, 1)]))       # test_graph.cpp:81-86
    assert tri.offsets.tolist() == [0, 2, 4, 6]
    d = W.build_csr(W.EdgeList.of([(0, 1, 3), (1, 0, 5)]))                    # :88-95
    assert (d.n, d.m, d.merged_duplicates) == (2, 1, 1) and d.weights.tolist() == [3.0, 3.0]
    h = W.build_csr(W.EdgeList.of([(0, 1, 4), (1, 2, 2)]))                    # :97-102
    assert h.min_incident_weight.tolist() == [4.0, 2.0, 2.0]
    c = W.build_csr(W.EdgeList.of([(7, 3, 1), (3, 900, 2)]))                  # :104-110
    assert c.original_id.tolist() == [7, 3, 900] and (c.edge_u[0], c.edge_v[0]) == (0, 1)
    e = W.build_csr(W.EdgeList())                                             # :112-120
    assert (e.n, e.m) == (0, 0) and e.offsets.tolist() == [0]
    s = W.graph_stats(e)
    assert s.max_degree == 0 and s.avg_degree == 0.0


def test_slot_symmetry_and_round_trip():
    el = W.assign_weights(W.gen_kronecker(8, 8.0, 3), 1, 20, 3)
    g = W.build_csr(el)
    assert int(g.offsets[-1]) == 2 * g.m
    cnt = np.bincount(g.edge_id, minlength=g.m)
    assert (cnt == 2).all()                                                   # two slots per edge
    back = W.to_edge_list(g)
    g2 = W.build_csr(back)
    for f in CSR_FIELDS:
        assert np.array_equal(getattr(g, f), getattr(g2, f)), f
    buf = io.StringIO()
    W.write_edge_list(buf, back, ["regen check"])
    g3 = W.build_csr(W.parse_edge_list(buf.getvalue()))
    assert np.array_equal(g3.weights, g.weights) and np.array_equal(g3.adjacency, g.adjacency)


@pytest.mark.parametrize("key", sorted(k for k in GOLD.files if k.startswith("stream/er_")))
def test_gen_er_stream(key):
    _, n, d, s = key.split("/")[1].split("_")
    el = W.gen_er(int(n), float(d), int(s))
    assert np.array_equal(np.stack([el.u, el.v]), GOLD[key])
    assert np.array_equal(W.assign_weights(el, 1, 10, int(s)).w, GOLD[key.replace("er_", "erw_")])


@pytest.mark.parametrize("key", sorted(k for k in GOLD.files if k.startswith("stream/kr_")))
def test_gen_kronecker_stream(key):
    _, sc, d, s = key.split("/")[1].split("_")
    el = W.gen_kronecker(int(sc), float(d), int(s))
    assert np.array_equal(np.stack([el.u, el.v]), GOLD[key])
    assert np.array_equal(W.assign_weights(el, 1, 255, int(s)).w, GOLD[key.replace("kr_", "krw_")])


@pytest.mark.parametrize("key", sorted(k for k in GOLD.files if k.startswith("stream/sample_")))
def test_sample_sources_stream(key):
    _, n, k, s = key.split("/")[1].split("_")
    assert np.array_equal(W.sample_sources(int(n), int(k), int(s)), GOLD[key])


def test_generator_contracts():                                              # acceptance.cpp:363-396
    assert len(W.gen_er(16, 4.0, 9)) == 32
    assert len(W.gen_er(10, 0.0, 9)) == 0
    assert len(W.gen_kronecker(4, 4.0, 9)) == 32
    big = W.assign_weights(W.gen_er(1000, 200.0, 12), 1, 10, 12)
    assert len(big) == 100000 and big.w.min() >= 1 and big.w.max() <= 10
    assert (big.w == np.floor(big.w)).all() and 5.4 < big.w.mean() < 5.6
    with pytest.raises(ValueError):
        W.gen_er(10, 20.0, 1)                                                # more edges than pairs
    with pytest.raises(ValueError):
        W.assign_weights(W.gen_er(10, 2.0, 1), 0, 5, 1)
    with pytest.raises(ValueError):
        W.gen_kronecker(0, 2.0, 1)


def test_ba_and_grid_generators():
    ba = W.gen_ba(65536, 10, 1)
    assert len(ba) == 10 * 11 // 2 + (65536 - 11) * 10 == 655305           # m = 655,305
    g = W.build_csr(ba)
    assert (g.n, g.m) == (65536, 655305)
    assert np.array_equal(W.gen_ba(2000, 4, 5).u, W.gen_ba(2000, 4, 5).u)  # deterministic
    gr = W.build_csr(W.gen_grid(64, 32))
    assert (gr.n, gr.m) == (64 * 32, 64 * 31 + 63 * 32)
    deg = np.diff(gr.offsets.astype(np.int64))
    assert deg.max() == 4 and deg.min() == 2


def test_parser_matches_reference():
    with open(os.path.join(HERE, "golden", "parse_cases.json")) as f:
        cases = json.load(f)
    for c in cases:
        if c["ok"]:
            el = W.parse_edge_list(c["text"], c["default_weight"])
            assert el.u.tolist() == c["u"] and el.v.tolist() == c["v"], c["text"]
            assert el.w.tolist() == c["w"] and el.self_loops_dropped == c["self_loops"], c["text"]
        else:
            with pytest.raises(W.ParseError) as ex:
                W.parse_edge_list(c["text"], c["default_weight"])
            assert str(ex.value) == c["error"], c["text"]
            assert ex.value.line == int(c["error"].split(":")[0].split()[1])
    with pytest.raises(ValueError):
        W.parse_edge_list("0 1", 0.0)                                        # default weight > 0
    assert len(W.parse_edge_list(io.StringIO("0 1 2\n"))) == 1              # stream input


_PAR_SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1701_05975_b200 as W
el = W.assign_weights(W.gen_kronecker(13, 24.0, 5), 1, 9, 5)
# duplicates (min weight wins, first orientation kept), reversed pairs and sparse raw ids
u = np.concatenate([el.u, el.v[:500], el.u[:300] * 7 + 11])
v = np.concatenate([el.v, el.u[:500], el.v[:300] * 7 + 11])
w = np.concatenate([el.w, np.full(500, 0.5), el.w[:300]])
e2 = W.EdgeList(); e2.u, e2.v, e2.w = u.astype(np.uint64), v.astype(np.uint64), w
g = W.build_csr(e2)
np.savez(sys.argv[2], gu=el.u, gv=el.v, gw=el.w, off=g.offsets, adj=g.adjacency, wt=g.weights, eid=g.edge_id,
         mw=g.min_incident_weight, oid=g.original_id, eu=g.edge_u, ev=g.edge_v, merged=[g.merged_duplicates])
'''


def test_parallel_builders_identical_to_serial(tmp_path):
    """gen_kronecker and build_csr take thread-parallel paths above
    WBC_HOST_PARALLEL_MIN; their output must equal the serial paths
    (the reference's stream and first-appearance orders) array for array."""
    import subprocess
    import sys
    from conftest import ROOT
    script = tmp_path / "par.py"
    script.write_text(_PAR_SCRIPT)
    res = {}
    for mode, thr in (("serial", str(1 << 40)), ("parallel", "1000")):
        out = tmp_path / f"{mode}.npz"
        env = dict(os.environ, WBC_HOST_PARALLEL_MIN=thr, WBC_HOST_THREADS="4")
        subprocess.run([sys.executable, str(script), ROOT, str(out)], env=env, check=True)
        res[mode] = np.load(out)
    a, b = res["serial"], res["parallel"]
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
    assert a["merged"][0] > 0
