"""Pins the CPU oracle (oracle/wbc_oracle.c) to the reference.

1. Against tests/golden/ (made by tests/golden/make_golden.py from the
   compiled reference library): bit-exact CSR arrays, bit-exact
   brandes_sequential node/edge BC, bit-exact Eq. 4 per-source state and
   depth_per_source, brute-force agreement at 1e-9.
2. Against the reference's hard-coded known answers (test_brandes.cpp,
   test_engine.cpp, acceptance.cpp).
3. Live against oracle/_ref when it was built (build container).
"""
import os

import numpy as np
import pytest

from conftest import approx_rel

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden.npz"))
NAMES = sorted({k.split("/")[0] for k in GOLD.files if "/csr_nm" in k})


class G:
    """CsrGraph view over the golden arrays."""

    def __init__(self, name):
        n, m, merged = (int(x) for x in GOLD[f"{name}/csr_nm"])
        self.n, self.m, self.merged = n, m, merged
        for f in ("offsets", "adjacency", "weights", "edge_id", "min_incident_weight", "original_id", "edge_u",
                  "edge_v"):
            setattr(self, f, GOLD[f"{name}/csr_{f}"])


@pytest.mark.parametrize("name", NAMES)
def test_build_csr_bit_exact(oracle, name):
    g = oracle.build_csr(GOLD[f"{name}/u"], GOLD[f"{name}/v"], GOLD[f"{name}/w"])
    ref = G(name)
    assert (g.n, g.m, g.merged_duplicates) == (ref.n, ref.m, ref.merged)
    for f in ("offsets", "adjacency", "weights", "edge_id", "min_incident_weight", "original_id", "edge_u",
              "edge_v"):
        assert np.array_equal(getattr(g, f), getattr(ref, f)), f


@pytest.mark.parametrize("name", NAMES)
def test_brandes_bit_exact(oracle, name):
    g = G(name)
    node, edge = oracle.brandes(g, edge_bc=True)
    assert np.array_equal(node, GOLD[f"{name}/brandes_node"])
    assert np.array_equal(edge, GOLD[f"{name}/brandes_edge"])
    assert np.array_equal(oracle.brandes(g, halved=True), GOLD[f"{name}/brandes_halved"])
    if f"{name}/brute_node" in GOLD.files:  # brandes == brute force (test_brandes.cpp:69-81)
        assert approx_rel(node, GOLD[f"{name}/brute_node"], 1e-9).all()


@pytest.mark.parametrize("name", NAMES)
def test_eq4_process_bit_exact(oracle, name):
    g = G(name)
    node, _, depth = oracle.bc_eq4(g)
    assert np.array_equal(node, GOLD[f"{name}/bcpar_node"])      # bc_parallel(we, 1 worker)
    assert np.array_equal(depth, GOLD[f"{name}/bcpar_depth"])
    for s in (0, 1, 5, 17):
        if f"{name}/src{s}_dist" not in GOLD.files:
            continue
        o = oracle.eq4_source(g, s)
        for k in ("dist", "sigma", "delta", "order", "ends"):
            assert np.array_equal(o[k], GOLD[f"{name}/src{s}_{k}"]), (s, k)
        assert o["depth"] == int(GOLD[f"{name}/src{s}_depth"][0])


def test_known_answers(oracle):
    """Hard-coded values of the reference's own tests."""
    p3 = G("path3")
    assert oracle.brandes(p3).tolist() == [0.0, 2.0, 0.0]                        # test_brandes.cpp:24-31
    assert oracle.brandes(p3, halved=True).tolist() == [0.0, 1.0, 0.0]
    assert oracle.brandes(p3, edge_bc=True)[1].tolist() == [4.0, 4.0]            # :39-44
    assert oracle.bc_eq4(p3)[2].tolist() == [3, 2, 3]                            # test_engine.cpp:376-380
    ts = G("tie_square")
    node, edge = oracle.brandes(ts, edge_bc=True)
    assert approx_rel(node, [0, 2, 4, 0], 1e-12).all()                           # test_brandes.cpp:48-56
    assert approx_rel(edge, [4, 2, 6, 6], 1e-12).all()
    st = oracle.eq4_source(ts, 0)
    assert st["dist"].tolist() == [0, 1, 2, 3] and st["sigma"][3] == 2.0          # test_engine.cpp:137-140
    assert oracle.eq4_source(ts, 0, less_equal=True)["sigma"][3] == 1.0          # the LessEqual undercount
    assert st["delta"][1:].tolist() == [1.0, 1.0, 0.0]                           # :183-193
    race = G("race64")
    st = oracle.eq4_source(race, 0)
    assert st["sigma"][65] == 64.0 and st["dist"][65] == 2.0 and st["depth"] == 3  # :304-326
    assert oracle.eq4_source(G("diamond"), 0)["sigma"][3] == 2.0                 # :156-162
    for k, name in ((6, "path6"), (17, "path17")):                               # acceptance.cpp:200-231
        assert np.allclose(oracle.brandes(G(name)), [2.0 * i * (k - 1 - i) for i in range(k)], atol=1e-9)
    for n, name in ((4, "star4"), (9, "star9")):
        assert oracle.brandes(G(name))[0] == (n - 1) * (n - 2)
    assert approx_rel(oracle.brandes(G("cycle4")), [1] * 4, 1e-12).all()
    for name in ("complete4", "complete7"):
        assert not oracle.brandes(G(name)).any()
    assert oracle.brandes(G("two_paths")).tolist() == [0, 2, 0, 0, 2, 0]        # test_brandes.cpp:101-106


def test_er4096_sample_and_all_source_depth(oracle):
    g = G("er4096") if "er4096/csr_nm" in GOLD.files else None
    if g is None:
        import paper_1701_05975_b200 as W
        el = W.assign_weights(W.gen_er(4096, 8.0, 1), 1, 64, 1)
        g = oracle.build_csr(el.u, el.v, el.w)
    src = GOLD["er4096/sample32_src"]
    node, edge = oracle.brandes(g, sources=src, edge_bc=True)
    assert np.array_equal(node, GOLD["er4096/sample32_node"])
    assert np.array_equal(edge, GOLD["er4096/sample32_edge"])
    allnode, _, depth = oracle.bc_eq4(g)
    assert approx_rel(allnode, GOLD["er4096/node_bc"], 1e-9).all()   # reference ran 8 workers
    assert np.array_equal(depth, GOLD["er4096/depth"])


def test_source_errors(oracle):
    g = G("path3")
    with pytest.raises(ValueError):
        oracle.brandes(g, sources=[3])
    with pytest.raises(ValueError):
        oracle.bc_eq4(g, sources=[0, 9])
    node, _, depth = oracle.bc_eq4(g, sources=[0, 0])              # duplicates count twice
    assert node.tolist() == [0.0, 2.0, 0.0] and depth[0] == 3


def test_oracle_vs_live_reference_random(oracle, ref):
    rng = np.random.default_rng(7)
    for i in range(12):
        seed = int(rng.integers(1, 2**40))
        if i % 2:
            n = int(rng.integers(10, 120))
            u, v, w = ref.gen_er(n, float(rng.uniform(1, min(8.0, n - 1.0))), seed)
        else:
            u, v, w = ref.gen_kronecker(int(rng.integers(3, 7)), float(rng.uniform(1, 12)), seed)
        u, v, w = ref.assign_weights(u, v, w, 1, 10, seed)
        rg = ref.build_csr(u, v, w)
        og = oracle.build_csr(u, v, w)
        if og.n:
            assert np.array_equal(oracle.brandes(og), ref.brandes(rg))
            r = ref.bc_parallel(rg, "we", 1)
            node, _, depth = oracle.bc_eq4(og)
            assert np.array_equal(node, r["node_bc"]) and np.array_equal(depth, r["depth"])
        ref.free_csr(rg)
