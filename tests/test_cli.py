"""Black-box tests of the `wbc` command-line drop-in (paper_1701_05975_b200/bin/wbc),
mirroring the reference's proj/tests/test_cli.cpp (exact output bytes, exit
code 2 on every failure path, generator determinism).  `compute` and
`stats --depth` run on the GPU and are marked accordingly.
"""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, approx_rel

CLI = os.path.join(ROOT, "paper_1701_05975_b200", "bin", "wbc")


def run(args, tmp_path=None):
    p = subprocess.run([CLI] + args, capture_output=True, text=True)
    return p.returncode, p.stdout, p.stderr


@pytest.fixture(scope="module")
def files(tmp_path_factory):
    d = tmp_path_factory.mktemp("cli")

    def w(name, text):
        p = d / name
        p.write_text(text)
        return str(p)

    return dict(d=d, p3=w("p3.txt", "0 1 1\n1 2 1\n"), p3w=w("p3w.txt", "0 1 5\n1 2 9\n"),
                sparse=w("sparse_ids.txt", "900 7 1\n7 30 1\n"), bad=w("bad.txt", "0 1 1\nnot numbers\n"),
                tri=w("tri.txt", "0 1 1\n1 2 1\n0 2 1\n"))


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(CLI):
        pytest.skip("bin/wbc not built (make -C paper_1701_05975_b200)")


# ---------------------------------------------------------------- CPU: failure modes, generate, stats

def test_compute_failure_modes_exit_2(files):                 # test_cli.cpp:102-112
    assert run(["compute", "/tmp/definitely_missing_wbc.txt"])[0] == 2
    rc, _, err = run(["compute", files["bad"]])
    assert rc == 2 and "line 2" in err
    assert run(["compute", files["p3"], "--strategy", "bogus"])[0] == 2
    assert run(["compute", files["p3"], "--lane-width", "5"])[0] == 2
    assert run(["compute", files["p3"], "--unknown-flag"])[0] == 2
    assert run(["compute", files["p3"], "--normalize", "third"])[0] == 2
    assert run([])[0] == 2
    assert run(["bench", files["p3"]])[0] == 2                # CPU strategy bench: not part of the GPU engine


def test_generate_er_deterministic_and_matches_reference(files, ref):  # test_cli.cpp:114-137
    out1, out2 = str(files["d"] / "g1.txt"), str(files["d"] / "g2.txt")
    flags = ["generate", "--model", "er", "--nodes", "16", "--avg-degree", "4", "--seed", "7", "-o"]
    assert run(flags + [out1])[0] == 0 and run(flags + [out2])[0] == 0
    a = open(out1).read()
    assert a == open(out2).read()
    lines = a.splitlines()
    assert lines[0] == "# model=er nodes=16 avg_degree=4 seed=7 weight_lo=1 weight_hi=10"
    assert lines[1] == "# edges_requested=32 edges_achieved=32"
    data = [ln for ln in lines if not ln.startswith("#")]
    assert len(data) == 32
    # the reference's own generator stream, same seed, formatted as write_edge_list does
    u, v, w = ref.gen_er(16, 4.0, 7)
    u, v, w = ref.assign_weights(u, v, w, 1, 10, 7)
    assert data == [f"{a_} {b_} {c_:.17g}" for a_, b_, c_ in zip(u.tolist(), v.tolist(), w.tolist())]


def test_generate_kronecker_ids_and_weights(files):           # test_cli.cpp:139-156
    out = str(files["d"] / "k.txt")
    assert run(["generate", "--model", "kronecker", "--scale", "4", "--avg-degree", "4", "--seed", "3",
                "-o", out])[0] == 0
    for ln in open(out).read().splitlines():
        if ln.startswith("#"):
            continue
        u, v, w = ln.split()
        assert int(u) < 16 and int(v) < 16 and 1.0 <= float(w) <= 10.0


def test_generate_new_models(files):
    rc, out, _ = run(["generate", "--model", "grid", "--rows", "3", "--cols", "4", "--seed", "1"])
    assert rc == 0 and len([x for x in out.splitlines() if not x.startswith("#")]) == 3 * 3 + 2 * 4
    rc, out, _ = run(["generate", "--model", "ba", "--nodes", "50", "--m-per", "3", "--seed", "1"])
    assert rc == 0 and "model=ba" in out


def test_generate_validates_the_model():                      # test_cli.cpp:158-161
    assert run(["generate", "--model", "banana", "--avg-degree", "4"])[0] == 2
    assert run(["generate", "--model", "er", "--avg-degree", "4"])[0] == 2


def test_stats_pinned_format(files):                          # test_cli.cpp:163-168
    rc, out, _ = run(["stats", files["tri"]])
    assert rc == 0 and out == "n=3 m=3 max_degree=2 avg_degree=2.0\n"


# ---------------------------------------------------------------- GPU: compute

@pytest.mark.gpu
def test_compute_p3_variants(files):                          # test_cli.cpp:61-92
    rc, out, err = run(["compute", files["p3"], "--strategy", "we-warp", "--lane-width", "4"])
    assert rc == 0 and out == "0\t0\n1\t2\n2\t0\n"
    assert "n=3 m=2" in err and "we-warp4" in err
    assert run(["compute", files["p3"], "--normalize", "half", "--strategy", "we"])[1] == "0\t0\n1\t1\n2\t0\n"
    assert run(["compute", files["p3"], "--strategy", "sequential"])[1] == "0\t0\n1\t2\n2\t0\n"
    assert run(["compute", files["p3w"], "--unit-weights", "--strategy", "np"])[1] == "0\t0\n1\t2\n2\t0\n"
    assert run(["compute", files["p3"], "--edge-bc", "--strategy", "we"])[1] == \
        "0\t0\n1\t2\n2\t0\n0\t1\t4\n1\t2\t4\n"


@pytest.mark.gpu
def test_compute_output_file_and_original_ids(files):         # test_cli.cpp:94-100
    out = str(files["d"] / "out.tsv")
    assert run(["compute", files["sparse"], "-o", out, "--strategy", "we"])[0] == 0
    assert open(out).read() == "7\t2\n30\t0\n900\t0\n"


@pytest.mark.gpu
def test_compute_matches_reference_report(files, ref):
    """A random weighted graph through the CLI against the compiled reference's
    bc_parallel + format_node_bc_tsv: same id order, scores within 1e-9."""
    u, v, w = ref.gen_er(300, 6.0, 5)
    u, v, w = ref.assign_weights(u, v, w, 1, 20, 5)
    path = str(files["d"] / "er300.txt")
    with open(path, "w") as f:
        f.write("".join(f"{a} {b} {c:.17g}\n" for a, b, c in zip(u.tolist(), v.tolist(), w.tolist())))
    rc, out, _ = run(["compute", path, "--sources-sample", "40", "--seed", "3"])
    assert rc == 0
    rg = ref.build_csr(u, v, w)
    want = ref.bc_parallel(rg, "we", 4, sources=ref.sample_sources(rg.n, 40, 3))
    ref_tsv = ref.format_node_tsv(rg, want["node_bc"])
    ref.free_csr(rg)
    got = [ln.split("\t") for ln in out.splitlines()]
    exp = [ln.split("\t") for ln in ref_tsv.splitlines()]
    assert [g[0] for g in got] == [e[0] for e in exp]
    assert approx_rel(np.array([float(g[1]) for g in got]), np.array([float(e[1]) for e in exp]), 1e-9).all()


@pytest.mark.gpu
def test_stats_depth(files):                                  # test_cli.cpp:170-175
    rc, out, _ = run(["stats", files["p3"], "--depth", "--seed", "1"])
    # depth_per_source of P3 is [3, 2, 3] (test_engine.cpp:376-380)
    assert rc == 0 and out == "n=3 m=2 max_degree=2 avg_degree=1.33333 avg_depth=2.66667\n"


@pytest.mark.gpu
def test_compute_strict_is_byte_identical_to_reference(files, ref):
    """`--strict` (strict_merge): the TSV is byte-for-byte the reference's
    bc_parallel + format_node_bc_tsv / format_edge_bc_tsv for the same lane width."""
    u, v, w = ref.gen_er(250, 5.0, 9)
    u, v, w = ref.assign_weights(u, v, w, 1, 12, 9)
    path = str(files["d"] / "er250.txt")
    with open(path, "w") as f:
        f.write("".join(f"{a} {b} {c:.17g}\n" for a, b, c in zip(u.tolist(), v.tolist(), w.tolist())))
    rc, out, _ = run(["compute", path, "--strict", "--strategy", "we-warp", "--lane-width", "8", "--edge-bc",
                      "--sources-sample", "60", "--seed", "2"])
    assert rc == 0
    rg = ref.build_csr(u, v, w)
    want = ref.bc_parallel(rg, "we-warp8", 4, sources=ref.sample_sources(rg.n, 60, 2), edge_bc=True,
                           strict_merge=True)
    exp = ref.format_node_tsv(rg, want["node_bc"]) + ref.format_edge_tsv(rg, want["edge_bc"])
    ref.free_csr(rg)
    assert out == exp
