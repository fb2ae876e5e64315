"""tools/cli/lamg_b200 -- the reference CLI's solve / info / bench subcommands
over the B200 facade (proj/tools/lamg.cpp:146-357).

CPU: the tool builds against include/lamg_b200/lamg.hpp, prints usage, and
reports file / argument errors with the reference's JSON error object and exit
codes (2 for I/O errors, 1 otherwise) before any device is touched.
GPU: `solve` reproduces the oracle's whole-problem driver bit for bit in
VALIDATE mode (x, cycles, levels, components, MVM work), `info` lists the
reference's levels, `bench` emits the reference's CSV columns.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1108_1310_b200 import graphs as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "cli", "lamg_b200_cli.cpp")
BIN = os.path.join(ROOT, "tools", "cli", "lamg_b200")


def build():
    lib = os.path.join(ROOT, "paper_1108_1310_b200")
    if os.path.exists(BIN) and os.path.getmtime(BIN) >= max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(ROOT, "include", "lamg_b200", "lamg.hpp"))):
        return
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", lib, "-llamg_b200", f"-Wl,-rpath,{lib}", "-lpthread", "-o", BIN], check=True)


def run(*args):
    p = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


def test_cli_builds_and_prints_usage():
    build()
    rc, out, _ = run("--help")
    assert rc == 0 and "solve" in out and "info" in out and "bench" in out
    assert run()[0] == 1


def test_cli_error_objects_and_exit_codes(tmp_path):
    build()
    rc, out, _ = run("solve", "--matrix", str(tmp_path / "missing.mtx"), "--stats", str(tmp_path / "s.json"))
    err = json.loads(out)
    assert rc == 2 and err["exit_code"] == 2 and err["error"].startswith("cannot open")
    assert json.load(open(tmp_path / "s.json")) == err  # the error object is also written to --stats
    bad = tmp_path / "bad.mtx"
    bad.write_text("not a matrix market file\n")
    rc, out, _ = run("info", "--matrix", str(bad))
    assert rc == 1 and json.loads(out)["exit_code"] == 1
    rc, out, _ = run("frob")
    assert rc == 1 and "unknown subcommand" in json.loads(out)["error"]
    rc, out, _ = run("solve")
    assert rc == 1 and "--matrix is required" in json.loads(out)["error"]


def _disconnected():
    """A 16x16 grid, a 7-node path and an isolated node."""
    g, p = G.grid_5pt(16), G.path(7)
    n = g.n + p.n + 1
    u, v, w = [], [], []
    for a, off in ((g, 0), (p, g.n)):
        rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
        keep = rows < a.col
        u += list(rows[keep] + off)
        v += list(a.col[keep] + off)
        w += list(-a.val[keep])
    return G.assemble_laplacian(n, u, v, w)


@pytest.mark.gpu
def test_cli_solve_info_bench_match_the_oracle(tmp_path):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    from paper_1108_1310_b200 import lamg as L
    build()
    a = _disconnected()
    mtx = str(tmp_path / "a.mtx")
    L.write_matrix_market(mtx, a)
    b = np.zeros(a.n)
    b[:256] = G.gaussian_rhs(256, 7)
    b[256:263] = [1.0, 0.0, -1.0, 0.5, -0.25, -0.25, 0.0]
    bfile = tmp_path / "b.txt"
    bfile.write_text("\n".join(repr(float(v)) for v in b) + "\n")
    xfile, sfile = str(tmp_path / "x.txt"), str(tmp_path / "s.json")
    rc, out, err = run("solve", "--matrix", mtx, "--rhs", f"file:{bfile}", "--out-x", xfile, "--stats", sfile,
                       "--seed", "1")
    assert rc == 0, (out, err)
    st = json.loads(out)
    assert st == json.load(open(sfile))
    o = Oracle("port")
    op = o.prepare(a)
    xo, rep = op.solve(b)
    x = np.loadtxt(xfile)
    assert np.array_equal(x, xo)  # VALIDATE: the reference's iterate, bit for bit
    assert (st["n"], st["m"], st["components"]) == (a.n, a.m, 3)
    assert st["converged"] is True and st["cycles"] == int(rep["cycles"][0])
    assert st["solve_mvm"] == pytest.approx(float(rep["total_solve_work"][0]), rel=1e-12)
    assert st["setup_mvm"] == pytest.approx(float(op.export()["setup_work"][0]), rel=1e-12)
    assert st["correction"] == "flat" and st["seed"] == 1
    for k in ("acf", "residual_initial", "residual_final", "reduction", "setup_mvm", "total_mvm", "t_setup",
              "t_solve", "t_total", "setup_fraction", "storage_per_edge", "edge_ratio", "recombinations",
              "recomb_max_growth", "wall_setup_seconds", "wall_solve_seconds", "gamma", "mu", "warnings", "levels"):
        assert k in st, k
    # the random right-hand side follows make_rhs (zero sum per component): a compatible solve
    rc, out, _ = run("solve", "--matrix", mtx, "--mode", "throughput")
    assert rc == 0 and json.loads(out)["converged"] is True
    # an incompatible file right-hand side: exit 1 with the reference's message
    bfile.write_text("\n".join("1.0" for _ in range(a.n)) + "\n")
    rc, out, _ = run("solve", "--matrix", mtx, "--rhs", f"file:{bfile}")
    assert rc == 1 and "rhs file sum is not zero" in json.loads(out)["error"]
    # info: the largest component's hierarchy, level by level
    rc, out, _ = run("info", "--matrix", mtx)
    info = json.loads(out)
    g12 = G.grid_5pt(16)
    assert rc == 0 and info["components"] == 3 and len(info["levels"]) >= 2
    assert (info["levels"][0]["n"], info["levels"][0]["m"], info["levels"][0]["kind"]) == (g12.n, g12.m, "finest")
    assert info["levels"][-1]["coarsest"] is True and info["setup_mvm"] == pytest.approx(st["setup_mvm"], rel=1e-12)
    # bench: the reference's CSV columns, one row per problem
    rc, out, _ = run("bench", "--problem", mtx, "--problem", mtx, "--jobs", "2")
    lines = out.strip().split("\n")
    assert rc == 0 and lines[0] == "name,n,m,L,t_setup,t_solve,t_total,acf,storage_per_edge,setup_pct"
    assert len(lines) == 3 and all(l.split(",")[1] == str(a.n) for l in lines[1:])
