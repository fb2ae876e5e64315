"""The C++ drop-in facade compiles against the C-ABI (CPU) and reproduces the
reference's results when run on the GPU.

tests/cpp/facade_demo.cpp is reference-style host code; tests/cpp/facade_api.cpp
calls every declaration of the reference's hierarchy.hpp, cycle.hpp and
solver.hpp (setup, Level::op/transfer/coarsest_solver, hierarchy_stats,
level_cycle_index, solve in both correction modes, DivergedError, recombine,
LevelCredit, flat_mu, prepare, Prepared::largest, solve_prepared,
performance_measures). Its outputs are compared with the CPU oracle bit for bit
(VALIDATE mode: the facade's default)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "facade_demo")
API = os.path.join(ROOT, "tests", "cpp", "facade_api")


def build(src="facade_demo.cpp", out=BIN):
    lib = os.path.join(ROOT, "paper_1108_1310_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", src), "-L", lib, "-llamg_b200",
                    f"-Wl,-rpath,{lib}", "-o", out], check=True)


def test_facade_compiles_and_links():
    build()
    assert os.path.exists(BIN)


def test_facade_api_compiles_and_links():
    build("facade_api.cpp", API)
    assert os.path.exists(API)


@pytest.mark.gpu
def test_facade_runs_on_gpu(port):
    import numpy as np
    from paper_1108_1310_b200 import graphs as G
    if not os.path.exists(BIN):
        build()
    out = subprocess.run([BIN], check=True, capture_output=True, text=True).stdout.splitlines()
    a = G.grid_5pt(64)
    b = np.zeros(a.n)
    b[0], b[-1] = 1.0, -1.0
    _, st = port.setup(a).solve(b, np.zeros(a.n))
    assert out[0].split()[3] == str(int(st["cycles"][0])), out[0]
    assert out[1].startswith("IncompatibleRhsError: right-hand side sum")
    assert out[2] == "components 3 converged 1 x6 0.0"
    assert out[3] == f"mm n {a.n} m {a.m} same 1 laplacian 0", out[3]
    assert out[4] == "IoError: cannot open: /nonexistent/x.mtx"


# ---------------------------------------------------------------- facade_api
def _write(d, name, arr):
    np.ascontiguousarray(arr).tofile(os.path.join(d, name))


def _csr_files(d, prefix, a):
    _write(d, f"{prefix}.row_ptr", np.asarray(a.row_ptr, np.int64))
    _write(d, f"{prefix}.col", np.asarray(a.col, np.int32))
    _write(d, f"{prefix}.val", np.asarray(a.val, np.float64))
    _write(d, f"{prefix}.diag", np.asarray(a.diag, np.float64))


def _meta(d):
    out = {}
    for line in open(os.path.join(d, "meta.txt")):
        k, _, v = line.rstrip("\n").partition(" ")
        out[k] = v
    return out


def _out(d, name, dt):
    return np.fromfile(os.path.join(d, "out." + name), dtype=dt)


def _disconnected():
    # test_cycle.cpp:349-362: a path, a triangle and an isolated node, plus a
    # 12x12 grid so one component has a real hierarchy
    from paper_1108_1310_b200 import graphs as G
    g = G.grid_5pt(12)
    u, v, w = [], [], []
    for r in range(g.n):
        for k in range(g.row_ptr[r], g.row_ptr[r + 1]):
            if g.col[k] > r:
                u.append(r), v.append(int(g.col[k])), w.append(-float(g.val[k]))
    o = g.n
    for a_, b_ in ((0, 1), (1, 2), (3, 4), (4, 5), (5, 3)):
        u.append(o + a_), v.append(o + b_), w.append(1.0)
    return G.assemble_laplacian(o + 7, np.array(u), np.array(v), np.array(w))


@pytest.mark.gpu
@pytest.mark.parametrize("graph", ["grid5_40", "chunglu_4k"])
def test_facade_api_matches_oracle(graph, tmp_path):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    from paper_1108_1310_b200 import graphs as G
    if not os.path.exists(API):
        build("facade_api.cpp", API)
    a = G.grid_5pt(40) if graph == "grid5_40" else G.chung_lu(4096, seed=4)
    if graph != "grid5_40":
        a = G.largest_component(a)[0]
    d = str(tmp_path)
    _csr_files(d, "in", a)
    b, x0 = G.gaussian_rhs(a.n, 31), G.default_x0(a.n, seed=5)
    _write(d, "in.b", b)
    _write(d, "in.x0", x0)
    rng = np.random.default_rng(3)
    sx = [rng.standard_normal(a.n) for _ in range(2)]
    o = Oracle("port")
    sr = [o.residual(a, b, s) for s in sx]
    rx = rng.standard_normal(a.n)
    for i in range(2):
        _write(d, f"in.sx{i}", sx[i])
        _write(d, f"in.sr{i}", sr[i])
    _write(d, "in.rx", rx)
    pa = _disconnected()
    _csr_files(d, "pin", pa)
    pb = np.zeros(pa.n)
    pb[:144] = G.gaussian_rhs(144, 7)
    pb[144:151] = [1.0, 0.0, -1.0, 0.5, -0.25, -0.25, 0.0]
    px0 = G.default_x0(pa.n, seed=9)
    _write(d, "pin.b", pb)
    _write(d, "pin.x0", px0)
    subprocess.run([API, d], check=True, timeout=600)
    m = _meta(d)

    # hierarchy.hpp: every level, operator and transfer equal the reference's
    oh = o.setup(a)
    e = oh.export()
    nl = int(e["nlevels"][0])
    assert int(m["nlevels"]) == nl and float(m["setup_work"]) == float(e["setup_work"][0])
    kinds = {0: "finest", 1: "elimination", 2: "aggregation", 3: "coarsest"}
    for l in range(nl):
        p = f"L{l}."
        assert m[p + "kind"] == kinds[int(e[p + "kind"][0])]
        assert int(m[p + "n"]) == int(e[p + "n"][0]) and int(m[p + "m"]) == int(e[p + "m"][0])
        assert float(m[p + "gamma"]) == float(e[p + "gamma"][0])
        assert int(m[p + "nu_pre"]) == int(e[p + "nu_pre"][0]) and int(m[p + "nu_post"]) == int(e[p + "nu_post"][0])
        assert int(m[p + "coarsest"]) == int(e[p + "coarsest"][0])
        assert float(m[p + "cycle_index"]) == oh.level_cycle_index(l, 1.5)
        for k, dt in (("row_ptr", np.int64), ("col", np.int32), ("val", np.float64), ("diag", np.float64)):
            assert np.array_equal(_out(d, p + k, dt), e[p + k]), (l, k)
        if int(e[p + "kind"][0]) == 2:
            assert np.array_equal(_out(d, p + "aggregate_of", np.int32), e[p + "aggregate_of"])
            assert np.array_equal(_out(d, p + "seed_of", np.int32), e[p + "seed_of"])
            assert float(m[p + "alpha"]) == float(e[p + "alpha"][0])
            assert int(m[p + "stage_used"]) == int(e[p + "stage_used"][0])
            assert int(m[p + "dummy_aggregate"]) == int(e[p + "dummy_aggregate"][0])
        if int(e[p + "kind"][0]) == 1:
            assert int(m[p + "nstages"]) == int(e[p + "nstages"][0])
            for s in range(int(e[p + "nstages"][0])):
                q = f"{p}S{s}."
                for k, dt in (("f_nodes", np.int32), ("f_diag", np.float64), ("f_ptr", np.int64),
                              ("f_nbr", np.int32), ("f_val", np.float64), ("coarse_of_parent", np.int32),
                              ("parent_of_coarse", np.int32)):
                    assert np.array_equal(_out(d, q + k, dt), e[q + k]), (l, s, k)
        if int(e[p + "coarsest"][0]):
            cb = _out(d, p + "coarsest_b", np.float64)
            lo = G.SparseLaplacian(int(e[p + "n"][0]), int(e[p + "m"][0]), e[p + "row_ptr"], e[p + "col"],
                                   e[p + "val"], e[p + "diag"])
            want = o.coarsest_direct(lo, cb) if int(e[p + "coarsest"][0]) == 1 else o.coarsest_relax(lo, cb)
            assert np.array_equal(_out(d, p + "coarsest_x", np.float64), want), l
            assert m[p + "coarsest_same"] == "1"

    # cycle.hpp: solves bit-identical in both correction modes, DivergedError
    xf, sf = oh.solve(b, x0)
    assert np.array_equal(_out(d, "x_flat", np.float64), xf)
    assert np.array_equal(_out(d, "res_flat", np.float64), sf["residuals"])
    assert int(m["flat_cycles"]) == int(sf["cycles"][0]) and float(m["flat_acf"]) == float(sf["acf"][0])
    assert float(m["flat_solve_work"]) == float(sf["solve_work"][0])
    xr, srr = oh.solve(b, x0, correction=1)
    assert np.array_equal(_out(d, "x_recomb", np.float64), xr)
    assert int(m["recomb_cycles"]) == int(srr["cycles"][0])
    assert int(m["recomb_recombinations"]) == int(srr["recombinations"][0])
    if int(sf["cycles"][0]) == 1:
        # a one-cycle solve (relaxation coarsest) converges before the divergence
        # test is reached (cycle.cpp:252-267): neither side throws
        oh.solve(b, x0, divergence_factor=1e-6)
        assert m["diverged"] == "none"
    else:
        with pytest.raises(Exception) as ei:
            oh.solve(b, x0, divergence_factor=1e-6)
        assert m["diverged_message"].startswith("solve diverged: residual grew from ")
        assert m["diverged_message"] in str(ei.value)
        assert int(m["diverged_cycles"]) == int(ei.value.stats["cycles"][0])
        assert np.array_equal(_out(d, "res_diverged", np.float64), ei.value.stats["residuals"])
    y, before, after = o.recombine(a, b, sx, sr, rx)
    assert np.array_equal(_out(d, "recombine_x", np.float64), y)
    assert float(m["recombine_before"]) == before and float(m["recombine_after"]) == after
    assert np.array_equal(_out(d, "credit_takes", np.int32), o.credit_takes(1.5, 12))
    assert float(m["flat_mu"]) == o.flat_mu(2.0)

    # solver.hpp: the whole-problem driver on a disconnected graph with an isolated node
    op = o.prepare(pa)
    pe = op.export()
    assert int(m["prep_components"]) == 4
    assert float(m["prep_setup_work"]) == pytest.approx(float(pe["setup_work"][0]), rel=1e-12)
    xp, rp = op.solve(pb, px0)
    assert np.array_equal(_out(d, "prep_x", np.float64), xp)
    assert m["prep_converged"] == "1"
    assert float(m["prep_solve_work"]) == pytest.approx(float(rp["total_solve_work"][0]), rel=1e-12)
    assert float(m["prep_reduction"]) == float(rp["reduction"][0])
    xg, _ = op.solve(pb)
    assert np.array_equal(_out(d, "prep_x_random_guess", np.float64), xg)
    assert m["prep_bad"].startswith("nonzero rhs at isolated node")
    sizes = [int(m[f"prep_comp{c}"].split()[0]) for c in range(4)]
    big = int(np.argmax(sizes))
    assert int(m["prep_largest_levels"]) == int(m[f"prep_comp{big}"].split()[1]) == int(pe[f"C{big}.nlevels"][0])
    pk = [float(v) for v in m["pm_known"].split()]
    assert pk[0] == 200.0 and abs(pk[1] - 60.0) < 1e-12 and abs(pk[2] - 800.0) < 1e-12 and abs(pk[3] - 0.25) < 1e-14
    assert [float(v) for v in m["pm_degenerate"].split()] == [0.0, 10.0]
