"""Known-answer tests of the reference unit suite, restated.

Each test cites the reference test it restates (paths under
/root/reference/proj/tests/unit/). They run against every backend that
exposes the oracle API: the C restatement ("port"), the compiled reference
("ref", when present), and the CUDA path ("gpu", marked gpu), so the same
expectations pin the oracle and check the product.
"""
import math

import numpy as np
import pytest

from paper_1108_1310_b200 import graphs as G

BACKENDS = ["port", "ref", pytest.param("gpu", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS, scope="module")
def be(request):
    if request.param == "port":
        from oracle import Oracle
        return Oracle("port")
    if request.param == "ref":
        import os
        from oracle import LIBS, Oracle
        if not os.path.exists(LIBS["ref"][0]):
            pytest.skip("oracle/_ref not built")
        return Oracle("ref")
    from paper_1108_1310_b200.lamg import Kernels
    return Kernels()


def _err_kind(e):
    return getattr(e, "kind", type(e).__name__)


def five_node():
    # test_graph_core.cpp:17-24
    return G.assemble_laplacian(5, [0, 0, 0, 0, 1, 2], [1, 2, 3, 4, 3, 3], [1.0, 1.0, 1.0, 5.0, 1.0, 2.0])


def test_five_node_assembly_bit_exact(be):
    # test_graph_core.cpp:27-40
    a = five_node()
    want = np.array([[8, -1, -1, -1, -5], [-1, 2, 0, -1, 0], [-1, 0, 3, -2, 0], [-1, -1, -2, 4, 0],
                     [-5, 0, 0, 0, 5]], dtype=float)
    assert np.array_equal(a.to_dense(), want) and a.m == 6
    be.validate(a)


def test_mvm_known_answers(be):
    # test_graph_core.cpp:86-99
    a = five_node()
    assert np.all(np.abs(be.mvm(a, np.ones(5))) == 0.0)
    two = G.assemble_laplacian(2, [0], [1], [1.0])
    assert np.array_equal(be.mvm(two, np.array([1.0, 0.0])), np.array([1.0, -1.0]))


def test_residual_dense_oracle(be):
    # test_graph_core.cpp:101-113 (dense product to 1e-12)
    for seed in (11, 12, 13):
        a = G.random_connected(200 if seed == 13 else 50, 2.0, seed)
        x = G.random_vector(a.n, seed + 100)
        b = G.random_vector(a.n, seed + 7)
        r = be.residual(a, b, x)
        want = b - a.to_dense() @ x
        assert np.all(np.abs(r - want) <= 1e-12 * np.maximum(1.0, np.abs(want)))


def test_energy_known_answers(be):
    # test_graph_core.cpp:139-154
    a = G.random_connected(30, 1.5, 3)
    assert be.energy(a, np.full(30, 2.5)) == 0.0
    p = G.path(3)
    assert be.energy(p, np.array([0.0, 1.0, 2.0])) == 2.0


def test_gs_two_node_forward_backward(be):
    # test_smoothing.cpp:22-30, 66-74
    a = G.assemble_laplacian(2, [0], [1], [1.0])
    b = np.array([1.0, -1.0])
    assert np.array_equal(be.gs_sweep(a, b, np.zeros(2)), np.array([1.0, 0.0]))
    assert np.array_equal(be.gs_sweep(a, b, np.zeros(2), backward=True), np.array([0.0, -1.0]))


def test_gs_fixed_point_and_monotone(be):
    # test_smoothing.cpp:32-64
    a = G.random_connected(40, 1.5, 5)
    xs = G.random_vector(a.n, 55, True)
    b = be.mvm(a, xs)
    x = xs.copy()
    for _ in range(5):
        x = be.gs_sweep(a, b, x)
    assert np.linalg.norm(be.residual(a, b, x)) <= 1e-12 * max(np.linalg.norm(b), 1.0)
    for seed in range(0, 100, 7):
        a = G.random_connected(25, 1.2, 1000 + seed)
        xs = G.random_vector(a.n, seed, True)
        b = be.mvm(a, xs)
        x = G.random_vector(a.n, seed + 500)
        f = lambda v: 0.5 * be.energy(a, v) - v @ b  # noqa: E731
        before = f(x)
        after = f(be.gs_sweep(a, b, x))
        assert after <= before + 1e-10 * (abs(before) + 1.0)


def test_tvs_properties(be):
    # test_smoothing.cpp:76-105
    a = G.path(64)
    t = be.generate_tvs(a, 4, 0, 9)
    for col in t:
        assert np.max(np.abs(col)) <= 2.0
        assert abs(col.sum()) <= 1e-12 * np.max(np.abs(col)) * a.n
    g = G.grid_5pt(12)
    raw, relaxed = be.generate_tvs(g, 4, 0, 31), be.generate_tvs(g, 4, 3, 31)
    for k in range(4):
        assert be.energy(g, relaxed[k]) <= be.energy(g, raw[k]) + 1e-12
    g = G.grid_5pt(10)
    assert np.array_equal(be.generate_tvs(g, 6, 3, 12345), be.generate_tvs(g, 6, 3, 12345))
    assert not np.array_equal(be.generate_tvs(g, 6, 3, 12345)[0], be.generate_tvs(g, 6, 3, 54321)[0])


def test_probe_known_answers(be):
    # test_smoothing.cpp:107-130
    assert be.probe(G.complete(50), 8, 7) <= 0.3
    p = G.path(1000)
    assert be.probe(p, 16, 7) >= 0.9
    assert be.probe(p, 8, 7) > 0.7
    assert be.probe(G.assemble_laplacian(2, [0], [1], [1.0]), 8, 7) == 0.0


def test_select_known_answers(be):
    # test_elimination.cpp:14-36
    f, c = be.select_low_degree(G.path(5))
    assert list(f) == [0, 2, 4] and list(c) == [1, 3]
    f, c = be.select_low_degree(G.complete(10))
    assert len(f) == 0 and len(c) == 10
    f, c = be.select_low_degree(G.star(9))
    assert len(f) == 8 and list(c) == [0]


def test_schur_and_transfers_three_path(be):
    # test_elimination.cpp:38-45, 155-161, 192-199
    s = be.schur(G.path(3), [1], [0, 2])
    assert int(s["n"][0]) == 2
    assert abs(s["diag"][0] - 0.5) <= 1e-14 * 0.5
    assert abs(-s["val"][0] - 0.5) <= 1e-14 * 0.5
    st = {k[2:]: v for k, v in s.items() if k.startswith("S.")}
    assert np.array_equal(be.coarsen_rhs_stage(st, np.array([1.0, 0.0, -1.0])), np.array([1.0, -1.0]))
    x = be.backsub_stage(st, np.array([0.5, -0.5]), np.array([1.0, 0.0, -1.0]))
    assert x[0] == 0.5 and x[2] == -0.5 and abs(x[1]) <= 1e-15


def test_schur_rejects_dependent_f(be):
    # test_elimination.cpp:73-77
    with pytest.raises(Exception):
        be.schur(G.path(4), [0, 1], [2, 3])


def test_affinity_known_answers(be):
    # test_aggregation.cpp:39-68
    p2 = G.path(2)
    aff = lambda a, rows: be.affinities(a, np.array(rows, dtype=float).T.copy())  # noqa: E731
    assert abs(aff(p2, [[1.0, 2.0, -0.5], [2.0, 4.0, -1.0]])["edge_affinity"][0]) <= 1e-14
    assert aff(p2, [[1.0, 0.0], [0.0, 1.0]])["edge_affinity"][0] == 1.0
    assert abs(aff(p2, [[1.0, 0.0], [1.0, 1.0]])["edge_affinity"][0] - 0.5) <= 1e-15
    d = aff(G.path(3), [[1.0, 1.0], [0.0, 0.0], [1.0, -1.0]])
    assert list(d["degenerate"]) == [1] and np.all(d["edge_affinity"] == 1.0)


def test_hubs_known_answers(be):
    # test_aggregation.cpp:96-118
    assert len(be.detect_hubs(G.star(8))) == 0
    for n in (9, 12):
        assert list(be.detect_hubs(G.star(n))) == [0]
    assert len(be.detect_hubs(G.grid_5pt(8))) == 0
    assert list(be.detect_hubs(G.two_hubs(50))) == [0, 1]


def test_energy_ratio_known_answers(port):
    # test_aggregation.cpp:120-136 (oracle-only entry point, used by tests)
    q = port.energy_ratio_qus(G.star(4), np.array([[7.0, 0.0, 1.0, 2.0]]), 0, 2)
    assert abs(q - 1.0) <= 1e-14
    q = port.energy_ratio_qus(G.path(3), np.array([[0.0, 1.0, 2.0]]), 1, 0)
    assert abs(q - 0.5) <= 1e-14


def test_aggregate_path8_and_hubs_apart(be):
    # test_aggregation.cpp:181-214
    a = G.path(8)
    t = be.aggregate(a, be.generate_tvs(a, 4, 3, 11), 1.5, be.detect_hubs(a))
    assert int(t["stage_used"][0]) == 1 and 0.375 <= t["alpha"][0] <= 0.625
    a = G.two_hubs(50)
    t = be.aggregate(a, be.generate_tvs(a, 4, 3, 5), 1.5, be.detect_hubs(a))
    assert t["aggregate_of"][0] != t["aggregate_of"][1]


def test_galerkin_known_answers(be):
    # test_aggregation.cpp:216-268
    c = be.galerkin(G.path(4), np.array([0, 0, 1, 1]), 2)
    assert c.n == 2 and c.diag[0] == 1.0 and -c.val[0] == 1.0
    a = G.random_connected(25, 1.0, 77)
    c = be.galerkin(a, np.arange(a.n), a.n)
    assert np.array_equal(G.SparseLaplacian(c.n, c.m, c.row_ptr, c.col, c.val, c.diag).to_dense(), a.to_dense())
    for seed in range(3):
        a = G.random_connected(40, 1.5, 880 + seed)
        r = G.Rng(seed)
        cn = a.n // 3
        agg = np.array(list(range(cn)) + [r.next_u64() % cn for _ in range(a.n - cn)])
        c = be.galerkin(a, agg, cn)
        p = np.zeros((a.n, cn))
        p[np.arange(a.n), agg] = 1.0
        want = p.T @ a.to_dense() @ p
        got = G.SparseLaplacian(c.n, c.m, c.row_ptr, c.col, c.val, c.diag).to_dense()
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


def test_credit_and_flat_mu(be):
    # test_cycle.cpp:69-90
    assert list(be.credit_takes(1.5, 6)) == [1, 2, 1, 2, 1, 2]
    assert list(be.credit_takes(1.0, 5)) == [1] * 5
    assert be.flat_mu(2.0) == 4.0 / 3.0 and be.flat_mu(1.0) == 1.0 and be.flat_mu(3.0) == 1.5


def test_coarsest_direct_known_answers(be):
    # test_cycle.cpp:92-133
    a = G.assemble_laplacian(2, [0], [1], [1.0])
    x = be.coarsest_direct(a, np.array([1.0, -1.0]))
    assert abs(x[0] - 0.5) <= 1e-14 and abs(x[1] + 0.5) <= 1e-14
    a = G.random_connected(30, 1.0, 5)
    assert np.all(np.abs(be.coarsest_direct(a, np.zeros(30), np.full(30, 9.0))) <= 1e-14)
    for seed in range(0, 100, 9):
        n = 20 + (seed % 5) * 30
        a = G.random_connected(n, 1.2, 4000 + seed)
        b = G.random_vector(n, seed, True)
        x = be.coarsest_direct(a, b)
        assert np.linalg.norm(be.residual(a, b, x)) <= 1e-10 * np.linalg.norm(b)
        assert abs(x.sum()) <= 1e-10 * n
    a = G.assemble_laplacian(4, [0, 2], [1, 3], [1.0, 2.0])
    b = np.array([1.0, -1.0, 3.0, -3.0])
    x = be.coarsest_direct(a, b)
    assert np.linalg.norm(be.residual(a, b, x)) <= 1e-12
    assert abs(x[0] + x[1]) <= 1e-14 and abs(x[2] + x[3]) <= 1e-14


def test_recombine_unchanged_iterate(be):
    # test_cycle.cpp:135-146
    a = G.random_connected(25, 1.0, 8)
    b, x = G.random_vector(25, 9, True), G.random_vector(25, 10)
    r = be.residual(a, b, x)
    y, before, after = be.recombine(a, b, [x], [r], x)
    assert abs(after - before) <= 1e-14 * before and np.array_equal(y, x)


def test_setup_shapes(be):
    # test_hierarchy.cpp:10-32, 69-79
    h = be.setup(G.random_connected(100, 1.0, 2)).export()
    assert int(h["nlevels"][0]) == 1 and int(h["L0.coarsest"][0]) == 1
    h = be.setup(G.complete(200)).export()
    assert int(h["nlevels"][0]) == 1 and int(h["L0.coarsest"][0]) == 2
    h = be.setup(G.path(10000)).export()
    assert int(h["nlevels"][0]) >= 2 and int(h["L1.kind"][0]) == 1
    g = G.grid_5pt(24)
    h1, h2 = be.setup(g, seed=9).export(), be.setup(g, seed=9).export()
    assert all(np.array_equal(h1[k], h2[k]) for k in h1)


def test_solve_known_answers(be):
    # test_cycle.cpp:192-300
    a = G.grid_5pt(16)
    h = be.setup(a)
    x, st = h.solve(np.zeros(a.n), np.zeros(a.n))
    assert np.array_equal(x, np.zeros(a.n)) and st["converged"][0] == 1 and st["cycles"][0] <= 1
    assert st["residuals"][0] == 0.0 and st["acf"][0] == 0.0
    h8 = be.setup(G.grid_5pt(8))
    with pytest.raises(Exception) as e:
        h8.solve(np.ones(64), np.zeros(64))
    assert "IncompatibleRhs" in _err_kind(e.value) or "IncompatibleRhs" in str(e.value)
    a = G.grid_5pt(24)
    h = be.setup(a)
    with pytest.raises(Exception) as e:
        h.solve(G.random_vector(a.n, 3, True), np.zeros(a.n), mu=40.0)
    st = e.value.stats
    assert len(st["residuals"]) >= 2 and st["residuals"][-1] > 1e3 * st["residuals"][0]
    a = G.grid_5pt(64)
    h = be.setup(a)
    x, st = h.solve(G.random_vector(a.n, 17, True), G.random_vector(a.n, 18))
    assert st["converged"][0] == 1 and st["acf"][0] <= 0.35
    assert st["residuals"][0] / st["residuals"][-1] >= 1e10
    a = G.complete(200)
    h = be.setup(a)
    b = G.random_vector(a.n, 3, True)
    x, st = h.solve(b, np.zeros(a.n))
    assert st["converged"][0] == 1 and np.linalg.norm(be.residual(a, b, x)) <= 1e-10 * np.linalg.norm(b)


def test_adaptive_accelerates_grid(be):
    # test_cycle.cpp:284-302
    a = G.grid_5pt(48)
    h = be.setup(a)
    b, x0 = G.random_vector(a.n, 21, True), G.random_vector(a.n, 22)
    _, sf = h.solve(b, x0)
    _, sa = h.solve(b, x0, correction=1)
    assert sf["converged"][0] == 1 and sa["converged"][0] == 1
    assert sa["recombinations"][0] > 0 and sa["recomb_max_growth"][0] <= 1.0 + 1e-12
    assert sa["acf"][0] <= sf["acf"][0] + 1e-12


def test_solution_matches_dense_min_norm(be):
    # test_cycle.cpp:304-323
    for seed in range(2):
        a = G.random_connected(220, 2.0, 50 + seed)
        h = be.setup(a, seed=seed + 1)
        b = G.random_vector(a.n, seed + 5, True)
        x, st = h.solve(b, np.zeros(a.n), target_reduction=1e12)
        assert st["converged"][0] == 1
        xs = np.linalg.pinv(a.to_dense()) @ b
        d = x - xs
        err = math.sqrt(max(be.energy(a, d), 0.0))
        assert err <= 1e-8 * math.sqrt(max(be.energy(a, xs), 0.0))
