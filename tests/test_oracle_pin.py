"""Pins the C restatement oracle (oracle/lamg_oracle.c) before it is trusted.

1. Against the golden fixtures (tests/golden/*.npz), which were produced by the
   unmodified reference (tests/golden/make_golden.py): every kernel output, the
   whole hierarchy and the solve are compared BIT-FOR-BIT.
2. Live against the compiled reference (oracle/_ref) on further seeded graphs
   when it is present (skipped on the GPU box).
3. The numpy input builders (paper_1108_1310_b200/graphs.py) against the
   reference generators and assembly.
"""
import numpy as np
import pytest

from conftest import golden_cases, load_golden
from paper_1108_1310_b200 import graphs as G


class _A:
    def __init__(self, d, p="A."):
        self.n = int(d[p + "n"][0])
        self.m = int(d[p + "m"][0])
        self.row_ptr, self.col, self.val, self.diag = d[p + "row_ptr"], d[p + "col"], d[p + "val"], d[p + "diag"]


def _sub(d, prefix):
    return {k[len(prefix):]: v for k, v in d.items() if k.startswith(prefix)}


def _assert_bag_equal(got: dict, want: dict, what: str):
    assert set(got) == set(want), (what, sorted(set(got) ^ set(want)))
    for k in want:
        assert np.array_equal(got[k], want[k]), f"{what}: {k} differs"


@pytest.mark.parametrize("case", golden_cases())
def test_port_kernels_match_reference_golden(port, case):
    d = load_golden(case)
    a = _A(d)
    x, b = d["K.x"], d["K.b"]
    assert np.array_equal(port.residual(a, b, x), d["K.residual"])
    assert np.array_equal(port.mvm(a, x), d["K.mvm"])
    assert port.energy(a, x) == d["K.energy"][0]
    assert np.array_equal(port.gs_sweep(a, b, x), d["K.gs_fwd"])
    assert np.array_equal(port.gs_sweep(a, b, x, backward=True), d["K.gs_bwd"])
    assert np.array_equal(port.gs_sweep(a, None, x), d["K.gs_homog"])
    assert port.probe(a, 8, 77) == d["K.probe"][0]
    tvs = port.generate_tvs(a, 4, 3, 1234)
    assert np.array_equal(tvs, d["K.tvs"])
    _assert_bag_equal(port.affinities(a, tvs), _sub(d, "K.aff."), "affinities")
    assert np.array_equal(port.detect_hubs(a), d["K.hubs"])
    _assert_bag_equal(port.aggregate(a, tvs, 1.5, d["K.hubs"]), _sub(d, "K.agg."), "aggregate")
    f, c = port.select_low_degree(a)
    assert np.array_equal(f, d["K.sel.f"]) and np.array_equal(c, d["K.sel.c"])
    _assert_bag_equal(port.eliminate_rounds(a), _sub(d, "K.elim."), "eliminate_rounds")


@pytest.mark.parametrize("case", golden_cases())
def test_port_setup_and_solve_match_reference_golden(port, case):
    d = load_golden(case)
    a = _A(d)
    h = port.setup(a)
    _assert_bag_equal(h.export(), _sub(d, "H."), "hierarchy")
    x, stats = h.solve(d["S.b"], d["S.x0"], correction=int(d["S.correction"][0]))
    assert np.array_equal(x, d["S.x"])
    for k in ("residuals", "acf", "solve_work", "cycles", "converged", "recombinations", "recomb_max_growth"):
        assert np.array_equal(stats[k], d["S." + k]), k


LIVE = [
    ("grid5_96", lambda: G.grid_5pt(96)),
    ("rc_5000", lambda: G.random_connected(5000, 1.2, 31)),
    ("grid3d_20w", lambda: G.grid3d_7pt(20, seed=9)),
    ("anis_ag_40", lambda: G.grid_anis_rotated(40, 0.5, 0.02, False)),
    ("rgg_16k", lambda: G.rgg(1 << 14, seed=8)),
    ("chunglu_16k", lambda: G.chung_lu(1 << 14, seed=6)),
]


@pytest.mark.parametrize("name,build", LIVE, ids=[n for n, _ in LIVE])
def test_port_matches_live_reference(port, ref, name, build):
    a = build()
    h1, h2 = port.setup(a), ref.setup(a)
    _assert_bag_equal(h1.export(), h2.export(), "hierarchy")
    b, x0 = G.gaussian_rhs(a.n, 5), G.default_x0(a.n)
    for corr in (0, 1):
        x1, s1 = h1.solve(b, x0, correction=corr)
        x2, s2 = h2.solve(b, x0, correction=corr)
        assert np.array_equal(x1, x2)
        _assert_bag_equal(s1, s2, "stats")


def test_port_prepared_matches_reference(port, ref):
    # disconnected graph with an isolated node (test_cycle.cpp:336-351)
    a = G.assemble_laplacian(7, [0, 1, 3, 4, 5], [1, 2, 4, 5, 3], [1, 1, 1, 1, 1])
    b = np.array([1.0, 0.0, -1.0, 0.5, -0.25, -0.25, 0.0])
    p1, p2 = port.prepare(a), ref.prepare(a)
    _assert_bag_equal(p1.export(), p2.export(), "prepared")
    x1, r1 = p1.solve(b)
    x2, r2 = p2.solve(b)
    assert np.array_equal(x1, x2)
    for k in ("residuals", "cycles", "converged", "all_converged", "total_solve_work"):
        assert np.array_equal(r1[k], r2[k]), k


def test_errors_match_reference(port, ref):
    from oracle import OracleError
    a = G.grid_5pt(8)
    bad = G.SparseLaplacian(a.n, a.m, a.row_ptr, a.col, a.val.copy(), a.diag)
    bad.val[3] *= 2.0
    msgs = []
    for o in (port, ref):
        with pytest.raises(OracleError) as e:
            o.validate(bad)
        msgs.append((e.value.kind, e.value.msg))
    assert msgs[0] == msgs[1] and msgs[0][0] == "InvalidLaplacianError"
    h = port.setup(a), ref.setup(a)
    for hh in h:
        with pytest.raises(OracleError) as e:
            hh.solve(np.ones(a.n), np.zeros(a.n))
        assert e.value.kind == "IncompatibleRhsError"


def test_generators_match_reference(ref):
    from oracle import ref_assemble, ref_generator

    def same(x, y):
        return x.n == y.n and x.m == y.m and all(
            np.array_equal(getattr(x, k), getattr(y, k)) for k in ("row_ptr", "col", "val", "diag"))

    assert same(G.grid_5pt(33), ref_generator(ref, "grid_5pt", 33))
    assert same(G.grid_13pt_4th(20), ref_generator(ref, "grid_13pt_4th", 20))
    for ne in (0, 1):
        assert same(G.grid_anis_rotated(20, 0.785, 0.01, bool(ne)),
                    ref_generator(ref, "grid_anis_rotated", 20, 0.785, 0.01, ne))
    for nm in ("path", "star", "complete", "two_hubs", "binary_tree"):
        assert same(getattr(G, nm)(37), ref_generator(ref, nm, 37)), nm
    us, vs, ws = G.random_connected_edges(500, 2.0, 9)
    assert same(G.random_connected(500, 2.0, 9), ref_assemble(ref, 500, us, vs, ws))
    # duplicates and self-loops (test_graph_core.cpp:51-67)
    assert same(G.assemble_laplacian(3, [0, 2, 1, 1], [1, 2, 2, 0], [1.0, 4.0, 1.0, 2.0]),
                ref_assemble(ref, 3, [0, 2, 1, 1], [1, 2, 2, 0], [1.0, 4.0, 1.0, 2.0]))


def test_rng_counter_form_matches_reference(port, ref):
    for seed in (0, 1, 12345, 2 ** 63 + 5):
        want = ref.rng_draws(seed, 1000, "u64")
        assert np.array_equal(G.rng_u64(seed, 0, 1000), want)
        assert np.array_equal(port.rng_draws(seed, 1000, "u64"), want)
        assert np.array_equal(G.rng_pm1(seed, 0, 1000), ref.rng_draws(seed, 1000, "pm1"))
        for stream in (0, 7, 0x517):
            assert G.Rng.derive(seed, stream) == ref.rng_derive(seed, stream) == port.rng_derive(seed, stream)
