"""CUDA path vs the reference golden fixtures, bit-for-bit (VALIDATE mode).

Every array in tests/golden/*.npz was produced by the unmodified reference
(tests/golden/make_golden.py). The GPU kernels are called through the C-ABI
(paper_1108_1310_b200/lamg.py -> liblamg_b200.so) on the same inputs.
"""
import numpy as np
import pytest

from conftest import golden_cases, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    from paper_1108_1310_b200.lamg import Kernels
    return Kernels()


class _A:
    def __init__(self, d, p="A."):
        self.n = int(d[p + "n"][0])
        self.m = int(d[p + "m"][0])
        self.row_ptr, self.col, self.val, self.diag = d[p + "row_ptr"], d[p + "col"], d[p + "val"], d[p + "diag"]


def _sub(d, prefix):
    return {k[len(prefix):]: v for k, v in d.items() if k.startswith(prefix)}


def _eq_bag(got, want, what):
    missing = sorted(set(want) - set(got))
    assert not missing, (what, missing)
    bad = [k for k in want if not np.array_equal(np.asarray(got[k]), want[k])]
    assert not bad, f"{what}: {bad[:8]} differ"


@pytest.mark.parametrize("case", golden_cases())
def test_gpu_kernels_bitexact(gpu, case):
    d = load_golden(case)
    a = _A(d)
    x, b = d["K.x"], d["K.b"]
    assert np.array_equal(gpu.residual(a, b, x), d["K.residual"])
    assert np.array_equal(gpu.mvm(a, x), d["K.mvm"])
    assert gpu.energy(a, x) == d["K.energy"][0]
    assert np.array_equal(gpu.gs_sweep(a, b, x), d["K.gs_fwd"])
    assert np.array_equal(gpu.gs_sweep(a, b, x, backward=True), d["K.gs_bwd"])
    assert np.array_equal(gpu.gs_sweep(a, None, x), d["K.gs_homog"])
    assert gpu.probe(a, 8, 77) == d["K.probe"][0]
    tvs = gpu.generate_tvs(a, 4, 3, 1234)
    assert np.array_equal(tvs, d["K.tvs"])
    _eq_bag(gpu.affinities(a, tvs), _sub(d, "K.aff."), "affinities")
    assert np.array_equal(gpu.detect_hubs(a), d["K.hubs"])
    _eq_bag(gpu.aggregate(a, tvs, 1.5, d["K.hubs"]), _sub(d, "K.agg."), "aggregate")
    f, c = gpu.select_low_degree(a)
    assert np.array_equal(f, d["K.sel.f"]) and np.array_equal(c, d["K.sel.c"])
    _eq_bag(gpu.eliminate_rounds(a), _sub(d, "K.elim."), "eliminate_rounds")


@pytest.mark.parametrize("case", golden_cases())
def test_gpu_setup_solve_bitexact(gpu, case):
    d = load_golden(case)
    a = _A(d)
    h = gpu.setup(a)
    _eq_bag(h.export(), _sub(d, "H."), "hierarchy")
    x, st = h.solve(d["S.b"], d["S.x0"], correction=int(d["S.correction"][0]))
    for k in ("cycles", "converged", "residuals", "acf", "solve_work", "recombinations", "recomb_max_growth"):
        assert np.array_equal(st[k], d["S." + k]), k
    assert np.array_equal(x, d["S.x"])
