"""Hub rows (more than 2048 entries) on the VALIDATE path, bit-for-bit.

Rows longer than kHeavyRowExact are swept by a whole CTA (products in
parallel, the add chain in reference order), so these cases force that code
path: a random connected graph with three hubs of 2.5k-5k neighbours, and a
star. Every kernel, the hierarchy and the solve are compared with the C
restatement (oracle/, pinned to the reference's goldens) on the same inputs,
and the validation error for a corrupted hub row must name the same entry
with the same message (sparse_laplacian.cpp:194-234).
"""
import numpy as np
import pytest

from paper_1108_1310_b200 import graphs as G

pytestmark = pytest.mark.gpu


def hubby(n=12000, seed=21):
    us, vs, ws = G.random_connected_edges(n, 1.5, seed)
    rng = np.random.default_rng(seed)
    for hub, deg in ((0, 5000), (1, 3000), (n // 2, 2500)):
        nb = rng.choice(np.setdiff1d(np.arange(n), [hub]), deg, replace=False)
        us += [hub] * deg
        vs += nb.tolist()
        ws += rng.uniform(0.5, 2.0, deg).tolist()
    return G.assemble_laplacian(n, us, vs, ws)


CASES = {"hubby": hubby, "star": lambda: G.star(6000), "two_hubs": lambda: G.two_hubs(2600)}


@pytest.fixture(scope="module")
def backends():
    from oracle import Oracle
    from paper_1108_1310_b200.lamg import Kernels
    return Oracle("port"), Kernels()


@pytest.mark.parametrize("name", list(CASES))
def test_hub_kernels_bitexact(backends, name):
    port, gpu = backends
    a = CASES[name]()
    assert np.diff(a.row_ptr).max() > 2048
    x = G.random_vector(a.n, 5)
    b = G.random_vector(a.n, 6, zero_mean=True)
    gpu.validate(a)
    assert np.array_equal(gpu.residual(a, b, x), port.residual(a, b, x))
    for bb, bw in ((b, False), (b, True), (None, False)):
        assert np.array_equal(gpu.gs_sweep(a, bb, x, backward=bw), port.gs_sweep(a, bb, x, backward=bw))
    assert gpu.probe(a, 8, 77) == port.probe(a, 8, 77)
    assert np.array_equal(gpu.generate_tvs(a, 4, 3, 99), port.generate_tvs(a, 4, 3, 99))


@pytest.mark.parametrize("name", list(CASES))
def test_hub_setup_solve_bitexact(backends, name):
    port, gpu = backends
    a = CASES[name]()
    hg, hp = gpu.setup(a), port.setup(a)
    eg, ep = hg.export(), hp.export()
    assert set(eg) == set(ep)
    bad = [k for k in ep if not np.array_equal(np.asarray(eg[k]), np.asarray(ep[k]))]
    assert not bad, bad[:8]
    b = G.random_vector(a.n, 8, zero_mean=True)
    x0 = G.default_x0(a.n)
    xg, sg = hg.solve(b, x0)
    xp, sp = hp.solve(b, x0)
    for k in ("cycles", "converged", "residuals", "acf", "solve_work"):
        assert np.array_equal(sg[k], sp[k]), k
    assert np.array_equal(xg, xp)


class _Raw:
    def __init__(self, a):
        self.n, self.m = a.n, a.m
        self.row_ptr, self.col = a.row_ptr.copy(), a.col.copy()
        self.val, self.diag = a.val.copy(), a.diag.copy()


def _msg(f):
    try:
        f()
    except Exception as e:  # noqa: BLE001 - both backends raise their own type
        return getattr(e, "kind", type(e).__name__), str(e)
    return None


@pytest.mark.parametrize("corrupt", ["value", "rowsum", "sort"])
def test_hub_validation_errors_match(backends, corrupt):
    port, gpu = backends
    a = _Raw(hubby())
    s, e = int(a.row_ptr[0]), int(a.row_ptr[1])
    assert e - s > 2048
    k = s + 3000
    if corrupt == "value":
        a.val[k] *= 1.5  # asymmetric at position 3000 of hub row 0
    elif corrupt == "rowsum":
        a.diag[0] += 1.0
    else:
        a.col[k], a.col[k + 1] = a.col[k + 1], a.col[k]
    want = _msg(lambda: port.validate(a))
    assert want is not None
    assert _msg(lambda: gpu.validate(a)) == want
