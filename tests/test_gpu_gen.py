"""Graph ingest on the device (gen.cu) vs the host restatement (graphs.py).

BASELINE config 5's R-MAT, config 4's Chung-Lu and the largest-component extraction used by
configs 3-5 (components.cpp:35-56 keeps ascending node
order) must produce the same CSR Laplacian, bit for bit.
"""
import numpy as np
import pytest

from paper_1108_1310_b200 import graphs as G

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert (a.n, a.m) == (b.n, b.m)
    for f in ("row_ptr", "col", "val", "diag"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("scale", [6, 10, 13, 15])
def test_rmat_matches_host_generator(scale):
    from paper_1108_1310_b200 import lamg as L
    g = L.gen_rmat(scale, seed=5)
    _same(g.download(), G.rmat(scale, seed=5))
    g.close()


@pytest.mark.parametrize("n", [1000, 1 << 12, 50000, 1 << 17])
def test_chung_lu_matches_host_generator(n):
    from paper_1108_1310_b200 import lamg as L
    g = L.gen_chung_lu(n, seed=4)
    _same(g.download(), G.chung_lu(n, seed=4))
    g.close()


def test_rmat_without_lcc_and_other_seed():
    from paper_1108_1310_b200 import lamg as L
    g = L.gen_rmat(9, seed=77, edge_factor=4, lcc=False)
    d = g.download()
    # host restatement without the component step
    n, samples = 1 << 9, 4 << 9
    u = np.zeros(samples, dtype=np.int64)
    v = np.zeros(samples, dtype=np.int64)
    a, b, c = 0.57, 0.19, 0.19
    for bit in range(9):
        r = G.rng_unit(77, bit * samples, samples)
        u |= (r >= a + b).astype(np.int64) << bit
        v |= (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.int64) << bit
    keep = u != v
    lo, hi = np.minimum(u[keep], v[keep]), np.maximum(u[keep], v[keep])
    key, cnt = np.unique(lo * n + hi, return_counts=True)
    _same(d, G.assemble_canonical(n, key // n, key % n, cnt.astype(np.float64)))


def _disconnected(seed):
    rng = np.random.default_rng(seed)
    us, vs, ws = [], [], []
    off = 0
    for size in (40, 300, 300, 17, 1, 120):  # two equal largest parts: the first wins
        if size > 1:
            uu, vv, ww = G.random_connected_edges(size, 1.0, seed + size)
            us += [x + off for x in uu]
            vs += [x + off for x in vv]
            ws += ww
        off += size
    perm = rng.permutation(off)  # interleave the components' node ids
    return G.assemble_laplacian(off, perm[np.array(us)], perm[np.array(vs)], ws)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_largest_component_matches_host(seed):
    from paper_1108_1310_b200 import lamg as L
    full = _disconnected(seed)
    g = L.largest_component(full)
    _same(g.download(), G.largest_component(full)[0])


def test_device_graph_feeds_setup():
    from paper_1108_1310_b200 import lamg as L
    ctx = L.Context(0, L.MODE_VALIDATE)
    g = L.gen_rmat(12, seed=5, ctx=ctx)
    h_dev = L.setup(g, ctx=ctx)
    h_host = L.setup(G.rmat(12, seed=5), ctx=ctx)
    e1, e2 = h_dev.export(), h_host.export()
    assert set(e1) == set(e2)
    assert all(np.array_equal(np.asarray(e1[k]), np.asarray(e2[k])) for k in e1)
    ctx.close()
