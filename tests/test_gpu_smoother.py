"""THROUGHPUT-mode smoother parity (GPU).

The coloured Gauss-Seidel sweep is gauss_seidel_sweep (smoothing.cpp:13-40)
run in colour-permuted row order. For every smoothing level of a hierarchy:
  * the colouring is proper (no edge inside a colour) and, on small levels,
    equals the sequential first-fit colouring in index order;
  * one GPU sweep (one column and a 32-column node-major block) matches a
    scipy restatement of the sequential sweep in the same row order within
    1e-12 relative (row dot products are summed in a fixed tree, not in
    column order, so this is a tolerance, not bit parity);
  * a sweep never raises the energy 1/2 x'Ax - b'x (GS on an SPD-on-range
    operator is monotone for any row order).
"""
import numpy as np
import pytest
import scipy.sparse as sp

from paper_1108_1310_b200 import graphs as G

pytestmark = pytest.mark.gpu

GRAPHS = {
    "grid5_64": lambda: G.grid_5pt(64),
    "grid3d_24": lambda: G.grid3d_7pt(24),
    "rgg_16k": lambda: G.rgg(1 << 14, seed=3),
    "rgg_256k": lambda: G.rgg(1 << 18, seed=3),
    "chunglu_16k": lambda: G.chung_lu(1 << 14, seed=4),
    "rmat_13": lambda: G.rmat(13, seed=5),
}


def _offdiag(a):
    return sp.csr_matrix((a.val, a.col, a.row_ptr), shape=(a.n, a.n))


def _sweep(A, diag, rows, ptr, b, x):
    x = x.copy()
    for c in range(len(ptr) - 1):
        r = rows[ptr[c]:ptr[c + 1]]
        r = r[diag[r] != 0.0]  # isolated rows are skipped (smoothing.cpp:20-23)
        d = diag[r] if x.ndim == 1 else diag[r][:, None]
        x[r] = (b[r] - A[r] @ x) / d
    return x


def _energy(A, diag, b, x):
    ax = A @ x + diag * x
    return 0.5 * float(x @ ax) - float(b @ x)


def _greedy(a):
    color = np.full(a.n, -1, np.int64)
    for u in range(a.n):
        nb = a.col[a.row_ptr[u]:a.row_ptr[u + 1]]
        used = set(color[nb[nb < u]].tolist())
        c = 0
        while c in used:
            c += 1
        color[u] = c
    return color


@pytest.fixture(scope="module")
def ctx():
    from paper_1108_1310_b200 import lamg as L
    c = L.Context(0, L.MODE_THROUGHPUT)
    yield c
    c.close()


@pytest.mark.parametrize("name", list(GRAPHS))
def test_colored_sweep_matches_sequential_restatement(name, ctx):
    from paper_1108_1310_b200 import lamg as L
    a = GRAPHS[name]()
    h = L.setup(a, ctx=ctx)
    h.prepare_throughput()
    rng = np.random.default_rng(11)
    checked = 0
    for l, li in enumerate(h.levels):
        if li.colors == 0:
            continue
        op = h.op(l)
        A = _offdiag(op)
        rows, ptr = h.colors(l)
        assert ptr[0] == 0 and ptr[-1] == op.n and np.all(np.diff(ptr) >= 0)
        assert np.array_equal(np.sort(rows), np.arange(op.n))
        color = np.empty(op.n, np.int64)
        for c in range(len(ptr) - 1):
            color[rows[ptr[c]:ptr[c + 1]]] = c
        u = np.repeat(np.arange(op.n), np.diff(op.row_ptr))
        assert not np.any(color[u] == color[op.col]), f"level {l}: improper colouring"
        if op.n <= 70000:
            assert np.array_equal(color, _greedy(op)), f"level {l}: not the index-order greedy colouring"
        b = rng.standard_normal(op.n)
        b -= b.mean()
        x = rng.standard_normal(op.n)
        want = _sweep(A, op.diag, rows, ptr, b, x)
        got = h.smooth(l, b, x, 1)
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err <= 1e-12, f"level {l} (n={op.n}, colours {li.colors}): rel err {err:.3e}"
        assert _energy(A, op.diag, b, got) <= _energy(A, op.diag, b, x) * (1 - 1e-14) + 1e-9
        K = 32
        B = rng.standard_normal((op.n, K))
        B -= B.mean(axis=0)
        X = rng.standard_normal((op.n, K))
        want = _sweep(A, op.diag, rows, ptr, B, X)
        got = h.smooth(l, B, X, 1)
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err <= 1e-12, f"level {l} block: rel err {err:.3e}"
        checked += 1
    assert checked > 0


@pytest.mark.parametrize("n", [100, 128, 129, 140, 150])
def test_throughput_coarsest_inverse(n, ctx):
    """DirectSolver (coarse_solver.cpp:26-76) through the THROUGHPUT inverse:
    every inverse column is built (sizes straddling the 128-thread block)."""
    from oracle import Oracle
    from paper_1108_1310_b200.lamg import Kernels
    gpu = Kernels(ctx)
    port = Oracle("port")
    for seed in (1, 2):
        a = G.random_connected(n, 1.2, 700 + seed + n)
        b = G.random_vector(n, seed, True)
        x = gpu.coarsest_direct(a, b)
        want = port.coarsest_direct(a, b)
        assert np.all(np.isfinite(x))
        assert np.linalg.norm(x - want) <= 1e-10 * np.linalg.norm(want)


RELAX_GRAPHS = {
    "rmat_12": lambda: G.rmat(12, seed=5),
    "chunglu_8k": lambda: G.chung_lu(1 << 13, seed=4),
    "rmat_14": lambda: G.rmat(14, seed=7),
    "rmat_17": lambda: G.rmat(17, seed=8),
}


@pytest.mark.parametrize("path", ["coop", "graph"])
@pytest.mark.parametrize("name", list(RELAX_GRAPHS))
def test_throughput_relaxation_coarsest(name, path, ctx, monkeypatch):
    """RelaxationSolver (coarse_solver.cpp:82-93) in THROUGHPUT mode, both the
    one-launch cooperative form and the per-sweep graph form: the iteration
    reaches the reference's stopping test (|r| <= 1e-12 |r0|) and lands on the
    reference's solution (different sweep order: within 1e-7 relative)."""
    from oracle import Oracle
    from paper_1108_1310_b200.lamg import Kernels
    monkeypatch.setenv("LAMG_RELAX_PATH", path)
    a = RELAX_GRAPHS[name]()
    b = G.random_vector(a.n, 3, True)
    x0 = G.random_vector(a.n, 4)
    gpu = Kernels(ctx)
    x = gpu.coarsest_relax(a, b, x0)
    r0 = np.linalg.norm(gpu.residual(a, b, x0))
    r = np.linalg.norm(gpu.residual(a, b, x))
    assert np.all(np.isfinite(x))
    assert r <= 2e-12 * r0, (r, r0)
    want = Oracle("port").coarsest_relax(a, b, x0)
    dx, dw = x - x.mean(), want - want.mean()
    assert np.linalg.norm(dx - dw) <= 1e-7 * np.linalg.norm(dw)


def test_concurrent_contexts_share_a_power_law_hierarchy():
    """Two contexts (threads/streams) solving over one hierarchy at the same
    time -- the relaxation's chunk counters and sweep graphs are per context,
    so each solve equals the lone solve bit for bit."""
    import threading

    from paper_1108_1310_b200 import lamg as L
    a = G.rmat(17, seed=5)
    c0 = L.Context(0, L.MODE_THROUGHPUT)
    h = L.setup(a, ctx=c0)
    h.prepare_throughput()
    assert h.levels[-1].coarsest == 2 and h.levels[-1].n > 40000
    bs = [G.gaussian_rhs(a.n, 30 + j) for j in range(2)]
    x0 = G.default_x0(a.n)
    want = [L.solve(h, b, x0, ctx=c0)[0] for b in bs]
    ctxs = [L.Context(0, L.MODE_THROUGHPUT) for _ in range(2)]
    got = [[None] * 3 for _ in range(2)]

    def run(j):
        for rep in range(3):
            got[j][rep] = L.solve(h, bs[j], x0, ctx=ctxs[j])[0]

    th = [threading.Thread(target=run, args=(j,)) for j in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for j in range(2):
        for rep in range(3):
            assert np.array_equal(got[j][rep], want[j]), (j, rep)
    for c in ctxs + [c0]:
        c.close()
