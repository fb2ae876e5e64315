"""Blocks of right-hand sides (lamg_solve_batch), GPU.

The reference solves one b per lamg::solve call (cycle.cpp:221-273); a batch
is nrhs such calls on one hierarchy. VALIDATE mode must return, per column,
exactly what the single solve returns (bit-identical to the reference).
THROUGHPUT mode runs up to 32 columns through one cycle schedule; per column
it must converge to the reference tolerance (r <= r0/1e10) in the reference's
cycle count +-1, land within 1e-8 relative of the reference solution (the
finest smoothing level is swept in the reference's order by bgs_exact), and
-- because every kernel folds a
column independently of the others -- give the same bits whatever the
batch it rides in.
"""
import numpy as np
import pytest

from paper_1108_1310_b200 import graphs as G

pytestmark = pytest.mark.gpu

CASES = {
    "grid5_128": lambda: G.grid_5pt(128),
    "rgg_64k": lambda: G.rgg(1 << 16, seed=3),
    "rmat_14": lambda: G.rmat(14, seed=5),
}


def rhs_block(n, nrhs, seed0=300):
    B = np.stack([G.gaussian_rhs(n, seed0 + j) for j in range(nrhs)])
    X0 = np.stack([G.default_x0(n, seed=1 + j) for j in range(nrhs)])
    return B, X0


@pytest.fixture(scope="module", params=list(CASES))
def problem(request):
    from paper_1108_1310_b200 import lamg as L
    a = CASES[request.param]()
    ctx = L.Context(0, L.MODE_VALIDATE)
    h = L.setup(a, ctx=ctx)
    yield request.param, a, ctx, h
    ctx.close()


def test_validate_batch_is_per_column_reference_solve(problem):
    from paper_1108_1310_b200 import lamg as L
    _, a, ctx, h = problem
    ctx.set_mode(L.MODE_VALIDATE)
    B, X0 = rhs_block(a.n, 3)
    X, st = L.solve_batch(h, B, X0, ctx=ctx)
    for j in range(3):
        x, s = L.solve(h, B[j], X0[j], ctx=ctx)
        assert np.array_equal(X[j], x)
        assert s.cycles == st[j].cycles and s.residuals == st[j].residuals


def test_throughput_batch_converges_to_reference_solution(problem):
    from paper_1108_1310_b200 import lamg as L
    name, a, ctx, h = problem
    B, X0 = rhs_block(a.n, 6)
    ctx.set_mode(L.MODE_VALIDATE)
    ref = [L.solve(h, B[j], X0[j], ctx=ctx) for j in range(6)]
    ctx.set_mode(L.MODE_THROUGHPUT)
    X, st = L.solve_batch(h, B, X0, ctx=ctx)
    for j in range(6):
        xr, sr = ref[j]
        s = st[j]
        assert s.converged and s.residuals[-1] <= s.residuals[0] / 1e10, (name, j)
        assert s.residuals[0] == pytest.approx(sr.residuals[0], rel=1e-12)
        # north_star's solve rule: the reference's cycle count +-1, x within 1e-8
        assert np.linalg.norm(X[j] - xr) / np.linalg.norm(xr) <= 1e-8, (name, j)
        assert abs(s.cycles - sr.cycles) <= 1, (name, j, s.cycles, sr.cycles)


def test_throughput_column_independent_of_batch(problem):
    from paper_1108_1310_b200 import lamg as L
    _, a, ctx, h = problem
    ctx.set_mode(L.MODE_THROUGHPUT)
    B, X0 = rhs_block(a.n, 32)
    X32, s32 = L.solve_batch(h, B, X0, ctx=ctx)
    for idx in ([0, 5], [3, 9, 17, 30, 31], list(range(10, 19))):
        Xs, ss = L.solve_batch(h, B[idx], X0[idx], ctx=ctx)
        for i, j in enumerate(idx):
            assert np.array_equal(Xs[i], X32[j]), (idx, j)
            assert ss[i].residuals == s32[j].residuals


def test_throughput_wide_blocks_equal_narrow_blocks(problem):
    # 64- and 128-column blocks run the same per-column arithmetic (one cycle
    # schedule, entry-order folds) as 32-column blocks: identical bits
    from paper_1108_1310_b200 import lamg as L
    _, a, ctx, h = problem
    ctx.set_mode(L.MODE_THROUGHPUT)
    B, X0 = rhs_block(a.n, 72)
    X32, s32 = L.solve_batch(h, B[:32], X0[:32], ctx=ctx)
    X72, s72 = L.solve_batch(h, B, X0, ctx=ctx)  # one 128-wide block
    X40, s40 = L.solve_batch(h, B[32:72], X0[32:72], ctx=ctx)  # one 64-wide block
    for j in range(32):
        assert np.array_equal(X72[j], X32[j]), j
        assert s72[j].residuals == s32[j].residuals
    for j in range(40):
        assert np.array_equal(X72[32 + j], X40[j]), j
        assert s72[32 + j].cycles == s40[j].cycles


def test_throughput_batch_zero_and_incompatible_rhs(problem):
    from paper_1108_1310_b200 import lamg as L
    _, a, ctx, h = problem
    ctx.set_mode(L.MODE_THROUGHPUT)
    B, X0 = rhs_block(a.n, 3)
    B[1] = 0.0
    X0[1] = 0.0
    X, st = L.solve_batch(h, B, X0, ctx=ctx)
    # cycle.cpp:234-238: r0 == 0 returns x0 minus its mean after 0 cycles
    assert st[1].converged and st[1].cycles == 0
    assert np.array_equal(X[1], np.zeros(a.n))
    assert st[0].converged and st[2].converged
    B[2] += 1.0  # sum(b) != 0: IncompatibleRhsError, as lamg::solve raises
    with pytest.raises(L.IncompatibleRhsError):
        L.solve_batch(h, B, X0, ctx=ctx)
