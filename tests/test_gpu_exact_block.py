"""Exact-order K-column Gauss-Seidel (bgs_exact), GPU.

The THROUGHPUT block solve sweeps its exact levels (the finest smoothing
level by default) in the reference's row order (gauss_seidel_sweep,
smoothing.cpp:29-40) for K columns at once, with ticketed wavefront items
instead of a grid barrier. Every column must equal, bit for bit, the
reference sweep applied to that column alone (the oracle's C restatement,
itself pinned to the compiled reference in test_oracle_pin.py) -- on grids,
geometric graphs and power-law levels with hub rows, for 2 sweeps in one
launch (the done counters chain the sweeps) and for every block width.
"""
import os
import sys

import numpy as np
import pytest

from paper_1108_1310_b200 import graphs as G

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))

GRAPHS = {
    "grid3d_20": lambda: G.grid3d_7pt(20),
    "grid5_64": lambda: G.grid_5pt(64),
    "rgg_16k": lambda: G.rgg(1 << 14, seed=3),
    "chunglu_16k": lambda: G.chung_lu(1 << 14, seed=4),
    "rmat_12": lambda: G.rmat(12, seed=5),
}


@pytest.fixture(scope="module", params=list(GRAPHS))
def hier(request):
    from paper_1108_1310_b200 import lamg as L
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    a = GRAPHS[request.param]()
    h = L.setup(a, ctx=ctx)
    yield request.param, a, h
    ctx.close()


def _levels(h):
    # every level the solve could sweep in exact order: levels with an
    # aggregation child (at most the two finest such), plus the finest level
    out = [0]
    for l in range(h.nlevels - 1):
        if h.levels[l + 1].kind == 2 and l not in out:
            out.append(l)
        if len(out) >= 3:
            break
    return out


@pytest.mark.parametrize("K", [128, 32, 8])
def test_block_exact_sweep_is_reference_sweep_per_column(hier, K):
    from oracle import Oracle
    name, _, h = hier
    o = Oracle("port")
    rng = np.random.default_rng(11)
    for l in _levels(h):
        a = h.op(l)
        B = rng.standard_normal((a.n, K))
        X = rng.standard_normal((a.n, K))
        got = h.smooth_exact(l, B, X, sweeps=2)
        for k in range(K):
            want = o.gs_sweep(a, B[:, k], o.gs_sweep(a, B[:, k], X[:, k]))
            assert np.array_equal(got[:, k], want), (name, l, k, float(np.max(np.abs(got[:, k] - want))))


def test_one_column_exact_sweep_is_reference_sweep(hier):
    from oracle import Oracle
    name, _, h = hier
    o = Oracle("port")
    rng = np.random.default_rng(12)
    for l in _levels(h):
        a = h.op(l)
        b, x = rng.standard_normal(a.n), rng.standard_normal(a.n)
        assert np.array_equal(h.smooth_exact(l, b, x, sweeps=3), o.gs_sweep(a, b, o.gs_sweep(a, b, o.gs_sweep(a, b, x))))
