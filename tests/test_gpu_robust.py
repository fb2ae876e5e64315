"""Error paths and cached-state hazards (GPU).

* DivergedError (cycle.cpp:257-267): raised with the reference's message and
  the partial statistics -- VALIDATE mode bit-identical to the oracle
  (message text, cycle count, residual history, acf), THROUGHPUT mode the
  same type, message format and cycle count; a diverged column of a block
  reports its own error while the others converge.
* Captured cycle graphs and relaxation sweep graphs are keyed on everything
  they bake in: a solve with mu = 1 after a solve with mu = 4/3 on the same
  context equals the solve of a fresh context, and
  back-to-back relaxation-coarsest solves of different operators on one
  context equal fresh-context solves.
"""
import os
import sys

import numpy as np
import pytest

from paper_1108_1310_b200 import graphs as G

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


@pytest.mark.parametrize("graph", ["grid5_40", "grid3d_16", "rgg_16k"])
def test_diverged_error_matches_oracle(graph):
    from oracle import Oracle
    from paper_1108_1310_b200 import lamg as L
    a = {"grid5_40": lambda: G.grid_5pt(40), "grid3d_16": lambda: G.grid3d_7pt(16),
         "rgg_16k": lambda: G.rgg(1 << 14, seed=3)}[graph]()
    b, x0 = G.gaussian_rhs(a.n, 17), G.default_x0(a.n, seed=2)
    oh = Oracle("port").setup(a)
    with pytest.raises(Exception) as oe:
        oh.solve(b, x0, divergence_factor=1e-6)
    want = oe.value.stats
    ctx = L.Context(0, L.MODE_VALIDATE)
    h = L.setup(a, ctx=ctx)
    cfg = L.CycleConfig(divergence_factor=1e-6)
    with pytest.raises(L.DivergedError) as ge:
        L.solve(h, b, x0, cfg, ctx=ctx)
    msg = ge.value.msg
    assert msg.startswith("solve diverged: residual grew from ") and msg in str(oe.value)
    st = ge.value.stats
    assert int(st["cycles"][0]) == int(want["cycles"][0]) == 1
    assert np.array_equal(np.asarray(st["residuals"]), want["residuals"])
    assert float(st["acf"][0]) == float(want["acf"][0])
    ctx.set_mode(L.MODE_THROUGHPUT)
    with pytest.raises(L.DivergedError) as te:
        L.solve(h, b, x0, cfg, ctx=ctx)
    assert te.value.msg.startswith("solve diverged: residual grew from ")
    assert int(te.value.stats["cycles"][0]) == 1
    # a block: every column diverges at cycle 1 and reports its own stats
    B = np.stack([b, G.gaussian_rhs(a.n, 18)])
    X0 = np.stack([x0, x0])
    with pytest.raises(L.DivergedError):
        L.solve_batch(h, B, X0, cfg, ctx=ctx)
    ctx.close()


def test_cycle_graphs_keyed_on_mu():
    from paper_1108_1310_b200 import lamg as L
    a = G.grid3d_7pt(24)
    b, x0 = G.gaussian_rhs(a.n, 5), G.default_x0(a.n, seed=3)
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    h = L.setup(a, ctx=ctx)
    x43, s43 = L.solve(h, b, x0, L.CycleConfig(mu=4.0 / 3.0), ctx=ctx)
    x1, s1 = L.solve(h, b, x0, L.CycleConfig(mu=1.0), ctx=ctx)
    B = np.stack([b] * 4)
    X0 = np.stack([x0] * 4)
    XB43, _ = L.solve_batch(h, B, X0, L.CycleConfig(mu=4.0 / 3.0), ctx=ctx)
    XB1, sb1 = L.solve_batch(h, B, X0, L.CycleConfig(mu=1.0), ctx=ctx)
    fresh = L.Context(0, L.MODE_THROUGHPUT)
    xf, sf = L.solve(h, b, x0, L.CycleConfig(mu=1.0), ctx=fresh)
    XBf, sbf = L.solve_batch(h, B, X0, L.CycleConfig(mu=1.0), ctx=fresh)
    assert np.array_equal(x1, xf) and s1.residuals == sf.residuals
    assert np.array_equal(XB1, XBf) and sb1[0].residuals == sbf[0].residuals
    assert s1.cycles != s43.cycles or not np.array_equal(x1, x43)  # mu matters
    fresh.close()
    ctx.close()


def test_relaxation_graph_not_reused_across_operators():
    from paper_1108_1310_b200 import lamg as L
    ops = [G.largest_component(G.chung_lu(1 << 13, seed=s))[0] for s in (4, 6)]
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    k = L.Kernels(ctx=ctx)
    got = []
    for rep in range(2):
        for a in ops:
            b = G.gaussian_rhs(a.n, 9)
            got.append(k.coarsest_relax(a, b))
    for i, a in enumerate(ops):
        c = L.Context(0, L.MODE_THROUGHPUT)
        want = L.Kernels(ctx=c).coarsest_relax(a, G.gaussian_rhs(a.n, 9))
        c.close()
        assert np.array_equal(got[i], want) and np.array_equal(got[i + 2], want), i
    ctx.close()
