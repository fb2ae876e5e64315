"""Debug: a column's result in a batch of 2 vs a batch of 32 (THROUGHPUT)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

a = G.rgg(1 << 16, seed=3) if len(sys.argv) < 2 else G.grid_5pt(128)
ctx = L.Context(0, L.MODE_VALIDATE)
h = L.setup(a, ctx=ctx)
if os.environ.get("ORDER"):
    B6 = np.stack([G.gaussian_rhs(a.n, 300 + j) for j in range(6)])
    X6 = np.stack([G.default_x0(a.n, seed=1 + j) for j in range(6)])
    L.solve_batch(h, B6[:3], X6[:3], ctx=ctx)
    for j in range(6):
        L.solve(h, B6[j], X6[j], ctx=ctx)
    ctx.set_mode(L.MODE_THROUGHPUT)
    L.solve_batch(h, B6, X6, ctx=ctx)
ctx.set_mode(L.MODE_THROUGHPUT)
for l in range(h.nlevels):
    li = h.level_info(l)
    print(l, li.kind, li.n, li.m, "coarsest", li.coarsest, "colors", li.colors)
B = np.stack([G.gaussian_rhs(a.n, 300 + j) for j in range(32)])
X0 = np.stack([G.default_x0(a.n, seed=1 + j) for j in range(32)])
X32, s32 = L.solve_batch(h, B, X0, ctx=ctx)
for idx in ([0, 5], [0, 1, 2, 3, 4, 5, 6, 7], list(range(16))):
    Xs, ss = L.solve_batch(h, B[idx], X0[idx], ctx=ctx)
    for i, j in enumerate(idx[:3]):
        r1, r2 = ss[i].residuals, s32[j].residuals
        k = next((q for q in range(min(len(r1), len(r2))) if r1[q] != r2[q]), None)
        print(len(idx), j, "cycles", ss[i].cycles, s32[j].cycles, "first diff at", k,
              "maxdiff", np.abs(Xs[i] - X32[j]).max())
