"""THROUGHPUT solve of RGG 256k (seed 3) for race/initcheck hunting."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 3
a = G.rgg(1 << 18, seed=3)
b, x0 = G.gaussian_rhs(a.n, 1), G.default_x0(a.n)
ctx = L.Context(0, L.MODE_THROUGHPUT)
h = L.setup(a, ctx=ctx)
try:
    x, st = L.solve(h, b, x0, L.CycleConfig(max_cycles=cyc), ctx=ctx)
    print("residuals", st.residuals, flush=True)
except L.DivergedError as e:
    print("diverged", e.stats["residuals"], flush=True)
