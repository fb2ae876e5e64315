"""LAMG_TRACE=1 one-cycle traces of the RGG 256k solve in both modes (debugging aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

a = G.rgg(1 << 18, seed=3)
b, x0 = G.gaussian_rhs(a.n, 1), G.default_x0(a.n)
ctx = L.Context(0, L.MODE_VALIDATE)
h = L.setup(a, ctx=ctx)
for mode in (L.MODE_VALIDATE, L.MODE_THROUGHPUT):
    ctx.set_mode(mode)
    print(f"===== mode {mode}", file=sys.stderr, flush=True)
    try:
        x, st = L.solve(h, b, x0, L.CycleConfig(max_cycles=2), ctx=ctx)
        print("residuals", st.residuals, file=sys.stderr, flush=True)
    except L.DivergedError as e:
        print("diverged", e.stats["residuals"], file=sys.stderr, flush=True)
