"""Cycle count and time of a THROUGHPUT one-column solve for exact_levels 0..3
vs the VALIDATE (reference) cycle count: tools/exact_levels.py GRAPH"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

name = sys.argv[1]
a = {"cfg1": lambda: G.make_config(1), "g64": lambda: G.grid3d_7pt(64), "rgg18": lambda: G.rgg(1 << 18, seed=3),
     "rgg20": lambda: G.rgg(1 << 20, seed=3), "cl18": lambda: G.chung_lu(1 << 18, seed=4)}[name]()
b, x0 = G.gaussian_rhs(a.n, 102), G.default_x0(a.n)
ctx = L.Context(0, L.MODE_VALIDATE)
h = L.setup(a, ctx=ctx)
xv, sv = L.solve(h, b, x0, ctx=ctx)
ctx.set_mode(L.MODE_THROUGHPUT)
out = [f"{name}: reference cycles {sv.cycles}; levels {[li.kind for li in h.levels][:6]}"]
for k in (0, 1, 2, 3):
    ctx.set_exact_levels(k)
    L.solve(h, b, x0, ctx=ctx)
    torch.cuda.synchronize()
    t = time.time()
    x, st = L.solve(h, b, x0, ctx=ctx)
    torch.cuda.synchronize()
    out.append(f"  k={k}: {st.cycles} cycles {time.time() - t:.3f}s dx {np.linalg.norm(x - xv) / np.linalg.norm(xv):.2e}")
print("\n".join(out), flush=True)
