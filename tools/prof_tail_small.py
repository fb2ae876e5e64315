"""Tail-kernel-only workload for ncu: a level stack that lives entirely in
the CTA-0 shared-memory path (g32: 3D 32^3 grid, tail from the first level)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

a = G.grid3d_7pt(int(sys.argv[1]) if len(sys.argv) > 1 else 32)
b, x0 = G.gaussian_rhs(a.n, 102), G.default_x0(a.n)
ctx = L.Context(0, L.MODE_THROUGHPUT)
h = L.setup(a, ctx=ctx)
L.solve(h, b, x0, L.CycleConfig(max_cycles=2), ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, st = L.solve(h, b, x0, L.CycleConfig(max_cycles=3), ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("cycles", st.cycles)
