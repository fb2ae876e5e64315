"""Solve-only workload for ncu: setup outside the profiled range, then a
short throughput-mode solve between cudaProfilerStart/Stop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = L.MODE_VALIDATE if len(sys.argv) > 3 and sys.argv[3] == "validate" else L.MODE_THROUGHPUT
a = G.make_config(cfg)
b, x0 = G.gaussian_rhs(a.n, 102), G.default_x0(a.n)
ctx = L.Context(0, mode)
h = L.setup(a, ctx=ctx)
L._check(ctx.lib.lamg_hier_prepare_throughput(ctx.p, h.h))
L.solve(h, b, x0, L.CycleConfig(max_cycles=1), ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, st = L.solve(h, b, x0, L.CycleConfig(max_cycles=cycles), ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("cycles", st.cycles)
