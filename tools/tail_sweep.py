"""Single-RHS steady-state cycle time (THROUGHPUT) for a graph under the
current LAMG_TAIL_* environment: tools/tail_sweep.py GRAPH [cycles]
GRAPH in {cfg1, cfg2, g64, rgg20, rgg22}."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

name = sys.argv[1]
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 10
a = {"cfg1": lambda: G.make_config(1), "cfg2": lambda: G.make_config(2), "g64": lambda: G.grid3d_7pt(64),
     "rgg20": lambda: G.rgg(1 << 20, seed=3), "rgg22": lambda: G.make_config(3)}[name]()
b, x0 = G.gaussian_rhs(a.n, 102), G.default_x0(a.n)
ctx = L.Context(0, L.MODE_THROUGHPUT)
h = L.setup(a, ctx=ctx)
x, st = L.solve(h, b, x0, ctx=ctx)
full = st.cycles
torch.cuda.synchronize()
t = time.time()
x, st = L.solve(h, b, x0, L.CycleConfig(max_cycles=cycles), ctx=ctx)
torch.cuda.synchronize()
print(f"{name}: {(time.time() - t) / st.cycles * 1e3:.2f} ms/cycle, full solve {full} cycles, "
      f"levels {h.nlevels}", flush=True)
