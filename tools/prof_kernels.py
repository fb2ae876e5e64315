"""ncu workload for the per-kernel HBM table: config-2 setup (VALIDATE, the
bit-exact setup kernels), then one THROUGHPUT cycle of a 32-column block, all
between cudaProfilerStart/Stop. Summarise the launch list with
tools/kernel_table.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

a = G.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
ctx = L.Context(0, L.MODE_VALIDATE)
L.setup(G.grid_5pt(8), ctx=ctx)
B = np.stack([G.gaussian_rhs(a.n, 100 + j) for j in range(32)])
X0 = np.stack([G.default_x0(a.n, seed=1 + j) for j in range(32)])
torch.cuda.synchronize()
torch.cuda.profiler.start()
h = L.setup(a, ctx=ctx)
ctx.set_mode(L.MODE_THROUGHPUT)
h.prepare_throughput()
L.solve_batch(h, B, X0, L.CycleConfig(max_cycles=1), ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("levels", h.nlevels)
