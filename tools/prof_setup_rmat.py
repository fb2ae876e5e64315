"""ncu workload: the GPU setup of a device R-MAT graph (config-5 shape at a
reduced scale) between cudaProfilerStart/Stop."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 21
ctx = L.Context(0, L.MODE_VALIDATE)
L.setup(G.grid_5pt(8), ctx=ctx)
a = L.gen_rmat(scale, seed=5, ctx=ctx)
torch.cuda.synchronize()
t = time.time()
torch.cuda.profiler.start()
h = L.setup(a, ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("levels", h.nlevels, "setup_s", round(time.time() - t, 2), [(li.kind, li.n) for li in h.levels])
