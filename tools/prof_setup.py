"""Setup-only workload for ncu (power-law graph): the setup runs between
cudaProfilerStart/Stop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

a = G.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 18)
ctx = L.Context(0, L.MODE_VALIDATE)
L.setup(G.grid_5pt(8), ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.start()
h = L.setup(a, ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("levels", h.nlevels, "setup_s", h.setup_seconds)
