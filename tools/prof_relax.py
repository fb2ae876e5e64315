"""ncu workload: one THROUGHPUT solve of R-MAT (reduced config 5) between
cudaProfilerStart/Stop; the relaxation-coarsest cooperative kernel dominates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
ctx = L.Context(0, L.MODE_THROUGHPUT)
a = G.chung_lu(1 << scale, seed=4) if "--chunglu" in sys.argv else L.gen_rmat(scale, seed=5, ctx=ctx)
h = L.setup(a, ctx=ctx)
h.prepare_throughput()
b, x0 = G.gaussian_rhs(a.n, 500), G.default_x0(a.n)
b -= b.sum() / a.n
L.solve(h, b, x0, ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, st = L.solve(h, b, x0, ctx=ctx)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("sweeps", st.relax_sweeps, "converged", st.converged)
