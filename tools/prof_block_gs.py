"""ncu workload: one 32-column coloured sweep of the config-2 finest level
(bgs_kernel<32>, the bench's roofline kernel) between cudaProfilerStart/Stop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

a = G.make_config(2)
ctx = L.Context(0, L.MODE_THROUGHPUT)
h = L.setup(a, ctx=ctx)
h.prepare_throughput()
rng = np.random.default_rng(1)
B = rng.standard_normal((a.n, 32))
X = rng.standard_normal((a.n, 32))
h.smooth(0, B, X, 1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
h.smooth(0, B, X, 1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
