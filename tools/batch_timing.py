"""Batched (K right-hand sides) THROUGHPUT solve timing on a BASELINE config.

usage: python tools/batch_timing.py [cfg] [nrhs] [reps] [max_cycles]
The last rep runs between cudaProfilerStart/Stop (ncu --profile-from-start off).
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
max_cycles = int(sys.argv[4]) if len(sys.argv) > 4 else 300
lanes = int(os.environ.get("LANES", "1"))
a = G.grid3d_7pt(int(cfg[1:])) if cfg.startswith("g") else G.make_config(int(cfg))
# (zero_sum: about 1 seed in 128 leaves |sum b| over the reference's 1e-10 max|b| threshold at n = 2M)
B = G.zero_sum(np.stack([G.gaussian_rhs(a.n, 1000 + j) for j in range(nrhs)]))
X0 = np.stack([G.default_x0(a.n, seed=1 + j) for j in range(nrhs)])
ctx = L.Context(0, L.MODE_THROUGHPUT)
t = time.time()
h = L.setup(a, ctx=ctx)
print(f"setup {time.time() - t:.2f}s levels {h.nlevels} n {a.n} m {a.m}", flush=True)
import torch  # noqa: E402

if lanes > 1:  # concurrent blocks, one context (stream + workspace) per lane
    import threading
    ctxs = [L.Context(0, L.MODE_THROUGHPUT) for _ in range(lanes)]
    out = [None] * lanes

    def go(i):
        out[i] = L.solve_batch(h, B, X0, L.CycleConfig(max_cycles=max_cycles), ctx=ctxs[i])

    for r in range(reps):
        t = time.time()
        ths = [threading.Thread(target=go, args=(i,)) for i in range(lanes)]
        [th.start() for th in ths]
        [th.join() for th in ths]
        dt = time.time() - t
        cyc = sum(s.cycles for o in out for s in o[1])
        print(f"lanes {lanes} rep {r}: {lanes * nrhs} rhs in {dt * 1e3:.1f} ms; edges*cycles/s {a.m * cyc / dt:.3e}",
              flush=True)
    sys.exit(0)

for r in range(reps):
    last = r == reps - 1
    if last:
        torch.cuda.profiler.start()
    t = time.time()
    X, st = L.solve_batch(h, B, X0, L.CycleConfig(max_cycles=max_cycles), ctx=ctx)
    dt = time.time() - t
    if last:
        torch.cuda.profiler.stop()
    cyc = [s.cycles for s in st]
    print(f"rep {r}: {nrhs} rhs in {dt * 1e3:.1f} ms; cycles min {min(cyc)} max {max(cyc)} mean {np.mean(cyc):.1f}; "
          f"all converged {all(s.converged for s in st)}; edges*cycles/s {a.m * sum(cyc) / dt:.3e}; "
          f"ms per block cycle {dt / max(cyc) * 1e3:.2f}", flush=True)
