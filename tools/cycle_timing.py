"""Steady-state cycle timing (throughput mode): setup, one warm solve that
captures every cycle graph, then K timed cycles; the timed solve is bracketed
by cudaProfilerStart/Stop so `ncu --profile-from-start off` sees only it."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 20
a = G.grid3d_7pt(int(cfg[1:])) if cfg.startswith("g") else G.make_config(int(cfg))
b, x0 = G.gaussian_rhs(a.n, 102), G.default_x0(a.n)
ctx = L.Context(0, L.MODE_THROUGHPUT)
t = time.time()
h = L.setup(a, ctx=ctx)
print(f"setup {time.time() - t:.2f}s levels {h.nlevels}", flush=True)
x, st = L.solve(h, b, x0, ctx=ctx)
print(f"warm solve: cycles {st.cycles}", flush=True)
for rep in range(2):
    torch.cuda.synchronize()
    if rep == 1:
        torch.cuda.profiler.start()
    t = time.time()
    x, st = L.solve(h, b, x0, L.CycleConfig(max_cycles=cycles), ctx=ctx)
    dt = time.time() - t
    if rep == 1:
        torch.cuda.profiler.stop()
    print(f"rep {rep}: {cycles} cycles {dt * 1e3:.1f} ms = {dt / cycles * 1e3:.2f} ms/cycle", flush=True)
