"""GPU timing of setup + solve (both modes) on BASELINE configs 3-5 (cfg5 at reduced scale)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

for name in sys.argv[1:]:
    t = time.time()
    a = {"cfg3": lambda: G.make_config(3), "cfg4": lambda: G.make_config(4),
         "rmat22": lambda: G.rmat(22), "rmat20": lambda: G.rmat(20)}[name]()
    tg = time.time() - t
    b, x0 = G.gaussian_rhs(a.n, 7), G.default_x0(a.n)
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    t = time.time()
    h = L.setup(a, ctx=ctx)
    ts = time.time() - t
    L._check(ctx.lib.lamg_hier_prepare_throughput(ctx.p, h.h))
    h.levels = [h.level_info(l) for l in range(h.nlevels)]
    print(f"{name}: n={a.n} m={a.m} gen {tg:.1f}s setup {ts:.2f}s levels "
          f"{[(li.kind, li.n, li.gs_fronts, li.colors, li.coarsest) for li in h.levels]}", flush=True)
    for mode in (L.MODE_THROUGHPUT, L.MODE_VALIDATE):
        ctx.set_mode(mode)
        t = time.time()
        x, st = L.solve(h, b, x0, ctx=ctx)
        dt = time.time() - t
        print(f"  mode {mode}: {dt:.3f}s cycles {st.cycles} relax sweeps {st.relax_sweeps} conv {st.converged} "
              f"edges*cycles/s {a.m * st.cycles / dt:.3e}", flush=True)
    ctx.close()
