"""GPU diagnostics: hierarchy shape, GS fronts/colours per level, solve timing by mode."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
a = G.grid3d_7pt(int(cfg[1:])) if cfg.startswith("g") else G.make_config(int(cfg))
b = G.gaussian_rhs(a.n, 102)
x0 = G.default_x0(a.n)
ctx = L.Context(0, L.MODE_THROUGHPUT)
t = time.time()
h = L.setup(a, ctx=ctx)
print(f"setup {time.time() - t:.2f}s levels {h.nlevels}", flush=True)
t = time.time()
L._check(ctx.lib.lamg_hier_prepare_throughput(ctx.p, h.h))
print(f"prepare_throughput {time.time() - t:.2f}s", flush=True)
h.levels = [h.level_info(l) for l in range(h.nlevels)]
for l, li in enumerate(h.levels):
    print(l, li.kind, li.n, li.m, "fronts", li.gs_fronts, "colors", li.colors, "coarsest", li.coarsest, flush=True)
xs = {}
for mode in (L.MODE_THROUGHPUT, L.MODE_VALIDATE):
    ctx.set_mode(mode)
    for mc in ((1, 3, 300) if mode == L.MODE_THROUGHPUT else (300,)):
        if mode == L.MODE_VALIDATE and a.n > 300000 and len(sys.argv) < 3:
            mc = 3
        l0 = ctx.lib.lamg_launch_count()
        t = time.time()
        x, st = L.solve(h, b, x0, L.CycleConfig(max_cycles=mc), ctx=ctx)
        dt = time.time() - t
        print(f"mode={mode} max_cycles={mc}: {dt:.3f}s cycles {st.cycles} conv {st.converged} "
              f"launches {ctx.lib.lamg_launch_count() - l0} per-cycle {dt / max(st.cycles, 1) * 1e3:.2f} ms "
              f"acf {st.acf:.4f}", flush=True)
        xs[(mode, mc)] = x
k1, k2 = (L.MODE_THROUGHPUT, 300), (L.MODE_VALIDATE, 300)
if k1 in xs and k2 in xs:
    print("rel x diff throughput vs validate:", np.linalg.norm(xs[k1] - xs[k2]) / np.linalg.norm(xs[k2]))
