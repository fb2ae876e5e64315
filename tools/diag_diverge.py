"""THROUGHPUT-mode divergence hunt: one graph, the solve repeated under
environment toggles (tail rows, graphs) in fresh subprocesses.

usage: python tools/diag_diverge.py [graph]   graph in {rgg18, chunglu18, rmat16}
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np
sys.path.insert(0, %r)
from paper_1108_1310_b200 import graphs as G, lamg as L
name = %r
a = {"rgg18": lambda: G.rgg(1 << 18, seed=3), "chunglu18": lambda: G.chung_lu(1 << 18, seed=4),
     "rmat16": lambda: G.rmat(16, seed=5)}[name]()
b, x0 = G.gaussian_rhs(a.n, 1), G.default_x0(a.n)
ctx = L.Context(0, L.MODE_THROUGHPUT)
h = L.setup(a, ctx=ctx)
L._check(ctx.lib.lamg_hier_prepare_throughput(ctx.p, h.h))
lv = [h.level_info(l) for l in range(h.nlevels)]
print("levels", [(li.kind, li.n, li.colors, li.coarsest) for li in lv])
for rep in range(3):
    try:
        x, st = L.solve(h, b, x0, ctx=ctx)
        print("rep", rep, "cycles", st.cycles, "conv", st.converged, "res", st.residuals[:4], st.residuals[-1])
    except L.DivergedError as e:
        print("rep", rep, "DIVERGED", e.stats["residuals"][:8])
'''
name = sys.argv[1] if len(sys.argv) > 1 else "rgg18"
for env in ({}, {"LAMG_GRAPHS": "0"}, {"LAMG_TAIL_ROWS": "0"}, {"LAMG_TAIL_ROWS": "4096"},
            {"LAMG_TAIL_CTAS": "1"}, {"LAMG_TAIL_SMALL": "0"}):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, name)], env=e, capture_output=True, text=True,
                       timeout=600)
    print("==", env, "rc", r.returncode, flush=True)
    print(r.stdout[-3000:], r.stderr[-2000:], flush=True)
