"""Full-scale runs of BASELINE.json configs 3-5 (THROUGHPUT mode): input
generation (config 5 on the device, lamg_gen_rmat), GPU setup, one
single-RHS solve and one 32-column block solve, timed with CUDA events.

usage: python tools/config_runs.py CFG [scale_down] > line.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

cfg = int(sys.argv[1])
sd = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = L.Context(0, L.MODE_THROUGHPUT)
t = time.time()
if cfg == 5:
    a = L.gen_rmat(25 - 2 * sd, seed=5, ctx=ctx)
    torch.cuda.synchronize()
    gen = {"where": "device (lamg_gen_rmat: samples, radix sort, run-length merge, union-find LCC, assembly)"}
elif cfg == 4:
    a = L.gen_chung_lu(1 << (24 - 2 * sd), seed=4, ctx=ctx)
    torch.cuda.synchronize()
    gen = {"where": "device (lamg_gen_chung_lu: host CDF, device inverse-CDF samples, radix sort, merge, "
                    "union-find LCC, assembly)"}
else:
    a = G.make_config(cfg, sd)
    gen = {"where": "host numpy (graphs.py)"}
gen["seconds"] = round(time.time() - t, 2)
print(f"cfg{cfg}: n={a.n} m={a.m} generated in {gen['seconds']}s ({gen['where']})", file=sys.stderr, flush=True)
t = time.time()
h = L.setup(a, ctx=ctx)
torch.cuda.synchronize()
setup_s = time.time() - t
levels = [h.level_info(l) for l in range(h.nlevels)]
print(f"setup {setup_s:.2f}s, {h.nlevels} levels", file=sys.stderr, flush=True)
t = time.time()
L._check(ctx.lib.lamg_hier_prepare_throughput(ctx.p, h.h))
torch.cuda.synchronize()
prep_s = time.time() - t
lv = [{"kind": li.kind, "n": li.n, "m": li.m, "colors": li.colors, "coarsest": li.coarsest} for li in levels]
nrhs = 32
B = np.stack([G.gaussian_rhs(a.n, 500 + j) for j in range(nrhs)])
# at n ~ 1e7 the reference's sequential mean subtraction leaves |sum b| ~ 3e-10,
# at the 1e-10 * max|b| compatibility threshold (cycle.cpp:226-230): project
# once more with a pairwise sum so every column is a zero-sum b
for _ in range(2):
    B -= (B.sum(axis=1) / a.n)[:, None]
X0 = np.stack([G.default_x0(a.n, seed=1 + j) for j in range(nrhs)])


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.time()
    r = fn()
    torch.cuda.synchronize()
    return r, time.time() - t0


L.solve(h, B[0], X0[0], ctx=ctx)  # first call: workspace, graphs
(x1, s1), single_s = timed(lambda: L.solve(h, B[0], X0[0], ctx=ctx))
(xb, sb), block_s = timed(lambda: L.solve_batch(h, B, X0, ctx=ctx))
(xb, sb), block_s2 = timed(lambda: L.solve_batch(h, B, X0, ctx=ctx))  # graphs captured
cyc = [s.cycles for s in sb]
sweeps = [s.relax_sweeps for s in sb]
out = {"config": cfg, "scale_down": sd, "n": a.n, "m": a.m, "generation": gen, "setup_s": round(setup_s, 2),
       "prepare_throughput_s": round(prep_s, 2), "levels": lv,
       "single": {"seconds": round(single_s, 3), "cycles": s1.cycles, "relax_sweeps": s1.relax_sweeps,
                  "converged": s1.converged, "edges_cycles_per_s": a.m * s1.cycles / single_s},
       "block32": {"seconds": round(block_s2, 3), "first_call_seconds": round(block_s, 3), "cycles": cyc,
                   "relax_sweeps": sweeps, "all_converged": all(s.converged for s in sb),
                   "edges_cycles_per_s": a.m * sum(cyc) / block_s2,
                   "edges_sweeps_per_s": a.m * sum(sweeps) / block_s2 if sum(sweeps) else None}}
print(json.dumps(out), flush=True)
