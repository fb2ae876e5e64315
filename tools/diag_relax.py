"""Relaxation-coarsest diagnostics on a power-law graph (BASELINE config 5 shape
at a reduced R-MAT scale): level structure, colour count, row-length
distribution of the relaxation level, single and 32-column solve times.

usage: python tools/diag_relax.py [scale] [--profile]   (--profile: brackets one
       block solve with cudaProfilerStart/Stop for an ncu launch list)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 22
chung = "--chunglu" in sys.argv  # config 4 shape (Chung-Lu, beta 2.1) at 2^scale nodes
prof = "--profile" in sys.argv
ctx = L.Context(0, L.MODE_THROUGHPUT)
t = time.time()
a = G.chung_lu(1 << scale, seed=4) if chung else L.gen_rmat(scale, seed=5, ctx=ctx)
torch.cuda.synchronize()
print(f"{'chunglu' if chung else 'rmat'}{scale}: n={a.n} m={a.m} gen {time.time() - t:.2f}s", flush=True)
t = time.time()
h = L.setup(a, ctx=ctx)
torch.cuda.synchronize()
ts = time.time() - t
t = time.time()
L._check(ctx.lib.lamg_hier_prepare_throughput(ctx.p, h.h))
torch.cuda.synchronize()
tp = time.time() - t
h.levels = [h.level_info(l) for l in range(h.nlevels)]
print(f"setup {ts:.2f}s prepare {tp:.2f}s levels "
      f"{[(li.kind, li.n, li.m, li.colors, li.coarsest) for li in h.levels]}", flush=True)
for l, li in enumerate(h.levels):
    if li.coarsest != 2:
        continue
    op = h.op(l)
    deg = np.diff(op.row_ptr)
    q = np.percentile(deg, [50, 90, 99, 99.9, 100])
    heavy = deg[deg > 2048]
    print(f"level {l}: n={li.n} nnz={deg.sum()} deg p50/90/99/99.9/max {q.tolist()} "
          f"rows>64 {int((deg > 64).sum())} ({int(deg[deg > 64].sum())} entries) "
          f"rows>2048 {heavy.size} ({int(heavy.sum())} entries) colours {li.colors}", flush=True)
nrhs = 32
B = np.stack([G.gaussian_rhs(a.n, 500 + j) for j in range(nrhs)])
for _ in range(2):
    B -= (B.sum(axis=1) / a.n)[:, None]
X0 = np.stack([G.default_x0(a.n, seed=1 + j) for j in range(nrhs)])


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.time()
    r = fn()
    torch.cuda.synchronize()
    return r, time.time() - t0


(x1, s1), t1 = timed(lambda: L.solve(h, B[0], X0[0], ctx=ctx))
(x1, s1), t1 = timed(lambda: L.solve(h, B[0], X0[0], ctx=ctx))
print(f"single: {t1:.3f}s cycles {s1.cycles} sweeps {s1.relax_sweeps} conv {s1.converged}", flush=True)
(xb, sb), tb = timed(lambda: L.solve_batch(h, B, X0, ctx=ctx))
if prof:
    torch.cuda.profiler.start()
(xb, sb), tb = timed(lambda: L.solve_batch(h, B, X0, ctx=ctx))
if prof:
    torch.cuda.profiler.stop()
sw = [s.relax_sweeps for s in sb]
print(f"block32: {tb:.3f}s cycles {[s.cycles for s in sb][:4]} sweeps max {max(sw)} "
      f"conv {all(s.converged for s in sb)}", flush=True)
