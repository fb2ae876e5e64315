"""Memory-safety workload. compute-sanitizer is closed on the GPU pool, so the
library's own guard mode stands in: LAMG_GUARD=1 puts 256-byte pattern bands
around every device buffer and checks them at release (LAMG_POISON=1 also
fills fresh floating-point buffers with NaN, so reads of never-written memory
surface in the compared results). Where compute-sanitizer is available the
same script is the workload for --tool memcheck / racecheck / synccheck.

    LAMG_GUARD=1 LAMG_POISON=1 python tools/sanitize_workload.py

The workload: the smoke solve, one power-law THROUGHPUT solve (relaxation
coarsest with chunked hub rows and acq_rel chunk counters, two contexts
sharing the hierarchy), and one 32-column THROUGHPUT block (bgs_exact tickets,
the node-major cluster tail).

    compute-sanitizer --tool memcheck python tools/sanitize_workload.py
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

__graft_entry__.smoke()

a = G.largest_component(G.chung_lu(1 << 12, seed=4))[0]
ctx = L.Context(0, L.MODE_THROUGHPUT)
h = L.setup(a, ctx=ctx)
b, x0 = G.gaussian_rhs(a.n, 3), G.default_x0(a.n)
x1, s1 = L.solve(h, b, x0, ctx=ctx)
c2 = L.Context(0, L.MODE_THROUGHPUT)
out = {}
ths = [threading.Thread(target=lambda c, k: out.__setitem__(k, L.solve(h, b, x0, ctx=c)), args=(c, k))
       for k, c in enumerate((ctx, c2))]
for t in ths:
    t.start()
for t in ths:
    t.join()
assert all(np.array_equal(out[k][0], x1) for k in out)
print(f"power-law THROUGHPUT solve: n={a.n} cycles={s1.cycles} relax_sweeps={s1.relax_sweeps}")

g = G.grid3d_7pt(16)
hg = L.setup(g, ctx=ctx)
B = np.stack([G.gaussian_rhs(g.n, 40 + j) for j in range(32)])
X0 = np.stack([G.default_x0(g.n, seed=1 + j) for j in range(32)])
X, st = L.solve_batch(hg, B, X0, ctx=ctx)
assert all(s.converged for s in st)
print(f"32-column block: n={g.n} cycles={st[0].cycles}..{max(s.cycles for s in st)}")
c2.close()
ctx.close()
del h, hg
import ctypes as C  # noqa: E402
import gc  # noqa: E402

gc.collect()
chk, ovr = C.c_int64(), C.c_int64()
L._lib.lib().lamg_guard_report(C.byref(chk), C.byref(ovr))
print(f"guard bands: {chk.value} buffers checked, {ovr.value} overruns"
      + ("" if os.environ.get("LAMG_GUARD") == "1" else " (LAMG_GUARD not set: nothing checked)"))
assert ovr.value == 0
print("sanitize workload ok")
