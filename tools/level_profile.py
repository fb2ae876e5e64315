"""Per-level time breakdown of one THROUGHPUT solve (lamg_ctx_profile
classes 2 + 4 l + {gs, residual, transfers, tail}); CUDA events around
each kernel group, graphs off.

    python tools/level_profile.py [cfg] [K]     (K = 1: one-column solve)
LANES=n runs n profiled block solves concurrently (one context each, the
bench's arrangement) and prints lane 0's table: how much each group stretches
under contention.
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402
from xb_time import config  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    a = config(cfg)
    validate = os.environ.get("MODE", "throughput") == "validate"  # MODE=validate: the exact-order solve (K = 1)
    ctx = L.Context(0, L.MODE_VALIDATE if validate else L.MODE_THROUGHPUT)
    h = L.setup(a, ctx=ctx)
    if not validate:
        h.prepare_throughput()
    B = np.stack([G.gaussian_rhs(a.n, 100 + cfg + 7 * i) for i in range(K)])
    X0 = np.stack([G.default_x0(a.n, seed=1 + 97 * i) for i in range(K)])
    lib = ctx.lib
    lanes = int(os.environ.get("LANES", "1"))
    mc = int(os.environ.get("MAX_CYCLES", "300"))
    others = [L.Context(0, L.MODE_THROUGHPUT) for _ in range(lanes - 1)]
    for c in [ctx] + others:
        lib.lamg_ctx_profile(c.p, 1)
    import threading
    ths = [threading.Thread(target=lambda c=c: L.solve_batch(h, B, X0, L.CycleConfig(max_cycles=mc), ctx=c))
           for c in others]
    t = time.time()
    [th.start() for th in ths]
    if K == 1:
        x, st = L.solve(h, B[0], X0[0], L.CycleConfig(max_cycles=mc), ctx=ctx)
        cyc = st.cycles
    else:
        X, st = L.solve_batch(h, B, X0, L.CycleConfig(max_cycles=mc), ctx=ctx)
        cyc = max(s.cycles for s in st)
    [th.join() for th in ths]
    wall = time.time() - t
    rows = []
    tot = 0.0
    for l in range(h.nlevels):
        r = [l, h.levels[l].n]
        for k in range(4):
            nl, tm, by = C.c_int64(), C.c_double(), C.c_double()
            lib.lamg_ctx_profile_read(ctx.p, C.c_int(2 + 4 * l + k), C.byref(nl), C.byref(tm), C.byref(by))
            gbs = by.value * nl.value / (tm.value / 1e3) / 1e9 if tm.value > 0 and by.value > 0 else 0.0
            r += [nl.value, tm.value, gbs]
            tot += tm.value
        rows.append(r)
    lib.lamg_ctx_profile(ctx.p, 0)
    print(f"cfg {cfg} K {K}: {cyc} cycles, wall {wall:.2f}s (profiled), sum of groups {tot:.0f} ms "
          f"= {tot / cyc:.2f} ms/cycle")
    print(f"{'lvl':>3} {'n':>8} | {'gs n':>6} {'gs ms':>8} {'GB/s':>6} | {'res n':>6} {'res ms':>7} {'GB/s':>6} | "
          f"{'xfer n':>6} {'xfer ms':>7} | {'tail n':>6} {'tail ms':>8} | ms/cycle")
    for r in rows:
        l, n, gn, gt, gg, rn, rt, rg, xn, xt, _, tn, tt, _ = r
        s = gt + rt + xt + tt
        if s == 0:
            continue
        print(f"{l:>3} {n:>8} | {gn:>6} {gt:>8.1f} {gg:>6.0f} | {rn:>6} {rt:>7.1f} {rg:>6.0f} | {xn:>6} {xt:>7.1f} | "
              f"{tn:>6} {tt:>8.1f} | {s / cyc:8.3f}")


if __name__ == "__main__":
    main()
