"""Timing of one 32-column THROUGHPUT block solve on config 2: cycles, solve
time and the finest-level sweep/residual launch times (lamg_ctx_profile CUDA
events). The input is cached in /tmp between runs on one box.

    python tools/xb_time.py [cfg] [K] [lanes]
"""
import ctypes as C
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402


def config(cfg):
    p = f"/tmp/lamg_cfg{cfg}.npz"
    if os.path.exists(p):
        z = np.load(p)
        return G.SparseLaplacian(int(z["n"]), int(z["m"]), z["row_ptr"], z["col"], z["val"], z["diag"])
    a = G.make_config(cfg)
    np.savez(p, n=a.n, m=a.m, row_ptr=a.row_ptr, col=a.col, val=a.val, diag=a.diag)
    return a


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    lanes = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    a = config(cfg)
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    h = L.setup(a, ctx=ctx)
    h.prepare_throughput()
    B = np.stack([G.gaussian_rhs(a.n, 100 + cfg + 7 * i) for i in range(K)])
    X0 = np.stack([G.default_x0(a.n, seed=1 + 97 * i) for i in range(K)])
    lib = ctx.lib
    # profiled solve: finest-level launch times
    lib.lamg_ctx_profile(ctx.p, 1)
    t = time.time()
    X, st = L.solve_batch(h, B, X0, ctx=ctx)
    tp = time.time() - t
    out = {"cycles0": st[0].cycles, "cycles_mean": float(np.mean([s.cycles for s in st]))}
    for k, name in ((0, "gs"), (1, "res")):
        nl, tm, by = C.c_int64(), C.c_double(), C.c_double()
        lib.lamg_ctx_profile_read(ctx.p, C.c_int(k), C.byref(nl), C.byref(tm), C.byref(by))
        if nl.value:
            avg = tm.value / nl.value
            out[name] = {"n": nl.value, "avg_ms": round(avg, 4), "gbs": round(by.value / (avg / 1e3) / 1e9, 1)}
    lib.lamg_ctx_profile(ctx.p, 0)
    L.solve_batch(h, B, X0, ctx=ctx)  # graphs captured
    torch.cuda.synchronize()
    t = time.time()
    L.solve_batch(h, B, X0, ctx=ctx)
    out["block_solve_s"] = round(time.time() - t, 3)
    out["profiled_solve_s"] = round(tp, 3)
    if lanes > 1:
        ctxs = [L.Context(0, L.MODE_THROUGHPUT) for _ in range(lanes)]
        for c in ctxs:
            L.solve_batch(h, B, X0, ctx=c)
        torch.cuda.synchronize()
        t = time.time()
        th = [threading.Thread(target=L.solve_batch, args=(h, B, X0), kwargs={"ctx": c}) for c in ctxs]
        for x in th:
            x.start()
        for x in th:
            x.join()
        out[f"{lanes}_lanes_s"] = round(time.time() - t, 3)
    env = {k: v for k, v in os.environ.items() if k.startswith("LAMG_")}
    print(env, out, flush=True)


if __name__ == "__main__":
    main()
