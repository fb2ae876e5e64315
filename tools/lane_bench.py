"""Concurrent K-column block solves with device-resident inputs (CUDA-event
timing, bounded cycles): ms per block cycle alone and with N lanes in flight.

    python tools/lane_bench.py [cfg] [block] [lanes] [max_cycles]
Environment knobs of the block tail apply (LAMG_BATCH_TAIL=slice|cluster|subtree,
LAMG_BATCH_TAIL_ROWS, LAMG_BATCH_CTAS, ...).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    KB = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    NL = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    mc = int(sys.argv[4]) if len(sys.argv) > 4 else 12
    ctx0 = L.Context(0, L.MODE_THROUGHPUT)
    a = bench.build_operator(cfg, ctx0)
    h = L.setup(a, ctx=ctx0)
    L._check(ctx0.lib.lamg_hier_prepare_throughput(ctx0.p, h.h))
    # one block of right-hand sides, shared by the lanes (each lane has its own device copy)
    B = np.stack([G.gaussian_rhs(a.n, 100 + cfg + 7 * i) for i in range(KB)])
    X0 = np.stack([G.default_x0(a.n, seed=1 + 97 * i) for i in range(KB)])
    if cfg >= 4:
        B = G.zero_sum(B)
    lanes = [bench.Lane(L, torch, 0, h, L.MODE_THROUGHPUT, B, X0) for _ in range(NL)]
    for ln in lanes:
        ln.cfg.max_cycles = mc
        if "LAMG_EXACT_LEVELS" in os.environ:  # 0: every level coloured
            ln.ctx.set_exact_levels(int(os.environ["LAMG_EXACT_LEVELS"]))
    s0 = lanes[0].stream
    out = []
    for n in sorted({1, NL}):
        sub = lanes[:n]
        bench.run_lanes(sub, bench.Lane.solve_dev, torch, s0)
        ms, cyc = bench.run_lanes(sub, bench.Lane.solve_dev, torch, s0)
        out.append(f"{n} lanes: {ms / max(cyc):8.2f} ms per block cycle, {a.m * sum(cyc) / ms * 1e3:.3e} edges*cycles/s")
    print(f"cfg {cfg} block {KB} cycles {mc}: " + "; ".join(out), flush=True)
    for ln in lanes:
        ln.ctx.close()


if __name__ == "__main__":
    main()
