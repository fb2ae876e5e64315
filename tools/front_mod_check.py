"""Per-column cycle counts of a K-column block solve with the front-modulo
colouring (default) against the exact-order block sweep (LAMG_FRONT_MOD=0),
each in its own process (the setting is read once).

    python tools/front_mod_check.py [cfg|gN] [nrhs] [C]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys
sys.path.insert(0, %r)
import numpy as np
from paper_1108_1310_b200 import graphs as G, lamg as L
cfg, nrhs = sys.argv[1], int(sys.argv[2])
a = G.grid3d_7pt(int(cfg[1:])) if cfg.startswith("g") else G.make_config(int(cfg))
B = G.zero_sum(np.stack([G.gaussian_rhs(a.n, 1000 + j) for j in range(nrhs)]))
X0 = np.stack([G.default_x0(a.n, seed=1 + j) for j in range(nrhs)])
ctx = L.Context(0, L.MODE_THROUGHPUT)
h = L.setup(a, ctx=ctx)
X, st = L.solve_batch(h, B, X0, ctx=ctx)
print(json.dumps({"cycles": [s.cycles for s in st], "norm": [float(np.linalg.norm(x)) for x in X],
                  "x0": X[0][:: max(1, a.n // 64)].tolist()}))
''' % ROOT


def run(mod, cfg, nrhs):
    env = dict(os.environ, LAMG_FRONT_MOD=str(mod))
    p = subprocess.run([sys.executable, "-c", CHILD, cfg, str(nrhs)], env=env, capture_output=True, text=True,
                       timeout=1200)
    if p.returncode:
        raise RuntimeError(p.stderr[-2000:])
    return json.loads(p.stdout.strip().split("\n")[-1])


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
    nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    C = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    ex, fm = run(0, cfg, nrhs), run(C, cfg, nrhs)
    d = [a - b for a, b in zip(fm["cycles"], ex["cycles"])]
    print(f"config {cfg}, {nrhs} right-hand sides")
    print("exact-order block sweep :", ex["cycles"])
    print(f"front-modulo, C = {C:<6}:", fm["cycles"])
    print("difference per column   :", d, " max |diff| =", max(abs(v) for v in d))
    rel = max(abs(a - b) / b for a, b in zip(fm["norm"], ex["norm"]))
    print(f"max relative difference of ||x|| per column: {rel:.3e}")


if __name__ == "__main__":
    main()
