"""Checksum fixtures of the REFERENCE at BASELINE.json scale.

Runs the unmodified reference (oracle/_ref) on the configuration inputs built
by paper_1108_1310_b200/graphs.py and stores, per configuration, the SHA-256 of
every hierarchy artefact (all level operators, aggregate maps, elimination
stages), the solve's cycle count and residual history, and the SHA-256 of the
solution -- a size-independent "checksum of checksums" the GPU test compares
against without needing the reference on the GPU box.

    python tests/golden/make_golden_large.py [names...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Oracle  # noqa: E402
from paper_1108_1310_b200 import graphs as G  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "large.json")

# name -> (builder, rhs seed)
CASES = {
    "cfg1_grid5_256": (lambda: G.make_config(1), 101),
    "cfg2_grid3d_128": (lambda: G.make_config(2), 102),
    "cfg2s_grid3d_64": (lambda: G.grid3d_7pt(64), 102),
    "cfg3s_rgg_256k": (lambda: G.rgg(1 << 18, seed=3), 103),
    "cfg4s_chunglu_256k": (lambda: G.chung_lu(1 << 18, seed=4), 104),
    "cfg5s_rmat_16": (lambda: G.rmat(16, seed=5), 105),
    # full BASELINE.json sizes (configs 3-5; the GPU tests generate 4 and 5 on
    # the device and check the input digests against these)
    "cfg3_rgg_4M": (lambda: G.make_config(3), 103),
    "cfg4_chunglu_16M": (lambda: G.make_config(4), 104),
    "cfg5_rmat_25": (lambda: G.make_config(5), 105),
    # config 5 at 1/8 size (the full R-MAT 25 reference run needs more host
    # memory than the build box has): hubs of ~10^5 entries
    "cfg5m_rmat_22": (lambda: G.rmat(22, seed=5), 105),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def digest_export(d: dict) -> dict:
    return {k: sha(v) for k, v in sorted(d.items())}


def main(names):
    ref = Oracle("ref")
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names or list(CASES):
        build, seed = CASES[name]
        a = build()
        b = G.gaussian_rhs(a.n, seed)
        if name in ("cfg3_rgg_4M", "cfg4_chunglu_16M", "cfg5_rmat_25", "cfg5m_rmat_22"):
            b = G.zero_sum(b[None])[0]  # as bench.py does for the full-size configs 3-5
        x0 = G.default_x0(a.n)
        t0 = time.time()
        h = ref.setup(a)
        t1 = time.time()
        x, st = h.solve(b, x0)
        t2 = time.time()
        e = h.export()
        data[name] = {
            "n": a.n, "m": a.m, "rhs_seed": seed,
            "input_sha": {k: sha(getattr(a, k)) for k in ("row_ptr", "col", "val", "diag")},
            "b_sha": sha(b), "x0_sha": sha(x0),
            "nlevels": int(e["nlevels"][0]),
            "levels": [{"kind": int(e[f"L{l}.kind"][0]), "n": int(e[f"L{l}.n"][0]), "m": int(e[f"L{l}.m"][0])}
                       for l in range(int(e["nlevels"][0]))],
            "hier_sha": digest_export(e),
            "cycles": int(st["cycles"][0]), "residuals": [float(r) for r in st["residuals"]],
            "acf": float(st["acf"][0]), "solve_work": float(st["solve_work"][0]),
            "x_sha": sha(x), "x_norm": float(np.linalg.norm(x)),
            # every stride-th entry of x: lets a THROUGHPUT solve be compared with the
            # reference's solution where a VALIDATE solve is too slow to produce it
            "x_sample_stride": max(1, a.n // 4096), "x_sample": [float(v) for v in x[::max(1, a.n // 4096)]],
            "ref_setup_s": t1 - t0, "ref_solve_s": t2 - t1,
        }
        print(f"{name}: n={a.n} m={a.m} levels={data[name]['nlevels']} cycles={data[name]['cycles']} "
              f"setup {t1 - t0:.1f}s solve {t2 - t1:.1f}s", flush=True)
        json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
