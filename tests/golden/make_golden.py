"""Generates the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists) after `make -C oracle`:

    python tests/golden/make_golden.py

Every array in the fixtures is produced by oracle/_ref/liblamg_ref.so, i.e. the
unmodified reference core (/root/reference/proj/core/src) compiled by
oracle/Makefile. Inputs are built with paper_1108_1310_b200/graphs.py, whose
generators are themselves pinned against the reference generators by
tests/test_oracle_pin.py. The fixtures travel with the repo so the GPU box
(which has no /root/reference) can check the CUDA path against reference
outputs directly.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Oracle  # noqa: E402
from paper_1108_1310_b200 import graphs as G  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, builder, solve-config overrides)
CASES = [
    ("grid5_32", lambda: G.grid_5pt(32), {}),
    ("grid5_64", lambda: G.grid_5pt(64), {}),
    ("grid3d_12w", lambda: G.grid3d_7pt(12), {}),
    ("grid13_24", lambda: G.grid_13pt_4th(24), {}),
    ("anis_ne_32", lambda: G.grid_anis_rotated(32, 0.7853981633974483, 0.01, True), {}),
    ("rc_300", lambda: G.random_connected(300, 1.5, 7), {}),
    ("rc_2000", lambda: G.random_connected(2000, 2.0, 2), {}),
    ("path_1000", lambda: G.path(1000), {}),
    ("tree_500", lambda: G.binary_tree(500), {}),
    ("two_hubs_80", lambda: G.two_hubs(80), {}),
    ("complete_200", lambda: G.complete(200), {}),
    ("rgg_4k", lambda: G.rgg(4096, seed=3), {}),
    ("chunglu_4k", lambda: G.chung_lu(4096, seed=4), {}),
    ("rmat_11", lambda: G.rmat(11, seed=5), {}),
    ("grid5_48_adaptive", lambda: G.grid_5pt(48), {"correction": 1}),
]


def put(d, prefix, bag):
    for k, v in bag.items():
        d[prefix + k] = v


def csr_dict(a):
    return {"A.n": np.array([a.n], np.int32), "A.m": np.array([a.m], np.int64), "A.row_ptr": a.row_ptr,
            "A.col": a.col, "A.val": a.val, "A.diag": a.diag}


def main():
    ref = Oracle("ref")
    for name, build, cyc in CASES:
        a = build()
        d = csr_dict(a)
        # kernel-level vectors on the finest level
        x = G.random_vector(a.n, 101)
        b = G.gaussian_rhs(a.n, 102)
        d["K.x"], d["K.b"] = x, b
        d["K.residual"] = ref.residual(a, b, x)
        d["K.mvm"] = ref.mvm(a, x)
        d["K.energy"] = np.array([ref.energy(a, x)])
        d["K.gs_fwd"] = ref.gs_sweep(a, b, x)
        d["K.gs_bwd"] = ref.gs_sweep(a, b, x, backward=True)
        d["K.gs_homog"] = ref.gs_sweep(a, None, x)
        d["K.probe"] = np.array([ref.probe(a, 8, 77)])
        tvs = ref.generate_tvs(a, 4, 3, 1234)
        d["K.tvs"] = tvs
        put(d, "K.aff.", ref.affinities(a, tvs))
        d["K.hubs"] = ref.detect_hubs(a)
        put(d, "K.agg.", ref.aggregate(a, tvs, 1.5, d["K.hubs"]))
        f, c = ref.select_low_degree(a)
        d["K.sel.f"], d["K.sel.c"] = f, c
        put(d, "K.elim.", ref.eliminate_rounds(a))
        # whole setup + solve with the reference's default configuration
        h = ref.setup(a)
        put(d, "H.", h.export())
        x0 = G.default_x0(a.n)
        d["S.b"], d["S.x0"] = b, x0
        xs, stats = h.solve(b, x0, **cyc)
        d["S.x"] = xs
        d["S.correction"] = np.array([cyc.get("correction", 0)], np.int32)
        put(d, "S.", stats)
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **d)
        print(f"{name}: n={a.n} m={a.m} levels={int(d['H.nlevels'][0])} cycles={int(stats['cycles'][0])} "
              f"{os.path.getsize(path) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
