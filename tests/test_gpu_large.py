"""Size-independent parity at BASELINE.json scale (GPU).

tests/golden/large.json holds SHA-256 digests of every hierarchy artefact and
of the solution computed by the unmodified reference (make_golden_large.py).
The GPU setup must reproduce every digest (bit-exact hierarchy), and the
VALIDATE-mode solve must reproduce the cycle count, the residual history and
the solution digest. THROUGHPUT-mode solves -- one column and a 4-column
block -- must converge to the same tolerance in the reference's cycle count
+-1 with x within 1e-8 relative of the reference (north_star's solve rule).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_1108_1310_b200 import graphs as G

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "large.json")
CASES = {
    "cfg1_grid5_256": lambda: G.make_config(1),
    "cfg2s_grid3d_64": lambda: G.grid3d_7pt(64),
    "cfg3s_rgg_256k": lambda: G.rgg(1 << 18, seed=3),
    "cfg4s_chunglu_256k": lambda: G.chung_lu(1 << 18, seed=4),
    "cfg5s_rmat_16": lambda: G.rmat(16, seed=5),
    "cfg2_grid3d_128": lambda: G.make_config(2),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


@pytest.mark.parametrize("name", list(CASES))
def test_large_config_matches_reference_digests(name):
    from paper_1108_1310_b200 import lamg as L
    g = json.load(open(GOLD))[name]
    a = CASES[name]()
    assert {k: sha(getattr(a, k)) for k in ("row_ptr", "col", "val", "diag")} == g["input_sha"]
    b = G.gaussian_rhs(a.n, g["rhs_seed"])
    x0 = G.default_x0(a.n)
    assert sha(b) == g["b_sha"] and sha(x0) == g["x0_sha"]
    ctx = L.Context(0, L.MODE_VALIDATE)
    h = L.setup(a, ctx=ctx)
    e = h.export()
    got = {k: sha(v) for k, v in e.items()}
    bad = [k for k, v in g["hier_sha"].items() if got.get(k) != v]
    assert not bad, bad[:10]
    x, st = L.solve(h, b, x0, ctx=ctx)
    assert st.cycles == g["cycles"]
    assert np.array_equal(np.array(st.residuals), np.array(g["residuals"]))
    assert sha(x) == g["x_sha"]
    # THROUGHPUT (north_star's solve rule): converged to 1e-10 in the
    # reference's cycle count +-1, ||x - x_ref|| / ||x_ref|| <= 1e-8 -- one
    # column, and column 0 of a 4-column block (the benchmarked path: the
    # finest smoothing level swept in exact order by bgs_exact)
    ctx.set_mode(L.MODE_THROUGHPUT)
    xt, stt = L.solve(h, b, x0, ctx=ctx)
    assert stt.converged and stt.residuals[-1] <= stt.residuals[0] / 1e10
    assert abs(stt.cycles - g["cycles"]) <= 1, (stt.cycles, g["cycles"])
    assert np.linalg.norm(xt - x) / np.linalg.norm(x) <= 1e-8
    B = np.stack([b] + [G.gaussian_rhs(a.n, 900 + j) for j in range(3)])
    X0 = np.stack([x0] * 4)
    XB, sb = L.solve_batch(h, B, X0, ctx=ctx)
    assert sb[0].converged and sb[0].residuals[-1] <= sb[0].residuals[0] / 1e10
    assert abs(sb[0].cycles - g["cycles"]) <= 1, (sb[0].cycles, g["cycles"])
    assert np.linalg.norm(XB[0] - x) / np.linalg.norm(x) <= 1e-8
    ctx.close()


# ---------------------------------------------------------------------------
# BASELINE.json configs 3-5 at full size (config 5 at 1/8 size: the reference
# run of R-MAT 25 needs more host memory than the build box has). Configs 4/5
# are generated on the device and their digests checked against the host
# restatement the reference consumed.
FULL = {
    "cfg3_rgg_4M": dict(host=lambda: G.make_config(3), zero_sum=True, validate=True),
    "cfg4_chunglu_16M": dict(dev=lambda L, ctx: L.gen_chung_lu(1 << 24, seed=4, ctx=ctx), zero_sum=True,
                             validate=False),
    "cfg5m_rmat_22": dict(dev=lambda L, ctx: L.gen_rmat(22, seed=5, ctx=ctx), zero_sum=True, validate=False),
}


@pytest.mark.parametrize("name", list(FULL))
def test_full_scale_config_matches_reference(name):
    """Hierarchy digests (every operator, aggregate map and elimination stage
    of every level) equal the unmodified reference's at BASELINE size; the
    VALIDATE solve is bit-identical where it is run (LAMG_TEST_VALIDATE_BIG=1
    forces it on the power-law configs, whose exact-order sweeps over 8M-row
    hub levels take minutes); the THROUGHPUT solve meets north_star's rule
    (cycle count +-1, x within 1e-8) against the reference's solution."""
    from paper_1108_1310_b200 import lamg as L
    gold = json.load(open(GOLD))
    if name not in gold:
        pytest.skip(f"{name}: no reference digests in large.json")
    g, spec = gold[name], FULL[name]
    ctx = L.Context(0, L.MODE_VALIDATE)
    a = spec["dev"](L, ctx) if "dev" in spec else spec["host"]()
    ha = a.download() if hasattr(a, "download") else a
    assert (ha.n, ha.m) == (g["n"], g["m"])
    assert {k: sha(getattr(ha, k)) for k in ("row_ptr", "col", "val", "diag")} == g["input_sha"]
    b = G.gaussian_rhs(ha.n, g["rhs_seed"])
    if spec.get("zero_sum"):
        b = G.zero_sum(b[None])[0]
    x0 = G.default_x0(ha.n)
    assert sha(b) == g["b_sha"] and sha(x0) == g["x0_sha"]
    del ha
    h = L.setup(a, ctx=ctx)
    assert h.nlevels == g["nlevels"]
    for l, want in enumerate(g["levels"]):
        li = h.level_info(l)
        assert (li.kind, li.n, li.m) == (want["kind"], want["n"], want["m"]), l
    e = h.export()
    got = {k: sha(v) for k, v in e.items()}
    del e
    bad = [k for k, v in g["hier_sha"].items() if got.get(k) != v]
    assert not bad, bad[:10]
    xref = None
    if spec["validate"] or os.environ.get("LAMG_TEST_VALIDATE_BIG") == "1":
        xref, st = L.solve(h, b, x0, ctx=ctx)
        assert st.cycles == g["cycles"]
        assert np.array_equal(np.array(st.residuals), np.array(g["residuals"]))
        assert sha(xref) == g["x_sha"]
    ctx.set_mode(L.MODE_THROUGHPUT)
    xt, stt = L.solve(h, b, x0, ctx=ctx)
    assert stt.converged and stt.residuals[-1] <= stt.residuals[0] / 1e10
    assert abs(stt.cycles - g["cycles"]) <= 1, (stt.cycles, g["cycles"])
    B = np.stack([b] + [G.gaussian_rhs(len(b), 900 + j) for j in range(3)])
    if spec.get("zero_sum"):
        B = G.zero_sum(B)
    XB, sb = L.solve_batch(h, B, np.stack([x0] * 4), ctx=ctx)
    assert sb[0].converged and abs(sb[0].cycles - g["cycles"]) <= 1, (sb[0].cycles, g["cycles"])
    for x in (xt, XB[0]):
        if xref is not None:
            assert np.linalg.norm(x - xref) / np.linalg.norm(xref) <= 1e-8
        else:
            assert abs(np.linalg.norm(x) - g["x_norm"]) / g["x_norm"] <= 1e-8
            if "x_sample" in g:  # every stride-th entry of the reference's x
                xs = np.array(g["x_sample"])
                d = x[::g["x_sample_stride"]] - xs
                assert np.linalg.norm(d) / np.linalg.norm(xs) <= 1e-8
    ctx.close()
