"""Fine-level node-block partition with halo exchange (SURVEY.md 8(e) mode 2).

CPU (no GPU): the host partition plan of liblamg_b200.so -- bounds cover
[0, n) in balanced contiguous blocks, the local CSR maps back to the global
rows entry for entry, every part's send list to q is exactly q's ghosts from
it (same order), and a residual computed block by block from owned values
plus exchanged ghosts equals the global residual. The exchange runs once in
process and once between two gloo ranks (the N>1 path of the NCCL transport).

GPU: the partitioned coloured sweep and residual (in-process transport, all
parts on one device) are bit-identical to the single-part ones for 2-4 parts
(the single-part residual is checked against scipy), and the NCCL transport
builds a communicator and sweeps on one rank.
"""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

from paper_1108_1310_b200 import graphs as G

GRAPHS = {
    "grid5_24": lambda: G.grid_5pt(24),
    "grid3d_12": lambda: G.grid3d_7pt(12),
    "rgg_4k": lambda: G.rgg(1 << 12, seed=3),
    "rmat_11": lambda: G.rmat(11, seed=5),
}


def _residual(a, b, x):
    A = sp.csr_matrix((a.val, a.col, a.row_ptr), shape=(a.n, a.n))
    return b - (a.diag * x + A @ x)


def _local_residual(a, d, b, xfull_owned, ghosts):
    lo, hi = d["lo"], d["hi"]
    nloc = hi - lo
    xl = np.concatenate([xfull_owned, ghosts])
    val = a.val[a.row_ptr[lo]:a.row_ptr[hi]]
    A = sp.csr_matrix((val, d["col"], d["row_ptr"]), shape=(nloc, nloc + len(d["ghost_gid"])))
    return b[lo:hi] - (a.diag[lo:hi] * xl[:nloc] + A @ xl)


@pytest.mark.parametrize("P", [1, 2, 3, 5])
@pytest.mark.parametrize("name", list(GRAPHS))
def test_plan_invariants_and_exchange(name, P):
    from paper_1108_1310_b200 import lamg as L
    a = GRAPHS[name]()
    bounds = L.part_bounds(a, P)
    assert bounds[0] == 0 and bounds[-1] == a.n and np.all(np.diff(bounds) >= 0)
    cost = np.diff(a.row_ptr) + 1
    per = [cost[bounds[p]:bounds[p + 1]].sum() for p in range(P)]
    assert max(per) <= cost.sum() / P + cost.max() + 1
    plans = [L.part_plan(a, bounds, p) for p in range(P)]
    for p, d in enumerate(plans):
        lo, hi = d["lo"], d["hi"]
        nloc = hi - lo
        gid = np.concatenate([np.arange(lo, hi), d["ghost_gid"]]).astype(np.int64)
        assert np.array_equal(gid[d["col"]], a.col[a.row_ptr[lo]:a.row_ptr[hi]])
        assert np.array_equal(d["row_ptr"], a.row_ptr[lo:hi + 1] - a.row_ptr[lo])
        assert np.all(np.diff(d["ghost_gid"]) > 0)
        assert not np.any((d["ghost_gid"] >= lo) & (d["ghost_gid"] < hi))
        for q in range(P):
            ghosts_from_q = d["ghost_gid"][d["recv_ptr"][q]:d["recv_ptr"][q + 1]]
            assert np.all((ghosts_from_q >= bounds[q]) & (ghosts_from_q < bounds[q + 1]))
            e = plans[q]
            sent = e["send_idx"][e["send_ptr"][p]:e["send_ptr"][p + 1]] + e["lo"]
            assert np.array_equal(sent, ghosts_from_q), (p, q)
        assert d["send_ptr"][p + 1] == d["send_ptr"][p] and d["recv_ptr"][p + 1] == d["recv_ptr"][p]
    rng = np.random.default_rng(5)
    b, x = rng.standard_normal(a.n), rng.standard_normal(a.n)
    want = _residual(a, b, x)
    got = np.empty(a.n)
    for p, d in enumerate(plans):
        ghosts = np.empty(len(d["ghost_gid"]))
        for q in range(P):  # exchange: q's send list lands in p's ghost range
            e = plans[q]
            ghosts[d["recv_ptr"][q]:d["recv_ptr"][q + 1]] = x[e["lo"] + e["send_idx"][e["send_ptr"][p]:e["send_ptr"][p + 1]]]
        got[d["lo"]:d["hi"]] = _local_residual(a, d, b, x[d["lo"]:d["hi"]], ghosts)
    assert np.allclose(got, want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_1108_1310_b200 import graphs as G2
    from paper_1108_1310_b200 import lamg as L
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = G2.rmat(10, seed=5)
    bounds = L.part_bounds(a, world)
    d = L.part_plan(a, bounds, rank)
    rng = np.random.default_rng(9)
    b, x = rng.standard_normal(a.n), rng.standard_normal(a.n)
    own = x[d["lo"]:d["hi"]]  # a rank knows only its own rows
    ghosts = torch.zeros(len(d["ghost_gid"]), dtype=torch.float64)
    ops = []
    for peer in range(world):
        if peer == rank:
            continue
        s0, s1 = d["send_ptr"][peer], d["send_ptr"][peer + 1]
        r0, r1 = d["recv_ptr"][peer], d["recv_ptr"][peer + 1]
        if s1 > s0:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(own[d["send_idx"][s0:s1]].copy()), peer))
        if r1 > r0:
            buf = torch.zeros(r1 - r0, dtype=torch.float64)
            ops.append((dist.P2POp(dist.irecv, buf, peer), r0, r1, buf))
    reqs = dist.batch_isend_irecv([o if isinstance(o, dist.P2POp) else o[0] for o in ops])
    for r in reqs:
        r.wait()
    for o in ops:
        if not isinstance(o, dist.P2POp):
            ghosts[o[1]:o[2]] = o[3]
    r_loc = _local_residual(a, d, b, own, ghosts.numpy())
    parts = [None] * world
    dist.all_gather_object(parts, (d["lo"], r_loc))
    if rank == 0:
        got = np.empty(a.n)
        for lo, rl in parts:
            got[lo:lo + len(rl)] = rl
        want = _residual(a, b, x)
        q.put(float(np.abs(got - want).max() / np.abs(want).max()))
    dist.destroy_process_group()


def test_two_rank_gloo_halo_exchange():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["grid3d_40", "rgg_64k", "rmat_15"])
def test_partitioned_sweep_bit_identical(name):
    from paper_1108_1310_b200 import lamg as L
    a = {"grid3d_40": lambda: G.grid3d_7pt(40), "rgg_64k": lambda: G.rgg(1 << 16, seed=3),
         "rmat_15": lambda: G.rmat(15, seed=5)}[name]()
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    rng = np.random.default_rng(3)
    b = rng.standard_normal(a.n)
    b -= b.mean()
    x = rng.standard_normal(a.n)
    one = L.PartLevel(a, 1, ctx=ctx)
    want_x = one.smooth(b, x, 2)
    want_r = one.residual(b, want_x)
    assert np.allclose(want_r, _residual(a, b, want_x), rtol=1e-12, atol=1e-12 * np.abs(want_r).max())
    for P in (2, 3, 4):
        pl = L.PartLevel(a, P, ctx=ctx)
        got_x = pl.smooth(b, x, 2)
        assert np.array_equal(got_x, want_x), (P, float(np.abs(got_x - want_x).max()))
        assert np.array_equal(pl.residual(b, want_x), want_r), P
        pl.close()
    one.close()
    ctx.close()


@pytest.mark.gpu
def test_nccl_transport_single_rank():
    """The NCCL transport on one rank (the multi-rank exchange needs more GPUs
    than this box has; its host side is the gloo test above): the library
    loads libnccl, builds a communicator and sweeps like the in-process form."""
    from paper_1108_1310_b200 import lamg as L
    a = G.grid3d_7pt(30)
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    rng = np.random.default_rng(4)
    b = rng.standard_normal(a.n)
    b -= b.mean()
    x = rng.standard_normal(a.n)
    want = L.PartLevel(a, 1, ctx=ctx).smooth(b, x, 2)
    comm = L.Comm(1, 0, L.Comm.unique_id(), ctx=ctx)
    pl = L.PartLevel(a, 1, ctx=ctx, comm=comm)
    assert np.array_equal(pl.smooth(b, x, 2), want)
    pl.close()
    # the partitioned solve over the NCCL transport (allgathers by ncclBroadcast)
    ctx.set_exact_levels(0)
    h = L.setup(a, ctx=ctx)
    bb, x0 = G.gaussian_rhs(a.n, 5), G.default_x0(a.n)
    x1, s1 = L.solve(h, bb, x0, ctx=ctx)
    ps = L.PartLevel.from_hierarchy(h, 1, comm=comm)
    xp, sp_ = ps.solve(h, bb, x0)
    assert sp_.cycles == s1.cycles and np.array_equal(xp, x1)
    ps.close()
    comm.close()
    ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["grid3d_48", "cfg2_128"])
def test_partitioned_solve_bit_identical(name):
    """lamg_part_solve: the finest level on 2-4 parts, coarse levels replicated
    -- the iterate, the residual history and the cycle count equal lamg_solve's
    bit for bit (THROUGHPUT), and the solve reaches the 1e-10 target."""
    from paper_1108_1310_b200 import lamg as L
    a = G.grid3d_7pt(48) if name == "grid3d_48" else G.make_config(2)
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    ctx.set_exact_levels(0)  # the partitioned finest level sweeps coloured
    h = L.setup(a, ctx=ctx)
    assert h.levels[1].kind == 2
    b, x0 = G.gaussian_rhs(a.n, 17), G.default_x0(a.n)
    x1, s1 = L.solve(h, b, x0, ctx=ctx)
    assert s1.converged and s1.residuals[-1] <= s1.residuals[0] / 1e10
    for P in ((2, 3) if name == "cfg2_128" else (1, 2, 4)):
        pl = L.PartLevel.from_hierarchy(h, P)
        xp, sp_ = pl.solve(h, b, x0)
        assert sp_.cycles == s1.cycles, P
        assert np.array_equal(np.array(sp_.residuals), np.array(s1.residuals)), P
        assert np.array_equal(xp, x1), P
        pl.close()
    ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["grid5_128", "rgg_64k"])
def test_partitioned_solve_below_a_finest_elimination(name):
    """Hierarchies whose finest level is reduced by elimination first (2D grids,
    geometric graphs: BASELINE configs 1 and 3): lamg_part_solve partitions
    level 1, the first level that smooths; the finest level's RHS coarsening,
    injection and back-substitution run replicated. Bit-identical to
    lamg_solve (exact_levels = 0) for 1-3 parts."""
    from paper_1108_1310_b200 import lamg as L
    a = G.grid_5pt(128) if name == "grid5_128" else G.largest_component(G.rgg(1 << 16, seed=3))[0]
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    ctx.set_exact_levels(0)
    h = L.setup(a, ctx=ctx)
    assert h.levels[1].kind == 1 and h.levels[2].kind == 2
    b, x0 = G.gaussian_rhs(a.n, 23), G.default_x0(a.n)
    x1, s1 = L.solve(h, b, x0, ctx=ctx)
    assert s1.converged and s1.residuals[-1] <= s1.residuals[0] / 1e10
    for P in (1, 2, 3):
        pl = L.PartLevel.from_hierarchy(h, P)
        assert pl.n == h.levels[1].n
        xp, sp_ = pl.solve(h, b, x0)
        assert sp_.cycles == s1.cycles, P
        assert np.array_equal(np.array(sp_.residuals), np.array(s1.residuals)), P
        assert np.array_equal(xp, x1), P
        pl.close()
    ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["chunglu_64k", "rmat_14"])
def test_partitioned_relaxation_coarsest(name):
    """Configs 4 and 5 in small: finest -> elimination -> a relaxation-coarsest
    level (coarse_solver.cpp:82-93). lamg_part_solve relaxes that level on the
    parts (halo exchange after every colour, mean and norm over the allgathered
    vectors): same cycle and sweep counts as lamg_solve, x within 1e-9, and
    bit-identical for 1, 2 and 4 parts."""
    from paper_1108_1310_b200 import lamg as L
    a = G.largest_component(G.chung_lu(1 << 16, seed=4) if name == "chunglu_64k" else G.rmat(14, seed=5))[0]
    ctx = L.Context(0, L.MODE_THROUGHPUT)
    h = L.setup(a, ctx=ctx)
    assert h.nlevels == 2 and h.levels[1].kind == 1 and h.levels[1].coarsest == 2
    b, x0 = G.gaussian_rhs(a.n, 29), G.default_x0(a.n)
    x1, s1 = L.solve(h, b, x0, ctx=ctx)
    assert s1.converged
    xs = []
    for P in (1, 2, 4):
        pl = L.PartLevel.from_hierarchy(h, P)
        xp, sp_ = pl.solve(h, b, x0)
        assert sp_.converged and sp_.cycles == s1.cycles, P
        assert abs(sp_.relax_sweeps - s1.relax_sweeps) <= 1, (P, sp_.relax_sweeps, s1.relax_sweeps)
        assert np.linalg.norm(xp - x1) / np.linalg.norm(x1) <= 1e-9, P
        xs.append(xp)
        pl.close()
    assert np.array_equal(xs[0], xs[1]) and np.array_equal(xs[0], xs[2])
    ctx.close()
