"""Partitioned finest level (SURVEY.md 8(e) mode 2): coloured sweeps + residual
with halo exchange, timed on the device.

  python tools/part_bench.py [cfg] [parts] [--solve] one GPU, all parts in process
                                                   (--solve: a whole lamg_part_solve)
  torchrun --nproc-per-node N tools/part_bench.py   one part per GPU over NCCL
                                                   (max over ranks)
Prints one JSON line: level size, parts, sweeps, ms per sweep, exchange bytes.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
parts = world if world > 1 else (int(sys.argv[2]) if len(sys.argv) > 2 else 1)
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
a = G.make_config(cfg)
ctx = L.Context(torch.cuda.current_device(), L.MODE_THROUGHPUT)
comm = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl")
    uid = [L.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = L.Comm(world, rank, uid[0], ctx=ctx)
if "--solve" in sys.argv:
    # one right-hand side solved with the finest level partitioned (lamg_part_solve)
    import time
    h = L.setup(a, ctx=ctx)
    pls = L.PartLevel.from_hierarchy(h, parts, comm=comm)
    b, x0 = G.gaussian_rhs(a.n, 17), G.default_x0(a.n)
    pls.solve(h, b, x0)
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.time()
        x, st = pls.solve(h, b, x0)
        torch.cuda.synchronize()
        times.append(time.time() - t0)
    sec = min(times)
    if comm is not None:
        t = torch.tensor([sec], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    if rank == 0:
        print(json.dumps({"config": cfg, "n": a.n, "m": a.m, "parts": parts,
                          "transport": "nccl" if comm else "in-process", "solve_s": sec, "cycles": st.cycles,
                          "edges_cycles_per_s": a.m * st.cycles / sec}))
    pls.close()
    if comm is not None:
        comm.close()
        dist.destroy_process_group()
    sys.exit(0)
pl = L.PartLevel(a, parts, ctx=ctx, comm=comm)
bounds = L.part_bounds(a, parts)
halo = sum(len(L.part_plan(a, bounds, p)["ghost_gid"]) for p in range(parts)) if parts <= 8 else -1
rng = np.random.default_rng(1)
b = rng.standard_normal(a.n)
b -= b.mean()
pl.smooth(b, rng.standard_normal(a.n), 1)
sweeps = 20
pl.time(2)
ms = pl.time(sweeps)
if comm is not None:
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
if rank == 0:
    print(json.dumps({"config": cfg, "n": a.n, "m": a.m, "parts": parts, "transport": "nccl" if comm else "in-process",
                      "sweeps": sweeps, "ms_per_sweep": ms / sweeps,
                      "edges_sweeps_per_s": a.m * sweeps / (ms * 1e-3),
                      "halo_doubles_per_exchange": halo}))
pl.close()
if comm is not None:
    comm.close()
    dist.destroy_process_group()
