"""The N>1 path on CPU: two gloo ranks shard a batch of right-hand sides,
solve their slices (with the CPU oracle standing in for the device solve),
and reduce timings and work exactly as bench.py does under torchrun."""
import os
import socket

import numpy as np
import pytest

from paper_1108_1310_b200.dist import rhs_shard


def test_rhs_shard_partitions():
    for total in (1, 7, 32, 33):
        for world in (1, 2, 3, 8):
            parts = [list(rhs_shard(total, r, world)) for r in range(world)]
            assert sum(parts, []) == list(range(total))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    from oracle import Oracle
    from paper_1108_1310_b200 import graphs as G
    from paper_1108_1310_b200.dist import Dist, rhs_shard
    d = Dist(want_gpu=False)
    a = G.grid_5pt(24)
    h = Oracle("port").setup(a)
    units, xs = 0.0, {}
    for i in rhs_shard(5, d.rank, d.world):
        x, st = h.solve(G.gaussian_rhs(a.n, 10 + i), G.default_x0(a.n, seed=1 + i))
        units += a.m * float(st["cycles"][0])
        xs[i] = float(np.linalg.norm(x))
    d.barrier()
    tot = d.allreduce(units, "SUM")
    mx = d.allreduce(float(d.rank + 1), "MAX")
    d.close()
    q.put((rank, tot, mx, xs))


def test_two_rank_gloo_sharded_solve():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    tots = {r[1] for r in res}
    assert len(tots) == 1 and {r[2] for r in res} == {2.0}
    xs = {}
    for r in res:
        xs.update(r[3])
    assert sorted(xs) == [0, 1, 2, 3, 4]
    # the sharded total equals the single-process total
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    from oracle import Oracle
    from paper_1108_1310_b200 import graphs as G
    a = G.grid_5pt(24)
    h = Oracle("port").setup(a)
    single = sum(a.m * float(h.solve(G.gaussian_rhs(a.n, 10 + i), G.default_x0(a.n, seed=1 + i))[1]["cycles"][0])
                 for i in range(5))
    assert tots.pop() == single


def test_bench_launcher_two_ranks():
    """bench.py --gpus 2 without WORLD_SIZE relaunches itself under
    torch.distributed.run (two ranks, gloo here: the reference arm needs no
    GPU); rank 0 alone prints the JSON line, the other rank exits 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not os.path.exists(os.path.join(root, "oracle", "_ref", "liblamg_ref.so")) and \
            not os.path.exists(os.path.join(root, "oracle", "liblamg_oracle.so")):
        pytest.skip("oracle not built")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "1", "--steps", "1", "--warmup", "0", "--cpu-cycles", "1"],
                       capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["n_gpus"] == 2 and out["value"] > 0
