"""Multi-GPU plumbing for right-hand-side sharding (SURVEY.md 8(e) mode 1).

The solve shards naturally over independent right-hand sides: every rank
(one process per GPU) holds a replica of the device hierarchy and solves its
own slice of the RHS batch; there is no data-path collective. torch.distributed
(NCCL on GPUs, gloo on CPU) only provides the barrier around the timed region
and the reductions of the per-rank timings and work counts (max of time, sum
of edge*cycles).
"""
from __future__ import annotations

import os


def rhs_shard(total: int, rank: int, world: int) -> range:
    """Contiguous, balanced slice of [0, total) owned by `rank`."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


class Dist:
    """torch.distributed wrapper (single process when WORLD_SIZE is unset)."""

    def __init__(self, want_gpu: bool):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            self.backend = "nccl" if (want_gpu and torch.cuda.is_available()) else "gloo"
            if self.backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend=self.backend)
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def allreduce(self, v: float, op: str) -> float:
        if self.world == 1:
            return v
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=getattr(self.dist.ReduceOp, op))
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()
