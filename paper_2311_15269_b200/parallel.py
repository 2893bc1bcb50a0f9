"""Multi-GPU sharding of the repetend search.

One process per GPU (``torch.distributed``; NCCL over NVLink on the B200 box,
gloo for CPU tests).  Every window of candidate ranks is split by rank prefix
across the processes; during the level-synchronous scan the processes
exchange ONE packed vector per stage with an all-reduce-min:

    [lowest completion-feasible SAT global index, -(active candidates)]

so each rank retires its candidates above the global first feasible SAT (a
bound that flows from lower to higher indices only) and all
ranks agree on when the window's scan ends.  After the window the SAT rows
are all-gathered and every rank runs the same deterministic ordered replay,
so the result (improvements, repetend, schedule, records) is identical on all
ranks and equal to the single-GPU / reference result.
"""

from __future__ import annotations

from typing import Optional

BIG = (1 << 62)


class Comm:
    """Thin collective layer over torch.distributed (NCCL or gloo)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.dist, self.torch, self.group = dist, torch, group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        backend = dist.get_backend(group)
        if backend == "nccl":
            self.device = device if device is not None else torch.device(
                "cuda", torch.cuda.current_device())
        else:
            self.device = torch.device("cpu")
        self.collectives = 0

    def allreduce_min(self, vals):
        t = self.torch.tensor(list(vals), dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        self.collectives += 1
        return [int(v) for v in t.tolist()]

    def allreduce_sum(self, vals):
        t = self.torch.tensor(list(vals), dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        self.collectives += 1
        return [int(v) for v in t.tolist()]

    def allgather(self, obj):
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.group)
        self.collectives += 1
        return out

    def barrier(self):
        self.dist.barrier(group=self.group)


def split_range(r0: int, r1: int, rank: int, size: int) -> tuple:
    """Contiguous rank-prefix share [a, b) of [r0, r1) for `rank`."""
    n = r1 - r0
    a = r0 + (n * rank) // size
    b = r0 + (n * (rank + 1)) // size
    return a, b


class LevelSync:
    """Per-stage bound exchange for one rank's share of a window."""

    def __init__(self, comm: Comm, offset: int):
        self.comm, self.offset = comm, offset

    def __call__(self, first_feasible: Optional[int], limit: int, n_active: int):
        mine = BIG if first_feasible is None else self.offset + first_feasible
        g_first, neg_active = self.comm.allreduce_min([mine, -n_active])
        if g_first < BIG:
            limit = min(limit, g_first - self.offset - 1)
        return limit, -neg_active > 0

    def any(self, flag: bool) -> bool:
        """True on every rank if any rank raised `flag` (speculation verdicts)."""
        return self.comm.allreduce_min([-int(bool(flag))])[0] < 0
