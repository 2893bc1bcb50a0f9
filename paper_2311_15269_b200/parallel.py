"""Multi-GPU sharding of the repetend search.

One process per GPU (``torch.distributed``; NCCL over NVLink on the B200 box,
gloo for CPU tests).  Every window of candidate ranks is split by rank prefix
across the processes and each process scans its share on its own GPU with no
collective inside the scan (the reference's only parallelism is a process pool
over candidates, completion.py:316-349).  Per window:

* one all-gather of fixed-width int64 rows — a 2-int header per rank
  (row count, first undetermined index, deadline flag) followed by the
  shard's first-SAT rows ``[window index, period, starts[K]]`` padded to the
  largest shard;
* rank 0 runs the ordered replay (the improvement rule and the completion
  checks, completion.py:351-382) and broadcasts its decisions as one int64
  vector (length-prefixed), so every rank applies the identical
  improvements, records and bound without re-running completion checks.

The bound a shard is scanned under is the one in force at the window start: a
shard above an improvement found in the same window only does extra work
(its outcomes are facts about (candidate, period) pairs and the replay
applies the true bound), never gives a different answer.  Status counts and
reference decide counts are reduced once at the end of the search.
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

    def gather_rows(self, rows, header):
        """All-gather every rank's int64 ``rows`` (n_i x w) and 2-int
        ``header``: returns (rows of all ranks in rank order, [header_i]).
        Two fixed-size collectives: the headers + counts, then the rows
        padded to the largest count."""
        import numpy as np

        torch = self.torch
        rows = np.asarray(rows, dtype=np.int64)
        w = rows.shape[1]
        head = torch.tensor([rows.shape[0], *header], dtype=torch.int64, device=self.device)
        heads = [torch.empty_like(head) for _ in range(self.size)]
        self.dist.all_gather(heads, head, group=self.group)
        heads = [[int(v) for v in h.tolist()] for h in heads]
        n_max = max(h[0] for h in heads)
        self.collectives += 1
        if n_max == 0:
            return np.zeros((0, w), dtype=np.int64), [h[1:] for h in heads]
        buf = torch.zeros((n_max, w), dtype=torch.int64, device=self.device)
        if rows.shape[0]:
            buf[:rows.shape[0]] = torch.from_numpy(rows).to(self.device)
        parts = [torch.empty_like(buf) for _ in range(self.size)]
        self.dist.all_gather(parts, buf, group=self.group)
        self.collectives += 1
        out = np.concatenate([parts[r][:heads[r][0]].cpu().numpy() for r in range(self.size)])
        return out, [h[1:] for h in heads]

    def bcast_ints(self, vals):
        """Broadcast rank 0's int list (length-prefixed; others pass None)."""
        torch = self.torch
        n = torch.tensor([len(vals) if self.rank == 0 else 0], dtype=torch.int64,
                         device=self.device)
        self.dist.broadcast(n, 0, group=self.group)
        m = int(n.item())
        t = (torch.tensor(list(vals), dtype=torch.int64, device=self.device) if self.rank == 0
             else torch.empty(m, dtype=torch.int64, device=self.device))
        if m:
            self.dist.broadcast(t, 0, group=self.group)
        self.collectives += 2
        return [int(v) for v in t.tolist()]

    def bcast_obj(self, obj):
        """Broadcast one small picklable object from rank 0 (once per search:
        the completed schedule and report fields)."""
        box = [obj if self.rank == 0 else None]
        self.dist.broadcast_object_list(box, 0, group=self.group)
        self.collectives += 1
        return box[0]


class SoloComm:
    """The single-process stand-in: every collective is the identity."""

    rank, size, collectives = 0, 1, 0

    def gather_rows(self, rows, header):
        import numpy as np

        return np.asarray(rows, dtype=np.int64), [list(header)]

    def bcast_ints(self, vals):
        return list(vals)

    def bcast_obj(self, obj):
        return obj

    def allreduce_sum(self, vals):
        return list(vals)


def split_range(r0: int, r1: int, rank: int, size: int) -> tuple:
    """Contiguous rank-prefix share [a, b) of [r0, r1) for `rank`."""
    n = r1 - r0
    a = r0 + (n * rank) // size
    b = r0 + (n * (rank + 1)) // size
    return a, b
