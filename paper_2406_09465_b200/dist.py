"""Multi-GPU plumbing: one process per GPU, torch.distributed for the
process group.  The orchestrated executable itself has no data-path collective: ranks
run replicas (bs = 1 latency) or disjoint batch shards (throughput), and only per-rank
timings / outputs are gathered (G3/G4).  Backend-agnostic so the logic is testable with
gloo on CPU."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(global_batch: int, rank: int, world_size: int):
    """Contiguous batch shard [start, end) of rank r; shards differ by at most one item."""
    base, extra = divmod(global_batch, world_size)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_values(values, device=None):
    """All-gather a list of floats from every rank -> list (per rank) of lists."""
    if not dist.is_available() or not dist.is_initialized():
        return [list(values)]
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [x.tolist() for x in out]


def max_over_ranks(values, device=None):
    """Element-wise max over ranks (the timing rule: a multi-GPU step takes as long as its
    slowest rank)."""
    rows = gather_values(values, device)
    return [max(r[i] for r in rows) for i in range(len(values))]
