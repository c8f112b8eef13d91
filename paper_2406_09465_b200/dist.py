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


INF = (1 << 63) - 1


def my_share(n_items: int, rank: int, world_size: int):
    """Round-robin share of candidate indices profiled by this rank ("the tuning of
    candidate kernels can be parallelized across multiple GPUs")."""
    return [i for i in range(n_items) if i % world_size == rank]


def merge_costs(local_idx, local_costs, local_variants, n_items, device=None):
    """G1: combine per-rank profiling results.  Each rank fills the entries it profiled and
    leaves INF elsewhere; an element-wise MIN all-reduce yields the full cost vector on every
    rank, and the chosen launch variant travels with its cost (encoded in the low bits of
    a (cost << 8 | variant) key, so the MIN picks the variant of the rank that timed it)."""
    keys = torch.full((n_items,), INF, dtype=torch.int64, device=device)
    for i, c, v in zip(local_idx, local_costs, local_variants):
        if c < INF:
            if not 0 <= int(max(v, 0)) < 256:
                raise ValueError(f"candidate {i}: launch variant {v} does not fit the 8-bit key field")
            if int(c) >= 1 << 54:
                raise ValueError(f"candidate {i}: cost {c} ns does not fit the cost field")
            keys[i] = (int(c) << 8) | int(max(v, 0))
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(keys, op=dist.ReduceOp.MIN)
    costs, variants = [], []
    for k in keys.tolist():
        if k == INF:
            costs.append(INF)
            variants.append(-1)
        else:
            costs.append(k >> 8)
            variants.append(k & 0xFF)
    return costs, variants


def broadcast_selection(sel, src=0, device=None):
    """G2: rank `src` (which solved the BLP) broadcasts the chosen candidate indices."""
    if not dist.is_available() or not dist.is_initialized():
        return list(sel)
    n = torch.tensor([len(sel) if dist.get_rank() == src else 0], dtype=torch.int64, device=device)
    dist.broadcast(n, src)
    buf = torch.zeros(int(n.item()), dtype=torch.int64, device=device)
    if dist.get_rank() == src:
        buf[:] = torch.tensor(sel, dtype=torch.int64)
    dist.broadcast(buf, src)
    return buf.tolist()


def max_over_ranks(values, device=None):
    """Element-wise max over ranks (the timing rule: a multi-GPU step takes as long as its
    slowest rank)."""
    rows = gather_values(values, device)
    return [max(r[i] for r in rows) for i in range(len(values))]
