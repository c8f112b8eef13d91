"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host logic."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2406_09465_b200.dist import shard


def test_shard_covers_batch_exactly():
    for gb in range(0, 40):
        for w in range(1, 9):
            parts = [shard(gb, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == gb
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [e - s for s, e in parts]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2406_09465_b200.dist import (INF, broadcast_selection, gather_values, max_over_ranks, merge_costs,
                                            my_share)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mx = max_over_ranks([1.0 + rank, 10.0 - rank])
    rows = gather_values([float(rank)])
    # sharded profiling (G1): rank r "measures" items i % world == r
    n = 7
    idx = my_share(n, rank, world)
    costs = [1000 + 10 * i if i != 5 else INF for i in idx]     # item 5 is not generable
    variants = [i % 3 for i in idx]
    allc, allv = merge_costs(idx, costs, variants, n)
    sel = broadcast_selection([1, 4, 6] if rank == 0 else [9, 9], src=0)   # G2
    dist.destroy_process_group()
    q.put((rank, mx, rows, allc, allv, sel))


@pytest.mark.timeout(120)
def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=100) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    INF = (1 << 63) - 1
    for rank, mx, rows, allc, allv, sel in res:
        assert mx == [2.0, 10.0]
        assert rows == [[0.0], [1.0]]
        assert allc == [1000 + 10 * i if i != 5 else INF for i in range(7)]
        assert allv == [i % 3 if i != 5 else -1 for i in range(7)]
        assert sel == [1, 4, 6]
