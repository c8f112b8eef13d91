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
    from paper_2406_09465_b200.dist import gather_values, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mx = max_over_ranks([1.0 + rank, 10.0 - rank])
    rows = gather_values([float(rank)])
    dist.destroy_process_group()
    q.put((rank, mx, rows))


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
    for rank, mx, rows in res:
        assert mx == [2.0, 10.0]
        assert rows == [[0.0], [1.0]]
