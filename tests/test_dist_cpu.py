"""World-size-2 gloo tests of the multi-GPU host logic, on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_07624_b200 import dist as hd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ws, rk, lr = hd.env()
        lo, hi = hd.shard_range(N, rk, ws)
        # every rank's "device time" differs; the bench reports the max over ranks
        t = hd.max_over_ranks(1.5 + rank)
        # the union of the shards, gathered, must tile [0, N) exactly once
        cols = torch.zeros(N, dtype=torch.int64)
        cols[lo:hi] += 1
        dist.all_reduce(cols)
        hd.barrier()
        q.put((rank, ws, rk, lr, lo, hi, t, bool(torch.all(cols == 1))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N", [0, 1, 7, 262144])
def test_shard_and_max_world2(N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, N, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ws, rk, lr, lo, hi, t, tiled in out:
        assert (ws, rk, lr) == (2, rank, rank)
        assert t == 2.5                     # max over ranks
        assert tiled
    sizes = [hi - lo for _, _, _, _, lo, hi, _, _ in out]
    assert sum(sizes) == N and max(sizes) - min(sizes) <= 1


def test_shard_range_single_and_errors():
    assert hd.shard_range(10, 0, 1) == (0, 10)
    assert [hd.shard_range(10, r, 3) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ValueError):
        hd.shard_range(10, 3, 3)
    assert hd.max_over_ranks(3.0) == 3.0
