"""Multi-GPU host logic on CPU: shard-by-cloud partition and the layer-1
index gather, exercised with world_size 2 over gloo (the GPU path runs the
same code over NCCL)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_17720_b200.sharded import gather_rows, shard_range


@pytest.mark.parametrize("batch,world", [(64, 1), (64, 2), (64, 8), (7, 3), (2, 4), (0, 2)])
def test_shard_range_partitions_batch(batch, world):
    seen = []
    for r in range(world):
        lo, hi = shard_range(batch, world, r)
        assert 0 <= hi - lo <= -(-batch // world) if batch else hi == lo
        seen += list(range(lo, hi))
    assert seen == list(range(batch))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, batch, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(batch, world, rank)
        # stand-in for this rank's layer-1 indices: row b holds cloud id b
        local = torch.arange(lo, hi, dtype=torch.int64)[:, None] * 1000 + \
            torch.arange(5, dtype=torch.int64)[None, :]
        full = gather_rows(local, batch)
        q.put((rank, full.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [8, 7])
def test_gather_rows_world2_gloo(batch):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [[b * 1000 + j for j in range(5)] for b in range(batch)]
    assert got[0] == want and got[1] == want
