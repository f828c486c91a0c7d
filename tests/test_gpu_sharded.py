"""The NCCL branch of the layer-1 index gather (sharded.py) on the one GPU this
environment has: a world-size-1 NCCL group in a spawned process, so the
``all_gather_into_tensor`` path with CUDA tensors runs for real (the
world-size-2 logic is covered over gloo in test_sharded_gloo.py)."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(port, q):
    import torch.distributed as dist

    from paper_2604_17720_b200 import PruneConfig
    from paper_2604_17720_b200.batched import hierarchical_sample_batch
    from paper_2604_17720_b200.sharded import gather_rows, hierarchical_sample_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        g = torch.Generator(device="cuda").manual_seed(3)
        x = torch.rand((5, 4000, 3), generator=g, device="cuda")
        budgets, cfg = (1000, 250, 62), PruneConfig(p=0.75)
        layers, _, gathered = hierarchical_sample_sharded(x, budgets, cfg, batch=5)
        ref, _, _ = hierarchical_sample_batch(x, budgets, cfg, 0, True)
        ok_gather = gathered.device.type == "cuda" and gathered.dtype == torch.int64 and \
            torch.equal(gathered, ref[0].indices)
        # int64 rows travel as int32 and come back unchanged
        rows = torch.arange(15, dtype=torch.int64, device="cuda").view(3, 5) * 100_003
        ok_rows = torch.equal(gather_rows(rows, 3), rows)
        q.put((bool(ok_gather), bool(ok_rows), torch.equal(layers[0].indices, ref[0].indices)))
    finally:
        dist.destroy_process_group()


def test_gather_rows_nccl_world1():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    got = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert got == (True, True, True)
