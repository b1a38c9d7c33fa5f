"""Multi-GPU path (runs when >= 2 GPUs are visible): one process per GPU over
NCCL, rank-range sharding of the split population, one all-gather of the
40-byte winner records; the merged result equals the single-GPU sweep."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    import torch.distributed as dist
    from gen import big_instance
    from paper_2309_01172_b200 import dist as D
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200.tensorize import build_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    st, fl = big_instance(np.random.default_rng(5), 30, 24, dag=False, pressure=(0.1, 0.6))
    batch = engine.device_batch([build_host(st, fl)], device=torch.device("cuda", rank))
    total = engine.splits_total(30, 24)
    bufs = engine.enum(batch, "splits", 0, total, part=rank, nparts=world)
    merged = D.merge_records(D.all_gather_winner(bufs.out).cpu().numpy())
    if rank == 0:
        single = engine.enum(batch, "splits", 0, total).read()
        q.put((merged, single))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_nccl_sharded_sweep_matches_single_gpu(engine_ready):
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    merged, single = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert merged == single
