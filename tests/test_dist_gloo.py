"""Multi-rank path on CPU: world_size-2 gloo processes shard the rank space,
score their slices with the oracle, all-gather the 40-byte winner records and
merge — the result equals the single-process winner."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import struct
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from gen import big_instance
    from oracle import oracle
    from paper_2309_01172_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st, fl = big_instance(np.random.default_rng(3), 16, 9, dag=False, pressure=(0.1, 0.7))
    inst = oracle.Instance(st, fl)
    total = oracle.splits_total(16, 9)
    k0, k1 = D.shard(total, rank, world)
    w = inst.enum("splits", k0, k1)
    rec = torch.frombuffer(bytearray(struct.pack(D.WINNER_FMT, w["makespan"], w["rank"], w["n_evaluated"],
                                                 w["n_feasible"], w["checksum"])), dtype=torch.uint8)
    out = torch.empty(world * rec.numel(), dtype=torch.uint8)
    dist.all_gather_into_tensor(out, rec)
    merged = D.merge_records(out.numpy())
    if rank == 0:
        q.put((merged, inst.enum("splits", 0, total)))
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, single = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert merged == single
