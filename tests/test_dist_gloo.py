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


def _worker_random_and_c4(rank, world, port, q):
    """The bench's other sharded populations at N=2 on CPU: counter ranges of
    a random-placement stream (oracle restatement of the recipe) and
    contiguous slices of the C4 scenario draws."""
    import struct
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from gen import big_instance
    from oracle import oracle
    from paper_2309_01172_b200 import configs as CF
    from paper_2309_01172_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st, fl = big_instance(np.random.default_rng(5), 30, 40, dag=False, pressure=(0.05, 0.5))
    inst = oracle.Instance(st, fl)
    online = np.arange(0, 40, 2, dtype=np.int32)
    N = 40000
    k0, k1 = D.shard(N, rank, world)
    w = inst.enum_random(online, 99, k0, k1)
    rec = torch.frombuffer(bytearray(struct.pack(D.WINNER_FMT, w["makespan"], w["rank"], w["n_evaluated"],
                                                 w["n_feasible"], w["checksum"])), dtype=torch.uint8)
    out = torch.empty(world * rec.numel(), dtype=torch.uint8)
    dist.all_gather_into_tensor(out, rec)
    merged = D.merge_records(out.numpy())
    # C4 slices: every rank draws all scenarios' parameters and keeps its slice
    P = CF.c4_params(1000, seed=0)
    lo, hi = D.shard(1000, rank, world)
    mine = torch.from_numpy(np.concatenate([P["layers"][lo:hi], P["p"][lo:hi]]).astype(np.int64))
    sizes = [D.shard(1000, r, world)[1] - D.shard(1000, r, world)[0] for r in range(world)]
    gathered = [torch.empty(2 * s_, dtype=torch.int64) for s_ in sizes]
    dist.all_gather(gathered, mine)
    layers = np.concatenate([g[: s_].numpy() for g, s_ in zip(gathered, sizes)])
    if rank == 0:
        q.put((merged, inst.enum_random(online, 99, 0, N), layers.tolist(), P["layers"].tolist()))
    dist.destroy_process_group()


def test_two_rank_gloo_random_ranges_and_c4_slices():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_random_and_c4, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, single, layers, full = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
    assert merged == single
    assert layers == full
