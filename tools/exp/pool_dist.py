"""One C2 scenario swept by N GPUs: the pooled sweep (dm_enum_splits_pooled,
side tables shared over NVLink, one tile queue) against the block-part split
(dm_enum_splits_part: each rank builds the tables of its blocks) and the
single-GPU sweep.  Checks the merged winners against tests/golden/full_size.json.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/exp/pool_dist.py
"""
import json
import os
import pathlib
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2309_01172_b200 import configs as CF, engine, search  # noqa: E402
from paper_2309_01172_b200 import dist as D  # noqa: E402
from paper_2309_01172_b200.tensorize import build_host  # noqa: E402

KEYS = ("makespan", "rank", "n_evaluated", "n_feasible", "checksum")


def timed(fn, reps, stream):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    t = torch.tensor([float(np.median(ts))], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    gold = json.loads((ROOT / "tests" / "golden" / "full_size.json").read_text())["c2"]
    stages = CF.model_stages("llama2-7b-layers")
    fleets = {int(s): CF.load(CF.c2_fleet_doc(0, *CF.C2_LINKS[int(s)])) for s in gold}
    engine.warmup()
    pool = search.PooledSweep(stages, fleets[0])
    ok = True
    for s, f in sorted(fleets.items()):
        w = pool.sweep(f)
        got = dict(makespan=w.makespan, rank=w.rank, n_evaluated=w.n_evaluated, n_feasible=w.n_feasible,
                   checksum=w.checksum)
        want = {k: gold[str(s)][k] for k in KEYS}
        ok &= got == want
        if rank == 0 and got != want:
            print("MISMATCH", s, got, want, flush=True)
    stream = torch.cuda.current_stream()
    batch = engine.device_batch([build_host(stages, fleets[0], True)])
    total = engine.splits_total(len(stages), 32)
    bufs = engine.WinnerBuffers(batch.dev_buf.device)
    reps = 20
    t_pool = timed(lambda: engine.splits_pooled(batch, rank, world, pool.ptrs, pool.bytes, pool.bufs), reps, stream)
    t_part = timed(lambda: engine.enum(batch, "splits", 0, total, bufs=bufs, part=rank, nparts=world), reps, stream)
    t_one = timed(lambda: engine.enum(batch, "splits", 0, total, bufs=bufs), reps, stream)
    def burst(fn, k=10):
        return timed(lambda: [fn() for _ in range(k)], 5, stream) / k
    pool_fn = lambda: engine.splits_pooled(batch, rank, world, pool.ptrs, pool.bytes, pool.bufs)  # noqa: E731
    b_pool = burst(pool_fn)
    os.environ["DM_POOL_REPLICATE"] = "1"
    b_repl = burst(pool_fn)
    os.environ["DM_POOL_REPLICATE"] = "0"
    b_part = burst(lambda: engine.enum(batch, "splits", 0, total, bufs=bufs, part=rank, nparts=world))
    b_one = burst(lambda: engine.enum(batch, "splits", 0, total, bufs=bufs))
    import ctypes as C
    from paper_2309_01172_b200 import _lib
    lib = _lib.load()
    phases = {}
    part_fn = lambda: engine.enum(batch, "splits", 0, total, bufs=bufs, part=rank, nparts=world)  # noqa: E731
    one_fn = lambda: engine.enum(batch, "splits", 0, total, bufs=bufs)  # noqa: E731
    for name, env, fn in (("pooled", "0", pool_fn), ("pooled_replicated_tables", "1", pool_fn),
                          ("block_parts", "0", part_fn), ("single", "0", one_fn)):
        os.environ["DM_POOL_REPLICATE"] = env
        lib.dm_sweep_timing(1, None, None)
        acc = []
        for _ in range(5):
            dist.barrier()
            torch.cuda.synchronize()
            fn()
            a, b = C.c_float(0), C.c_float(0)
            _lib.check(lib.dm_sweep_timing(-1, C.byref(a), C.byref(b)))
            acc.append((a.value, b.value))
        lib.dm_sweep_timing(0, None, None)
        t = torch.tensor(np.median(np.array(acc), axis=0), dtype=torch.float64, device="cuda")
        g = torch.empty(2 * world, dtype=torch.float64, device="cuda")
        dist.all_gather_into_tensor(g, t)
        phases[name] = g.view(world, 2).tolist()
    os.environ["DM_POOL_REPLICATE"] = "0"
    if rank == 0:
        print(json.dumps({"phase_ms_per_rank [tables+barrier, plan+sweep]": phases}), flush=True)
    if rank == 0:
        print(json.dumps({"burst10_ms_per_sweep": {"pooled": b_pool, "pooled_replicated_tables": b_repl,
                                                   "block_parts": b_part, "single": b_one}}), flush=True)
    # the parts' records merge to the single sweep too
    engine.enum(batch, "splits", 0, total, bufs=bufs, part=rank, nparts=world)
    merged = D.merge_records(D.all_gather_winner(bufs.out).cpu().numpy())
    ok &= merged == {k: gold["0"][k] for k in KEYS}
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"world": world, "parity": bool(okt.item()), "scenarios_checked": len(fleets),
                          "single_gpu_ms": t_one, "pooled_ms": t_pool, "block_parts_ms": t_part,
                          "pooled_speedup": t_one / t_pool, "pooled_efficiency": t_one / t_pool / world,
                          "parts_speedup": t_one / t_part, "parts_efficiency": t_one / t_part / world}), flush=True)
    pool.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
