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
