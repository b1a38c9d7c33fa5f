"""Multi-GPU sharding of candidate populations (one process per GPU).

Each rank scores a contiguous slice [k0, k1) of the global rank space with
its own replica of the instance tables (built deterministically from the same
inputs — no broadcast), then ONE collective, an all-gather of the fixed-size
winner records, lets every rank take the lexicographic minimum by
(makespan, global rank).  The result is identical for any GPU count.
"""

from __future__ import annotations

import struct

import numpy as np

WINNER_FMT = "<dqqqQ"  # dm_winner: makespan, rank, n_evaluated, n_feasible, checksum
WINNER_BYTES = struct.calcsize(WINNER_FMT)


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced slice of [0, total) for `rank`."""
    base, extra = divmod(total, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def merge_records(raw: np.ndarray) -> dict:
    """Merge dm_winner records (rows of raw bytes) — first strict minimum by
    (makespan, rank), counts and checksums summed (mod 2^64)."""
    best_mk, best_rank = float("inf"), -1
    n_eval = n_feas = 0
    csum = 0
    for row in raw.reshape(-1, WINNER_BYTES):
        mk, rank, ne, nf, cs = struct.unpack(WINNER_FMT, row.tobytes())
        n_eval += ne
        n_feas += nf
        csum = (csum + cs) & ((1 << 64) - 1)
        if rank >= 0 and (best_rank < 0 or mk < best_mk or (mk == best_mk and rank < best_rank)):
            best_mk, best_rank = mk, rank
    return dict(makespan=best_mk, rank=best_rank, n_evaluated=n_eval, n_feasible=n_feas, checksum=csum)


def all_gather_winner(out_dev, group=None):
    """All-gather a device dm_winner record (uint8[40]) across the process
    group; returns a device tensor [world, 40]."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gathered = torch.empty(world * out_dev.numel(), dtype=torch.uint8, device=out_dev.device)
    dist.all_gather_into_tensor(gathered, out_dev, group=group)
    return gathered.view(world, -1)
