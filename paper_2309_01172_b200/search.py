"""Batched search APIs beyond the reference's per-call functions.

``split_sweep`` scores the whole identity-split population of a model on
each of several fleets — every contiguous split of the stages with run q on
worker q, brute_force_schedule's inner body (scheduling.py:264-272) for each
— and returns each fleet's first strict minimum (:271) as the reference
types.  It is the serving form of the headline sweep: stages and fleets in,
tensorised (stage side cached), one captured CUDA graph per input shape
(H2D of the tables, the meet-in-the-middle kernels of dm_mitm.cu, D2H of the
winner records), winners decoded on the host."""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import engine
from .tensorize import build_host


@dataclass(frozen=True)
class SplitWinner:
    """First strict minimum of one fleet's identity-split population."""
    runs: tuple               # Runs in the reference's form, () when nothing is feasible
    makespan: float           # inf when nothing is feasible
    rank: int                 # position in brute_force_schedule's order restricted to identity splits
    n_evaluated: int
    n_feasible: int
    checksum: int             # sum of every feasible candidate's makespan bits mod 2^64


def splits_total(n: int, p: int) -> int:
    return sum(math.comb(n - 1, r - 1) for r in range(1, min(n, p) + 1))


_GRAPHS: dict = {}


def _graph_for(hosts, total, units):
    key = (tuple(h.packed_size() for h in hosts), total, tuple(units))
    g = _GRAPHS.get(key)
    if g is not None and g.batch.repack(hosts):
        return g
    batch = engine.device_batch(hosts)
    g = engine.SweepGraph(batch, total, units=units)
    _GRAPHS[key] = g
    return g


def split_sweep(stages, fleets, *, include_comm: bool = True, part: int = 0, nparts: int = 1,
                records: bool = False):
    """Identity-split sweep of `stages` on every fleet in `fleets`.

    part/nparts: this caller's share of every population (block-level parts,
    merged with dist.merge_records); records=True returns the raw 40-byte
    winner records (uint8[len(fleets), 40], for a multi-GPU all-gather)
    instead of decoded winners."""
    stages = list(stages)
    hosts = [build_host(stages, f, include_comm) for f in fleets]
    n = len(stages)
    p = hosts[0].p
    if any(h.p != p for h in hosts):
        raise ValueError("split_sweep: every fleet needs the same number of workers")
    total = splits_total(n, p)
    units = [(i, part, nparts) for i in range(len(hosts))]
    g = _graph_for(hosts, total, units)
    g.launch()
    if records:
        g.read_all()
        return g.host_out.numpy().copy()
    out = []
    for h, w in zip(hosts, g.read_all()):
        runs = ()
        if w["rank"] >= 0:
            bounds, peers = engine.unrank(n, p, int(w["rank"]), "splits")
            runs = tuple((h.peer_ids[peers[q]], tuple(range(bounds[q], bounds[q + 1]))) for q in range(len(peers)))
        out.append(SplitWinner(runs, w["makespan"], int(w["rank"]), int(w["n_evaluated"]), int(w["n_feasible"]),
                               int(w["checksum"])))
    return out
