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
    if g is not None:                  # same shape, other scalars (e.g. default links): recapture
        del _GRAPHS[key]
        del g
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


class SplitSweeper:
    """Pipelined serving form of split_sweep for a stream of requests of one
    shape (same stages, same number of fleets and workers): two slots, each a
    pinned staging buffer + captured graph (H2D of the tables, the sweep
    kernels, D2H of the winner records).  submit() tensorises and packs the
    next request while the GPU still runs the previous one, then replays the
    free slot's graph; result() waits for that request and decodes it.  Every
    request still copies its own inputs in and its winners out."""

    def __init__(self, stages, fleets_example, *, include_comm: bool = True, slots: int = 2):
        torch = engine._torch()
        self.stages = list(stages)
        self.include_comm = include_comm
        hosts = [build_host(self.stages, f, include_comm) for f in fleets_example]
        self.n, self.p = len(self.stages), hosts[0].p
        self.total = splits_total(self.n, self.p)
        units = [(i, 0, 1) for i in range(len(hosts))]
        self.graphs = []
        for _ in range(slots):
            g = engine.SweepGraph(engine.device_batch(hosts), self.total, units=units)
            self.graphs.append(g)
        self.events = [None] * slots
        self.hosts = [None] * slots
        self.next = 0
        self.stream = torch.cuda.current_stream()

    def submit(self, fleets) -> int:
        torch = engine._torch()
        slot = self.next
        self.next = (slot + 1) % len(self.graphs)
        hosts = [build_host(self.stages, f, self.include_comm) for f in fleets]   # overlaps the GPU's work
        if self.events[slot] is not None:
            self.events[slot].synchronize()          # the slot's previous request has left its buffers
        g = self.graphs[slot]
        if not g.batch.repack(hosts):
            # other scalars (default link, flags) or shapes than the captured
            # graph: recapture this slot on the request's tables
            g = self.graphs[slot] = engine.SweepGraph(engine.device_batch(hosts), self.total,
                                                      units=[(i, 0, 1) for i in range(len(hosts))])
        g.launch()
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self.events[slot] = ev
        self.hosts[slot] = hosts
        return slot

    def gathered(self, slot: int, group=None):
        """Multi-GPU form of result(slot, records=True): the slot's DEVICE
        records all-gathered over the process group (one NCCL all-gather) on
        a stream of their own — it waits for this request's graph only, not
        for the request queued behind it on the main stream — then copied to
        the host: uint8[world, units, 40] (merge with dist.merge_records)."""
        torch = engine._torch()
        import torch.distributed as dist
        if not hasattr(self, "_gstream"):
            self._gstream = torch.cuda.Stream()
        g = self.graphs[slot]
        world = dist.get_world_size(group)
        with torch.cuda.stream(self._gstream):
            self._gstream.wait_event(self.events[slot])
            out = torch.empty(world * g.out.numel(), dtype=torch.uint8, device=g.out.device)
            dist.all_gather_into_tensor(out, g.out.reshape(-1), group=group)
            host = out.view(world, g.out.shape[0], -1).cpu()
        return host.numpy()

    def result(self, slot: int, records: bool = False):
        self.events[slot].synchronize()
        g = self.graphs[slot]
        if records:
            return g.host_out.numpy().copy()
        out = []
        raw = g.host_out.numpy().tobytes()
        from . import _lib
        for i, h in enumerate(self.hosts[slot]):
            w = _lib.DmWinner.from_buffer_copy(raw[i * _lib.C.sizeof(_lib.DmWinner):(i + 1) * _lib.C.sizeof(_lib.DmWinner)])
            runs = ()
            if w.rank >= 0:
                bounds, peers = engine.unrank(self.n, self.p, int(w.rank), "splits")
                runs = tuple((h.peer_ids[peers[q]], tuple(range(bounds[q], bounds[q + 1]))) for q in range(len(peers)))
            out.append(SplitWinner(runs, w.makespan, int(w.rank), int(w.n_evaluated), int(w.n_feasible),
                                   int(w.checksum)))
        return out
