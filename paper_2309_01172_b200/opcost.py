"""Operator-level PALEO costs on the GPU: mirror of hardware.op_time and
hardware.subgraph_time (pkg/src/dagmesh/hardware.py:180-226).

`op_time(graph, name, fleet, placement)` -> OpCost(read_s, compute_s, write_s)
`subgraph_time(graph, nodes, fleet, placement)` -> SubgraphTime(lower, upper, sequential)
`op_costs(table, fleet, placements)` -> [B, n_ops, 3] for a batch of placements.

The graph is read by attribute (`graph.node(name)` with `.args`, `.users`,
`.out_elements`; `graph.nodes` in authoring order).  Operator FLOPs come from
the graph's own catalog (`op_flops` of the module defining the graph class,
i.e. the reference's ir.op_flops) — the catalog is a host-side table producer;
all timing arithmetic runs in dm_op_costs / dm_subgraph_times.
"""

from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib
from .tensorize import build_host

ELEMENT_BYTES = 4


class OpCost(NamedTuple):
    read_s: float
    compute_s: float
    write_s: float

    @property
    def total_s(self) -> float:
        return self.read_s + self.compute_s + self.write_s


class SubgraphTime(NamedTuple):
    lower_s: float
    upper_s: float
    sequential_s: float


@dataclass
class OpTable:
    names: list
    flops: list          # op_flops per op (int)
    out_elements: list   # per op (int)
    args: list           # list of arg index lists
    users: list          # list of user index lists

    @property
    def index(self) -> dict:
        return {n: i for i, n in enumerate(self.names)}


def op_table_from_graph(graph, op_flops=None) -> OpTable:
    if op_flops is None:
        op_flops = getattr(sys.modules[type(graph).__module__], "op_flops")
    names = list(graph.nodes)
    idx = {n: i for i, n in enumerate(names)}
    nodes = [graph.node(n) for n in names]
    return OpTable(names=names, flops=[int(op_flops(nd)) for nd in nodes],
                   out_elements=[int(nd.out_elements) for nd in nodes],
                   args=[[idx[a] for a in nd.args] for nd in nodes],
                   users=[[idx[u] for u in nd.users] for nd in nodes])


def _csr(lists):
    ptr = np.zeros(len(lists) + 1, np.int32)
    flat = []
    for i, l in enumerate(lists):
        flat.extend(l)
        ptr[i + 1] = len(flat)
    return ptr, np.array(flat or [0], np.int32)


def op_costs(table: OpTable, fleet, placements) -> np.ndarray:
    """Per-op (read_s, compute_s, write_s) for each placement (dict op name ->
    peer id, covering every op)."""
    _, out, _, n = _op_costs_device(table, fleet, placements)
    return out.cpu().numpy()[: len(placements) * n * 3].reshape(len(placements), n, 3)


def _op_costs_device(table: OpTable, fleet, placements):
    """dm_op_costs launch; returns (input tensors, per-op costs, numpy-type
    flags, n_ops) on the device (reentrant: no state kept between calls)."""
    import torch
    lib = _lib.load()
    host = build_host([], fleet, True)
    n = len(table.names)
    ratio = fleet.msg_ratio
    mbytes = np.array([float(int(round(e * ELEMENT_BYTES * ratio))) for e in table.out_elements], np.float64)
    flops = np.array([float(f) for f in table.flops], np.float64)
    aptr, aidx = _csr(table.args)
    uptr, uidx = _csr(table.users)
    unknown: dict = {}
    place = np.zeros((len(placements), n), np.int32)
    for b, pl in enumerate(placements):
        for i, name in enumerate(table.names):
            pid = str(pl[name])
            place[b, i] = host.index_of[pid] if pid in host.index_of else unknown.setdefault(pid, host.P + len(unknown))
    wbw = [fleet.peers[p].write_bandwidth for p in host.peer_ids]
    write_bw = np.array([float(v) for v in wbw] or [1.0], np.float64)
    # CPython sum() in subgraph_time is compensated only over exact floats:
    # record which totals the reference computes as numpy floats
    write_np = np.array([0 if type(v) in (int, float, bool) else 1 for v in wbw] or [0], np.uint8)
    d = fleet.default_link
    np_links = any(type(v) not in (int, float, bool)
                   for v in [d.alpha, d.beta, *(x for lk in fleet.links.values() for x in (lk.alpha, lk.beta))])
    from .engine import device_batch
    batch = device_batch([host], pin=False)
    dev = batch.dev_buf.device
    arrs = [torch.from_numpy(a).to(dev)
            for a in (flops, mbytes, aptr, aidx, uptr, uidx, write_bw, place.reshape(-1), write_np)]
    ops = _lib.DmOps(n, _lib.DM_OPS_NP_LINKS if np_links else 0, *[a.data_ptr() for a in arrs[:6]],
                     arrs[8].data_ptr())
    out = torch.empty(max(len(placements) * n * 3, 1), dtype=torch.float64, device=dev)
    out_np = torch.empty(max(len(placements) * n, 1), dtype=torch.uint8, device=dev)
    st = batch.struct(0)
    _lib.check(lib.dm_op_costs(C.byref(ops), C.byref(st), arrs[6].data_ptr(), len(placements), arrs[7].data_ptr(),
                               out.data_ptr(), out_np.data_ptr(), _lib.stream_ptr()))
    return arrs, out, out_np, n


def subgraph_costs(table: OpTable, fleet, placements, cells) -> np.ndarray:
    """subgraph_time for every cell (list of op names) and placement: [B, n_cells, 3]."""
    import torch
    lib = _lib.load()
    arrs, out, out_np, n = _op_costs_device(table, fleet, placements)
    idx = table.index
    sptr, sidx = _csr([[idx[x] for x in cell] for cell in cells])
    sp, si = torch.from_numpy(sptr).to(out.device), torch.from_numpy(sidx).to(out.device)
    res = torch.empty(max(len(placements) * len(cells) * 3, 1), dtype=torch.float64, device=out.device)
    _lib.check(lib.dm_subgraph_times(n, len(placements), out.data_ptr(), out_np.data_ptr(), len(cells),
                                     sp.data_ptr(), si.data_ptr(),
                                     res.data_ptr(), _lib.stream_ptr()))
    return res.cpu().numpy()[: len(placements) * len(cells) * 3].reshape(len(placements), len(cells), 3)


def _full_placement(table, placement, needed):
    """Complete a (possibly partial) placement so every op has a peer; ops
    outside `needed` are parked on the first needed op's peer (unused)."""
    for name in needed:
        placement[name]  # KeyError exactly where the reference raises
    fill = str(placement[needed[0]])
    return {n: (placement[n] if n in placement else fill) for n in table.names}


def op_time(graph, name, fleet, placement) -> OpCost:
    """hardware.op_time (hardware.py:190-206) on the GPU."""
    table = op_table_from_graph(graph)
    node = graph.node(name)
    me = str(placement[name])
    fleet.peer(me)  # FleetError for an unknown peer, as the reference
    needed = [name, *node.args, *node.users]
    pl = _full_placement(table, dict(placement), needed)
    r, c, w = op_costs(table, fleet, [pl])[0, table.index[name]]
    return OpCost(float(r), float(c), float(w))


def subgraph_time(graph, nodes, fleet, placement) -> SubgraphTime:
    """hardware.subgraph_time (hardware.py:219-226) on the GPU."""
    nodes = list(nodes)
    if not nodes:
        return SubgraphTime(0.0, 0.0, 0.0)
    table = op_table_from_graph(graph)
    needed = []
    for nm in nodes:
        nd = graph.node(nm)
        fleet.peer(str(placement[nm]))
        needed += [nm, *nd.args, *nd.users]
    pl = _full_placement(table, dict(placement), needed)
    lo, up, sq = subgraph_costs(table, fleet, [pl], [nodes])[0, 0]
    return SubgraphTime(float(lo), float(up), float(sq))
