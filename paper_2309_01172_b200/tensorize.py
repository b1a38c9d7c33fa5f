"""Structure-of-arrays tensorisation of (stages, fleet) instances.

Turns the reference's ``list[Stage]`` + ``Fleet`` (pkg/src/dagmesh/
scheduling.py:32-42, hardware.py:103-144) into the ``dm_tables`` layout of
include/dagmesh_b200.h:

* stage columns as float64 plus exact int64 prefix sums when a column is
  integral with sum(|v|) < 2^53 (then every subset sum the reference forms is
  exact, whatever order CPython adds in);
* in-edges in stored order as CSR, message sizes ``nbytes * msg_ratio``
  evaluated with CPython's own float arithmetic (scheduling.py:168,301);
* peers in ``worker_ids()`` order followed by the other peers (backups) in
  ``peer_ids()`` order; capacities and ``effective_speed`` as float64;
* ``link_between`` (hardware.py:136-140) resolved into a dense P x P alpha/beta
  matrix when the fleet has pairwise overrides.

All segments of one instance are packed into one 256-byte aligned buffer so a
single host->device copy ships an instance (or a whole batch of instances).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .refapi import FleetError, effective_speed

_EXACT_LIMIT = 2 ** 53
_ALIGN = 256

TABLES_DTYPE = np.dtype([
    ("n", "<i4"), ("p", "<i4"), ("P", "<i4"), ("n_edges", "<i4"), ("flags", "<u4"), ("pad_", "<i4"),
    ("def_alpha", "<f8"), ("def_beta", "<f8"),
    ("flops", "<u8"), ("gpu", "<u8"), ("cpu", "<u8"), ("disk", "<u8"),
    ("pre_flops", "<u8"), ("pre_gpu", "<u8"), ("pre_cpu", "<u8"), ("pre_disk", "<u8"),
    ("edge_ptr", "<u8"), ("edge_src", "<u8"), ("edge_m", "<u8"),
    ("speed", "<u8"), ("cap_gpu", "<u8"), ("cap_cpu", "<u8"), ("cap_disk", "<u8"),
    ("link_alpha", "<u8"), ("link_beta", "<u8"), ("peer_np", "<u8"),
])
assert TABLES_DTYPE.itemsize == C.sizeof(_lib.DmTables)

_PTR_FIELDS = ("flops", "gpu", "cpu", "disk", "pre_flops", "pre_gpu", "pre_cpu", "pre_disk",
               "edge_ptr", "edge_src", "edge_m", "speed", "cap_gpu", "cap_cpu", "cap_disk",
               "link_alpha", "link_beta", "peer_np")


def _exact_column(values) -> tuple[np.ndarray, np.ndarray | None]:
    """float64 column and, when exact arithmetic is guaranteed, int64 prefix."""
    col = np.array([float(v) for v in values], dtype=np.float64)
    exact = True
    total = 0
    ints = []
    for v in values:
        if isinstance(v, bool):
            v = int(v)
        if isinstance(v, int):
            iv = v
        else:
            fv = float(v)
            if not fv.is_integer():
                exact = False
                break
            iv = int(fv)
        ints.append(iv)
        total += abs(iv)
    if not exact or total >= _EXACT_LIMIT:
        return col, None
    pre = np.zeros(len(ints) + 1, dtype=np.int64)
    if ints:
        pre[1:] = np.cumsum(np.array(ints, dtype=np.int64))
    return col, pre


@dataclass
class HostTables:
    """One (stages, fleet, include_comm) instance in SoA form (host memory)."""

    n: int
    p: int
    P: int
    flags: int
    def_alpha: float
    def_beta: float
    peer_ids: tuple          # index -> peer id (workers first)
    index_of: dict           # peer id -> index
    arrays: dict = field(default_factory=dict)

    @property
    def workers(self) -> tuple:
        return self.peer_ids[: self.p]

    def segments(self):
        """(name, ndarray) in a fixed order."""
        return [(k, self.arrays[k]) for k in _PTR_FIELDS if self.arrays.get(k) is not None]

    def packed_size(self) -> int:
        size = 0
        for _, a in self.segments():
            size = (size + _ALIGN - 1) // _ALIGN * _ALIGN + a.nbytes
        return (size + _ALIGN - 1) // _ALIGN * _ALIGN

    def pack_into(self, buf: np.ndarray, base: int) -> dict:
        """Copy the segments into buf[base:], return name -> byte offset."""
        off = base
        offsets = {}
        for name, a in self.segments():
            off = (off + _ALIGN - 1) // _ALIGN * _ALIGN
            raw = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
            buf[off: off + raw.size] = raw
            offsets[name] = off
            off += raw.size
        return offsets

    def struct_record(self, offsets: dict, dev_base: int) -> np.void:
        rec = np.zeros((), dtype=TABLES_DTYPE)
        rec["n"], rec["p"], rec["P"] = self.n, self.p, self.P
        rec["n_edges"] = int(self.arrays["edge_src"].size)
        rec["flags"] = self.flags
        rec["def_alpha"], rec["def_beta"] = self.def_alpha, self.def_beta
        for name in _PTR_FIELDS:
            rec[name] = dev_base + offsets[name] if name in offsets else 0
        return rec


def build_host(stages, fleet, include_comm: bool = True) -> HostTables:
    """Tensorise one instance on the host (O(n + E + P + |links|))."""
    stages = list(stages)
    n = len(stages)
    workers = tuple(fleet.worker_ids())
    wset = set(workers)
    others = tuple(pid for pid in fleet.peer_ids() if pid not in wset)
    order = workers + others
    index_of = {pid: i for i, pid in enumerate(order)}
    P = len(order)

    flops, pre_flops = _exact_column([s.flops for s in stages])
    gpu, pre_gpu = _exact_column([s.gpu_bytes for s in stages])
    cpu, pre_cpu = _exact_column([s.cpu_bytes for s in stages])
    disk, pre_disk = _exact_column([s.disk_bytes for s in stages])
    bytes_exact = pre_gpu is not None and pre_cpu is not None and pre_disk is not None

    edge_ptr = np.zeros(n + 1, dtype=np.int32)
    srcs, ms = [], []
    is_chain, backward = True, False
    ratio = fleet.msg_ratio
    for i, st in enumerate(stages):
        for src, nbytes in st.in_edges:
            src = int(src)
            if include_comm and not 0 <= src < n:
                raise KeyError(src)
            m = nbytes * ratio                   # CPython float product, as :168
            if include_comm and m < 0:
                raise FleetError("message size must be nonnegative")
            srcs.append(src)
            ms.append(float(m))
            if src != i - 1:
                is_chain = False
            if src >= i:
                backward = True
        edge_ptr[i + 1] = len(srcs)
    edge_src = np.array(srcs, dtype=np.int32)
    edge_m = np.array(ms, dtype=np.float64)

    peers = [fleet.peers[pid] for pid in order]
    speeds = [effective_speed(pe) for pe in peers]
    speed = np.array(speeds, dtype=np.float64)
    # CPython's sum() is compensated only over exact `float` items
    peer_np = np.array([0 if type(v) in (int, float, bool) else 1 for v in speeds] or [0], dtype=np.uint8)
    def _np(v):
        return type(v) not in (int, float, bool)
    np_flops = any(_np(s.flops) for s in stages)
    np_bytes = any(_np(s.gpu_bytes) or _np(s.cpu_bytes) or _np(s.disk_bytes) for s in stages)
    np_comm = (_np(fleet.msg_ratio) or _np(fleet.default_link.alpha) or _np(fleet.default_link.beta)
               or any(_np(lk.alpha) or _np(lk.beta) for lk in fleet.links.values())
               or any(_np(nb) for s in stages for _, nb in s.in_edges))
    cap_gpu = np.array([float(pe.gpu_bytes) for pe in peers], dtype=np.float64)
    cap_cpu = np.array([float(pe.cpu_bytes) for pe in peers], dtype=np.float64)
    cap_disk = np.array([float(pe.disk_bytes) for pe in peers], dtype=np.float64)

    d = fleet.default_link
    flags = 0
    link_alpha = link_beta = None
    if fleet.links:
        la = np.full((P, P), float(d.alpha), dtype=np.float64)
        lb = np.full((P, P), float(d.beta), dtype=np.float64)
        direct = set()
        for (a, b), lk in fleet.links.items():
            ia, ib = index_of.get(str(a)), index_of.get(str(b))
            if ia is None or ib is None:
                continue
            direct.add((ia, ib))
        for (a, b), lk in fleet.links.items():   # links[(a,b)] wins over links[(b,a)]
            ia, ib = index_of.get(str(a)), index_of.get(str(b))
            if ia is None or ib is None:
                continue
            la[ia, ib], lb[ia, ib] = lk.alpha, lk.beta
            if (ib, ia) not in direct:
                la[ib, ia], lb[ib, ia] = lk.alpha, lk.beta
        np.fill_diagonal(la, 0.0)
        np.fill_diagonal(lb, 0.0)
        link_alpha, link_beta = la.reshape(-1), lb.reshape(-1)
        flags |= _lib.DM_F_PAIR_LINKS

    if pre_flops is not None:
        flags |= _lib.DM_F_FLOPS_EXACT
    if bytes_exact:
        flags |= _lib.DM_F_BYTES_EXACT
    if is_chain:
        flags |= _lib.DM_F_CHAIN
    if backward:
        flags |= _lib.DM_F_BACKWARD
    if include_comm:
        flags |= _lib.DM_F_INCLUDE_COMM
    flags |= (_lib.DM_F_NP_FLOPS if np_flops else 0) | (_lib.DM_F_NP_BYTES if np_bytes else 0)
    flags |= _lib.DM_F_NP_COMM if np_comm else 0

    zero_pre = np.zeros(n + 1, dtype=np.int64)
    arrays = dict(flops=flops, gpu=gpu, cpu=cpu, disk=disk,
                  pre_flops=pre_flops if pre_flops is not None else zero_pre,
                  pre_gpu=pre_gpu if bytes_exact else zero_pre,
                  pre_cpu=pre_cpu if bytes_exact else zero_pre,
                  pre_disk=pre_disk if bytes_exact else zero_pre,
                  edge_ptr=edge_ptr, edge_src=edge_src if edge_src.size else np.zeros(1, np.int32),
                  edge_m=edge_m if edge_m.size else np.zeros(1, np.float64),
                  speed=speed, cap_gpu=cap_gpu, cap_cpu=cap_cpu, cap_disk=cap_disk,
                  link_alpha=link_alpha, link_beta=link_beta, peer_np=peer_np)
    return HostTables(n=n, p=len(workers), P=P, flags=flags, def_alpha=float(d.alpha),
                      def_beta=float(d.beta), peer_ids=order, index_of=index_of, arrays=arrays)


class DeviceBatch:
    """One or more HostTables resident on a CUDA device.

    ``struct(i)`` is the ctypes dm_tables (device pointers) of instance i,
    ``structs_dev`` a device array of all records (for the batched kernels)."""

    def __init__(self, hosts, device="cuda", stream=None, pin: bool = True):
        import torch

        hosts = list(hosts)
        self.hosts = hosts
        sizes = [h.packed_size() for h in hosts]
        total = sum(sizes) + _ALIGN
        # pinned staging for long-lived batches (re-uploaded every step by the
        # end-to-end benchmark); small per-call batches use pageable memory,
        # whose synchronous copy is cheaper than a cudaHostAlloc
        self.host_buf = torch.empty(total, dtype=torch.uint8, pin_memory=pin)
        hb = self.host_buf.numpy()
        offs = []
        base = 0
        for h, sz in zip(hosts, sizes):
            offs.append(h.pack_into(hb, base))
            base += sz
        self.nbytes = base
        self.dev_buf = torch.empty(total, dtype=torch.uint8, device=device)
        self.dev_buf.copy_(self.host_buf, non_blocking=True)
        dev_base = int(self.dev_buf.data_ptr())
        recs = np.zeros(len(hosts), dtype=TABLES_DTYPE)
        for i, (h, o) in enumerate(zip(hosts, offs)):
            recs[i] = h.struct_record(o, dev_base)
        self.records = recs
        self.records_host = torch.from_numpy(recs.view(np.uint8).copy())
        if pin:
            self.records_host = self.records_host.pin_memory()
        self.structs_dev = torch.empty(recs.nbytes, dtype=torch.uint8, device=device)
        self.structs_dev.copy_(self.records_host, non_blocking=True)
        self.h2d_bytes = total + recs.nbytes

    def struct(self, i: int = 0) -> _lib.DmTables:
        return _lib.DmTables.from_buffer_copy(self.records[i].tobytes())

    def struct_ptr(self) -> int:
        return int(self.structs_dev.data_ptr())
