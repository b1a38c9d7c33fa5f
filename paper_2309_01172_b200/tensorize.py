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


class _StageSide:
    """Fleet-independent part of an instance: stage columns, exact prefixes,
    CSR in-edges with the raw message sizes, structural flags."""

    __slots__ = ("stages", "n", "flops", "pre_flops", "gpu", "pre_gpu", "cpu", "pre_cpu", "disk", "pre_disk",
                 "bytes_exact", "edge_ptr", "edge_src", "nbytes", "nbytes_f64", "is_chain", "backward",
                 "np_flops", "np_bytes", "np_edges", "src_range_ok", "byte_pre")

    def __init__(self, stages):
        self.stages = stages                      # keeps the (immutable) Stage objects alive: ids stay unique
        n = self.n = len(stages)
        self.flops, self.pre_flops = _exact_column([s.flops for s in stages])
        self.gpu, self.pre_gpu = _exact_column([s.gpu_bytes for s in stages])
        self.cpu, self.pre_cpu = _exact_column([s.cpu_bytes for s in stages])
        self.disk, self.pre_disk = _exact_column([s.disk_bytes for s in stages])
        self.bytes_exact = self.pre_gpu is not None and self.pre_cpu is not None and self.pre_disk is not None
        edge_ptr = np.zeros(n + 1, dtype=np.int32)
        srcs, nbs = [], []
        is_chain, backward, ok = True, False, True
        for i, st in enumerate(stages):
            for src, nbytes in st.in_edges:
                src = int(src)
                ok &= 0 <= src < n
                srcs.append(src)
                nbs.append(nbytes)
                is_chain &= src == i - 1
                backward |= src >= i
            edge_ptr[i + 1] = len(srcs)
        self.edge_ptr, self.edge_src = edge_ptr, np.array(srcs, dtype=np.int32)
        self.nbytes = nbs
        # int message sizes below 2^53 multiply like CPython's int * float
        self.nbytes_f64 = (np.array(nbs, dtype=np.float64)
                           if all(type(v) is int and abs(v) < _EXACT_LIMIT for v in nbs) else None)
        self.is_chain, self.backward, self.src_range_ok = is_chain, backward, ok

        def _np(v):
            return type(v) not in (int, float, bool)
        # per byte column: int when every value is a Python int, float when
        # every value is a Python float, else None (range_bytes falls back)
        def _kind(vals):
            if all(type(v) is int for v in vals):
                return int
            if all(type(v) is float for v in vals):
                return float
            return None
        kinds = tuple(_kind([getattr(s_, a) for s_ in stages]) for a in ("gpu_bytes", "cpu_bytes", "disk_bytes"))
        pres = (self.pre_gpu, self.pre_cpu, self.pre_disk)
        # Python-int prefixes (fast scalar access) and result types, or None
        self.byte_pre = (tuple(pr.tolist() for pr in pres) + kinds
                         if all(pr is not None for pr in pres) and all(k is not None for k in kinds) else None)
        self.np_flops = any(_np(s.flops) for s in stages)
        self.np_bytes = any(_np(s.gpu_bytes) or _np(s.cpu_bytes) or _np(s.disk_bytes) for s in stages)
        self.np_edges = any(_np(nb) for nb in nbs)


    def range_bytes(self, a: int, b: int):
        """(Σ gpu_bytes, Σ cpu_bytes, Σ disk_bytes) over stages [a, b) with
        the value and type of the reference's sum() of the attributes
        (scheduling.py:228-230), from the exact prefixes; None when a column
        has no exact prefix or mixes types."""
        bp = self.byte_pre
        if bp is None:
            return None
        g, c, d, kg, kc, kd = bp
        return kg(g[b] - g[a]), kc(c[b] - c[a]), kd(d[b] - d[a])


_STAGE_CACHE: dict = {}
_STAGE_CACHE_MAX = 256


def _stage_side(stages) -> _StageSide:
    """Cached by the identity of the Stage objects: Stage is a frozen
    dataclass, so an instance's columns never change, and the cache entry
    holds the objects so their ids cannot be reused while cached.  (Fleet is
    mutable — its side is rebuilt every call.)"""
    key = tuple(map(id, stages))
    side = _STAGE_CACHE.get(key)
    if side is None:
        side = _StageSide(stages)
        if len(_STAGE_CACHE) >= _STAGE_CACHE_MAX:
            _STAGE_CACHE.pop(next(iter(_STAGE_CACHE)))
        _STAGE_CACHE[key] = side
    return side


def stage_side(stages) -> _StageSide:
    """Fleet-independent tables of a stage list (cached for frozen Stage objects)."""
    stages = list(stages)
    params = getattr(type(stages[0]), "__dataclass_params__", None) if stages else None
    return _stage_side(stages) if params is not None and params.frozen else _StageSide(stages)


def build_host(stages, fleet, include_comm: bool = True, link_pairs=None, workers=None) -> HostTables:
    """Tensorise one instance on the host (O(n + E + P + |links|); the stage
    side is cached per stage list).  ``link_pairs`` (peer-index pairs) limits
    the pairwise link matrix to the entries a caller's kernels will read
    (resolved with the fleet's own link_between, hardware.py:136-140; the
    rest holds the default link) instead of every override.  ``workers``:
    the caller's fleet.worker_ids() (the sort is not repeated)."""
    stages = list(stages)
    st = stage_side(stages)
    n = st.n
    workers = tuple(fleet.worker_ids() if workers is None else workers)
    if len(workers) == len(fleet.peers):
        order = workers
    else:
        wset = set(workers)
        order = workers + tuple(pid for pid in fleet.peer_ids() if pid not in wset)
    index_of = {pid: i for i, pid in enumerate(order)}
    P = len(order)

    ratio = fleet.msg_ratio
    if st.nbytes_f64 is not None and type(ratio) is float:
        edge_m = st.nbytes_f64 * ratio                  # = CPython's nbytes * msg_ratio (:168), exact int -> float
    else:
        edge_m = np.array([float(nb * ratio) for nb in st.nbytes], dtype=np.float64)
    if include_comm and (not st.src_range_ok or (edge_m.size and (edge_m < 0).any())):
        for s_ in stages:                               # the first offending edge decides the error
            for src, nbytes in s_.in_edges:
                if not 0 <= int(src) < n:
                    raise KeyError(int(src))
                if nbytes * ratio < 0:
                    raise FleetError("message size must be nonnegative")

    peers = [fleet.peers[pid] for pid in order]
    speeds = [effective_speed(pe) for pe in peers]
    speed = np.array(speeds, dtype=np.float64)
    # CPython's sum() is compensated only over exact `float` items
    peer_np = np.array([0 if type(v) in (int, float, bool) else 1 for v in speeds] or [0], dtype=np.uint8)

    def _np(v):
        return type(v) not in (int, float, bool)
    np_comm = _np(ratio) or _np(fleet.default_link.alpha) or _np(fleet.default_link.beta) or st.np_edges
    cap_gpu = np.array([float(pe.gpu_bytes) for pe in peers], dtype=np.float64)
    cap_cpu = np.array([float(pe.cpu_bytes) for pe in peers], dtype=np.float64)
    cap_disk = np.array([float(pe.disk_bytes) for pe in peers], dtype=np.float64)

    d = fleet.default_link
    flags = 0
    link_alpha = link_beta = None
    if fleet.links:
        la = np.full((P, P), float(d.alpha), dtype=np.float64)
        lb = np.full((P, P), float(d.beta), dtype=np.float64)
        if link_pairs is not None:
            for ia, ib in link_pairs:
                if ia != ib:
                    lk = fleet.link_between(order[ia], order[ib])
                    la[ia, ib], lb[ia, ib] = lk.alpha, lk.beta
                    np_comm = np_comm or _np(lk.alpha) or _np(lk.beta)
        else:
            ia_l, ib_l, al_l, be_l = [], [], [], []
            get = index_of.get
            for (a, b), lk in fleet.links.items():
                ia, ib = get(a if type(a) is str else str(a)), get(b if type(b) is str else str(b))
                al, be = lk.alpha, lk.beta
                if type(al) is not float or type(be) is not float:
                    np_comm = np_comm or _np(al) or _np(be)
                if ia is None or ib is None:
                    continue
                ia_l.append(ia)
                ib_l.append(ib)
                al_l.append(al)
                be_l.append(be)
            if ia_l:
                ia_a, ib_a = np.array(ia_l, np.int64), np.array(ib_l, np.int64)
                al_a, be_a = np.array(al_l, np.float64), np.array(be_l, np.float64)
                la[ib_a, ia_a], lb[ib_a, ia_a] = al_a, be_a      # links[(b, a)] serves (a, b) ...
                la[ia_a, ib_a], lb[ia_a, ib_a] = al_a, be_a      # ... unless links[(a, b)] exists
        np.fill_diagonal(la, 0.0)
        np.fill_diagonal(lb, 0.0)
        link_alpha, link_beta = la.reshape(-1), lb.reshape(-1)
        flags |= _lib.DM_F_PAIR_LINKS

    if st.pre_flops is not None:
        flags |= _lib.DM_F_FLOPS_EXACT
    if st.bytes_exact:
        flags |= _lib.DM_F_BYTES_EXACT
    if st.is_chain:
        flags |= _lib.DM_F_CHAIN
    if st.backward:
        flags |= _lib.DM_F_BACKWARD
    if include_comm:
        flags |= _lib.DM_F_INCLUDE_COMM
    flags |= (_lib.DM_F_NP_FLOPS if st.np_flops else 0) | (_lib.DM_F_NP_BYTES if st.np_bytes else 0)
    flags |= _lib.DM_F_NP_COMM if np_comm else 0

    zero_pre = np.zeros(n + 1, dtype=np.int64)
    arrays = dict(flops=st.flops, gpu=st.gpu, cpu=st.cpu, disk=st.disk,
                  pre_flops=st.pre_flops if st.pre_flops is not None else zero_pre,
                  pre_gpu=st.pre_gpu if st.bytes_exact else zero_pre,
                  pre_cpu=st.pre_cpu if st.bytes_exact else zero_pre,
                  pre_disk=st.pre_disk if st.bytes_exact else zero_pre,
                  edge_ptr=st.edge_ptr, edge_src=st.edge_src if st.edge_src.size else np.zeros(1, np.int32),
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

    def repack(self, hosts) -> bool:
        """Re-tensorised instances of the same shapes into the existing pinned
        staging buffer and records (the device addresses stay valid, so a
        captured graph that copies host_buf -> dev_buf can be replayed on the
        new inputs).  Returns False when a shape or a scalar field of a record
        differs (the caller then builds a new batch / graph)."""
        hosts = list(hosts)
        if len(hosts) != len(self.hosts) or any(a.packed_size() != b.packed_size() for a, b in zip(hosts, self.hosts)):
            return False
        # kernels receive dm_tables BY VALUE: a captured graph holds the scalar
        # fields (sizes, flags, default link) of the records it was captured
        # with, so only the device-resident columns may change
        for a, b in zip(hosts, self.hosts):
            if (a.n, a.p, a.P, a.flags, a.def_alpha, a.def_beta, int(a.arrays["edge_src"].size)) != \
                    (b.n, b.p, b.P, b.flags, b.def_alpha, b.def_beta, int(b.arrays["edge_src"].size)):
                return False
        hb = self.host_buf.numpy()
        base = 0
        dev_base = int(self.dev_buf.data_ptr())
        recs = self.records_host.numpy().view(TABLES_DTYPE)
        for i, h in enumerate(hosts):
            offs = h.pack_into(hb, base)
            recs[i] = h.struct_record(offs, dev_base)
            base += h.packed_size()
        self.records = recs.copy()
        self.hosts = hosts
        return True

    def struct(self, i: int = 0) -> _lib.DmTables:
        return _lib.DmTables.from_buffer_copy(self.records[i].tobytes())

    def struct_ptr(self) -> int:
        return int(self.structs_dev.data_ptr())
