"""Thin Python front of the C ABI: device buffers, stream handling, result
read-back.  Every function here launches CUDA work through
``libdagmesh_b200.so``; nothing computes cost-model values on the host."""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .tensorize import DeviceBatch, HostTables

_WINNER_BYTES = C.sizeof(_lib.DmWinner)


def _torch():
    import torch
    return torch


def device_batch(hosts, device=None, pin: bool = True) -> DeviceBatch:
    _lib.load()
    torch = _torch()
    return DeviceBatch(hosts, device=device or torch.device("cuda", torch.cuda.current_device()), pin=pin)


def warmup(device=None):
    """Create the CUDA context, load every kernel module and touch the
    allocator once, so the first API call does not pay initialisation."""
    lib = _lib.load()
    torch = _torch()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    ops = C.c_int64(0)
    _lib.check(lib.dm_microbench_fp64(1, sink.data_ptr(), C.byref(ops), _lib.stream_ptr()))
    torch.cuda.synchronize(dev)


# ------------------------------------------------------------ evaluate_runs
def eval_runs(hosts_or_batch, runs_per_cand, *, index: int = 0):
    """Score candidate Runs of ONE instance with dm_eval_runs.

    runs_per_cand: list (one per candidate) of lists of (peer_index, sorted
    tuple of stage indices).  Returns dict of numpy arrays.  A HostTables
    instance goes through the per-thread ScheduleSlot (one H2D of tables and
    runs, one launch, one D2H)."""
    if isinstance(hosts_or_batch, HostTables):
        return schedule_slot().eval_runs(hosts_or_batch, runs_per_cand)
    lib = _lib.load()
    torch = _torch()
    batch = hosts_or_batch
    n_cand = len(runs_per_cand)
    cand_ptr = [0]
    run_peer, run_ptr, run_idx = [], [0], []
    for runs in runs_per_cand:
        for pe, idxs in runs:
            run_peer.append(pe)
            run_idx.extend(idxs)
            run_ptr.append(len(run_idx))
        cand_ptr.append(len(run_peer))
    R = len(run_peer)
    ints = np.concatenate([np.array(cand_ptr, np.int32), np.array(run_peer or [0], np.int32),
                           np.array(run_ptr, np.int32), np.array(run_idx or [0], np.int32)])
    dev = batch.dev_buf.device
    ints_d = torch.from_numpy(ints).to(dev)
    o1 = len(cand_ptr)
    o2 = o1 + max(R, 1)
    o3 = o2 + len(run_ptr)
    out_f = torch.empty(2 * max(R, 1) + n_cand, dtype=torch.float64, device=dev)
    out_i = torch.empty(3 * n_cand, dtype=torch.int32, device=dev)
    base = ints_d.data_ptr()
    st = batch.struct(index)
    s = _lib.stream_ptr()
    _lib.check(lib.dm_eval_runs(C.byref(st), n_cand, base, base + 4 * o1, base + 4 * o2, base + 4 * o3,
                                out_f.data_ptr(), out_f.data_ptr() + 8 * max(R, 1),
                                out_f.data_ptr() + 16 * max(R, 1), out_i.data_ptr(),
                                out_i.data_ptr() + 4 * n_cand, out_i.data_ptr() + 8 * n_cand, s))
    both = torch.cat([out_f.view(torch.int32), out_i]).cpu()      # one D2H copy
    f = both[: out_f.numel() * 2].view(torch.float64).numpy()
    i = both[out_f.numel() * 2:].numpy()
    return dict(compute=f[:R], read=f[max(R, 1): max(R, 1) + R], makespan=f[2 * max(R, 1):],
                code=i[:n_cand], code_run=i[n_cand: 2 * n_cand], status=i[2 * n_cand:],
                cand_ptr=np.array(cand_ptr))


# ---------------------------------------------------------------- scoring
def eval_owner(batch: DeviceBatch, owner, index: int = 0):
    """Mode A: score a device tensor of owner vectors [n_cand, n] (uint8/int16)."""
    lib = _lib.load()
    torch = _torch()
    n_cand = owner.shape[0]
    ob = owner.element_size()
    mk = torch.empty(n_cand, dtype=torch.float64, device=owner.device)
    code = torch.empty(n_cand, dtype=torch.uint8, device=owner.device)
    st = batch.struct(index)
    _lib.check(lib.dm_eval_owner(C.byref(st), n_cand, owner.data_ptr(), ob, mk.data_ptr(), code.data_ptr(),
                                 _lib.stream_ptr()))
    return mk, code


def eval_owner_argmin(batch: DeviceBatch, owner, rank_base: int = 0, bufs=None, out=None, index: int = 0):
    """Mode A with the arg-min fused into the scoring kernel."""
    lib = _lib.load()
    torch = _torch()
    n_cand = owner.shape[0]
    if out is None:
        out = (torch.empty(n_cand, dtype=torch.float64, device=owner.device),
               torch.empty(n_cand, dtype=torch.uint8, device=owner.device))
    bufs = bufs or WinnerBuffers(owner.device)
    st = batch.struct(index)
    _lib.check(lib.dm_eval_owner_argmin(C.byref(st), n_cand, owner.data_ptr(), owner.element_size(),
                                        out[0].data_ptr(), out[1].data_ptr(), rank_base, bufs.out.data_ptr(),
                                        bufs.scratch.data_ptr(), _lib.stream_ptr()))
    return out, bufs


class WinnerBuffers:
    """Device scratch + one device dm_winner record for enumeration calls."""

    def __init__(self, device):
        lib = _lib.load()
        torch = _torch()
        self.scratch = torch.empty(int(lib.dm_enum_scratch_bytes()) + 256, dtype=torch.uint8, device=device)
        self.out = torch.empty(_WINNER_BYTES, dtype=torch.uint8, device=device)
        self.device = device
        self.workspace = None      # split-sweep side tables (dm_splits_workspace_bytes), grown on demand

    def workspace_for(self, nbytes: int):
        if nbytes <= 0:
            return None
        if self.workspace is None or self.workspace.numel() < nbytes:
            self.workspace = _torch().empty(nbytes, dtype=_torch().uint8, device=self.device)
        return self.workspace

    def read(self) -> dict:
        raw = self.out.cpu().numpy().tobytes()
        w = _lib.DmWinner.from_buffer_copy(raw)
        return dict(makespan=w.makespan, rank=w.rank, n_evaluated=w.n_evaluated,
                    n_feasible=w.n_feasible, checksum=w.checksum)


def argmin_scores(mk, code, rank_base: int = 0, bufs: WinnerBuffers | None = None):
    lib = _lib.load()
    bufs = bufs or WinnerBuffers(mk.device)
    _lib.check(lib.dm_argmin_scores(mk.data_ptr(), code.data_ptr(), mk.numel(), rank_base,
                                    bufs.out.data_ptr(), bufs.scratch.data_ptr(), _lib.stream_ptr()))
    return bufs


def enum(batch: DeviceBatch, mode: str, k0: int, k1: int, bufs: WinnerBuffers | None = None,
         index: int = 0, online=None, seed: int = 0, part: int = 0, nparts: int = 1,
         phase: int = 3):
    """Mode B enumeration: 'bruteforce' | 'splits' | 'random'. Returns bufs
    (call bufs.read() to synchronise and fetch the winner).  'splits' takes
    `phase` (dm_enum_splits_phase): 1 = side tables only, 2 = sweep only,
    3 = both; 2 splits into 4 (tile plan) then 8 (sweep kernel)."""
    lib = _lib.load()
    bufs = bufs or WinnerBuffers(batch.dev_buf.device)
    st = batch.struct(index)
    s = _lib.stream_ptr()
    if mode in ("bruteforce", "splits"):              # ranks beyond the population do not exist
        total = (bruteforce_total if mode == "bruteforce" else splits_total)(st.n, st.p)
        k1 = min(k1, total)
        k0 = min(k0, k1)
    if mode == "bruteforce":
        _lib.check(lib.dm_enum_bruteforce(C.byref(st), k0, k1, bufs.out.data_ptr(), bufs.scratch.data_ptr(), s))
    elif mode == "splits":
        need = int(lib.dm_splits_workspace_bytes(C.byref(st)))
        ws = bufs.workspace_for(need)
        _lib.check(lib.dm_enum_splits_phase(C.byref(st), k0, k1, part, nparts, bufs.out.data_ptr(),
                                            bufs.scratch.data_ptr(), ws.data_ptr() if ws is not None else None,
                                            max(need, 0), phase, s))
    elif mode == "random":
        _lib.check(lib.dm_enum_random(C.byref(st), online.data_ptr(), online.numel(), seed & 0xFFFFFFFFFFFFFFFF,
                                      k0, k1, bufs.out.data_ptr(), bufs.scratch.data_ptr(), s))
    else:
        raise ValueError(mode)
    return bufs


# ------------------------------------------------- one-instance API calls
class ScheduleSlot:
    """Reusable device staging for one-instance API calls (schedule()): a
    pinned host buffer and a device buffer for the packed tables plus their
    dm_tables record, the search outputs and the report record — one H2D,
    the kernels, one D2H, one synchronisation per call and no allocation
    once warm.  One slot per (thread, device)."""

    def __init__(self, device):
        self.device = device
        self.cap = 0
        self.n_cap = 0

    def _grow(self, nbytes, n, p):
        torch = _torch()
        lib = _lib.load()
        if nbytes > self.cap:
            self.cap = max(nbytes, 2 * self.cap, 64 * 1024)
            self.host = torch.empty(self.cap, dtype=torch.uint8, pin_memory=True)
            self.dev = torch.empty(self.cap, dtype=torch.uint8, device=self.device)
        if n > self.n_cap or p > getattr(self, "p_cap", 0):
            self.n_cap = max(n, self.n_cap)
            self.p_cap = max(p, getattr(self, "p_cap", 0))
            out_b = int(lib.dm_sched_out_bytes(self.n_cap))
            self.owner = torch.empty(self.n_cap, dtype=torch.int16, device=self.device)
            self.owner2 = torch.empty(self.n_cap, dtype=torch.int16, device=self.device)
            self.vals = torch.empty(2, dtype=torch.float64, device=self.device)
            self.ints = torch.empty(2, dtype=torch.int32, device=self.device)
            self.out = torch.empty(out_b, dtype=torch.uint8, device=self.device)
            self.out_host = torch.empty(out_b, dtype=torch.uint8, pin_memory=True)
            sb = int(lib.dm_subset_dp_scratch_bytes(self.n_cap, min(self.p_cap, 20), 1))
            self.scratch = torch.empty(max(sb, 256), dtype=torch.uint8, device=self.device)

    def upload(self, host: HostTables, extra: np.ndarray | None = None, dev_extra: int = 0):
        """Pack `host`, its dm_tables record and `extra` (int32 payload) into
        the pinned buffer, start one H2D copy; returns (device address of the
        record, struct, device address of the payload, device address of
        `dev_extra` scratch bytes after it)."""
        size = host.packed_size()
        rec_off = (size + 255) // 256 * 256
        ext_off = rec_off + 256
        ext_bytes = 0 if extra is None else extra.nbytes
        scr_off = (ext_off + ext_bytes + 255) // 256 * 256
        self._grow(max(ext_off + ext_bytes, scr_off + dev_extra), host.n, host.p)
        if scr_off + dev_extra > self.dev.numel():
            self.dev = _torch().empty(scr_off + dev_extra, dtype=_torch().uint8, device=self.device)
        hb = self.host.numpy()
        offs = host.pack_into(hb, 0)
        rec = host.struct_record(offs, int(self.dev.data_ptr()))
        hb[rec_off: rec_off + C.sizeof(_lib.DmTables)] = np.frombuffer(rec.tobytes(), np.uint8)
        if extra is not None:
            hb[ext_off: ext_off + ext_bytes] = extra.view(np.uint8).reshape(-1)
        total = ext_off + ext_bytes
        self.dev[:total].copy_(self.host[:total], non_blocking=True)
        base = int(self.dev.data_ptr())
        self.last_struct = _lib.DmTables.from_buffer_copy(rec.tobytes())
        return base + rec_off, base + ext_off, base + scr_off

    def eval_runs(self, host: HostTables, runs_per_cand) -> dict:
        """dm_eval_runs_ws on one instance: tables, record and the runs' CSR in
        one H2D, outputs in one D2H."""
        lib = _lib.load()
        torch = _torch()
        n_cand = len(runs_per_cand)
        cand_ptr = [0]
        run_peer, run_ptr, run_idx = [], [0], []
        for runs in runs_per_cand:
            for pe, idxs in runs:
                run_peer.append(pe)
                run_idx.extend(idxs)
                run_ptr.append(len(run_idx))
            cand_ptr.append(len(run_peer))
        R = len(run_peer)
        ints = np.concatenate([np.array(cand_ptr, np.int32), np.array(run_peer or [0], np.int32),
                               np.array(run_ptr, np.int32), np.array(run_idx or [0], np.int32)])
        o1 = len(cand_ptr)
        o2 = o1 + max(R, 1)
        o3 = o2 + len(run_ptr)
        ws = int(lib.dm_eval_runs_ws_bytes(host.n, n_cand, R))
        ws = (ws + 255) // 256 * 256
        nf = 2 * max(R, 1) + n_cand
        out_bytes = 8 * nf + 4 * 3 * n_cand
        rec, ext, scr = self.upload(host, ints, ws + out_bytes)
        out = scr + ws
        s = _lib.stream_ptr()
        _lib.check(lib.dm_eval_runs_ws(C.byref(self.last_struct), n_cand, ext, ext + 4 * o1, ext + 4 * o2,
                                       ext + 4 * o3, R, out, out + 8 * max(R, 1), out + 16 * max(R, 1),
                                       out + 8 * nf, out + 8 * nf + 4 * n_cand, out + 8 * nf + 8 * n_cand, scr, s))
        if getattr(self, "ev_host", None) is None or self.ev_host.numel() < out_bytes:
            self.ev_host = torch.empty(max(out_bytes, 4096), dtype=torch.uint8, pin_memory=True)
        off = out - int(self.dev.data_ptr())
        self.ev_host[:out_bytes].copy_(self.dev[off: off + out_bytes], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        raw = self.ev_host.numpy()[:out_bytes]
        f = raw[: 8 * nf].view(np.float64)
        i = raw[8 * nf:].view(np.int32)
        return dict(compute=f[:R].copy(), read=f[max(R, 1): max(R, 1) + R].copy(),
                    makespan=f[2 * max(R, 1):].copy(), code=i[:n_cand].copy(), code_run=i[n_cand: 2 * n_cand].copy(),
                    status=i[2 * n_cand:].copy(), cand_ptr=np.array(cand_ptr))

    def schedule(self, host: HostTables, use_dp: bool, hill_after_dp: bool) -> dict:
        """schedule()'s search (scheduling.py:404-419) and the _evaluate of its
        result (:210-232) on the device; returns the decoded report record."""
        lib = _lib.load()
        s = _lib.stream_ptr()
        rec, _, _ = self.upload(host)
        n, p = host.n, host.p
        found = None
        owner = self.owner
        if use_dp:
            found = self.ints
            _lib.check(lib.dm_subset_dp(rec, 1, n, p, owner.data_ptr(), self.vals.data_ptr(), found.data_ptr(),
                                        self.scratch.data_ptr(), s))
            if hill_after_dp:
                _lib.check(lib.dm_prop_hill(rec, 1, n, owner.data_ptr(), None, self.owner2.data_ptr(),
                                            self.vals.data_ptr() + 8, None, s))
                owner = self.owner2
        else:
            _lib.check(lib.dm_prop_hill(rec, 1, n, None, None, owner.data_ptr(), self.vals.data_ptr() + 8, None, s))
        _lib.check(lib.dm_schedule_report(rec, n, owner.data_ptr(), found.data_ptr() if found is not None else None,
                                          self.out.data_ptr(), s))
        ob = int(lib.dm_sched_out_bytes(n))
        self.out_host[:ob].copy_(self.out[:ob], non_blocking=True)
        _torch().cuda.current_stream().synchronize()
        raw = self.out_host.numpy()
        hdr = raw[:16].view(np.int32)
        r = int(hdr[1])
        off_p = 32 + ((n + 1) * 4 + 7) // 8 * 8
        off_c = off_p + (n * 4 + 7) // 8 * 8
        return dict(found=int(hdr[0]), n_runs=r, code=int(hdr[2]), bad_run=int(hdr[3]),
                    makespan=float(raw[16:24].view(np.float64)[0]),
                    bounds=raw[32: 32 + 4 * (r + 1)].view(np.int32).copy(),
                    peers=raw[off_p: off_p + 4 * r].view(np.int32).copy(),
                    compute=raw[off_c: off_c + 8 * r].view(np.float64).copy(),
                    read=raw[off_c + 8 * n: off_c + 8 * n + 8 * r].view(np.float64).copy())


_SLOTS = None


def schedule_slot(device=None) -> ScheduleSlot:
    import threading
    global _SLOTS
    if _SLOTS is None:
        _SLOTS = threading.local()
    torch = _torch()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    slots = getattr(_SLOTS, "by_dev", None)
    if slots is None:
        slots = _SLOTS.by_dev = {}
    key = str(dev)
    if key not in slots:
        slots[key] = ScheduleSlot(dev)
    return slots[key]


# ------------------------------------------------------------ partitioners
def subset_dp(batch: DeviceBatch, n_max: int, p_max: int):
    """Batched _subset_dp over every instance of the batch."""
    lib = _lib.load()
    torch = _torch()
    dev = batch.dev_buf.device
    ns = len(batch.hosts)
    owner = torch.empty((ns, n_max), dtype=torch.int16, device=dev)
    mk = torch.empty(ns, dtype=torch.float64, device=dev)
    found = torch.empty(ns, dtype=torch.int32, device=dev)
    sb = int(lib.dm_subset_dp_scratch_bytes(n_max, p_max, ns))
    if sb < 0:
        raise _lib.EngineError(_lib.DM_E_TOO_LARGE, "subset DP instance too large")
    scratch = torch.empty(max(sb, 256), dtype=torch.uint8, device=dev)
    _lib.check(lib.dm_subset_dp(batch.struct_ptr(), ns, n_max, p_max, owner.data_ptr(), mk.data_ptr(),
                                found.data_ptr(), scratch.data_ptr(), _lib.stream_ptr()))
    return owner, mk, found, scratch


def prop_hill(batch: DeviceBatch, n_max: int, init_owner=None, do_hill=None):
    lib = _lib.load()
    torch = _torch()
    dev = batch.dev_buf.device
    ns = len(batch.hosts)
    owner = torch.empty((ns, n_max), dtype=torch.int16, device=dev)
    score = torch.empty(ns, dtype=torch.float64, device=dev)
    moves = torch.empty(ns, dtype=torch.int32, device=dev)
    _lib.check(lib.dm_prop_hill(batch.struct_ptr(), ns, n_max, _lib.ptr(init_owner), _lib.ptr(do_hill),
                                owner.data_ptr(), score.data_ptr(), moves.data_ptr(), _lib.stream_ptr()))
    return owner, score, moves


def prop_hill_epilogue(batch: DeviceBatch, n_max: int, n_batches: int, samples_per_batch: int, init_owner=None,
                       do_hill=None):
    """Batched schedule() (proportional split + hill climb) and the Eq. 3/4
    epilogue of the final runs in one launch: (owner, score, moves, out[ns, 6])."""
    lib = _lib.load()
    torch = _torch()
    dev = batch.dev_buf.device
    ns = len(batch.hosts)
    owner = torch.empty((ns, n_max), dtype=torch.int16, device=dev)
    score = torch.empty(ns, dtype=torch.float64, device=dev)
    moves = torch.empty(ns, dtype=torch.int32, device=dev)
    out = torch.empty((ns, 6), dtype=torch.float64, device=dev)
    _lib.check(lib.dm_prop_hill_epilogue(batch.struct_ptr(), ns, n_max, _lib.ptr(init_owner), _lib.ptr(do_hill),
                                         owner.data_ptr(), score.data_ptr(), moves.data_ptr(), int(n_batches),
                                         int(samples_per_batch), out.data_ptr(), _lib.stream_ptr()))
    return owner, score, moves, out


def epilogue(batch: DeviceBatch, n_max: int, owner, n_batches: int, samples_per_batch: int):
    lib = _lib.load()
    torch = _torch()
    ns = len(batch.hosts)
    out = torch.empty((ns, 6), dtype=torch.float64, device=batch.dev_buf.device)
    _lib.check(lib.dm_pipeline_epilogue(batch.struct_ptr(), ns, n_max, owner.data_ptr(), int(n_batches),
                                        int(samples_per_batch), out.data_ptr(), _lib.stream_ptr()))
    return out


# ------------------------------------------------------------- rank codecs
def bruteforce_total(n: int, p: int) -> int:
    return sum(math.comb(n - 1, r - 1) * math.perm(p, r) for r in range(1, min(n, p) + 1))


def splits_total(n: int, p: int) -> int:
    return sum(math.comb(n - 1, r - 1) for r in range(1, min(n, p) + 1))


def unrank(n: int, p: int, k: int, mode: str):
    """Global rank -> (bounds, worker indices) in the reference's itertools
    order (scheduling.py:260-264); mode 'bruteforce' or 'splits'."""
    for r in range(1, min(n, p) + 1):
        npm = math.perm(p, r) if mode == "bruteforce" else 1
        blk = math.comb(n - 1, r - 1) * npm
        if k >= blk:
            k -= blk
            continue
        c, pi = divmod(k, npm)
        cuts, lo, m = [], 1, r - 1
        for q in range(m):
            for v in range(lo, n):
                cnt = math.comb(n - 1 - v, m - q - 1)
                if c < cnt:
                    cuts.append(v)
                    lo = v + 1
                    break
                c -= cnt
        if mode == "bruteforce":
            free = list(range(p))
            peers = []
            for q in range(r):
                blkp = math.perm(p - q - 1, r - q - 1)
                d, pi = divmod(pi, blkp)
                peers.append(free.pop(d))
        else:
            peers = list(range(r))
        return [0] + cuts + [n], peers
    raise IndexError(k)


def cross_peak(iters: int = 400, repeats: int = 3) -> float:
    """Measured candidate pairs per second of the split sweep's inner loop
    alone (dm_microbench_cross): the sweep's issue-bound roofline."""
    lib = _lib.load()
    torch = _torch()
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    pairs = C.c_int64(0)
    s = _lib.stream_ptr()
    _lib.check(lib.dm_microbench_cross(4, sink.data_ptr(), C.byref(pairs), s))
    best = 0.0
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.dm_microbench_cross(iters, sink.data_ptr(), C.byref(pairs), s))
        b.record()
        b.synchronize()
        best = max(best, pairs.value / (a.elapsed_time(b) / 1e3))
    return best


class SweepGraph:
    """Whole-population split sweeps captured as one CUDA graph (the serving
    form of `enum(batch, "splits", 0, total)`): the H2D copy of the instance
    tables from pinned host memory, the sweep kernels of every unit and — when
    every unit is a whole population — the D2H copy of the winner records into
    pinned host memory.  A unit is (instance index, part, nparts); the default
    is the single unit (0, part, nparts).  `launch()` replays the graph on the
    current stream; `read()` waits and returns the first unit's winner,
    `read_all()` every unit's.  `out` holds the units' device records
    (uint8[units, 40]) for a multi-GPU all-gather.  copy_inputs=False captures
    the kernels alone (tables already resident, records left in `out`)."""

    def __init__(self, batch: DeviceBatch, total: int, bufs: WinnerBuffers | None = None, part: int = 0,
                 nparts: int = 1, copy_inputs: bool = True, units=None, overlap: bool = True):
        torch = _torch()
        lib = _lib.load()
        self.batch, self.total = batch, total
        self.units = [tuple(u) for u in units] if units is not None else [(0, part, nparts)]
        self.copy_inputs = copy_inputs
        dev = batch.dev_buf.device
        # several units: unit i+1's table phase (side stream) overlaps unit
        # i's sweep (the table kernels are L1/latency bound, the sweep is
        # ALU bound); every unit has its own workspace
        self.overlap = overlap and len(self.units) > 1
        self.side = torch.cuda.Stream(device=dev) if self.overlap else None
        # each unit's one-CTA tile plan on a third stream: it waits for the
        # unit's tables and runs in the previous sweep's tail, neither
        # delaying the sweeps (main) nor holding back the next tables (side)
        self.plan = torch.cuda.Stream(device=dev) if self.overlap else None
        self.unit_bufs = [bufs if (i == 0 and bufs is not None) else WinnerBuffers(dev)
                          for i in range(len(self.units))]
        for (idx, _, _), ub in zip(self.units, self.unit_bufs):
            ub.workspace_for(int(lib.dm_splits_workspace_bytes(C.byref(batch.struct(idx)))))
        self.bufs = self.unit_bufs[0]
        self.whole = all(u[2] == 1 for u in self.units)
        self.out = torch.empty((len(self.units), _WINNER_BYTES), dtype=torch.uint8, device=dev)
        for i, ub in enumerate(self.unit_bufs):      # each unit's record lands in its row directly
            ub.out = self.out[i]
        self.host_out = torch.empty((len(self.units), _WINNER_BYTES), dtype=torch.uint8, pin_memory=True)
        self.h2d_bytes = int(batch.h2d_bytes) if copy_inputs else 0
        self.d2h_bytes = _WINNER_BYTES * len(self.units) if copy_inputs else 0
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):          # warm the plan cache and the kernels' attributes
            self._body()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._body()

    def _body(self):
        torch = _torch()
        b = self.batch
        if self.copy_inputs:
            b.dev_buf.copy_(b.host_buf, non_blocking=True)
            b.structs_dev.copy_(b.records_host, non_blocking=True)
        if self.overlap:
            main = torch.cuda.current_stream()
            self.side.wait_stream(main)
            self.plan.wait_stream(main)
            ready = []
            for (idx, part, nparts), ub in zip(self.units, self.unit_bufs):
                with torch.cuda.stream(self.side):
                    enum(b, "splits", 0, self.total, ub, index=idx, part=part, nparts=nparts, phase=1)
                    tables = torch.cuda.Event()
                    tables.record(self.side)
                with torch.cuda.stream(self.plan):
                    self.plan.wait_event(tables)
                    enum(b, "splits", 0, self.total, ub, index=idx, part=part, nparts=nparts, phase=4)
                    ev = torch.cuda.Event()
                    ev.record(self.plan)
                    ready.append(ev)
            for i, ((idx, part, nparts), ub) in enumerate(zip(self.units, self.unit_bufs)):
                main.wait_event(ready[i])
                enum(b, "splits", 0, self.total, ub, index=idx, part=part, nparts=nparts, phase=8)
            main.wait_stream(self.side)
            main.wait_stream(self.plan)
        else:
            for i, ((idx, part, nparts), ub) in enumerate(zip(self.units, self.unit_bufs)):
                enum(b, "splits", 0, self.total, ub, index=idx, part=part, nparts=nparts)
        if self.copy_inputs:
            self.host_out.copy_(self.out, non_blocking=True)

    def launch(self):
        self.graph.replay()

    def read_all(self) -> list:
        _torch().cuda.current_stream().synchronize()
        raw = self.host_out.numpy().tobytes()
        res = []
        for i in range(len(self.units)):
            w = _lib.DmWinner.from_buffer_copy(raw[i * _WINNER_BYTES:(i + 1) * _WINNER_BYTES])
            res.append(dict(makespan=w.makespan, rank=w.rank, n_evaluated=w.n_evaluated,
                            n_feasible=w.n_feasible, checksum=w.checksum))
        return res

    def read(self) -> dict:
        return self.read_all()[0]


def sweep_kernel_times(batch: DeviceBatch, total: int, steps: int = 5, bufs: WinnerBuffers | None = None,
                       part: int = 0, nparts: int = 1, index: int = 0) -> tuple:
    """Average (table phase ms, sweep kernel ms) of `steps` whole-population
    split sweeps, from CUDA events the library records around its kernels."""
    lib = _lib.load()
    bufs = bufs or WinnerBuffers(batch.dev_buf.device)
    _lib.check(lib.dm_sweep_timing(1, None, None))
    ta = tb = 0.0
    try:
        for _ in range(steps):
            enum(batch, "splits", 0, total, bufs, index=index, part=part, nparts=nparts)
            a, b = C.c_float(0), C.c_float(0)
            _lib.check(lib.dm_sweep_timing(-1, C.byref(a), C.byref(b)))
            ta += a.value
            tb += b.value
    finally:
        lib.dm_sweep_timing(0, None, None)
    return ta / steps, tb / steps


def alu_peak(iters: int = 20000, repeats: int = 3) -> float:
    """Measured ALU-pipe (LOP3) lane-operations per second on the current device."""
    lib = _lib.load()
    torch = _torch()
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    ops = C.c_int64(0)
    s = _lib.stream_ptr()
    _lib.check(lib.dm_microbench_alu(200, sink.data_ptr(), C.byref(ops), s))
    best = 0.0
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.dm_microbench_alu(iters, sink.data_ptr(), C.byref(ops), s))
        b.record()
        b.synchronize()
        best = max(best, ops.value / (a.elapsed_time(b) / 1e3))
    return best


def fp64_peak(iters: int = 20000, repeats: int = 3) -> float:
    """Measured fp64 (DMUL/DADD) operations per second on the current device."""
    lib = _lib.load()
    torch = _torch()
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    ops = C.c_int64(0)
    s = _lib.stream_ptr()
    _lib.check(lib.dm_microbench_fp64(200, sink.data_ptr(), C.byref(ops), s))
    best = 0.0
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.dm_microbench_fp64(iters, sink.data_ptr(), C.byref(ops), s))
        b.record()
        b.synchronize()
        best = max(best, ops.value / (a.elapsed_time(b) / 1e3))
    return best


def materialize(n: int, p: int, mode: str, k0: int, count: int, device="cuda", owner_bytes: int = 1):
    """Owner vectors of candidates [k0, k0+count) (mode 'bruteforce' | 'splits')."""
    lib = _lib.load()
    torch = _torch()
    out = torch.empty((count, n), dtype=torch.uint8 if owner_bytes == 1 else torch.int16, device=device)
    _lib.check(lib.dm_materialize(n, p, {"bruteforce": 0, "splits": 1}[mode], k0, count, out.data_ptr(),
                                  owner_bytes, _lib.stream_ptr()))
    return out
