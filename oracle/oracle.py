"""ctypes front of the CPU oracle (oracle/dm_oracle.c).

*** TEST INFRASTRUCTURE ONLY *** — imported by tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs, never by the product package.

The instance tables are built here independently of the product's
tensoriser (paper_2309_01172_b200/tensorize.py) so a tensorisation bug cannot
hide behind a shared helper: this builder follows the reference objects
field by field (scheduling.Stage, hardware.Fleet / Peer / Link,
link_between precedence hardware.py:136-140).
"""

from __future__ import annotations

import ctypes as C
import math
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

DM_F_FLOPS_EXACT, DM_F_BYTES_EXACT, DM_F_PAIR_LINKS = 1, 2, 4
DM_F_CHAIN, DM_F_BACKWARD, DM_F_INCLUDE_COMM = 8, 16, 32
DM_F_NP_FLOPS, DM_F_NP_COMM, DM_F_NP_BYTES = 64, 128, 256

_P = C.c_void_p


class Tables(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("p", C.c_int32), ("P", C.c_int32), ("n_edges", C.c_int32),
        ("flags", C.c_uint32), ("pad_", C.c_int32),
        ("def_alpha", C.c_double), ("def_beta", C.c_double),
        ("flops", _P), ("gpu", _P), ("cpu", _P), ("disk", _P),
        ("pre_flops", _P), ("pre_gpu", _P), ("pre_cpu", _P), ("pre_disk", _P),
        ("edge_ptr", _P), ("edge_src", _P), ("edge_m", _P),
        ("speed", _P), ("cap_gpu", _P), ("cap_cpu", _P), ("cap_disk", _P),
        ("link_alpha", _P), ("link_beta", _P), ("peer_np", _P),
    ]


class Winner(C.Structure):
    _fields_ = [("makespan", C.c_double), ("rank", C.c_int64), ("n_evaluated", C.c_int64),
                ("n_feasible", C.c_int64), ("checksum", C.c_uint64)]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        L.or_py_sum.restype = C.c_double
        L.or_py_sum.argtypes = [_P, C.c_int64]
        L.or_eval_runs.restype = C.c_int
        L.or_eval_runs.argtypes = [_P, C.c_int, _P, _P, _P, _P, _P, _P, _P, _P]
        L.or_verify_runs.restype = C.c_int
        L.or_verify_runs.argtypes = [_P, C.c_int, _P, _P, _P, _P]
        L.or_eval_owner.restype = C.c_int
        L.or_eval_owner.argtypes = [_P, _P, _P]
        L.or_enum.restype = None
        L.or_enum.argtypes = [_P, C.c_int, C.c_int64, C.c_int64, _P]
        L.or_unrank.restype = C.c_int
        L.or_unrank.argtypes = [_P, C.c_int, C.c_int64, _P, _P]
        L.or_random_candidate.restype = C.c_int
        L.or_random_candidate.argtypes = [C.c_int, C.c_int32, C.c_uint64, C.c_int64, _P, _P]
        L.or_enum_random.restype = None
        L.or_enum_random.argtypes = [_P, C.c_int32, _P, C.c_uint64, C.c_int64, C.c_int64, _P]
        L.or_subset_dp.restype = C.c_int
        L.or_subset_dp.argtypes = [_P, _P, _P]
        L.or_proportional.restype = C.c_int
        L.or_proportional.argtypes = [_P, _P]
        L.or_hill_climb.restype = C.c_int
        L.or_hill_climb.argtypes = [_P, C.c_int, _P, _P, C.c_int, _P]
        L.or_schedule.restype = C.c_int
        L.or_schedule.argtypes = [_P, C.c_int, _P]
        L.or_epilogue.restype = None
        L.or_epilogue.argtypes = [C.c_int, _P, _P, _P, C.c_int64, C.c_int64, _P]
        L.or_mitm_table.restype = None
        L.or_mitm_table.argtypes = [_P, _P]
        L.or_splits_mitm.restype = C.c_int64
        L.or_splits_mitm.argtypes = [_P, _P, C.c_int, C.c_int, _P]
        L.or_py_sum_items.restype = C.c_double
        L.or_py_sum_items.argtypes = [_P, _P, C.c_int64]
        _lib = L
    return _lib


def _ptr(a):
    return 0 if a is None else a.ctypes.data


def _sort_key(pid):
    s = str(pid)
    return (0, int(s), "") if s.isdigit() else (1, 0, s)


class Instance:
    """Oracle-side tables of one (stages, fleet, include_comm) instance."""

    def __init__(self, stages, fleet, include_comm=True):
        stages = list(stages)
        self.stages = stages
        self.fleet = fleet
        n = len(stages)
        pids = sorted(fleet.peers, key=_sort_key)
        backups = set(fleet.backup_pool)
        workers = [q for q in pids if q not in backups]
        order = workers + [q for q in pids if q in backups]
        self.order = order
        self.workers = workers
        self.idx = {q: i for i, q in enumerate(order)}
        P = len(order)

        def column(vals):
            col = np.array([float(v) for v in vals], dtype=np.float64)
            ok = all(float(v).is_integer() for v in vals) and sum(abs(int(float(v))) for v in vals) < 2 ** 53
            pre = np.zeros(n + 1, dtype=np.int64)
            if ok and n:
                pre[1:] = np.cumsum([int(float(v)) for v in vals])
            return col, pre, ok

        self.flops, self.pre_flops, fex = column([s.flops for s in stages])
        self.gpu, self.pre_gpu, g_ok = column([s.gpu_bytes for s in stages])
        self.cpu, self.pre_cpu, c_ok = column([s.cpu_bytes for s in stages])
        self.disk, self.pre_disk, d_ok = column([s.disk_bytes for s in stages])
        ptr = [0]
        src, m = [], []
        chain, backward = True, False
        for i, s in enumerate(stages):
            for a, nb in s.in_edges:
                src.append(int(a))
                m.append(float(nb * fleet.msg_ratio))
                chain &= (a == i - 1)
                backward |= (a >= i)
            ptr.append(len(src))
        self.edge_ptr = np.array(ptr, dtype=np.int32)
        self.edge_src = np.array(src or [0], dtype=np.int32)
        self.edge_m = np.array(m or [0.0], dtype=np.float64)
        peers = [fleet.peers[q] for q in order]
        sp = [pe.peak_flops * pe.lam for pe in peers]
        self.speed = np.array(sp, dtype=np.float64)
        self.peer_np = np.array([0 if type(v) in (int, float, bool) else 1 for v in sp] or [0], dtype=np.uint8)
        isnp = lambda v: type(v) not in (int, float, bool)
        np_flops = any(isnp(s.flops) for s in stages)
        np_bytes = any(isnp(s.gpu_bytes) or isnp(s.cpu_bytes) or isnp(s.disk_bytes) for s in stages)
        np_comm = (isnp(fleet.msg_ratio) or isnp(fleet.default_link.alpha) or isnp(fleet.default_link.beta)
                   or any(isnp(l.alpha) or isnp(l.beta) for l in fleet.links.values())
                   or any(isnp(nb) for s in stages for _, nb in s.in_edges))
        self.include_comm = include_comm
        self.np_flops, self.np_comm = np_flops, np_comm
        self.cap_gpu = np.array([float(pe.gpu_bytes) for pe in peers], dtype=np.float64)
        self.cap_cpu = np.array([float(pe.cpu_bytes) for pe in peers], dtype=np.float64)
        self.cap_disk = np.array([float(pe.disk_bytes) for pe in peers], dtype=np.float64)
        flags = DM_F_INCLUDE_COMM if include_comm else 0
        flags |= DM_F_FLOPS_EXACT if fex else 0
        flags |= DM_F_BYTES_EXACT if (g_ok and c_ok and d_ok) else 0
        flags |= DM_F_CHAIN if chain else 0
        flags |= DM_F_BACKWARD if backward else 0
        flags |= (DM_F_NP_FLOPS if np_flops else 0) | (DM_F_NP_BYTES if np_bytes else 0)
        flags |= DM_F_NP_COMM if np_comm else 0
        self.la = self.lb = None
        if fleet.links:
            flags |= DM_F_PAIR_LINKS
            la = np.zeros((P, P))
            lb = np.zeros((P, P))
            for a in range(P):
                for b in range(P):
                    lk = fleet.link_between(order[a], order[b])
                    la[a, b], lb[a, b] = lk.alpha, lk.beta
            self.la, self.lb = la.reshape(-1), lb.reshape(-1)
        t = Tables()
        t.n, t.p, t.P, t.n_edges, t.flags = n, len(workers), P, len(src), flags
        t.def_alpha, t.def_beta = fleet.default_link.alpha, fleet.default_link.beta
        for name in ("flops", "gpu", "cpu", "disk", "pre_flops", "pre_gpu", "pre_cpu", "pre_disk", "edge_ptr",
                     "edge_src", "edge_m", "speed", "cap_gpu", "cap_cpu", "cap_disk"):
            setattr(t, name, _ptr(getattr(self, name)))
        t.link_alpha, t.link_beta = _ptr(self.la), _ptr(self.lb)
        t.peer_np = _ptr(self.peer_np)
        self.t = t
        self.n, self.p, self.P = n, len(workers), P

    # ----------------------------------------------------------- helpers
    def _runs_csr(self, runs):
        unknown = {}
        peer, ptr, idx = [], [0], []
        for pe, ids in runs:
            if pe in self.idx:
                peer.append(self.idx[pe])
            else:
                peer.append(unknown.setdefault(pe, self.P + len(unknown)))
            idx.extend(sorted(ids))
            ptr.append(len(idx))
        return (np.array(peer or [0], np.int32), np.array(ptr, np.int32), np.array(idx or [0], np.int32))

    def load_np(self, runs):
        """Per run (first-stage order, as eval_runs): 1 when _evaluate's
        compute + read (scheduling.py:156-169, 220) is a numpy float — numpy
        speed or FLOPs, or a crossing read priced with numpy link/message
        values.  fp_latency's sum() (pipeline.py:43) turns naive there."""
        runs = sorted(((pe, tuple(sorted(ids))) for pe, ids in runs if ids), key=lambda r: r[1][0])
        out = []
        for pe, ids in runs:
            w = self.idx.get(pe)
            f = (w is not None and bool(self.peer_np[w])) or self.np_flops
            if self.np_comm and self.include_comm:
                inside = set(ids)
                f = f or any(a not in inside for i in ids for a, _ in self.stages[i].in_edges)
            out.append(1 if f else 0)
        return np.array(out, np.uint8)

    def eval_runs(self, runs):
        """(makespan, code, code_run, status, compute[], read[])"""
        runs = tuple(runs)
        peer, ptr, idx = self._runs_csr(runs)
        R = len(runs)
        comp = np.zeros(max(R, 1))
        read = np.zeros(max(R, 1))
        mk = np.zeros(1)
        code = np.zeros(1, np.int32)
        bad = np.zeros(1, np.int32)
        st = lib().or_eval_runs(C.byref(self.t), R, _ptr(peer), _ptr(ptr), _ptr(idx), _ptr(comp), _ptr(read),
                                _ptr(mk), _ptr(code), _ptr(bad))
        return float(mk[0]), int(code[0]), int(bad[0]), int(st), comp[:R], read[:R]

    def eval_owner(self, owner_row):
        o = np.ascontiguousarray(owner_row, dtype=np.int32)
        mk = np.zeros(1)
        code = lib().or_eval_owner(C.byref(self.t), _ptr(o), _ptr(mk))
        return float(mk[0]), int(code)

    def enum(self, mode, k0, k1):
        w = Winner()
        lib().or_enum(C.byref(self.t), {"bruteforce": 0, "splits": 1}[mode], k0, k1, C.byref(w))
        return dict(makespan=w.makespan, rank=w.rank, n_evaluated=w.n_evaluated, n_feasible=w.n_feasible,
                    checksum=w.checksum)

    def mitm_table(self):
        T = np.empty(self.p * (self.n + 1) * (self.n + 1), np.float64)
        lib().or_mitm_table(C.byref(self.t), _ptr(T))
        return T

    def splits_mitm(self, T, m_lo, m_hi):
        """Identity-split sweep over cut counts [m_lo, m_hi) with the GPU's
        meet-in-the-middle algorithm (or_splits_mitm)."""
        w = Winner()
        lib().or_splits_mitm(C.byref(self.t), _ptr(T), m_lo, m_hi, C.byref(w))
        return dict(makespan=w.makespan, rank=w.rank, n_evaluated=w.n_evaluated, n_feasible=w.n_feasible,
                    checksum=w.checksum)

    def unrank(self, mode, k):
        b = np.zeros(self.n + 2, np.int32)
        p = np.zeros(self.n + 1, np.int32)
        r = lib().or_unrank(C.byref(self.t), {"bruteforce": 0, "splits": 1}[mode], k, _ptr(b), _ptr(p))
        return b[: r + 1].tolist(), p[:r].tolist()

    def enum_random(self, online, seed, k0, k1):
        on = np.ascontiguousarray(online, np.int32)
        w = Winner()
        lib().or_enum_random(C.byref(self.t), on.size, _ptr(on), seed & 0xFFFFFFFFFFFFFFFF, k0, k1, C.byref(w))
        return dict(makespan=w.makespan, rank=w.rank, n_evaluated=w.n_evaluated, n_feasible=w.n_feasible,
                    checksum=w.checksum)

    def random_candidate(self, n_online, seed, k):
        b = np.zeros(self.n + 2, np.int32)
        q = np.zeros(self.n + 1, np.int32)
        r = lib().or_random_candidate(self.n, n_online, seed & 0xFFFFFFFFFFFFFFFF, k, _ptr(b), _ptr(q))
        return b[: r + 1].tolist(), q[:r].tolist()

    def subset_dp(self):
        own = np.full(self.n, -1, np.int32)
        mk = np.zeros(1)
        found = lib().or_subset_dp(C.byref(self.t), _ptr(own), _ptr(mk))
        return (own if found else None), float(mk[0])

    def proportional(self):
        b = np.zeros(self.n + self.p + 2, np.int32)
        r = lib().or_proportional(C.byref(self.t), _ptr(b))
        return b[: r + 1].tolist()

    def hill_climb(self, bounds, peers, rounds=200):
        b = np.array(bounds, np.int32)
        p = np.array(peers, np.int32)
        sc = np.zeros(1)
        moves = lib().or_hill_climb(C.byref(self.t), len(peers), _ptr(b), _ptr(p), rounds, _ptr(sc))
        return b.tolist(), float(sc[0]), int(moves)

    def schedule(self):
        """(path, owner vector of worker indices) — or_schedule semantics."""
        own = np.full(self.n, -1, np.int32)
        path = lib().or_schedule(C.byref(self.t), 1 if self.fleet.links else 0, _ptr(own))
        return path, own

    def owner_to_runs(self, own):
        runs = []
        a = 0
        n = len(own)
        for i in range(1, n + 1):
            if i == n or own[i] != own[a]:
                runs.append((self.workers[int(own[a])], tuple(range(a, i))))
                a = i
        return tuple(runs)


def py_sum(values) -> float:
    a = np.ascontiguousarray(values, dtype=np.float64)
    return float(lib().or_py_sum(_ptr(a), a.size))


def epilogue(compute, read, n_batches, samples_per_batch, np_load=None):
    """np_load[q]: profile q's compute_s + read_s is a numpy float
    (Instance.load_np); None = every load is an exact float."""
    c = np.ascontiguousarray(compute, np.float64)
    r = np.ascontiguousarray(read, np.float64)
    f = None if np_load is None else np.ascontiguousarray(np_load, np.uint8)
    out = np.zeros(4)
    lib().or_epilogue(c.size, _ptr(c), _ptr(r), _ptr(f), n_batches, samples_per_batch, _ptr(out))
    return tuple(float(x) for x in out)


def bruteforce_total(n, p):
    return sum(math.comb(n - 1, r - 1) * math.perm(p, r) for r in range(1, min(n, p) + 1))


def splits_total(n, p):
    return sum(math.comb(n - 1, r - 1) for r in range(1, min(n, p) + 1))
