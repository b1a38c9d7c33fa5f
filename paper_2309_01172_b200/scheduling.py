"""Drop-in replacement of the reference's ``dagmesh.scheduling`` hot path.

Same names, signatures, return types and error behaviour as
pkg/src/dagmesh/scheduling.py:179-474; every cost-model evaluation, search
and arg-min runs as CUDA on the B200 through the C ABI
(include/dagmesh_b200.h).  Host Python only tensorises inputs, launches, and
assembles the ``ScheduleReport`` (formatting the reason string, summing the
byte columns of the chosen runs for the report rows with the reference's
own expressions, so CSV/summary output is byte-identical).

There is no CPU fallback: without the built library or a CUDA device every
call raises ``EngineUnavailable``.
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

from . import _lib, engine
from . import refapi as _model
from .refapi import peer_sort_key
from .tensorize import build_host, stage_side

# Result/error classes; install() points these at the reference's own
# classes so reports built here are instances of dagmesh.scheduling types.
T = SimpleNamespace(ScheduleReport=_model.ScheduleReport, PeerLoad=_model.PeerLoad,
                    SchedulingError=_model.SchedulingError, FleetError=_model.FleetError)

_DIM = {_lib.DM_V_GPU: "gpu", _lib.DM_V_CPU: "cpu", _lib.DM_V_DISK: "disk"}
_INF = math.inf


def _peer_load(*vals):
    """T.PeerLoad(*vals).  The reference's PeerLoad is a frozen dataclass
    with a plain __dict__ and no __post_init__: its generated __init__ sets
    each field with object.__setattr__, so the same object is built by one
    __dict__ update (a report carries one row per worker: 256 on C3).  Any
    other class goes through its constructor."""
    cls = T.PeerLoad
    fields = getattr(cls, "__dataclass_fields__", None)
    if (fields is None or hasattr(cls, "__slots__") or hasattr(cls, "__post_init__")
            or len(fields) != len(vals)):
        return cls(*vals)
    obj = object.__new__(cls)
    obj.__dict__.update(zip(fields, vals))
    return obj


def _check_inputs(stages, workers):
    """scheduling.py:281-285."""
    if not stages:
        raise T.SchedulingError("empty stage list")
    if not workers:
        raise T.SchedulingError("empty fleet: no schedulable peers")


def _encode_runs(host, runs, str_keys: bool = True):
    """Runs -> [(peer index, sorted indices)]; unknown peers get indices >= P
    (distinct per distinct id, so 'holds two runs' and link_between's
    same-peer test keep working).  str_keys: a key that is not a fleet id
    but whose str() is (e.g. int 1 for '1') maps to that peer, as
    fleet.peer() str-converts for costing (hardware.py:122-126); with
    str_keys=False it stays unknown, as verify_assignment's `peer not in
    fleet.peers` sees it (:187-188)."""
    unknown: dict = {}
    out = []
    n = host.n
    for peer, idxs in runs:
        key = peer
        if key in host.index_of:
            pi = host.index_of[key]
        elif str_keys and str(key) in host.index_of:
            pi = host.index_of[str(key)]
        else:
            pi = unknown.setdefault(key, host.P + len(unknown))
        sidx = tuple(sorted(idxs))
        for i in sidx:
            if not 0 <= i < n:
                raise IndexError("list index out of range")
        out.append((pi, sidx))
    return out


def _mixed_keys(host, runs) -> bool:
    return any(peer not in host.index_of and str(peer) in host.index_of for peer, _ in runs)


def _raise_cost_error(stages, fleet, runs, include_comm):
    """Re-derive which exception the reference raises first while costing
    (ordered runs, scheduling.py:217-221): FleetError for an unknown run peer,
    KeyError for a crossing edge from an unassigned stage."""
    peer_of = {i: peer for peer, idxs in runs for i in idxs}
    ordered = sorted(((p, tuple(sorted(i))) for p, i in runs if i), key=lambda r: r[1][0])
    for peer, idxs in ordered:
        if str(peer) not in fleet.peers:
            raise T.FleetError(f"unknown peer {peer!r}")
        if include_comm:
            inside = set(idxs)
            for i in idxs:
                for src, _ in stages[i].in_edges:
                    if src not in inside and src not in peer_of:
                        raise KeyError(src)
    raise RuntimeError("engine reported a costing error the host cannot reproduce")


def _reason(stages, fleet, runs, code, bad):
    """verify_assignment's message for violation `code` at run `bad`
    (scheduling.py:179-207)."""
    if code == _lib.DM_V_OK:
        return ""
    if code == _lib.DM_V_UNASSIGNED:
        seen = {i for _, idxs in runs for i in idxs}
        missing = sorted(set(range(len(stages))) - seen)
        return f"stages {[m + 1 for m in missing]} unassigned"
    peer, indices = runs[bad]
    ordered = sorted(indices)
    if code == _lib.DM_V_TWO_RUNS:
        return f"peer {peer} holds two runs"
    if code == _lib.DM_V_UNKNOWN_PEER:
        return f"unknown peer {peer}"
    if code == _lib.DM_V_NOT_CONTIGUOUS:
        return f"peer {peer} run {ordered} is not contiguous"
    if code == _lib.DM_V_ASSIGNED_TWICE:
        before = {i for _, idxs in runs[:bad] for i in idxs}
        for i in ordered:
            if i in before:
                return f"stage {i + 1} assigned twice"
        return "stage assigned twice"
    dim = _DIM[code]
    p = fleet.peer(peer)
    cap = getattr(p, f"{dim}_bytes")
    used = sum(getattr(stages[i], f"{dim}_bytes") for i in ordered)
    return f"peer {peer} exceeds {dim} capacity: {used:.0f} > {cap:.0f} bytes"


def _cost_types(host, stages, peer, indices, include_comm):
    """Python types of _run_cost's (compute, read) (scheduling.py:156-169):
    numpy.float64 where the reference's arithmetic meets a numpy operand —
    a numpy speed or FLOP count for compute, a crossing read priced with
    numpy message/link values for read.  Later sum()s over these values
    (fp_latency, pipeline.py:43) are compensated only over exact floats, so
    the report carries the same types as the reference's."""
    f = host.flags
    pi = host.index_of.get(peer)
    cnp = bool(f & _lib.DM_F_NP_FLOPS) or (pi is not None and bool(host.arrays["peer_np"][pi]))
    rnp = False
    if include_comm and f & _lib.DM_F_NP_COMM:
        inside = set(indices)
        rnp = any(src not in inside for i in indices for src, _ in stages[i].in_edges)
    return cnp, rnp


def _report(stages, fleet, runs, include_comm, trace, res, c=0, host=None):
    """Assemble the ScheduleReport of candidate c from device results
    (scheduling.py:210-232)."""
    lo = int(res["cand_ptr"][c])
    code = int(res["code"][c])
    reason = _reason(stages, fleet, runs, code, int(res["code_run"][c]))
    comp = {}
    for r, (peer, idxs) in enumerate(runs):
        if idxs:
            comp[r] = (float(res["compute"][lo + r]), float(res["read"][lo + r]))
    order = sorted((r for r, (_, i) in enumerate(runs) if i), key=lambda r: min(runs[r][1]))
    rows, ordered_runs = [], []
    typed = host is not None and (bool(host.flags & (_lib.DM_F_NP_FLOPS | _lib.DM_F_NP_COMM))
                                  or bool(host.arrays["peer_np"].any()))
    makespan = 0.0
    side = stage_side(stages) if stages else None
    for r in order:
        peer, idxs = runs[r]
        indices = tuple(sorted(idxs))
        compute, read = comp[r]
        if typed:
            cnp, rnp = _cost_types(host, stages, peer, indices, include_comm)
            compute = np.float64(compute) if cnp else compute
            read = np.float64(read) if rnp else read
        ordered_runs.append((peer, indices))
        load = compute + read
        makespan = max(makespan, load)          # :222, keeps the first maximal value's type
        rb = None
        if side is not None and indices[-1] - indices[0] + 1 == len(indices) and 0 <= indices[0] \
                and indices[-1] < len(stages):
            rb = side.range_bytes(indices[0], indices[-1] + 1)       # contiguous run: exact prefixes
        if rb is None:
            rb = (sum(stages[i].gpu_bytes for i in indices), sum(stages[i].cpu_bytes for i in indices),
                  sum(stages[i].disk_bytes for i in indices))
        rows.append(_peer_load(peer, indices, compute, read, load, *rb))
    assigned = {peer for peer, idxs in runs if idxs}
    # the idle rows in worker order (the tensoriser's peer order starts with
    # fleet.worker_ids(), so the sort is not repeated)
    for peer in (host.peer_ids[:host.p] if host is not None else fleet.worker_ids()):
        if peer not in assigned:
            rows.append(_peer_load(peer, (), 0.0, 0.0, 0.0, 0.0, 0.0, 0.0))
    mk = float(res["makespan"][c])
    if typed and mk == makespan:
        mk = makespan
    return T.ScheduleReport(tuple(stages), tuple(ordered_runs), tuple(rows), mk,
                            feasible=(code == _lib.DM_V_OK), reason=reason,
                            include_comm=include_comm, trace=trace)


def _evaluate_many(stages, fleet, runs_list, include_comm, traces, host=None):
    """Score several candidate Runs of one instance in one dm_eval_runs launch."""
    host = host or build_host(stages, fleet, include_comm)
    enc = [_encode_runs(host, runs) for runs in runs_list]
    res = engine.eval_runs(host, enc)
    mixed = [c for c, runs in enumerate(runs_list) if _mixed_keys(host, runs)]
    if mixed:                     # verdicts with the raw keys (a second launch, rare)
        raw = engine.eval_runs(host, [_encode_runs(host, runs_list[c], str_keys=False) for c in mixed])
        for i, c in enumerate(mixed):
            res["code"][c], res["code_run"][c] = raw["code"][i], raw["code_run"][i]
    out = []
    for c, runs in enumerate(runs_list):
        if int(res["status"][c]) != _lib.DM_OK:
            out.append(None)
            continue
        out.append(_report(stages, fleet, tuple(runs), include_comm, traces[c], res, c, host))
    return out, res


def _evaluate(stages, fleet, runs, include_comm, trace=(), host=None):
    runs = tuple(runs)
    reps, res = _evaluate_many(stages, fleet, [runs], include_comm, [trace], host)
    if reps[0] is None:
        _raise_cost_error(stages, fleet, runs, include_comm)
    return reps[0]


def _mark_infeasible(report, reason):
    """scheduling.py:426-428."""
    return T.ScheduleReport(report.stages, report.runs, report.per_peer, _INF, False, reason,
                            report.include_comm, report.trace)


# ============================================================== public API
def evaluate_runs(stages, fleet, runs, *, include_comm: bool = True, trace: tuple = ()):
    """Score a concrete assignment without optimizing it (scheduling.py:235-239)."""
    return _evaluate(list(stages), fleet, runs, include_comm, trace)


def verify_assignment(stages, fleet, runs) -> str:
    """Feasibility check, '' or the violated constraint (scheduling.py:179-207)."""
    stages = list(stages)
    runs = tuple(runs)
    host = build_host(stages, fleet, include_comm=False)
    res = engine.eval_runs(host, [_encode_runs(host, runs, str_keys=False)])
    return _reason(stages, fleet, runs, int(res["code"][0]), int(res["code_run"][0]))


def brute_force_schedule(stages, fleet, *, include_comm: bool = True, limit: int = 1_000_000):
    """Exhaustive optimum over contiguous assignments (scheduling.py:245-278),
    enumerated on the GPU in the reference's itertools order."""
    stages = list(stages)
    workers = fleet.worker_ids()
    _check_inputs(stages, workers)
    n, p = len(stages), len(workers)
    total = engine.bruteforce_total(n, p)
    if total > limit:
        raise T.SchedulingError(f"instance too large for enumeration: "
                                f"{total} contiguous assignments > {limit}")
    host = build_host(stages, fleet, include_comm)
    batch = engine.device_batch([host], pin=False)
    win = engine.enum(batch, "bruteforce", 0, total).read()
    if win["rank"] < 0:
        report = _evaluate(stages, fleet, ((workers[0], tuple(range(n))),), include_comm,
                           ("enumeration: no feasible assignment",), host)
        return _mark_infeasible(report, "no feasible assignment under memory constraints")
    bounds, peers = engine.unrank(n, p, int(win["rank"]), "bruteforce")
    runs = tuple((workers[peers[q]], tuple(range(bounds[q], bounds[q + 1]))) for q in range(len(peers)))
    return _evaluate(stages, fleet, runs, include_comm, (f"enumeration over {total} assignments",), host)


def _owner_to_runs(workers, owner_row, n):
    runs = []
    a = 0
    for i in range(1, n + 1):
        if i == n or owner_row[i] != owner_row[a]:
            runs.append((workers[int(owner_row[a])], tuple(range(a, i))))
            a = i
    return tuple(runs)


def schedule(stages, fleet, *, include_comm: bool = True):
    """Assign stages to the fleet's workers minimising the makespan
    (scheduling.py:391-423): pinned runs, exact subset DP (+ exact-link hill
    climb when overrides exist), or proportional split + hill climb."""
    stages = list(stages)
    workers = fleet.worker_ids()
    _check_inputs(stages, workers)
    n, p = len(stages), len(workers)

    if fleet.pinned_runs is not None:
        if len(fleet.pinned_runs) > p:
            raise T.SchedulingError(f"{len(fleet.pinned_runs)} pinned runs but only {p} workers")
        runs = tuple((workers[k], tuple(run)) for k, run in enumerate(fleet.pinned_runs))
        return _evaluate(stages, fleet, runs, include_comm, ("pinned runs",))

    # one H2D, the search kernel(s), the report kernel, one D2H (engine.ScheduleSlot)
    use_dp = n * n * p * (2 ** p) <= 3_000_000                   # :406
    pairs = None
    if fleet.links and include_comm and not use_dp and stage_side(stages).is_chain:
        # proportional split + hill climb keep run q on worker q and chain
        # stages read only from the previous run: links (q-1, q) suffice
        pairs = [(q - 1, q) for q in range(1, min(n, p))]
    host = build_host(stages, fleet, include_comm, link_pairs=pairs, workers=workers)
    out = engine.schedule_slot().schedule(host, use_dp, use_dp and bool(fleet.links))
    b, pe = out["bounds"], out["peers"]
    runs = tuple((workers[int(pe[q])], tuple(range(int(b[q]), int(b[q + 1])))) for q in range(out["n_runs"]))
    r = out["n_runs"]
    res = dict(cand_ptr=np.array([0, r]), code=np.array([out["code"]]), code_run=np.array([out["bad_run"]]),
               compute=out["compute"], read=out["read"], makespan=np.array([out["makespan"]]))
    if use_dp:
        if not out["found"]:
            report = _report(stages, fleet, runs, include_comm, ("exact search: no feasible assignment",), res,
                             0, host)
            return _mark_infeasible(report, "no feasible assignment under memory constraints")
        return _report(stages, fleet, runs, include_comm, ("exact subset search",), res, 0, host)
    report = _report(stages, fleet, runs, include_comm, ("proportional split with boundary search",), res, 0, host)
    if not report.feasible:
        return _mark_infeasible(report, report.reason or "no feasible assignment under memory constraints")
    return report


def reschedule_on_failure(report, failed_peer, fleet):
    """Replace a failed peer's run with the best backup, or re-solve without
    it (scheduling.py:431-474).  All backups are scored in one launch."""
    failed_peer = str(failed_peer)
    stages = report.stages
    lost = tuple(idxs for peer, idxs in report.runs if peer == failed_peer)
    if not lost:
        return report
    survivors = {pid: p for pid, p in fleet.peers.items() if pid != failed_peer}
    assigned = {peer for peer, idxs in report.runs if idxs and peer != failed_peer}
    candidates = sorted((b for b in fleet.backup_pool
                         if b != failed_peer and b in survivors and b not in assigned), key=peer_sort_key)
    if candidates:
        runs_list = [tuple((b if peer == failed_peer else peer, idxs) for peer, idxs in report.runs)
                     for b in candidates]
        traces = [report.trace + (f"replaced {failed_peer} with {b}",) for b in candidates]
        reps, res = _evaluate_many(list(stages), fleet, runs_list, report.include_comm, traces)
        scored = []
        for b, rep, runs in zip(candidates, reps, runs_list):
            if rep is None:
                _raise_cost_error(list(stages), fleet, runs, report.include_comm)
            if rep.feasible:
                scored.append((rep.makespan, peer_sort_key(b), rep))
        if scored:
            scored.sort(key=lambda t: (t[0], t[1]))
            return scored[0][2]

    reduced = type(fleet)(peers=survivors, default_link=fleet.default_link,
                          links={k: v for k, v in fleet.links.items() if failed_peer not in k},
                          backup_pool=(), msg_ratio=fleet.msg_ratio, pinned_runs=None, name=fleet.name)
    if not reduced.peers:
        raise T.SchedulingError("no surviving peers to reschedule onto")
    solved = schedule(stages, reduced, include_comm=report.include_comm)
    if not solved.feasible:
        raise T.SchedulingError(f"no feasible recovery after losing {failed_peer}: {solved.reason}")
    return T.ScheduleReport(solved.stages, solved.runs, solved.per_peer, solved.makespan, True, "",
                            solved.include_comm, report.trace + (f"re-solved without {failed_peer}",))
