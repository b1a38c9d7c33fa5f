"""Neutral JSON form of instances and reports for the golden fixtures.

Ints stay ints and floats are written with repr (bit-exact round trip), so
the column types the reference's own sum()/compare expressions see are
preserved.  Loaders rebuild instances in any module that provides the
reference's type names (the reference package itself, or the engine's
mirror `paper_2309_01172_b200.model`)."""

from __future__ import annotations


def dump_stages(stages):
    return [[s.index, s.label, s.flops, s.gpu_bytes, s.cpu_bytes, s.disk_bytes, [list(e) for e in s.in_edges]]
            for s in stages]


def load_stages(rows, M):
    return [M.Stage(r[0], r[1], r[2], r[3], r[4], r[5], tuple(tuple(e) for e in r[6])) for r in rows]


def dump_fleet(f):
    return {"peers": [[pe.id, pe.role.value, pe.peak_flops, pe.lam, pe.gpu_bytes, pe.cpu_bytes, pe.disk_bytes,
                       pe.write_bandwidth] for pe in f.peers.values()],
            "default_link": [f.default_link.alpha, f.default_link.beta],
            "links": [[a, b, lk.alpha, lk.beta] for (a, b), lk in f.links.items()],
            "backup_pool": list(f.backup_pool), "msg_ratio": f.msg_ratio,
            "pinned_runs": None if f.pinned_runs is None else [list(r) for r in f.pinned_runs],
            "name": f.name}


def load_fleet(d, M):
    peers = {}
    for pid, role, pk, lam, g, c, dk, wb in d["peers"]:
        peers[pid] = M.Peer(pid, role=M.Role(role), peak_flops=pk, lam=lam, gpu_bytes=g, cpu_bytes=c,
                            disk_bytes=dk, write_bandwidth=wb)
    fl = M.Fleet(peers=peers, default_link=M.Link(*d["default_link"]),
                 links={(a, b): M.Link(al, be) for a, b, al, be in d["links"]},
                 backup_pool=tuple(d["backup_pool"]), msg_ratio=d["msg_ratio"], name=d["name"])
    if d["pinned_runs"] is not None:
        fl.pinned_runs = tuple(tuple(r) for r in d["pinned_runs"])
    return fl


def dump_report(r):
    return {"runs": [[p, list(i)] for p, i in r.runs], "makespan": r.makespan, "feasible": r.feasible,
            "reason": r.reason, "trace": list(r.trace), "include_comm": r.include_comm,
            "per_peer": [[x.peer, list(x.stage_indices), x.compute_s, x.read_s, x.load_s, x.gpu_bytes, x.cpu_bytes,
                          x.disk_bytes] for x in r.per_peer]}


def runs_of(d):
    return tuple((p, tuple(i)) for p, i in d)


def report_matches(got, want) -> list:
    """Field-by-field comparison of a report with its golden dump; returns
    the list of mismatching fields (empty = identical)."""
    bad = []
    g = dump_report(got)
    for key in ("runs", "feasible", "reason", "trace", "include_comm"):
        if g[key] != want[key]:
            bad.append(key)
    if not (g["makespan"] == want["makespan"]):
        bad.append("makespan")
    if len(g["per_peer"]) != len(want["per_peer"]):
        bad.append("per_peer")
    else:
        for a, b in zip(g["per_peer"], want["per_peer"]):
            if a[:5] != b[:5] or a[5:] != b[5:] or [type(x) for x in a[5:]] != [type(x) for x in b[5:]]:
                bad.append(f"row {b[0]}")
    return bad
