"""Neutral JSON form of instances and reports for the golden fixtures.

Ints stay ints and floats are written with repr (bit-exact round trip), so
the column types the reference's own sum()/compare expressions see are
preserved.  Loaders rebuild instances in any module that provides the
reference's type names (the reference package, directly or through
`paper_2309_01172_b200.refapi`)."""

from __future__ import annotations

import numpy as np


def _enc(v):
    """numpy scalars keep their type through the fixture: the reference's
    sum() is compensated only over exact `float` items, so the type of
    a speed or a FLOP count is part of the instance."""
    if isinstance(v, np.floating):
        return {"f64": float(v)}
    if isinstance(v, np.integer):
        return {"i64": int(v)}
    return v


def _dec(v):
    if isinstance(v, dict):
        return np.float64(v["f64"]) if "f64" in v else np.int64(v["i64"])
    return v


def dump_stages(stages):
    return [[s.index, s.label, _enc(s.flops), _enc(s.gpu_bytes), _enc(s.cpu_bytes), _enc(s.disk_bytes),
             [[e[0], _enc(e[1])] for e in s.in_edges]]
            for s in stages]


def load_stages(rows, M):
    return [M.Stage(r[0], r[1], _dec(r[2]), _dec(r[3]), _dec(r[4]), _dec(r[5]),
                    tuple((e[0], _dec(e[1])) for e in r[6])) for r in rows]


def dump_fleet(f):
    return {"peers": [[pe.id, pe.role.value] + [_enc(x) for x in (pe.peak_flops, pe.lam, pe.gpu_bytes, pe.cpu_bytes,
                                                                    pe.disk_bytes, pe.write_bandwidth)]
                      for pe in f.peers.values()],
            "default_link": [_enc(f.default_link.alpha), _enc(f.default_link.beta)],
            "links": [[a, b, _enc(lk.alpha), _enc(lk.beta)] for (a, b), lk in f.links.items()],
            "backup_pool": list(f.backup_pool), "msg_ratio": _enc(f.msg_ratio),
            "pinned_runs": None if f.pinned_runs is None else [list(r) for r in f.pinned_runs],
            "name": f.name}


def load_fleet(d, M):
    peers = {}
    for pid, role, *vals in d["peers"]:
        pk, lam, g, c, dk, wb = (_dec(x) for x in vals)
        peers[pid] = M.Peer(pid, role=M.Role(role), peak_flops=pk, lam=lam, gpu_bytes=g, cpu_bytes=c,
                            disk_bytes=dk, write_bandwidth=wb)
    fl = M.Fleet(peers=peers, default_link=M.Link(*(_dec(x) for x in d["default_link"])),
                 links={(a, b): M.Link(_dec(al), _dec(be)) for a, b, al, be in d["links"]},
                 backup_pool=tuple(d["backup_pool"]), msg_ratio=_dec(d["msg_ratio"]), name=d["name"])
    if d["pinned_runs"] is not None:
        fl.pinned_runs = tuple(tuple(r) for r in d["pinned_runs"])
    return fl


def dump_report(r):
    return {"runs": [[p, list(i)] for p, i in r.runs], "makespan": r.makespan, "feasible": r.feasible,
            "reason": r.reason, "trace": list(r.trace), "include_comm": r.include_comm,
            "per_peer": [[x.peer, list(x.stage_indices), x.compute_s, x.read_s, x.load_s, x.gpu_bytes, x.cpu_bytes,
                          x.disk_bytes] for x in r.per_peer],
            # Python types of the float fields (float vs numpy.float64)
            "types": [type(r.makespan).__name__] + [[type(v).__name__ for v in (x.compute_s, x.read_s, x.load_s)]
                                                    for x in r.per_peer]}


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
    if "types" in want and g["types"] != want["types"]:
        bad.append("types")
    return bad


def c4_record(owner, vals) -> bytes:
    """One C4 scenario in the full-size digest (tests/golden/make_full_size.py):
    the owner vector as little-endian int16 and six float64 values (makespan,
    Eq. 3 latency, bottleneck, Eq. 4 pipe time, throughput, violation code)."""
    import struct
    return np.asarray(owner, dtype="<i2").tobytes() + struct.pack("<6d", *[float(v) for v in vals])
