#!/usr/bin/env python3
"""Generate the golden fixtures of the hot path by running the REFERENCE
package (pkg/src/dagmesh, imported read-only from /root/reference) on the
reference's own test inputs and on seeded random instances.

Run in the build container (the reference is not present on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (committed): tests/golden/scheduling_cases.json,
tests/golden/pipeline_cases.json, tests/golden/stage_digests.json,
tests/golden/opcost_cases.json.

Instances are stored in a neutral JSON form (ints stay ints, floats are
written with repr so they round-trip bit-exactly; `tests/golden_io.py` reads
them back into either the reference's or the engine's types).
"""

from __future__ import annotations

import hashlib
import json
import math
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from dagmesh import hardware as hw, ir, pipeline as PL, scheduling as S  # noqa: E402

from golden_io import dump_fleet, dump_report, dump_stages  # noqa: E402


def ref_random_stages(rng, n):
    """pkg/tests/test_scheduling.py:26-37 (call-for-call)."""
    stages = []
    for i in range(n):
        edges = ()
        if i > 0:
            src = int(rng.integers(0, i))
            edges = ((src, int(rng.integers(256, 65536))),)
        stages.append(S.Stage(index=i, label=f"s{i}", flops=float(rng.integers(10**5, 10**8)),
                              gpu_bytes=float(rng.integers(2**10, 2**24)), cpu_bytes=1024.0, disk_bytes=512.0,
                              in_edges=edges))
    return stages


def ref_uniform_fleet(speeds, link=hw.ZERO_LINK, gpu_gb=64.0, backups=()):
    peers = {str(i + 1): hw.Peer(str(i + 1), peak_flops=s, gpu_bytes=gpu_gb * 2**30) for i, s in enumerate(speeds)}
    return hw.Fleet(peers=peers, default_link=link, backup_pool=tuple(backups))


def ref_big_instance(rng, n, p, *, dag=True, frac=False, links=False, pressure=(0.05, 0.6)):
    """Same draws as tests/gen.py:big_instance, built with reference types."""
    st = []
    for i in range(n):
        edges = ()
        if i > 0:
            if dag:
                k = int(rng.integers(1, 3))
                srcs = sorted(set(int(x) for x in rng.integers(max(0, i - 4), i, k)))
            else:
                srcs = [i - 1]
            edges = tuple((s, int(rng.integers(256, 2**22))) for s in srcs)
        fl = float(rng.integers(10**9, 10**12)) + (float(rng.random()) if frac else 0.0)
        st.append(S.Stage(i, f"s{i}", fl, float(rng.integers(2**20, 2**30)), float(rng.integers(1024, 2**20)),
                          512.0, edges))
    total = sum(s.gpu_bytes for s in st)
    peers = {str(k + 1): hw.Peer(str(k + 1), peak_flops=float(rng.choice([59.5e12, 97.5e12, 82.58e12, 155.92e12])),
                                 lam=float(rng.uniform(0.3, 1)), gpu_bytes=float(rng.uniform(*pressure)) * total)
             for k in range(p)}
    lk = {}
    if links:
        ids = list(peers)
        for _ in range(3 * p):
            a, b = rng.choice(ids, 2, replace=False)
            lk[(str(a), str(b))] = hw.Link(float(rng.uniform(0, 0.02)), 8 / (float(rng.uniform(0.1, 100)) * 1e9))
    fleet = hw.Fleet(peers=peers, default_link=hw.Link(float(rng.uniform(0, 0.01)), 8 / (float(rng.uniform(0.1, 10)) * 1e9)),
                     links=lk, msg_ratio=float(rng.choice([1.0, 0.5, 0.3])))
    return st, fleet


def case(kind, stages, fleet, **kw):
    out = {"kind": kind, "stages": dump_stages(stages), "fleet": dump_fleet(fleet)}
    out.update(kw)
    return out


def solve_cases(stages, fleet, tag, brute=True, evals=()):
    """One fixture entry per instance: schedule(), brute_force_schedule() and
    evaluate_runs() of the given candidate runs."""
    rep = S.schedule(stages, fleet)
    out = case("solve", stages, fleet, tag=tag, schedule=dump_report(rep))
    if rep.feasible:   # Eq. 3 / Eq. 4 over the schedule (pipeline.py:41-62), n_b = 64, 4 samples per batch
        prof = PL.profiles_from_report(rep)
        out["epilogue"] = [PL.fp_latency(prof), PL.bottleneck(prof), PL.pipeline_time(prof, 64),
                           PL.throughput(prof, 64, 4)]
    if brute:
        try:
            out["brute_force"] = dump_report(S.brute_force_schedule(stages, fleet))
        except Exception as exc:  # oversize
            out["brute_force_error"] = [type(exc).__name__, str(exc)]
    out["evals"] = [{"runs": runs, "report": dump_report(S.evaluate_runs(stages, fleet, runs))} for runs in evals]
    return [out]


def scheduling_cases():
    cases = []
    demo = ir.load_job(REF / "jobs" / "demo.json")
    trio = hw.load_fleet(REF / "fleets" / "trio.json")
    demo_cells = (("Input", "Conv", "Add", "Pool"), ("TensorA", "Multiply"),
                  ("Label", "Concat", "Linear", "CrossEntropy"))
    ds = S.build_stages(demo, demo_cells)
    topo = S.build_stages(demo, S.topological_cells(demo))
    three = (("1", (0,)), ("2", (1,)), ("3", (2,)))
    # test_scheduling.py:82-138 evaluate / verify
    for inc in (True, False):
        cases.append(case("evaluate", ds, trio, runs=three, include_comm=inc,
                          report=dump_report(S.evaluate_runs(ds, trio, three, include_comm=inc)), tag="demo-three"))
    for runs in [(("1", (0, 1, 2)),), (("1", (0, 2)), ("2", (1,))), (("1", (0, 1)), ("2", (1, 2))),
                 (("1", (0, 1)),), (("1", (0,)), ("1", (1, 2))), three]:
        cases.append(case("verify", ds, trio, runs=runs, reason=S.verify_assignment(ds, trio, runs), tag="demo-verify"))
    tiny = ref_uniform_fleet([1e6], gpu_gb=30000 / 2**30)
    cases.append(case("verify", ds, tiny, runs=(("1", (0, 1, 2)),),
                      reason=S.verify_assignment(ds, tiny, (("1", (0, 1, 2)),)), tag="demo-cap"))
    # demo optimum + CSV golden (test_scheduling.py:142-150, 283-292)
    cases += solve_cases(topo, trio, "demo-topo")
    # two-stage split (152-159), infeasible (191-197), pinned (206-220)
    two = [S.Stage(0, "a", 1e8, 1024, 64, 64), S.Stage(1, "b", 1e8, 1024, 64, 64)]
    cases += solve_cases(two, ref_uniform_fleet([1e9, 1e9]), "two-stage")
    inf1 = [S.Stage(0, "a", 1e6, 2**34, 64, 64)]
    cases += solve_cases(inf1, ref_uniform_fleet([1e9], gpu_gb=1.0), "infeasible")
    pin_st = [S.Stage(i, f"s{i}", 1e6 * (i + 1), 1024, 64, 64) for i in range(3)]
    pin_fl = ref_uniform_fleet([1e9, 1e9])
    pin_fl.pinned_runs = ((0,), (1, 2))
    cases.append(case("schedule", pin_st, pin_fl, tag="pinned", report=dump_report(S.schedule(pin_st, pin_fl))))
    # random instances (test_scheduling.py:161-189, 222-231)
    rng = np.random.default_rng(404)
    for trial in range(30):
        n = int(rng.integers(3, 9))
        p = int(rng.integers(2, 4))
        st = ref_random_stages(rng, n)
        link = hw.Link(float(rng.uniform(0, 1e-3)), float(rng.uniform(0, 1e-7)))
        fl = ref_uniform_fleet(list(rng.uniform(1e8, 1e9, p)), link=link)
        cases += solve_cases(st, fl, f"seed404-{trial}")
    rng = np.random.default_rng(77)
    for trial in range(15):
        n = int(rng.integers(3, 8))
        st = ref_random_stages(rng, n)
        cap_gb = (0.7 * sum(s.gpu_bytes for s in st)) / 2**30
        fl = ref_uniform_fleet(list(rng.uniform(1e8, 1e9, 3)), gpu_gb=cap_gb)
        cases += solve_cases(st, fl, f"seed77-{trial}")
    # acceptance criterion 6 (test_acceptance.py:141-156)
    rng = np.random.default_rng(2024)
    for trial in range(200):
        n = int(rng.integers(2, 13))
        p = int(rng.integers(2, 5))
        st = ref_random_stages(rng, n)
        link = hw.Link(float(rng.uniform(0, 1e-3)), float(rng.uniform(0, 1e-7)))
        cap_gb = float(rng.uniform(0.7, 1.6)) * sum(s.gpu_bytes for s in st) / 2**30
        fl = ref_uniform_fleet(list(rng.uniform(1e8, 1e9, p)), link=link, gpu_gb=cap_gb)
        cases += solve_cases(st, fl, f"crit6-{trial}")
    # larger instances: proportional + hill climb, DAG edges, pair links,
    # non-integral flops, msg_ratio != 1
    rng = np.random.default_rng(7)
    for k in range(40):
        st, fl = ref_big_instance(rng, int(rng.integers(15, 70)), int(rng.integers(6, 24)), dag=k % 2 == 0,
                                  frac=k % 4 == 1, links=k % 3 == 0)
        evals = []
        for j in range(3):
            own = rng.integers(0, len(fl.peers), len(st))
            grp = {}
            for i, o in enumerate(own):
                grp.setdefault(str(o + 1), []).append(i)
            evals.append(tuple((pid, tuple(v)) for pid, v in grp.items()))
        cases += solve_cases(st, fl, f"big-{k}", brute=False, evals=evals)
    # reschedule_on_failure (test_scheduling.py:240-279)
    rep = S.evaluate_runs(ds, trio, three)
    twin = hw.Peer("5", peak_flops=1.5e6, gpu_bytes=2**30, cpu_bytes=4 * 2**30, disk_bytes=16 * 2**30)
    tie = hw.Fleet(peers=dict(trio.peers, **{"5": twin}), default_link=trio.default_link, links=dict(trio.links),
                   backup_pool=("5", "4"), msg_ratio=1.0)
    nob = hw.Fleet(peers={k: v for k, v in trio.peers.items() if k != "4"}, default_link=trio.default_link,
                   links=dict(trio.links))
    for tag, fl in (("backup", trio), ("tie", tie), ("no-backups", nob)):
        healed = S.reschedule_on_failure(rep, "2", fl)
        cases.append(case("reschedule", ds, fl, runs=three, failed="2", tag=f"resched-{tag}",
                          report=dump_report(healed)))
    return cases


def pipeline_cases():
    bert = PL.build_bert_large()
    stages = S.build_stages(bert.graph, bert.cells)
    out = {"stages": dump_stages(stages), "model": bert.name, "samples_per_batch": bert.samples_per_batch,
           "sweeps": []}
    grids = [([1.0, 2.0, 5.0, 10.0], [0.0, 5e-3, 1e-2], 512),
             ([float(b) for b in np.geomspace(0.1, 10.0, 10)], [float(a) for a in np.linspace(0.0, 9e-3, 10)], 2),
             ([1.0, 5.0], [0.0, 5e-3], 512)]
    for bws, alphas, nb in grids:
        res = PL.sweep(bert, PL.reference_fleets(), bws, alphas, nb)
        out["sweeps"].append({"bw": bws, "alpha": alphas, "n_b": nb,
                              "rows": [[r.fleet, r.bandwidth_gbps, r.alpha_ms, r.n_batches, repr(r.latency_s),
                                        repr(r.pipe_time_s), repr(r.throughput)] for r in res.rows],
                              "infeasible": res.infeasible})
    return out


def opcost_cases():
    """hardware.op_time / subgraph_time (hardware.py:190-226) on the demo job:
    the reference's own test placements (test_hardware.py:100-129) plus
    seeded random placements, slow-writer and msg_ratio variants."""
    demo = ir.load_job(REF / "jobs" / "demo.json")
    trio = hw.load_fleet(REF / "fleets" / "trio.json")
    names = list(demo.nodes)
    table = {"names": names,
             "flops": [int(ir.op_flops(demo.node(n))) for n in names],
             "out_elements": [int(demo.node(n).out_elements) for n in names],
             "args": [[names.index(a) for a in demo.node(n).args] for n in names],
             "users": [[names.index(u) for u in demo.node(n).users] for n in names]}
    slow = hw.Fleet(dict(trio.peers, **{"1": hw.Peer("1", peak_flops=2e6, write_bandwidth=1024.0)}),
                    default_link=trio.default_link, links=trio.links)
    halfmsg = hw.Fleet(dict(trio.peers), default_link=trio.default_link, links=trio.links, msg_ratio=0.37)
    # numpy-typed peer values (as the reference's own tests build fleets from
    # rng draws): sum() over numpy totals is not compensated
    npeers = dict(trio.peers)
    for pid in ("2", "3"):
        pe = npeers[pid]
        npeers[pid] = hw.Peer(pid, role=pe.role, peak_flops=np.float64(pe.peak_flops) * np.float64(1.0 / 3.0),
                              lam=pe.lam, gpu_bytes=pe.gpu_bytes, cpu_bytes=pe.cpu_bytes, disk_bytes=pe.disk_bytes,
                              write_bandwidth=np.float64(pe.write_bandwidth) / 7.0)
    numpy_fl = hw.Fleet(npeers, default_link=hw.Link(np.float64(trio.default_link.alpha) + 1e-4,
                                                     trio.default_link.beta),
                        links={k: hw.Link(np.float64(v.alpha), v.beta) for k, v in trio.links.items()},
                        msg_ratio=0.61)
    rng = np.random.default_rng(91)
    placements = [dict(demo.placement)]
    for _ in range(12):
        placements.append({n: str(int(rng.integers(1, 5))) for n in names})
    cells = [("TensorA", "Multiply"), tuple(names), ("Conv", "Add", "Pool"), ("Label",)]
    out = {"table": table, "placements": placements, "cells": [list(c) for c in cells], "fleets": []}
    for fl in (trio, slow, halfmsg, numpy_fl):
        rows, subs = [], []
        for pl in placements:
            rows.append([list(hw.op_time(demo, n, fl, pl)) for n in names])
            subs.append([list(hw.subgraph_time(demo, c, fl, pl)) for c in cells])
        out["fleets"].append({"fleet": dump_fleet(fl), "ops": rows, "subgraphs": subs})
    return out


def stage_digests():
    from paper_2309_01172_b200 import configs as CF
    out = {}
    for name, kw in CF.MODELS.items():
        job, cells = CF.encoder_job(**kw)
        st = S.build_stages(ir.parse_job_definition(job), cells)
        blob = repr([(s.index, s.label, s.flops, s.gpu_bytes, s.cpu_bytes, s.disk_bytes, s.in_edges) for s in st])
        out[name] = {"n": len(st), "sha256": hashlib.sha256(blob.encode()).hexdigest(),
                     "total_flops": sum(s.flops for s in st)}
    for L in (32, 57, 80):
        for h in CF.C4_HIDDEN:
            kw = dict(hidden=h, layers=L, vocab=32000, batch=4, seq=1024)
            job, cells = CF.encoder_job(**kw)
            st = S.build_stages(ir.parse_job_definition(job), cells)
            blob = repr([(s.index, s.label, s.flops, s.gpu_bytes, s.cpu_bytes, s.disk_bytes, s.in_edges) for s in st])
            out[f"c4-L{L}-h{h}"] = {"n": len(st), "sha256": hashlib.sha256(blob.encode()).hexdigest(), "kw": kw}
    return out


def main():
    (HERE / "scheduling_cases.json").write_text(json.dumps({"python": sys.version, "cases": scheduling_cases()}))
    (HERE / "pipeline_cases.json").write_text(json.dumps(pipeline_cases()))
    (HERE / "stage_digests.json").write_text(json.dumps(stage_digests(), indent=1))
    (HERE / "opcost_cases.json").write_text(json.dumps(opcost_cases()))
    for f in ("scheduling_cases.json", "pipeline_cases.json", "stage_digests.json", "opcost_cases.json"):
        print(f, (HERE / f).stat().st_size, "bytes")


if __name__ == "__main__":
    main()
