"""The CPU oracle (oracle/dm_oracle.c) against golden fixtures produced by
the reference itself (tests/golden/make_golden.py): this pins the oracle
before it is trusted as the GPU checker."""

import json
import pathlib

import pytest

from golden_io import load_fleet, load_stages, runs_of
from paper_2309_01172_b200 import refapi as M

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
CASES = json.loads((GOLD / "scheduling_cases.json").read_text())["cases"]

KEYWORD = {0: "", 1: "holds two runs", 2: "unknown peer", 3: "not contiguous", 4: "assigned twice",
           5: "exceeds gpu capacity", 6: "exceeds cpu capacity", 7: "exceeds disk capacity", 8: "unassigned"}


def _inst(oracle_mod, c, include_comm=True):
    st = load_stages(c["stages"], M)
    fl = load_fleet(c["fleet"], M)
    return st, fl, oracle_mod.Instance(st, fl, include_comm)


def _check_eval(inst, runs, want):
    mk, code, bad, status, comp, read = inst.eval_runs(runs)
    assert status == 0
    assert mk == want["makespan"] or (not want["feasible"] and want["makespan"] == float("inf"))
    assert (code == 0) == want["feasible"]
    if code:
        assert KEYWORD[code] in want["reason"]
    rows = {(r[0], tuple(r[1])): r for r in want["per_peer"] if r[1]}
    for (pe, ix), c, r in zip(runs, comp, read):
        if ix:
            row = rows[(pe, tuple(sorted(ix)))]
            assert (c, r) == (row[2], row[3])


def test_oracle_evaluate_and_verify(oracle_mod):
    n = 0
    for c in CASES:
        if c["kind"] == "evaluate":
            _, _, inst = _inst(oracle_mod, c, c["include_comm"])
            _check_eval(inst, runs_of(c["runs"]), c["report"])
            n += 1
        elif c["kind"] == "verify":
            _, _, inst = _inst(oracle_mod, c)
            _, code, _, _, _, _ = inst.eval_runs(runs_of(c["runs"]))
            assert (code == 0) == (c["reason"] == "")
            assert KEYWORD[code] in c["reason"]
            n += 1
        elif c["kind"] == "solve":
            _, _, inst = _inst(oracle_mod, c)
            for e in c["evals"]:
                _check_eval(inst, runs_of(e["runs"]), e["report"])
                n += 1
    assert n > 100


def test_oracle_schedule(oracle_mod):
    n = 0
    for c in CASES:
        if c["kind"] != "solve":
            continue
        _, _, inst = _inst(oracle_mod, c)
        want = c["schedule"]
        path, own = inst.schedule()
        if path < 0:
            assert not want["feasible"]
            continue
        runs = inst.owner_to_runs(own)
        assert runs == runs_of(want["runs"]), c["tag"]
        assert (path > 0) == want["feasible"], c["tag"]
        n += 1
    assert n > 250


def test_oracle_brute_force(oracle_mod):
    n = 0
    for c in CASES:
        if c["kind"] != "solve" or "brute_force" not in c:
            continue
        _, _, inst = _inst(oracle_mod, c)
        want = c["brute_force"]
        w = inst.enum("bruteforce", 0, oracle_mod.bruteforce_total(inst.n, inst.p))
        if w["rank"] < 0:
            assert not want["feasible"]
            continue
        b, pe = inst.unrank("bruteforce", w["rank"])
        runs = tuple(sorted(((inst.workers[pe[q]], tuple(range(b[q], b[q + 1]))) for q in range(len(pe))),
                            key=lambda r: r[1][0]))
        assert runs == runs_of(want["runs"]), c["tag"]
        assert w["makespan"] == want["makespan"]
        n += 1
    assert n > 200


def test_oracle_pipeline_epilogue(oracle_mod):
    """Eq. 3/4 restatement against the reference's sweep rows (pinned presets)."""
    from paper_2309_01172_b200 import configs as CF
    data = json.loads((GOLD / "pipeline_cases.json").read_text())
    st = load_stages(data["stages"], M)
    presets = {"rtx3080-x50": (59.5e12, 50, [(i,) for i in range(50)]),
               "h100-x4": (756e12, 4, [(0,), tuple(range(1, 25)), tuple(range(25, 49)), (49,)])}
    checked = 0
    for sw in data["sweeps"]:
        for fleet_name, bw, alpha_ms, nb, lat, pipe, thr in sw["rows"]:
            speed, count, pins = presets[fleet_name]
            peers = {str(k): M.Peer(str(k), peak_flops=speed, gpu_bytes=(80 if count == 4 else 10) * 2**30,
                                    cpu_bytes=32 * 2**30, disk_bytes=256 * 2**30) for k in range(1, count + 1)}
            alpha = [a for a in sw["alpha"] if a * 1e3 == alpha_ms][0]
            fl = M.Fleet(peers=peers, default_link=M.Link(alpha, M.bandwidth_to_beta(bw)))
            inst = oracle_mod.Instance(st, fl)
            runs = tuple((str(k + 1), pins[k]) for k in range(count))
            mk, code, _, _, comp, read = inst.eval_runs(runs)
            got = oracle_mod.epilogue(comp, read, nb, data["samples_per_batch"])
            assert (repr(got[0]), repr(got[2]), repr(got[3])) == (lat, pipe, thr)
            checked += 1
    assert checked >= 100 * 2


def test_py_sum_restatement(oracle_mod):
    import numpy as np
    rng = np.random.default_rng(1)
    for _ in range(20000):
        k = int(rng.integers(1, 40))
        v = [float(x) for x in rng.standard_normal(k) * 10.0 ** rng.integers(-5, 20, k)]
        assert oracle_mod.py_sum(v) == sum(v)


def test_oracle_schedule_epilogue(oracle_mod):
    """Eq. 3 / Eq. 4 over every feasible golden schedule, against the
    reference's fp_latency / bottleneck / pipeline_time / throughput
    (pipeline.py:41-62) — fleets with numpy speeds included, where fp_latency's
    sum() runs uncompensated."""
    n = 0
    for c in CASES:
        if c["kind"] != "solve" or "epilogue" not in c:
            continue
        _, _, inst = _inst(oracle_mod, c)
        runs = runs_of(c["schedule"]["runs"])
        mk, code, _, _, comp, read = inst.eval_runs(runs)
        assert code == 0
        got = oracle_mod.epilogue(comp, read, 64, 4, inst.load_np(runs))
        assert list(got) == c["epilogue"], c["tag"]
        n += 1
    assert n > 250
