"""The engine's public API (GPU path) against reports produced by the
reference itself (tests/golden/*.json): runs, makespan bits, feasibility,
reason strings, per-peer rows (values and Python types), traces — i.e. the
reports are interchangeable with the reference's, including CSV output."""

import json
import pathlib

import pytest

from golden_io import load_fleet, load_stages, report_matches, runs_of
from paper_2309_01172_b200 import refapi as M
from paper_2309_01172_b200 import pipeline as P
from paper_2309_01172_b200 import scheduling as S

pytestmark = pytest.mark.gpu
GOLD = pathlib.Path(__file__).resolve().parent / "golden"
CASES = json.loads((GOLD / "scheduling_cases.json").read_text())["cases"]


def _inst(c):
    return load_stages(c["stages"], M), load_fleet(c["fleet"], M)


def test_evaluate_verify_golden(engine_ready):
    n = 0
    for c in CASES:
        st, fl = _inst(c)
        if c["kind"] == "evaluate":
            rep = S.evaluate_runs(st, fl, runs_of(c["runs"]), include_comm=c["include_comm"])
            assert report_matches(rep, c["report"]) == [], c["tag"]
            n += 1
        elif c["kind"] == "verify":
            assert S.verify_assignment(st, fl, runs_of(c["runs"])) == c["reason"], c["tag"]
            n += 1
        elif c["kind"] == "solve":
            for e in c["evals"]:
                rep = S.evaluate_runs(st, fl, runs_of(e["runs"]))
                assert report_matches(rep, e["report"]) == [], c["tag"]
                n += 1
    assert n > 100


def test_schedule_and_brute_force_golden(engine_ready):
    n = 0
    for c in CASES:
        if c["kind"] == "schedule":
            st, fl = _inst(c)
            assert report_matches(S.schedule(st, fl), c["report"]) == [], c["tag"]
        if c["kind"] != "solve":
            continue
        st, fl = _inst(c)
        assert report_matches(S.schedule(st, fl), c["schedule"]) == [], c["tag"]
        if "brute_force" in c:
            assert report_matches(S.brute_force_schedule(st, fl), c["brute_force"]) == [], c["tag"]
        n += 1
    assert n > 280


def test_schedule_epilogue_golden(engine_ready):
    """dm_pipeline_epilogue over every feasible golden schedule, batched, bit
    for bit against the reference's Eq. 3 / Eq. 4 values (numpy-typed fleets
    included)."""
    import torch
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200.tensorize import build_host
    hosts, owners, want = [], [], []
    for c in CASES:
        if c["kind"] != "solve" or "epilogue" not in c:
            continue
        st, fl = _inst(c)
        h = build_host(st, fl)
        own = [0] * len(st)
        for pe, ix in runs_of(c["schedule"]["runs"]):
            for i in ix:
                own[i] = h.index_of[pe]
        hosts.append(h)
        owners.append(own)
        want.append(c["epilogue"])
    n_max = max(len(o) for o in owners)
    own = torch.full((len(owners), n_max), -1, dtype=torch.int16)
    for s_, o in enumerate(owners):
        own[s_, :len(o)] = torch.tensor(o, dtype=torch.int16)
    batch = engine.device_batch(hosts)
    out = engine.epilogue(batch, n_max, own.cuda(), 64, 4).cpu().numpy()
    for s_, w in enumerate(want):
        assert out[s_, 1:5].tolist() == w, s_
    assert len(want) > 250


def test_reschedule_golden(engine_ready):
    for c in CASES:
        if c["kind"] != "reschedule":
            continue
        st, fl = _inst(c)
        trio = load_fleet(next(x for x in CASES if x["tag"] == "demo-three")["fleet"], M)
        base = S.evaluate_runs(st, trio, runs_of(c["runs"]))
        healed = S.reschedule_on_failure(base, c["failed"], fl)
        assert report_matches(healed, c["report"]) == [], c["tag"]


def test_csv_golden(engine_ready, tmp_path):
    c = next(x for x in CASES if x["tag"] == "demo-topo")
    st, fl = _inst(c)
    rep = S.schedule(st, fl)
    rep.to_csv(tmp_path / "s.csv")
    lines = (tmp_path / "s.csv").read_text().splitlines()
    assert lines[1] == "1,1-2,0.020736,0,0.020736,9552"   # pkg/tests/test_scheduling.py:291
    assert rep.makespan == 0.020736 or abs(rep.makespan - 0.020736) < 1e-15


def test_error_conventions(engine_ready):
    c = next(x for x in CASES if x["tag"] == "demo-topo")
    st, fl = _inst(c)
    with pytest.raises(M.SchedulingError, match="empty stage list"):
        S.schedule([], fl)
    with pytest.raises(M.SchedulingError, match="empty fleet"):
        S.schedule(st, M.Fleet(peers={}))
    with pytest.raises(M.SchedulingError, match="too large for enumeration"):
        S.brute_force_schedule(st, fl, limit=10)
    pf = M.Fleet(peers={"1": M.Peer("1")})
    pf.pinned_runs = ((0,), (1,))
    with pytest.raises(M.SchedulingError, match="pinned runs but only"):
        S.schedule(st, pf)
    rep = S.schedule(st[:1], M.Fleet(peers={"1": M.Peer("1")}))
    with pytest.raises(M.SchedulingError, match="no surviving peers"):
        S.reschedule_on_failure(rep, "1", M.Fleet(peers={"1": M.Peer("1")}))


def test_sweep_golden(engine_ready):
    """Batched Eq. 3/4 sweep (pipeline.sweep) against the reference's rows
    for the acceptance-criteria grids (test_acceptance.py:31-86)."""
    data = json.loads((GOLD / "pipeline_cases.json").read_text())
    st = load_stages(data["stages"], M)
    fleets = [P_fleet for P_fleet in _reference_fleets()]
    for sw in data["sweeps"]:
        res = P.sweep_stages(st, data["model"], data["samples_per_batch"], fleets, sw["bw"], sw["alpha"], sw["n_b"])
        got = [[r.fleet, r.bandwidth_gbps, r.alpha_ms, r.n_batches, repr(r.latency_s), repr(r.pipe_time_s),
                repr(r.throughput)] for r in res.rows]
        assert got == sw["rows"]
        assert res.infeasible == sw["infeasible"]


def _reference_fleets():
    """pipeline.reference_fleets() presets (pipeline.py:140-191): 50 x rtx3080
    one stage each, 4 x h100 with the published four-run split."""
    def gpu_fleet(name, model, count, pinned):
        spec = M.GPU_TABLE[model]
        peers = {str(k): M.Peer(str(k), peak_flops=spec.tflops_tensor * 1e12, lam=1.0,
                                gpu_bytes=spec.memory_gb * 2**30, cpu_bytes=32 * 2**30, disk_bytes=256 * 2**30)
                 for k in range(1, count + 1)}
        return M.Fleet(peers=peers, default_link=M.Link(5e-3, M.bandwidth_to_beta(1.0)), pinned_runs=pinned, name=name)
    return [gpu_fleet("rtx3080-x50", "rtx3080", 50, tuple((i,) for i in range(50))),
            gpu_fleet("h100-x4", "h100", 4, ((0,), tuple(range(1, 25)), tuple(range(25, 49)), (49,)))]
