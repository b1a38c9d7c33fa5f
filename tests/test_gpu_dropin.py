"""Drop-in: the reference package itself (installed unmodified into
baseline/_ref with pip) runs its hot path on the engine after
paper_2309_01172_b200.install(): its own scheduling.schedule / evaluate_runs /
brute_force_schedule / pipeline.sweep now launch the CUDA kernels, return the
reference's own ScheduleReport instances, and reproduce the reference's
golden results."""

import json
import pathlib
import sys
from types import SimpleNamespace

import pytest

from golden_io import load_fleet, load_stages, report_matches, runs_of

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parent.parent
REF_INSTALL = ROOT / "baseline" / "_ref"
GOLD = ROOT / "tests" / "golden"


@pytest.fixture(scope="module")
def dagmesh_installed(engine_ready):
    if not (REF_INSTALL / "dagmesh").exists():
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, str(REF_INSTALL))
    import dagmesh
    import paper_2309_01172_b200 as eng
    uninstall = eng.install(dagmesh)
    yield dagmesh
    uninstall()


def _types(dm):
    return SimpleNamespace(Stage=dm.scheduling.Stage, Peer=dm.hardware.Peer, Role=dm.hardware.Role,
                           Fleet=dm.hardware.Fleet, Link=dm.hardware.Link)


def test_reference_api_is_rebound(dagmesh_installed):
    import paper_2309_01172_b200.scheduling as eng_sched
    dm = dagmesh_installed
    assert dm.scheduling.schedule is eng_sched.schedule
    assert dm.schedule is eng_sched.schedule
    assert dm.scheduling.evaluate_runs is eng_sched.evaluate_runs


def test_reference_types_through_engine(dagmesh_installed):
    dm = dagmesh_installed
    T = _types(dm)
    cases = json.loads((GOLD / "scheduling_cases.json").read_text())["cases"]
    n = 0
    for c in cases:
        if c["kind"] != "solve":
            continue
        st, fl = load_stages(c["stages"], T), load_fleet(c["fleet"], T)
        rep = dm.scheduling.schedule(st, fl)
        assert isinstance(rep, dm.scheduling.ScheduleReport)
        assert report_matches(rep, c["schedule"]) == [], c["tag"]
        if "brute_force" in c and n % 5 == 0:
            assert report_matches(dm.scheduling.brute_force_schedule(st, fl), c["brute_force"]) == []
        n += 1
        if n >= 120:
            break


def test_reference_sweep_through_engine(dagmesh_installed):
    dm = dagmesh_installed
    data = json.loads((GOLD / "pipeline_cases.json").read_text())
    bert = dm.pipeline.build_bert_large()
    for sw in data["sweeps"]:
        res = dm.pipeline.sweep(bert, dm.pipeline.reference_fleets(), sw["bw"], sw["alpha"], sw["n_b"])
        got = [[r.fleet, r.bandwidth_gbps, r.alpha_ms, r.n_batches, repr(r.latency_s), repr(r.pipe_time_s),
                repr(r.throughput)] for r in res.rows]
        assert got == sw["rows"]
