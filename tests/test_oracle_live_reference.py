"""The oracle against the LIVE reference package (build container only:
/root/reference is absent on the GPU box, where the committed golden fixtures
take over).  Fresh seeded instances each run — DAG and chain stages, pairwise
links, non-integral FLOPs, msg_ratio != 1, memory pressure — compared on
schedule(), brute_force_schedule(), evaluate_runs() and the Eq. 3/4 epilogue."""

import numpy as np
import pytest

from golden_io import dump_fleet, dump_stages, load_fleet, load_stages

pytestmark = pytest.mark.reference


@pytest.fixture(scope="module")
def ref(dagmesh_ref):
    return dagmesh_ref


def _ref_types(dm):
    from types import SimpleNamespace
    return SimpleNamespace(Stage=dm.scheduling.Stage, Peer=dm.hardware.Peer, Role=dm.hardware.Role,
                           Fleet=dm.hardware.Fleet, Link=dm.hardware.Link)


def test_oracle_matches_live_reference(ref, oracle_mod):
    from gen import big_instance, random_stages, uniform_fleet
    from paper_2309_01172_b200 import refapi as M
    rng = np.random.default_rng(20261018)
    RT = _ref_types(ref)
    S, PL = ref.scheduling, ref.pipeline
    n_checked = 0
    for k in range(60):
        if k % 2:
            st, fl = big_instance(rng, int(rng.integers(12, 50)), int(rng.integers(4, 20)), dag=k % 4 == 1,
                                  frac=k % 6 == 1, links=k % 3 == 0)
        else:
            st = random_stages(rng, int(rng.integers(3, 11)))
            fl = uniform_fleet(list(rng.uniform(1e8, 1e9, int(rng.integers(2, 5)))),
                               link=M.Link(float(rng.uniform(0, 1e-3)), float(rng.uniform(0, 1e-7))),
                               gpu_gb=float(rng.uniform(0.5, 1.5)) * sum(s.gpu_bytes for s in st) / 2**30)
        rst, rfl = load_stages(dump_stages(st), RT), load_fleet(dump_fleet(fl), RT)
        inst = oracle_mod.Instance(st, fl)
        want = S.schedule(rst, rfl)
        path, own = inst.schedule()
        if path > 0:
            assert inst.owner_to_runs(own) == want.runs, k
        else:
            assert not want.feasible, k
        if want.feasible:
            prof = PL.profiles_from_report(want)
            mk, code, _, _, comp, read = inst.eval_runs(want.runs)
            assert mk == want.makespan and code == 0
            assert oracle_mod.epilogue(comp, read, 64, 4, inst.load_np(want.runs)) == (PL.fp_latency(prof), PL.bottleneck(prof),
                                                               PL.pipeline_time(prof, 64),
                                                               PL.throughput(prof, 64, 4))
        if len(st) <= 10 and len(fl.worker_ids()) <= 4:
            bf = S.brute_force_schedule(rst, rfl)
            w = inst.enum("bruteforce", 0, oracle_mod.bruteforce_total(inst.n, inst.p))
            assert (w["rank"] < 0) == (not bf.feasible)
            if w["rank"] >= 0:
                assert w["makespan"] == bf.makespan
        n_checked += 1
    assert n_checked == 60
