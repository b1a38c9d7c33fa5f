"""Full-size parity: the engine on the exact populations the bench reports,
against tests/golden/full_size.json (computed on CPU by
tests/golden/make_full_size.py from instances built with the reference
package: the reference's own schedule() where it finishes in minutes, the
oracle's per-candidate restatement of brute_force_schedule's inner body for
the 8.6e9-candidate sweeps and the random-placement streams).

Bar: winner makespan bits, winner rank (the reference's first strict
minimum, scheduling.py:271), evaluated / feasible counts and the checksum of
every feasible candidate's makespan bits — identical."""

import hashlib
import json
import pathlib

import numpy as np
import pytest

from golden_io import c4_record

pytestmark = pytest.mark.gpu
GOLD = json.loads((pathlib.Path(__file__).resolve().parent / "golden" / "full_size.json").read_text())
KEYS = ("makespan", "rank", "n_evaluated", "n_feasible", "checksum")


def _w(d):
    return {k: d[k] for k in KEYS}


@pytest.fixture(scope="module")
def c2(engine_ready):
    from paper_2309_01172_b200 import configs as CF, engine
    from paper_2309_01172_b200.tensorize import build_host
    stages = CF.model_stages("llama2-7b-layers")
    fleets = [CF.load(CF.c2_fleet_doc(0, a, bw)) for a, bw in CF.C2_LINKS]
    batch = engine.device_batch([build_host(stages, f, True) for f in fleets])
    return engine, batch, engine.splits_total(len(stages), 32)


@pytest.mark.parametrize("scen", sorted(GOLD["c2"], key=int))
def test_c2_whole_population_sweep(c2, scen):
    """The headline meet-in-the-middle sweep over all 8,589,934,558 splits of
    a C2 scenario (the bench's per-scenario unit) equals the oracle's
    rank-order enumeration of the same population."""
    engine, batch, total = c2
    got = engine.enum(batch, "splits", 0, total, index=int(scen)).read()
    assert got == _w(GOLD["c2"][scen])


def test_c2_bench_graph_units(c2):
    """The bench's own timed object (engine.SweepGraph over the 16 link
    settings, one unit per scenario) reports the pinned winners."""
    engine, batch, total = c2
    g = engine.SweepGraph(batch, total, units=[(s, 0, 1) for s in range(len(batch.hosts))])
    g.launch()
    res = g.read_all()
    for scen, want in GOLD["c2"].items():
        assert res[int(scen)] == _w(want), scen


def test_c2_block_parts_merge_to_pinned(c2):
    """Multi-GPU form: the block-level parts of a scenario (dealt to 3 ranks)
    merge to the pinned whole-population result."""
    from paper_2309_01172_b200 import dist as D
    engine, batch, total = c2
    recs = []
    for part in range(3):
        bufs = engine.enum(batch, "splits", 0, total, part=part, nparts=3)
        recs.append(bufs.out.cpu().numpy())
    m = D.merge_records(np.stack(recs))
    assert {k: m[k] for k in KEYS} == _w(GOLD["c2"]["0"])


def test_c2_rank_range_above_2_32(c2):
    """A sub-range whose ranks all exceed 2^32 (rank-order kernel)."""
    engine, batch, _ = c2
    g = GOLD["c2_hi_range"]
    got = engine.enum(batch, "splits", g["k0"], g["k1"], index=0).read()
    assert got == _w(g) and got["rank"] > 2 ** 32


@pytest.fixture(scope="module")
def c1(engine_ready):
    from paper_2309_01172_b200 import configs as CF
    stages = CF.model_stages("gpt2-small")
    bws, alphas = CF.c1_link_grid()
    fleets = [CF.load(CF.c1_fleet_doc(bw, al)) for bw in bws for al in alphas]
    return stages, fleets


def test_c1_schedule_api_all_fleets(c1):
    """The reference's own schedule() on all 1024 link-grid fleets vs the
    engine's public schedule()."""
    from paper_2309_01172_b200 import scheduling as S
    stages, fleets = c1
    for i, f in enumerate(fleets):
        rep = S.schedule(stages, f)
        want = GOLD["c1"]["schedule"][i]
        assert [[p, list(x)] for p, x in rep.runs] == want["runs"], i
        assert rep.makespan == want["makespan"] and rep.feasible == want["feasible"], i
        assert list(rep.trace) == want["trace"], i


def test_c1_batched_dp_all_fleets(c1):
    """The bench's batched subset DP (one warp per fleet) picks the
    reference's schedule on every fleet."""
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200.tensorize import build_host
    stages, fleets = c1
    hosts = [build_host(stages, f, True) for f in fleets]
    batch = engine.device_batch(hosts)
    own, mk, found, _ = engine.subset_dp(batch, 26, 4)
    own, found = own.cpu().numpy(), found.cpu().numpy()
    for i, h in enumerate(hosts):
        want = GOLD["c1"]["schedule"][i]
        runs, a = [], 0
        for s in range(1, 27):
            if s == 26 or own[i, s] != own[i, a]:
                runs.append([h.peer_ids[int(own[i, a])], list(range(a, s))])
                a = s
        assert found[i] and runs == want["runs"], i


def test_c1_bruteforce_all_fleets(c1):
    """Brute-force order (all 62,704 candidates, itertools order) per fleet."""
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200.tensorize import build_host
    stages, fleets = c1
    batch = engine.device_batch([build_host(stages, f, True) for f in fleets])
    total = engine.bruteforce_total(26, 4)
    bufs = engine.WinnerBuffers(batch.dev_buf.device)
    for i in range(len(fleets)):
        assert engine.enum(batch, "bruteforce", 0, total, bufs, index=i).read() == _w(GOLD["c1"]["bruteforce"][i]), i


def test_c3_schedule_api(engine_ready):
    """C3 (Llama-2-70B x 256 workers, 32,640 pairwise links): schedule()."""
    from paper_2309_01172_b200 import configs as CF, scheduling as S
    rep = S.schedule(CF.model_stages("llama2-70b"), CF.load(CF.c3_fleet_doc(0)))
    want = GOLD["c3_schedule"]
    assert [[p, list(x)] for p, x in rep.runs] == want["runs"]
    assert rep.makespan == want["makespan"] and rep.feasible == want["feasible"] and rep.reason == want["reason"]
    assert list(rep.trace) == want["trace"]


@pytest.mark.parametrize("name", ["c3_random", "c5_random"])
def test_random_population(engine_ready, name):
    """The whole random-placement stream the bench scores (C3: 2^28
    candidates with pairwise links; C5: 10^9 over 922 online peers)."""
    from paper_2309_01172_b200 import configs as CF, engine
    from paper_2309_01172_b200.tensorize import build_host
    import torch
    want = GOLD[name]
    if name == "c3_random":
        stages, fleet = CF.model_stages("llama2-70b"), CF.load(CF.c3_fleet_doc(0))
        online_ids = list(fleet.worker_ids())
    else:
        stages, fleet = CF.model_stages("opt-175b"), CF.load(CF.c5_fleet_doc(0))
        online_ids = CF.c5_churn(1024, 0.1, 0)[1]
    host = build_host(stages, fleet, True)
    batch = engine.device_batch([host])
    online = torch.tensor([host.index_of[i] for i in online_ids], dtype=torch.int32, device=batch.dev_buf.device)
    got = engine.enum(batch, "random", 0, want["candidates"], online=online, seed=want["seed"]).read()
    assert got == _w(want)


def test_c4_million_scenarios(engine_ready):
    """10^6 C4 scenarios through the batched schedule() path (proportional
    split + hill climb + Eq. 3/4 epilogue): per-4096-scenario sha256 of every
    owner vector and its six result values equals the oracle's."""
    from paper_2309_01172_b200 import batch as B, engine
    g = GOLD["c4"]
    sb = B.c4_batch(g["scenarios"], seed=0)
    owner, _, _, epi_f = engine.prop_hill_epilogue(sb, sb.n_max, g["n_batches"], g["samples_per_batch"])
    epi = engine.epilogue(sb, sb.n_max, owner, g["n_batches"], g["samples_per_batch"]).cpu().numpy()
    assert np.array_equal(epi_f.cpu().numpy().view(np.uint64), epi.view(np.uint64))   # fused == separate
    owner = owner.cpu().numpy()
    ns = sb.records["n"]
    bad = []
    for c, lo in enumerate(range(0, g["scenarios"], g["chunk"])):
        h = hashlib.sha256()
        for s in range(lo, min(lo + g["chunk"], g["scenarios"])):
            h.update(c4_record(owner[s, :ns[s]], epi[s]))
        if h.hexdigest() != g["chunk_digests"][c]:
            bad.append(c)
    assert not bad, f"chunks differing: {bad[:10]}"
    assert int((epi[:, 5] == 0).sum()) == g["n_feasible"]


def test_split_sweep_public_api(c2):
    """search.split_sweep (stages + fleets in, decoded winners out) on the
    pinned C2 scenarios; the winner's runs re-scored by evaluate_runs give
    the pinned makespan; block parts over 2 callers merge to the same."""
    from paper_2309_01172_b200 import configs as CF, dist as D, scheduling as S, search
    stages = CF.model_stages("llama2-7b-layers")
    idx = sorted(int(s) for s in GOLD["c2"])
    fleets = [CF.load(CF.c2_fleet_doc(0, *CF.C2_LINKS[i])) for i in idx]
    for rev in (False, False, True):    # replay on repacked inputs; reordered fleets (other default links)
        res = search.split_sweep(stages, fleets[::-1] if rev else fleets)
        for i, w in zip(idx[::-1] if rev else idx, res):
            want = GOLD["c2"][str(i)]
            assert (w.makespan, w.rank, w.n_evaluated, w.n_feasible, w.checksum) == tuple(want[k] for k in KEYS)
            assert S.evaluate_runs(stages, fleets[idx.index(i)], w.runs).makespan == want["makespan"]
    parts = [search.split_sweep(stages, fleets[:1], part=k, nparts=2, records=True) for k in range(2)]
    m = D.merge_records(np.stack([p_[0] for p_ in parts]))
    assert {k: m[k] for k in KEYS} == _w(GOLD["c2"][str(idx[0])])


def test_split_sweeper_pipelined(c2):
    """search.SplitSweeper (two slots, request k+1 prepared while k runs):
    every request's winners equal the pinned ones."""
    from paper_2309_01172_b200 import configs as CF, search
    stages = CF.model_stages("llama2-7b-layers")
    idx = sorted(int(s) for s in GOLD["c2"])
    fleets = [CF.load(CF.c2_fleet_doc(0, *CF.C2_LINKS[i])) for i in idx]
    sw = search.SplitSweeper(stages, fleets)
    tickets = [sw.submit(fleets)]
    for k in range(3):
        tickets.append(sw.submit(fleets[::-1] if k % 2 == 0 else fleets))
        res = sw.result(tickets[k])
        order = idx if k % 2 == 0 else idx[::-1]
        for i, w in zip(order, res):
            want = GOLD["c2"][str(i)]
            assert (w.makespan, w.rank, w.n_evaluated, w.n_feasible, w.checksum) == tuple(want[k_] for k_ in KEYS)
    sw.result(tickets[-1])
