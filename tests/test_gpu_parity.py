"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle on
identical seeded inputs.  Bar: bit-identical float64 values, identical
violation codes, identical chosen runs (the reference's tie-breaks)."""

import math

import numpy as np
import pytest

from gen import big_instance, criterion6_instances, random_stages, uniform_fleet
from paper_2309_01172_b200 import engine, refapi as M, rng as R, scheduling as S
from paper_2309_01172_b200.tensorize import build_host

pytestmark = pytest.mark.gpu


def same(a, b):
    return (math.isnan(a) and math.isnan(b)) or a == b


def _oracle_runs(inst, own):
    return inst.owner_to_runs(own)


# ------------------------------------------------------------ evaluate_runs
def _random_runs(rng, stages, fleet, kind):
    n = len(stages)
    workers = list(fleet.worker_ids())
    if kind == "contig":
        r = int(rng.integers(1, min(n, len(workers)) + 1))
        cuts = sorted(rng.choice(np.arange(1, n), r - 1, replace=False).tolist()) if r > 1 else []
        b = [0] + cuts + [n]
        peers = rng.choice(workers, r, replace=False).tolist()
        return tuple((peers[q], tuple(range(b[q], b[q + 1]))) for q in range(r))
    if kind == "owner":
        own = rng.integers(0, len(workers), n)
        d = {}
        for i, o in enumerate(own):
            d.setdefault(workers[o], []).append(i)
        return tuple((k, tuple(v)) for k, v in d.items())
    if kind == "twice":
        runs = list(_random_runs(rng, stages, fleet, "contig"))
        if len(runs) > 1:
            pe, idx = runs[1]
            runs[1] = (pe, idx + (runs[0][1][-1],))
        return tuple(runs)
    if kind == "gap":
        runs = list(_random_runs(rng, stages, fleet, "contig"))
        pe, idx = runs[-1]
        runs[-1] = (pe, idx[:-1])
        return tuple(runs)
    raise ValueError(kind)


def test_evaluate_runs_matches_oracle(oracle_mod, engine_ready):
    rng = np.random.default_rng(5)
    insts = criterion6_instances(count=60)
    for k in range(12):
        insts.append(big_instance(rng, int(rng.integers(10, 60)), int(rng.integers(3, 20)), dag=k % 2 == 0,
                                  frac=k % 3 == 0, links=k % 4 == 0))
    checked = 0
    for stages, fleet in insts:
        inst = oracle_mod.Instance(stages, fleet)
        for kind in ("contig", "owner", "twice", "gap"):
            for _ in range(4):
                runs = _random_runs(rng, stages, fleet, kind)
                mk, code, bad, status, comp, read = inst.eval_runs(runs)
                if status != 0:
                    with pytest.raises((KeyError, M.FleetError)):
                        S.evaluate_runs(stages, fleet, runs)
                    continue
                rep = S.evaluate_runs(stages, fleet, runs)
                assert same(rep.makespan, mk), (kind, runs, rep.makespan.hex(), mk.hex())
                assert rep.feasible == (code == 0), (kind, runs, rep.reason, code)
                by_run = {(pe, tuple(sorted(ix))): (c, r) for (pe, ix), c, r in zip(runs, comp, read) if ix}
                for row in rep.per_peer:
                    if row.stage_indices and (row.peer, row.stage_indices) in by_run:
                        c, r = by_run[(row.peer, row.stage_indices)]
                        assert row.compute_s == c and row.read_s == r
                checked += 1
    assert checked > 500


def test_unknown_peer_raises(engine_ready):
    stages = random_stages(np.random.default_rng(1), 4)
    fleet = uniform_fleet([1e9, 2e9])
    with pytest.raises(M.FleetError, match="unknown peer"):
        S.evaluate_runs(stages, fleet, (("9", (0, 1, 2, 3)),))
    assert "unknown peer" in S.verify_assignment(stages, fleet, (("9", (0, 1, 2, 3)),))


# ---------------------------------------------------------------- solvers
def test_schedule_matches_oracle_dp_path(oracle_mod, engine_ready):
    for stages, fleet in criterion6_instances():
        inst = oracle_mod.Instance(stages, fleet)
        path, own = inst.schedule()
        rep = S.schedule(stages, fleet)
        if path < 0:
            assert not rep.feasible and rep.makespan == math.inf
            continue
        assert rep.runs == inst.owner_to_runs(own)
        assert rep.trace == ("exact subset search",)


def test_schedule_matches_oracle_hill_path(oracle_mod, engine_ready):
    rng = np.random.default_rng(7)
    for k in range(40):
        stages, fleet = big_instance(rng, int(rng.integers(15, 70)), int(rng.integers(6, 24)), dag=k % 2 == 0,
                                     frac=k % 4 == 1, links=k % 3 == 0)
        inst = oracle_mod.Instance(stages, fleet)
        path, own = inst.schedule()
        rep = S.schedule(stages, fleet)
        assert rep.runs == inst.owner_to_runs(own), k
        assert rep.feasible == (path > 0), k


def test_schedule_dp_with_pair_links(oracle_mod, engine_ready):
    rng = np.random.default_rng(99)
    for k in range(30):
        stages = random_stages(rng, int(rng.integers(3, 10)))
        fleet = uniform_fleet(list(rng.uniform(1e8, 1e9, int(rng.integers(2, 5)))),
                              link=M.Link(float(rng.uniform(0, 1e-3)), float(rng.uniform(0, 1e-7))))
        ids = fleet.worker_ids()
        fleet.links[(ids[0], ids[-1])] = M.Link(float(rng.uniform(0, 1e-3)), float(rng.uniform(0, 1e-7)))
        inst = oracle_mod.Instance(stages, fleet)
        path, own = inst.schedule()
        rep = S.schedule(stages, fleet)
        assert rep.runs == inst.owner_to_runs(own)


def test_brute_force_matches_oracle(oracle_mod, engine_ready):
    for stages, fleet in criterion6_instances(count=120):
        inst = oracle_mod.Instance(stages, fleet)
        total = oracle_mod.bruteforce_total(inst.n, inst.p)
        w = inst.enum("bruteforce", 0, total)
        rep = S.brute_force_schedule(stages, fleet)
        if w["rank"] < 0:
            assert not rep.feasible
            continue
        b, pe = inst.unrank("bruteforce", w["rank"])
        runs = tuple((inst.workers[pe[q]], tuple(range(b[q], b[q + 1]))) for q in range(len(pe)))
        assert rep.runs == tuple(sorted(runs, key=lambda r: r[1][0]))
        assert rep.makespan == w["makespan"]


def test_enumeration_winner_checksum_and_sharding(oracle_mod, engine_ready):
    rng = np.random.default_rng(11)
    stages = random_stages(rng, 9)
    fleet = uniform_fleet(list(rng.uniform(1e8, 1e9, 5)), link=M.Link(2e-4, 3e-8), gpu_gb=0.02)
    inst = oracle_mod.Instance(stages, fleet)
    host = build_host(stages, fleet)
    batch = engine.device_batch([host])
    total = engine.bruteforce_total(9, 5)
    for k0, k1 in [(0, total), (0, 1), (17, 4000), (total // 3, total)]:
        want = inst.enum("bruteforce", k0, k1)
        got = engine.enum(batch, "bruteforce", k0, k1).read()
        assert got == want, (k0, k1)
    total_s = engine.splits_total(9, 5)
    assert engine.enum(batch, "splits", 0, total_s).read() == inst.enum("splits", 0, total_s)


def test_splits_enumeration_larger(oracle_mod, engine_ready):
    rng = np.random.default_rng(12)
    st, fleet = big_instance(rng, 20, 12, dag=False, pressure=(0.2, 0.9))
    inst = oracle_mod.Instance(st, fleet)
    batch = engine.device_batch([build_host(st, fleet)])
    total = engine.splits_total(20, 12)
    assert engine.enum(batch, "splits", 0, total).read() == inst.enum("splits", 0, total)
    st2, fleet2 = big_instance(rng, 14, 6, dag=True, links=True, pressure=(0.3, 0.9))
    inst2 = oracle_mod.Instance(st2, fleet2)
    batch2 = engine.device_batch([build_host(st2, fleet2)])
    total2 = engine.splits_total(14, 6)
    assert engine.enum(batch2, "splits", 0, total2).read() == inst2.enum("splits", 0, total2)


def test_random_placements(oracle_mod, engine_ready):
    import torch
    rng = np.random.default_rng(13)
    for links in (True, False):
        _random_case(oracle_mod, rng, links)


def _random_case(oracle_mod, rng, links):
    import torch
    st, fleet = big_instance(rng, 60, 256, dag=False, links=links, pressure=(0.05, 0.4))
    inst = oracle_mod.Instance(st, fleet)
    host = build_host(st, fleet)
    batch = engine.device_batch([host])
    online = np.sort(rng.choice(256, 200, replace=False)).astype(np.int32)
    dev = batch.dev_buf.device
    on_d = torch.from_numpy(online).to(dev)
    for seed, k0, k1 in [(1, 0, 30000), (2, 1000, 21000), (3, 2**33, 2**33 + 5000)]:
        got = engine.enum(batch, "random", k0, k1, online=on_d, seed=seed).read()
        want = inst.enum_random(online, seed, k0, k1)
        assert got == want
        if got["rank"] >= 0:
            b, pe = R.candidate(60, len(online), seed, got["rank"])
            runs = tuple((host.peer_ids[online[pe[q]]], tuple(range(b[q], b[q + 1]))) for q in range(len(pe)))
            assert S.evaluate_runs(st, fleet, runs).makespan == got["makespan"]


# --------------------------------------------------------------- Mode A
@pytest.mark.parametrize("dag,links,wide", [(False, False, False), (True, True, False), (False, True, True),
                                            (False, True, False), (True, False, False)])
def test_eval_owner_stream(oracle_mod, engine_ready, dag, links, wide):
    import torch
    rng = np.random.default_rng(21)
    n, p = 34, (300 if wide else 32)
    st, fleet = big_instance(rng, n, p, dag=dag, links=links, pressure=(0.05, 0.5))
    inst = oracle_mod.Instance(st, fleet)
    host = build_host(st, fleet)
    batch = engine.device_batch([host])
    N = 3000
    own = np.zeros((N, n), np.int64)
    for c in range(N):
        kind = c % 3
        if kind == 0:
            own[c] = rng.integers(0, p, n)
        else:
            r = int(rng.integers(1, 20))
            cuts = sorted(rng.choice(np.arange(1, n), r - 1, replace=False).tolist())
            b = [0] + cuts + [n]
            pe = rng.choice(p, r, replace=False)
            for q in range(r):
                own[c, b[q]:b[q + 1]] = pe[q]
    own[7, 3] = host.P + 2  # unknown peer
    dt = torch.int16 if wide else torch.uint8
    o_d = torch.from_numpy(own.astype(np.int16 if wide else np.uint8)).to(batch.dev_buf.device).to(dt)
    mk, code = engine.eval_owner(batch, o_d)
    mk, code = mk.cpu().numpy(), code.cpu().numpy()
    for c in range(N):
        m_o, c_o = inst.eval_owner(own[c])
        assert int(code[c]) == c_o, c
        assert same(float(mk[c]), m_o), (c, float(mk[c]).hex(), m_o.hex())


def test_argmin_scores(engine_ready):
    import torch
    rng = np.random.default_rng(3)
    mk = rng.integers(0, 50, 100000).astype(np.float64) / 7.0
    code = (rng.random(100000) < 0.3).astype(np.uint8)
    bufs = engine.argmin_scores(torch.from_numpy(mk).cuda(), torch.from_numpy(code).cuda(), rank_base=1000)
    got = bufs.read()
    ok = np.where(code == 0)[0]
    best = ok[np.argmin(mk[ok])]
    assert got["rank"] == 1000 + best and got["makespan"] == mk[best]
    assert got["n_feasible"] == ok.size and got["n_evaluated"] == 100000


# ------------------------------------------------------------ batched solvers
@pytest.mark.parametrize("form", ["default", "cta", "warp", "generic"])
def test_subset_dp_batch(oracle_mod, engine_ready, monkeypatch, form):
    """Every DP kernel form on the criterion-6 instances vs the oracle:
    the launcher's choice, the 4-warp CTA form, the warp form and the generic
    one-CTA-per-scenario kernel."""
    if form == "cta":
        monkeypatch.setenv("DM_DP_CTA", "1")
    elif form == "warp":
        monkeypatch.setenv("DM_DP_CTA", "0")
    elif form == "generic":
        monkeypatch.setenv("DM_DISABLE_DP_WARP", "1")
        monkeypatch.setenv("DM_DISABLE_DP_LANE", "1")
    insts = [i for i in criterion6_instances(count=80)]
    hosts = [build_host(s, f) for s, f in insts]
    batch = engine.device_batch(hosts)
    n_max = max(h.n for h in hosts)
    p_max = max(h.p for h in hosts)
    owner, mk, found, _ = engine.subset_dp(batch, n_max, p_max)
    owner, mk, found = owner.cpu().numpy(), mk.cpu().numpy(), found.cpu().numpy()
    for s, (st, fl) in enumerate(insts):
        own, m = oracle_mod.Instance(st, fl).subset_dp()
        if own is None:
            assert found[s] == 0
            continue
        assert found[s] == 1 and mk[s] == m
        assert owner[s, :len(st)].tolist() == own.tolist()


@pytest.mark.parametrize("knob", [None, "DM_DISABLE_DP_LANE"])
def test_subset_dp_mid_fleets(oracle_mod, engine_ready, monkeypatch, knob):
    """Fleets of 6-8 workers (the thread-per-(mask, worker) DP kernel, and
    with DM_DISABLE_DP_LANE the generic one-CTA-per-scenario kernel): chosen
    runs and makespans equal the oracle's _subset_dp restatement, including
    forced ties (identical peers, uniform stages) and infeasible instances."""
    if knob:
        monkeypatch.setenv(knob, "1")
    rng = np.random.default_rng(66)
    insts = []
    for k in range(48):
        n, p = int(rng.integers(8, 39)), int(rng.integers(6, 9))
        st, fl = big_instance(rng, n, p, dag=k % 4 == 1, pressure=(0.02, 0.5) if k % 6 else (0.001, 0.01))
        insts.append((st, fl))
    for p in (6, 7, 8):                                          # ties: equal speeds, equal stages
        st = [M.Stage(i, f"s{i}", 1e12, 2.0**20, 1024.0, 512.0, ((i - 1, 1 << 20),) if i else ())
              for i in range(int(rng.integers(p, 30)))]
        insts.append((st, uniform_fleet([50e12] * p, link=M.Link(1e-3, 8 / 1e10))))
    hosts = [build_host(s, f) for s, f in insts]
    batch = engine.device_batch(hosts)
    n_max = max(h.n for h in hosts)
    owner, mk, found, _ = engine.subset_dp(batch, n_max, 8)
    owner, mk, found = owner.cpu().numpy(), mk.cpu().numpy(), found.cpu().numpy()
    n_found = 0
    for s, (st, fl) in enumerate(insts):
        own, m = oracle_mod.Instance(st, fl).subset_dp()
        if own is None:
            assert found[s] == 0, s
            continue
        n_found += 1
        assert found[s] == 1 and mk[s] == m, s
        assert owner[s, :len(st)].tolist() == own.tolist(), s
    assert n_found >= 20


def test_prop_hill_batch_and_epilogue(oracle_mod, engine_ready):
    rng = np.random.default_rng(31)
    insts = [big_instance(rng, int(rng.integers(20, 80)), int(rng.integers(12, 40)), dag=k % 2 == 1, links=k % 5 == 0)
             for k in range(64)]
    hosts = [build_host(s, f) for s, f in insts]
    batch = engine.device_batch(hosts)
    n_max = max(h.n for h in hosts)
    owner, score, moves = engine.prop_hill(batch, n_max)
    epi = engine.epilogue(batch, n_max, owner, 512, 8).cpu().numpy()
    owner = owner.cpu().numpy()
    for s, (st, fl) in enumerate(insts):
        inst = oracle_mod.Instance(st, fl)
        path, own = inst.schedule()
        assert owner[s, :len(st)].tolist() == own.tolist(), s
        runs = inst.owner_to_runs(own)
        mk, code, _, _, comp, read = inst.eval_runs(runs)
        assert epi[s, 0] == mk and int(epi[s, 5]) == code
        lat, bn, pipe, thr = oracle_mod.epilogue(comp, read, 512, 8)
        assert (epi[s, 1], epi[s, 2], epi[s, 3], epi[s, 4]) == (lat, bn, pipe, thr)


def test_splits_memo_matches_generic(engine_ready, monkeypatch):
    """The shared-memory memo kernel and the generic per-run kernel agree
    (winner, counts, checksum) on chain, DAG and no-comm instances."""
    rng = np.random.default_rng(44)
    for dag, links, inc in [(False, False, True), (False, True, True), (True, False, True), (True, True, False)]:
        st, fleet = big_instance(rng, 22, 14, dag=dag, links=links, pressure=(0.1, 0.8))
        batch = engine.device_batch([build_host(st, fleet, inc)])
        total = engine.splits_total(22, 14)
        a = engine.enum(batch, "splits", 0, total).read()
        b = engine.enum(batch, "splits", 12345, total - 999).read()
        monkeypatch.setenv("DM_DISABLE_MEMO", "1")
        a2 = engine.enum(batch, "splits", 0, total).read()
        b2 = engine.enum(batch, "splits", 12345, total - 999).read()
        monkeypatch.delenv("DM_DISABLE_MEMO")
        assert a == a2 and b == b2


def test_materialized_stream_matches_enumeration(engine_ready):
    """Mode A (materialised owner vectors scored from HBM + arg-min) and Mode B
    (in-kernel enumeration) agree on the same rank range: winner, counts and
    the checksum of every feasible candidate's makespan."""
    rng = np.random.default_rng(8)
    for dag, links in [(False, False), (False, True), (True, False)]:
        st, fleet = big_instance(rng, 30, 24, dag=dag, links=links, pressure=(0.1, 0.6))
        batch = engine.device_batch([build_host(st, fleet)])
        total = engine.splits_total(30, 24)
        k0, cnt = total // 3, 2_000_000
        own = engine.materialize(30, 24, "splits", k0, cnt)
        mk, code = engine.eval_owner(batch, own)
        a = engine.argmin_scores(mk, code, rank_base=k0).read()
        b = engine.enum(batch, "splits", k0, k0 + cnt).read()
        assert a == b
        (mk2, code2), bufs = engine.eval_owner_argmin(batch, own, rank_base=k0)
        assert bufs.read() == b
        assert bool((mk2 == mk).all()) and bool((code2 == code).all())
    bf_total = engine.bruteforce_total(9, 5)
    st, fleet = big_instance(rng, 9, 5, dag=False, links=True, pressure=(0.2, 0.9))
    batch = engine.device_batch([build_host(st, fleet)])
    own = engine.materialize(9, 5, "bruteforce", 0, bf_total)
    mk, code = engine.eval_owner(batch, own)
    assert engine.argmin_scores(mk, code).read() == engine.enum(batch, "bruteforce", 0, bf_total).read()


def test_split_parts_partition_the_population(engine_ready):
    """dm_enum_splits_part: the interleaved parts are disjoint and cover the
    population; merging their records equals the single sweep."""
    import struct
    from paper_2309_01172_b200 import dist as D
    rng = np.random.default_rng(17)
    for dag, links in ((False, False), (True, False), (True, True)):
        st, fleet = big_instance(rng, 26 if not links else 20, 20 if not links else 9, dag=dag, links=links,
                                 pressure=(0.1, 0.7))
        batch = engine.device_batch([build_host(st, fleet)])
        total = engine.splits_total(len(st), len(fleet.worker_ids()))
        full = engine.enum(batch, "splits", 0, total).read()
        for nparts in (2, 3, 8):
            recs = []
            for part in range(nparts):
                w = engine.enum(batch, "splits", 0, total, part=part, nparts=nparts).read()
                recs.append(struct.pack(D.WINNER_FMT, w["makespan"], w["rank"], w["n_evaluated"], w["n_feasible"],
                                        w["checksum"]))
            assert D.merge_records(np.frombuffer(b"".join(recs), np.uint8)) == full


def test_splits_mitm_matches_memo_and_oracle(oracle_mod, engine_ready, monkeypatch):
    """The whole-population meet-in-the-middle sweep (dm_mitm.cu) against the
    oracle (small shapes, incl. n = 1, p = 1, n < p, n > p) and against the
    rank-range memo kernel (larger shapes, memory pressure, DAG with a uniform
    link, no-comm); part-wise sweeps merge to the same record."""
    import struct
    from paper_2309_01172_b200 import dist as D
    rng = np.random.default_rng(2309)
    shapes = [(1, 1), (1, 4), (2, 1), (2, 2), (3, 5), (6, 3), (9, 9), (12, 5), (16, 16), (18, 7)]
    for i, (n, p) in enumerate(shapes):
        st, fleet = big_instance(rng, n, p, dag=i % 3 == 1, links=False, pressure=(0.05, 0.9))
        inst = oracle_mod.Instance(st, fleet)
        batch = engine.device_batch([build_host(st, fleet)])
        total = engine.splits_total(n, p)
        assert engine.enum(batch, "splits", 0, total).read() == inst.enum("splits", 0, total), (n, p)
    for n, p, dag, links, inc, pr in [(30, 24, False, True, True, (0.1, 0.6)), (28, 28, True, False, True, (0.05, 0.5)),
                                      (26, 12, True, True, False, (0.2, 0.9)), (34, 32, False, False, True, (0.3, 1.2))]:
        st, fleet = big_instance(rng, n, p, dag=dag, links=links, pressure=pr)
        batch = engine.device_batch([build_host(st, fleet, inc)])
        total = engine.splits_total(n, p)
        a = engine.enum(batch, "splits", 0, total).read()
        monkeypatch.setenv("DM_DISABLE_MITM", "1")
        b = engine.enum(batch, "splits", 0, total).read()
        monkeypatch.delenv("DM_DISABLE_MITM")
        assert a == b and a["n_evaluated"] == total, (n, p)
        recs = []
        for part in range(3):
            w = engine.enum(batch, "splits", 0, total, part=part, nparts=3).read()
            recs.append(struct.pack(D.WINNER_FMT, w["makespan"], w["rank"], w["n_evaluated"], w["n_feasible"],
                                    w["checksum"]))
        assert D.merge_records(np.frombuffer(b"".join(recs), np.uint8)) == a


def test_splits_c_abi_without_workspace(engine_ready):
    """dm_enum_splits / dm_enum_splits_part called directly through the C ABI
    (no caller workspace: the library allocates its side tables
    stream-ordered) return the same record as the engine's workspace path."""
    import ctypes as C
    import torch
    from paper_2309_01172_b200 import _lib
    rng = np.random.default_rng(5)
    st, fleet = big_instance(rng, 24, 20, dag=False, links=True, pressure=(0.1, 0.7))
    batch = engine.device_batch([build_host(st, fleet)])
    total = engine.splits_total(24, 20)
    want = engine.enum(batch, "splits", 0, total).read()
    lib = _lib.load()
    bufs = engine.WinnerBuffers(batch.dev_buf.device)
    stt = batch.struct(0)
    _lib.check(lib.dm_enum_splits(C.byref(stt), 0, total, bufs.out.data_ptr(), bufs.scratch.data_ptr(),
                                  _lib.stream_ptr()))
    assert bufs.read() == want
    _lib.check(lib.dm_enum_splits_part(C.byref(stt), 0, total, 0, 1, bufs.out.data_ptr(), bufs.scratch.data_ptr(),
                                       _lib.stream_ptr()))
    assert bufs.read() == want
    torch.cuda.synchronize()


def test_sweep_graph_matches_enum(engine_ready):
    """engine.SweepGraph (H2D + sweep kernels + D2H captured as one CUDA graph)
    returns the enumeration's record on every replay."""
    rng = np.random.default_rng(9)
    st, fleet = big_instance(rng, 22, 16, dag=False, links=True, pressure=(0.1, 0.7))
    batch = engine.device_batch([build_host(st, fleet)])
    total = engine.splits_total(22, 16)
    want = engine.enum(batch, "splits", 0, total).read()
    g = engine.SweepGraph(batch, total)
    for _ in range(3):
        g.launch()
        assert g.read() == want


def test_sweep_graph_units_overlap_matches_enum(engine_ready):
    """A SweepGraph over several instances (unit i+1's side tables on a side
    stream, overlapping unit i's sweep) returns every instance's own record,
    and dm_enum_splits_phase 1 then 2 equals the one-call sweep."""
    import torch
    rng = np.random.default_rng(11)
    hosts = []
    for _ in range(3):
        st, fleet = big_instance(rng, 22, 16, dag=False, links=True, pressure=(0.1, 0.7))
        hosts.append(build_host(st, fleet))
    batch = engine.device_batch(hosts)
    total = engine.splits_total(22, 16)
    want = [engine.enum(batch, "splits", 0, total, index=i).read() for i in range(3)]
    g = engine.SweepGraph(batch, total, units=[(0, 0, 1), (1, 0, 1), (2, 0, 1)])
    assert g.overlap
    for _ in range(2):
        g.launch()
        assert g.read_all() == want
    bufs = engine.WinnerBuffers(batch.dev_buf.device)
    engine.enum(batch, "splits", 0, total, bufs, index=1, phase=1)
    engine.enum(batch, "splits", 0, total, bufs, index=1, phase=2)
    assert bufs.read() == want[1]
    torch.cuda.synchronize()


def test_splits_phase_needs_workspace(engine_ready):
    """dm_enum_splits_phase: the split halves (1, 2) need the caller's
    workspace (the tables live there between the calls) and fail loudly
    without one; phase 3 without a workspace allocates its own."""
    import ctypes as C
    import torch
    from paper_2309_01172_b200 import _lib
    rng = np.random.default_rng(5)
    st, fleet = big_instance(rng, 16, 8, dag=False, links=False, pressure=(0.1, 0.7))
    batch = engine.device_batch([build_host(st, fleet)])
    total = engine.splits_total(16, 8)
    lib = _lib.load()
    bufs = engine.WinnerBuffers(batch.dev_buf.device)
    stt = batch.struct(0)
    for phase in (1, 2):
        rc = lib.dm_enum_splits_phase(C.byref(stt), 0, total, 0, 1, bufs.out.data_ptr(), bufs.scratch.data_ptr(),
                                      None, 0, phase, _lib.stream_ptr())
        assert rc != 0
    rc = lib.dm_enum_splits_phase(C.byref(stt), 0, total, 0, 1, bufs.out.data_ptr(), bufs.scratch.data_ptr(),
                                  None, 0, 3, _lib.stream_ptr())
    assert rc == 0
    assert bufs.read() == engine.enum(batch, "splits", 0, total).read()
    # the phase sequences 1+2 and 1+4+8 (plan and sweep apart) equal phase 3,
    # for the whole population and for block parts
    for nparts in (1, 3):
        want = [engine.enum(batch, "splits", 0, total, part=q, nparts=nparts).read() for q in range(nparts)]
        for seq in ((1, 2), (1, 4, 8)):
            got = []
            for q in range(nparts):
                b2 = engine.WinnerBuffers(batch.dev_buf.device)
                for ph in seq:
                    engine.enum(batch, "splits", 0, total, b2, part=q, nparts=nparts, phase=ph)
                got.append(b2.read())
            assert got == want, (nparts, seq)
    torch.cuda.synchronize()


def test_sweep_graph_part_units_merge(engine_ready):
    """A SweepGraph of block-level parts of one instance (the bench's units
    when the scenario batch does not divide the GPUs): the parts' records
    merge to the whole sweep's."""
    import torch
    from paper_2309_01172_b200 import dist as D
    rng = np.random.default_rng(13)
    st, fleet = big_instance(rng, 24, 14, dag=False, links=True, pressure=(0.1, 0.7))
    batch = engine.device_batch([build_host(st, fleet)])
    total = engine.splits_total(24, 14)
    want = engine.enum(batch, "splits", 0, total).read()
    g = engine.SweepGraph(batch, total, units=[(0, 0, 3), (0, 1, 3), (0, 2, 3)], copy_inputs=False)
    g.launch()
    torch.cuda.synchronize()
    assert D.merge_records(g.out.cpu().numpy()) == want


# Every Mode A stream configuration (threads, CTAs/SM, candidates per thread,
# ring stages, square/triangular table) against the oracle, with contiguous,
# non-contiguous and out-of-range owners (P <= w < 32 and w >= 32), a ragged
# last tile and the fused arg-min.
MODEA_CFGS = ["256,4,2,3,1", "256,3,2,3,1", "256,2,4,3,1", "128,8,2,3,1", "512,2,1,2,1",
              "768,1,1,2,0", "512,1,1,2,0", "1024,1,1,2,0", "256,2,2,3,0"]


@pytest.mark.parametrize("cfg", MODEA_CFGS)
@pytest.mark.parametrize("shape", [(26, 4), (34, 32), (12, 7), (64, 9)])
def test_eval_owner_stream_configs(oracle_mod, engine_ready, monkeypatch, cfg, shape):
    import torch
    n, p = shape
    rng = np.random.default_rng(1000 + n * p)
    st, fleet = big_instance(rng, n, p, dag=False, links=False, pressure=(0.1, 0.6))
    inst = oracle_mod.Instance(st, fleet)
    host = build_host(st, fleet)
    batch = engine.device_batch([host])
    N = 4099
    own = np.zeros((N, n), np.int64)
    for c in range(N):
        r = int(rng.integers(1, min(n, p) + 1))
        cuts = sorted(rng.choice(np.arange(1, n), r - 1, replace=False).tolist()) if r > 1 else []
        b = [0] + cuts + [n]
        pe = rng.choice(p, r, replace=False)
        for q in range(r):
            own[c, b[q]:b[q + 1]] = pe[q]
        if c % 97 == 5:
            own[c] = rng.integers(0, p, n)                     # non-contiguous
    own[11, n // 2] = p + 1                                    # P <= w < 32
    own[12, n - 1] = 200                                       # w >= 32
    own[13, 0] = 255
    monkeypatch.setenv("DM_MODEA_CFG", cfg)
    o_d = torch.from_numpy(own.astype(np.uint8)).cuda()
    (mk, code), bufs = engine.eval_owner_argmin(batch, o_d, rank_base=77)
    win = bufs.read()
    mk, code = mk.cpu().numpy(), code.cpu().numpy()
    best, feas, csum = None, 0, 0
    for c in range(N):
        m_o, c_o = inst.eval_owner(own[c])
        assert int(code[c]) == c_o, (cfg, c)
        assert same(float(mk[c]), m_o), (cfg, c, float(mk[c]).hex(), m_o.hex())
        if c_o == 0:
            feas += 1
            csum = (csum + int(np.float64(m_o).view(np.uint64))) % (1 << 64)
            if best is None or m_o < best[0]:
                best = (m_o, 77 + c)
    assert win["n_evaluated"] == N and win["n_feasible"] == feas and win["checksum"] == csum
    if best:
        assert (win["makespan"], win["rank"]) == best


@pytest.mark.parametrize("shape", [(18, 12, False), (26, 9, True), (34, 32, True), (40, 64, False)])
def test_splits_direct_kernel_matches_oracle(oracle_mod, engine_ready, monkeypatch, shape):
    """The per-candidate split evaluator (splits_direct_kernel: staged tables,
    Markstein-corrected division) equals the oracle's per-candidate
    enumeration bit for bit (winner, counts, checksum of every feasible
    makespan), on sub-ranges and across block boundaries."""
    n, p, links = shape
    rng = np.random.default_rng(500 + n)
    st, fleet = big_instance(rng, n, p, dag=False, links=False, pressure=(0.1, 0.8))
    inst = oracle_mod.Instance(st, fleet)
    batch = engine.device_batch([build_host(st, fleet)])
    total = engine.splits_total(n, p)
    monkeypatch.setenv("DM_DISABLE_MEMO", "1")
    for k0, k1 in ((0, min(total, 300000)), (total // 2 - 150000, total // 2 + 150000), (max(total - 200000, 0), total),
                   (total - 1000, total + 5000)):
        k0 = max(k0, 0)
        assert engine.enum(batch, "splits", k0, k1).read() == inst.enum("splits", k0, k1), (k0, k1)
