"""Host-side logic that runs without a GPU: the mirror types and fleet
parser, the rank codecs against itertools, the counter RNG (Python vs C
oracle), sharding/merging, closed-form stage tables against the reference's
build_stages digests, and the tensoriser's flags."""

import hashlib
import itertools
import json
import math
import pathlib

import numpy as np
import pytest

from paper_2309_01172_b200 import configs as CF
from paper_2309_01172_b200 import dist as D
from paper_2309_01172_b200 import engine, refapi as M, rng as R
from paper_2309_01172_b200.tensorize import build_host

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


def test_unrank_matches_itertools_order():
    for n in range(1, 8):
        for p in range(1, 5):
            k = 0
            for r in range(1, min(n, p) + 1):
                for cuts in itertools.combinations(range(1, n), r - 1):
                    for chosen in itertools.permutations(range(p), r):
                        b, pe = engine.unrank(n, p, k, "bruteforce")
                        assert b == [0, *cuts, n] and pe == list(chosen)
                        k += 1
            assert k == engine.bruteforce_total(n, p)


def test_oracle_unrank_matches_python(oracle_mod):
    rng = np.random.default_rng(0)
    st = [M.Stage(i, "s", 1.0, 1, 1, 1) for i in range(12)]
    fl = M.Fleet(peers={str(i): M.Peer(str(i)) for i in range(1, 6)})
    inst = oracle_mod.Instance(st, fl)
    for mode, tot in (("bruteforce", engine.bruteforce_total(12, 5)), ("splits", engine.splits_total(12, 5))):
        for k in rng.integers(0, tot, 200):
            assert inst.unrank(mode, int(k)) == engine.unrank(12, 5, int(k), mode)


def test_rng_python_matches_c(oracle_mod):
    """rng.py (product-side restatement of the candidate recipe) and the
    oracle's C restatement draw identical candidates."""
    L = oracle_mod.lib()
    b = np.zeros(300, np.int32)
    pe = np.zeros(300, np.int32)
    for n, n_online in ((194, 922), (162, 256), (5, 3), (1, 1), (40, 1000), (257, 300)):
        for k in [0, 1, 2, 17, 10**9, 2**40 + 3]:
            r = L.or_random_candidate(n, n_online, 12345, k, b.ctypes.data, pe.ctypes.data)
            bb, pp = R.candidate(n, n_online, 12345, k)
            assert b[: r + 1].tolist() == bb and pe[:r].tolist() == pp
            assert len(set(pp)) == len(pp) and all(0 <= x < n_online for x in pp)
            assert 1 <= r <= min(n, n_online) and bb == sorted(set(bb)) and bb[0] == 0 and bb[-1] == n


def test_rng_distribution_matches_survey():
    """r ~ U{1..min(n, n_online)} and, given r, every
    (r-1)-subset of the cut positions equally likely (chi-square on a small
    shape), r distinct peers."""
    from collections import Counter
    n, n_online, N = 6, 4, 24000
    by_r, subsets = Counter(), Counter()
    for k in range(N):
        bb, pp = R.candidate(n, n_online, 7, k)
        by_r[len(pp)] += 1
        subsets[tuple(bb)] += 1
        assert len(set(pp)) == len(pp)
    assert set(by_r) == {1, 2, 3, 4}
    assert all(abs(c - N / 4) < 5 * math.sqrt(N / 4) for c in by_r.values())
    for r in (2, 3, 4):
        cells = [c for s, c in subsets.items() if len(s) == r + 1]
        assert len(cells) == math.comb(n - 1, r - 1)
        exp = by_r[r] / len(cells)
        chi2 = sum((c - exp) ** 2 / exp for c in cells)
        assert chi2 < 3 * len(cells) + 20
    # peers: every online index appears as run 0 about equally often
    first = Counter(R.candidate(10, 5, 3, k)[1][0] for k in range(5000))
    assert set(first) == set(range(5)) and max(first.values()) < 1.25 * min(first.values())


def test_shard_covers_range():
    for total in (0, 1, 7, 1000, 8589934558):
        for world in (1, 2, 3, 8):
            parts = [D.shard(total, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))


def test_merge_records_first_strict_min():
    import struct
    recs = [(2.0, 10, 5, 4, 7), (1.0, 30, 5, 5, 9), (1.0, 20, 5, 5, 1), (math.inf, -1, 3, 0, 0)]
    raw = np.frombuffer(b"".join(struct.pack(D.WINNER_FMT, *r) for r in recs), np.uint8)
    m = D.merge_records(raw)
    assert (m["makespan"], m["rank"], m["n_evaluated"], m["n_feasible"], m["checksum"]) == (1.0, 20, 18, 14, 17)


def test_closed_form_stages_match_reference_digests():
    digests = json.loads((GOLD / "stage_digests.json").read_text())
    for name, d in digests.items():
        st = CF.model_stages(name) if name in CF.MODELS else CF.encoder_stages(**d["kw"])
        blob = repr([(s.index, s.label, s.flops, s.gpu_bytes, s.cpu_bytes, s.disk_bytes, s.in_edges) for s in st])
        assert len(st) == d["n"] and hashlib.sha256(blob.encode()).hexdigest() == d["sha256"], name


def test_fleet_parser_and_tensoriser_flags():
    doc = {"name": "t", "peers": [{"id": "10", "gpu": "h100"}, {"id": "2", "gpu": "rtx3080", "lambda": 0.5},
                                  {"id": "b", "tflops_tensor": 1.0, "gpu_gb": 2}],
           "links": {"default_alpha_s": 0.001, "bandwidth_gbps": 2.0,
                     "overrides": [{"src": "2", "dst": "10", "alpha_s": 0.5, "bandwidth_gbps": 1.0}]},
           "backup_pool": ["2"], "pinned_runs": [[1, 2], [3]]}
    fl = M.parse_fleet(json.dumps(doc))
    assert fl.worker_ids() == ("10", "b") and fl.peer_ids() == ("2", "10", "b")
    assert fl.pinned_runs == ((0, 1), (2,))
    assert fl.link_between("10", "2").alpha == 0.5 and fl.link_between("b", "2").alpha == 0.001
    st = [M.Stage(0, "a", 3.0, 10, 10, 10), M.Stage(1, "b", 4.0, 10, 10, 10, ((0, 100),))]
    h = build_host(st, fl)
    assert h.peer_ids == ("10", "b", "2") and h.p == 2 and h.P == 3
    from paper_2309_01172_b200 import _lib
    assert h.flags & _lib.DM_F_CHAIN and h.flags & _lib.DM_F_PAIR_LINKS and h.flags & _lib.DM_F_FLOPS_EXACT
    la = h.arrays["link_alpha"].reshape(3, 3)
    assert la[2, 0] == 0.5 and la[0, 2] == 0.5 and la[1, 2] == 0.001 and la[0, 0] == 0.0
    with pytest.raises(M.FleetError):
        M.parse_fleet({"peers": [{"id": "1", "gpu": "nope"}]})
    frac = [M.Stage(0, "a", 0.5, 1, 1, 1)]
    assert not build_host(frac, fl).flags & _lib.DM_F_FLOPS_EXACT


def test_reference_fleet_files_parse_identically(dagmesh_ref):
    from golden_io import dump_fleet
    for f in pathlib.Path("/root/reference/pkg/fleets").glob("*.json"):
        a = dump_fleet(dagmesh_ref.hardware.load_fleet(f))
        b = dump_fleet(M.load_fleet(f))
        assert a == b, f


def test_report_assembly_types_golden():
    """scheduling._report (host-side report assembly) fed with the oracle's
    per-run costs reproduces the reference's reports field for field —
    including which floats are numpy.float64 (fleets built from rng draws):
    CPython's sum() over report values is compensated only over exact floats,
    so the types are part of parity."""
    import json
    import pathlib

    import numpy as np

    from golden_io import load_fleet, load_stages, report_matches, runs_of
    from oracle import oracle as O
    from paper_2309_01172_b200 import refapi as M
    from paper_2309_01172_b200 import scheduling as S
    from paper_2309_01172_b200.tensorize import build_host

    O.build()
    cases = json.loads((pathlib.Path(__file__).parent / "golden" / "scheduling_cases.json").read_text())["cases"]
    n_np = n = 0
    for c in cases:
        if c["kind"] != "solve":
            continue
        st, fl = load_stages(c["stages"], M), load_fleet(c["fleet"], M)
        want = c["schedule"]
        if not want["feasible"]:
            continue
        runs = runs_of(want["runs"])
        inst = O.Instance(st, fl)
        mk, code, bad, status, comp, read = inst.eval_runs(runs)
        res = dict(compute=np.asarray(comp), read=np.asarray(read), makespan=np.array([mk]),
                   code=np.array([code]), code_run=np.array([bad]), status=np.array([status]),
                   cand_ptr=np.array([0, len(runs)]))
        rep = S._report(st, fl, runs, True, tuple(want["trace"]), res, 0, build_host(st, fl))
        assert report_matches(rep, want) == [], c["tag"]
        n += 1
        n_np += "float64" in json.dumps(want["types"])
    assert n > 250 and n_np > 200


def test_bench_scenario_units_cover_every_scenario_once():
    """bench.units_for: every (scenario, part) of the batch is owned by exactly
    one rank, for any GPU count, and every rank holds the same number of units
    (the winner all-gather's fixed record count)."""
    import bench
    for n_scen in (1, 3, 8):
        for world in range(1, 9):
            owned = [bench.units_for(r, world, n_scen) for r in range(world)]
            assert len({len(u) for u in owned}) == 1
            flat = [u for us in owned for u in us]
            assert len(flat) == len(set(flat))
            for s in range(n_scen):
                parts = sorted((p, k) for (sc, p, k) in flat if sc == s)
                assert parts and [p for p, _ in parts] == list(range(parts[0][1]))


def test_stage_fast_path_equals_reference_build_stages():
    """Tensoriser fast path (configs.stages_for: encoder chains in closed
    form) against the reference's own build_stages on every model the
    benchmark builds — all 196 C4 models (block cells), the C4b layer-cell
    chains, the named configs — and the reference's own MODELS; a graph
    that is not an encoder chain falls back to build_stages."""
    from dagmesh import ir, pipeline as PL, scheduling as RS
    jobs = []
    for L in range(32, 81):
        for h in CF.C4_HIDDEN:
            jobs.append(CF.encoder_job(h, L, 32000, 4, 1024))
    for L in range(24, 37):
        jobs.append(CF.encoder_job(4096, L, 32000, 4, 1024, cells="layer"))
    for kw in CF.MODELS.values():
        jobs.append(CF.encoder_job(**kw))
    for job, cells in jobs:
        g = ir.parse_job_definition(job)
        assert CF.encoder_params(g, cells) is not None
        assert CF.stages_for(g, cells) == RS.build_stages(g, cells)
    for mdl in (PL.build_bert_large(), PL.build_gpt3_24(), PL.build_bert_large(2, 64)):
        assert CF.encoder_params(mdl.graph, mdl.cells) is not None
        assert CF.stages_for(mdl.graph, mdl.cells) == RS.build_stages(mdl.graph, mdl.cells)
    job, cells = CF.encoder_job(1024, 3, 30522, 2, 64)
    g = ir.parse_job_definition(job)
    topo = RS.topological_cells(g)
    assert CF.encoder_params(g, topo) is None and CF.stages_for(g, topo) == RS.build_stages(g, topo)
    job["nodes"][3]["kwargs"] = {"inner_features": 77}          # one ffn differs from the others
    g = ir.parse_job_definition(job)
    assert CF.encoder_params(g, cells) is None and CF.stages_for(g, cells) == RS.build_stages(g, cells)


def test_tensoriser_link_matrix_and_stage_cache():
    """Vectorised link matrix == the fleet's own link_between for every pair
    (asymmetric overrides, both orders present, unknown ids skipped); the
    lazy form (link_pairs) matches on the requested pairs; the stage side is
    shared between fleets while fleet columns follow each fleet."""
    import itertools
    from paper_2309_01172_b200 import tensorize as TZ
    doc = {"name": "t", "peers": [{"id": str(i), "gpu": g} for i, g in
                                  enumerate(["h100", "rtx3080", "a100", "rtx4090", "rtx4080"], 1)],
           "links": {"default_alpha_s": 0.002, "bandwidth_gbps": 3.0,
                     "overrides": [{"src": "1", "dst": "2", "alpha_s": 0.5, "bandwidth_gbps": 1.0},
                                   {"src": "2", "dst": "1", "alpha_s": 0.25, "bandwidth_gbps": 2.0},
                                   {"src": "3", "dst": "5", "alpha_s": 0.125, "bandwidth_gbps": 4.0}]},
           "backup_pool": ["4"]}
    fl = M.parse_fleet(json.dumps(doc))
    st = CF.model_stages("gpt2-small")
    h = build_host(st, fl)
    P = h.P
    la, lb = h.arrays["link_alpha"].reshape(P, P), h.arrays["link_beta"].reshape(P, P)
    for i, j in itertools.product(range(P), range(P)):
        lk = fl.link_between(h.peer_ids[i], h.peer_ids[j])
        assert (la[i, j], lb[i, j]) == ((0.0, 0.0) if i == j else (lk.alpha, lk.beta))
    pairs = [(0, 1), (1, 0), (2, 3)]
    hl = build_host(st, fl, link_pairs=pairs)
    lla = hl.arrays["link_alpha"].reshape(P, P)
    assert all(lla[i, j] == la[i, j] for i, j in pairs)
    fl2 = M.parse_fleet(json.dumps({**doc, "links": {"default_alpha_s": 0.001}}))
    h2 = build_host(st, fl2)
    assert h2.arrays["pre_flops"] is h.arrays["pre_flops"]              # cached stage side
    assert h2.def_alpha == 0.001 and "link_alpha" not in dict(h2.segments())
    assert TZ.stage_side(st) is TZ.stage_side(list(st))


def test_report_fast_paths_match_reference_semantics():
    """The report assembly's shortcuts build the same values and objects as
    the reference's own code: per-run byte sums from the exact prefixes have
    the value AND type of sum() over the stage attributes (ints stay ints,
    floats stay floats, mixed columns fall back), and PeerLoad rows built
    without the frozen dataclass's __init__ are equal, hash-equal and still
    frozen."""
    import dataclasses

    from paper_2309_01172_b200 import scheduling as SCH
    from paper_2309_01172_b200.tensorize import stage_side

    def stages_of(vals):
        return [M.Stage(i, f"s{i}", 1e9, g, c, d, ((i - 1, 8),) if i else ()) for i, (g, c, d) in enumerate(vals)]

    rng = np.random.default_rng(3)
    ints = [(int(rng.integers(1, 2**40)), int(rng.integers(1, 2**30)), int(rng.integers(0, 2**20))) for _ in range(40)]
    floats = [(float(g), float(c), float(d)) for g, c, d in ints]
    mixed = [(g if i % 2 else float(g), c, d) for i, (g, c, d) in enumerate(ints)]
    for vals, exact in ((ints, True), (floats, True), (mixed, False)):
        st = stages_of(vals)
        side = stage_side(st)
        for a, b in ((0, 1), (3, 17), (0, 40), (39, 40)):
            got = side.range_bytes(a, b)
            want = tuple(sum(getattr(st[i], f) for i in range(a, b)) for f in ("gpu_bytes", "cpu_bytes", "disk_bytes"))
            if not exact:
                assert got is None
                continue
            assert got == want and [type(x) for x in got] == [type(x) for x in want]
    vals = ("7", (1, 2), 0.5, 0.25, 0.75, 10, 20.0, 30)
    fast, ref = SCH._peer_load(*vals), M.PeerLoad(*vals)
    assert type(fast) is type(ref) and fast == ref and hash(fast) == hash(ref) and repr(fast) == repr(ref)
    assert dataclasses.astuple(fast) == dataclasses.astuple(ref)
    with pytest.raises(dataclasses.FrozenInstanceError):
        fast.peer = "8"
