#!/usr/bin/env python3
"""Full-size parity pins for the benchmarked configurations.

The bench reports winners, feasible counts and checksums over whole
populations (C2: 8,589,934,558 splits per scenario; C1: the 1024-fleet link
grid; C3/C5: random-placement streams; C4: batched schedule()).  This script
computes the same quantities on CPU, independently of the engine, and writes
them to tests/golden/full_size.json, which the -m gpu tests compare with the
engine bit for bit.

Instances are built with the REFERENCE package (pkg/src/dagmesh imported
read-only from /root/reference): `ir.parse_job_definition` + `build_stages`
(scheduling.py:107-145) for the jobs, `hardware.parse_fleet`
(hardware.py:315-354) for the fleets.  Scoring is done by

* the reference's own functions where they finish in minutes
  (`schedule()` scheduling.py:391-423 on all 1024 C1 fleets and on C3), and
* the oracle (oracle/dm_oracle.c, the C restatement pinned to the reference
  by tests/test_oracle_golden.py) for the populations the Python reference
  would need days for: `or_enum` mode 1 = brute_force_schedule's inner body
  (scheduling.py:264-272) in the identity-split order, threaded over rank
  ranges and merged by (makespan, rank) = the reference's first strict
  minimum (:271).

Run in the build container (all host cores; C2 takes ~10 min per scenario):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_full_size.py [part ...]

parts: c2 c2hi c1 c3sched c3rand c5rand c4   (default: all)
Existing entries of full_size.json are kept unless recomputed.
"""

from __future__ import annotations

import json
import os
import pathlib
import sys
import time
from concurrent.futures import ThreadPoolExecutor

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = pathlib.Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
from dagmesh import hardware as hw, ir, scheduling as S  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2309_01172_b200 import configs as CF  # noqa: E402

OUT = HERE / "full_size.json"
THREADS = os.cpu_count() or 1
M64 = (1 << 64) - 1

# C2 scenarios pinned at full size (indices into configs.C2_LINKS)
C2_PINNED = (0, 5, 10, 15)
# a rank sub-range of C2 scenario 0 entirely above 2^32
C2_HI_RANGE = (5_000_000_000, 5_000_000_000 + 200_000_000)


def ref_stages(name):
    job, cells = CF.encoder_job(**CF.MODELS[name])
    return S.build_stages(ir.parse_job_definition(job), cells)


def ref_fleet(doc):
    return hw.parse_fleet(json.dumps(doc))


def merge(parts):
    best = None
    tot_e = tot_f = cs = 0
    for w in parts:
        tot_e += w["n_evaluated"]
        tot_f += w["n_feasible"]
        cs = (cs + w["checksum"]) & M64
        if w["rank"] >= 0 and (best is None or (w["makespan"], w["rank"]) < (best["makespan"], best["rank"])):
            best = w
    return {"makespan": best["makespan"] if best else float("inf"), "rank": best["rank"] if best else -1,
            "n_evaluated": tot_e, "n_feasible": tot_f, "checksum": cs}


def threaded(fn, k0, k1, chunks=None):
    """fn(a, b) over [k0, k1) split into chunks on all host threads (the
    oracle releases the GIL inside ctypes)."""
    chunks = chunks or THREADS * 8
    step = max((k1 - k0 + chunks - 1) // chunks, 1)
    ranges = [(a, min(a + step, k1)) for a in range(k0, k1, step)]
    with ThreadPoolExecutor(THREADS) as ex:
        return merge(list(ex.map(lambda ab: fn(*ab), ranges)))


def c2(res):
    stages = ref_stages("llama2-7b-layers")
    out = res.setdefault("c2", {})
    for s in C2_PINNED:
        a, bw = CF.C2_LINKS[s]
        inst = oracle.Instance(stages, ref_fleet(CF.c2_fleet_doc(0, a, bw)))
        total = oracle.splits_total(inst.n, inst.p)
        t0 = time.time()
        w = threaded(lambda k0, k1: inst.enum("splits", k0, k1), 0, total)
        w["seconds"] = time.time() - t0
        w["scenario"], w["alpha_s"], w["bandwidth_gbps"] = s, a, bw
        out[str(s)] = w
        print(f"c2 scenario {s}: {w}", flush=True)
        save(res)


def c2hi(res):
    stages = ref_stages("llama2-7b-layers")
    inst = oracle.Instance(stages, ref_fleet(CF.c2_fleet_doc(0, *CF.C2_LINKS[0])))
    k0, k1 = C2_HI_RANGE
    w = threaded(lambda a, b: inst.enum("splits", a, b), k0, k1)
    w["k0"], w["k1"] = k0, k1
    res["c2_hi_range"] = w
    print("c2 hi range:", w, flush=True)
    save(res)


def c1(res):
    """Reference schedule() on every fleet of the 32 x 32 link grid, and the
    oracle's brute-force winner over the 62,704-candidate population of each."""
    stages = ref_stages("gpt2-small")
    bws, alphas = CF.c1_link_grid()
    docs = [CF.c1_fleet_doc(bw, al) for bw in bws for al in alphas]
    t0 = time.time()
    sched = []
    for d in docs:
        rep = S.schedule(stages, ref_fleet(d))
        sched.append({"runs": [[p, list(i)] for p, i in rep.runs], "makespan": rep.makespan,
                      "feasible": rep.feasible, "trace": list(rep.trace)})
    t_sched = time.time() - t0

    def bf(i):
        inst = oracle.Instance(stages, ref_fleet(docs[i]))
        return inst.enum("bruteforce", 0, oracle.bruteforce_total(inst.n, inst.p))
    with ThreadPoolExecutor(THREADS) as ex:
        brute = list(ex.map(bf, range(len(docs))))
    res["c1"] = {"schedule": sched, "bruteforce": brute, "reference_schedule_seconds": t_sched,
                 "fleets": len(docs)}
    print(f"c1: {len(docs)} schedules in {t_sched:.1f}s", flush=True)
    save(res)


def c3sched(res):
    """The reference's own schedule() on C3 (Llama-2-70B x 256 workers with
    32,640 pairwise links): proportional split + hill climb."""
    stages = ref_stages("llama2-70b")
    fleet = ref_fleet(CF.c3_fleet_doc(0))
    t0 = time.time()
    rep = S.schedule(stages, fleet)
    res["c3_schedule"] = {"runs": [[p, list(i)] for p, i in rep.runs], "makespan": rep.makespan,
                          "feasible": rep.feasible, "reason": rep.reason, "trace": list(rep.trace),
                          "reference_seconds": time.time() - t0}
    print("c3 schedule:", rep.makespan, rep.feasible, len(rep.runs), flush=True)
    save(res)


RANDOM_SEED = 20260
C3_RANDOM_N = 1 << 28
C5_RANDOM_N = 10 ** 9


def _random(res, name, stages, fleet, online_ids, N):
    inst = oracle.Instance(stages, fleet)
    online = np.array([inst.idx[i] for i in online_ids], np.int32)
    t0 = time.time()
    w = threaded(lambda a, b: inst.enum_random(online, RANDOM_SEED, a, b), 0, N)
    w.update(seed=RANDOM_SEED, candidates=N, seconds=time.time() - t0, n_online=int(online.size))
    res[name] = w
    print(name, w, flush=True)
    save(res)


def c3rand(res):
    fleet = ref_fleet(CF.c3_fleet_doc(0))
    _random(res, "c3_random", ref_stages("llama2-70b"), fleet, list(fleet.worker_ids()), C3_RANDOM_N)


def c5rand(res):
    _, online_ids = CF.c5_churn(1024, 0.1, 0)
    _random(res, "c5_random", ref_stages("opt-175b"), ref_fleet(CF.c5_fleet_doc(0)), online_ids, C5_RANDOM_N)


# ------------------------------------------------------------------ C4
C4_SCENARIOS = 10 ** 6
C4_CHUNK = 4096
C4_NB, C4_SPB = 512, 4
GPU_KINDS = tuple(hw.GPU_TABLE)
_C4 = {}


def c4_params(n_scen, seed=0):
    """The same draws as paper_2309_01172_b200/batch.c4_batch, in the same order."""
    rng = np.random.default_rng(seed)
    layers = rng.integers(32, 81, n_scen)
    hid = rng.integers(0, len(CF.C4_HIDDEN), n_scen)
    p = rng.integers(8, 65, n_scen)
    alpha = rng.uniform(0.0, 1e-2, n_scen)
    bw = 10.0 ** rng.uniform(-1.0, 1.0, n_scen)
    kinds = rng.integers(0, len(GPU_KINDS), int(p.sum()))
    lam = rng.uniform(0.3, 1.0, int(p.sum()))
    poff = np.concatenate([[0], np.cumsum(p)])
    return dict(layers=layers, hid=hid, p=p, alpha=alpha, bw=bw, kinds=kinds, lam=lam, poff=poff)


def c4_instance(P, s):
    """Scenario s through the reference: job -> parse_job_definition ->
    build_stages; fleet document -> parse_fleet."""
    L, h = int(P["layers"][s]), CF.C4_HIDDEN[int(P["hid"][s])]
    key = (L, h)
    if key not in _C4:
        job, cells = CF.encoder_job(h, L, 32000, 4, 1024)
        _C4[key] = S.build_stages(ir.parse_job_definition(job), cells)
    a, b = int(P["poff"][s]), int(P["poff"][s + 1])
    peers = [{"id": str(j - a + 1), "gpu": GPU_KINDS[int(P["kinds"][j])], "lambda": float(P["lam"][j])}
             for j in range(a, b)]
    doc = CF.fleet_doc(peers, float(P["alpha"][s]), float(P["bw"][s]), name="c4")
    return _C4[key], ref_fleet(doc)


def c4_chunk(args):
    """sha256 over the chunk's scenarios of (owner int16[n] | mk, latency,
    bottleneck, pipe, throughput, violation code as 6 float64) — the values the
    engine's prop_hill + epilogue produce (tests/golden_io.c4_record)."""
    from golden_io import c4_record
    import hashlib
    lo, hi = args
    P = _C4["params"]
    h = hashlib.sha256()
    feas = 0
    for s in range(lo, hi):
        stages, fleet = c4_instance(P, s)
        inst = oracle.Instance(stages, fleet)
        path, own = inst.schedule()
        runs = inst.owner_to_runs(own)
        mk, code, _, _, comp, read = inst.eval_runs(runs)
        lat, bn, pipe, thr = oracle.epilogue(comp, read, C4_NB, C4_SPB)
        h.update(c4_record(own, (mk, lat, bn, pipe, thr, float(code))))
        feas += code == 0
    return h.hexdigest(), feas


def c4(res):
    import multiprocessing as mp
    P = c4_params(C4_SCENARIOS)
    _C4["params"] = P
    chunks = [(a, min(a + C4_CHUNK, C4_SCENARIOS)) for a in range(0, C4_SCENARIOS, C4_CHUNK)]
    t0 = time.time()
    with mp.get_context("fork").Pool(THREADS) as pool:
        out = pool.map(c4_chunk, chunks, chunksize=1)
    import hashlib
    top = hashlib.sha256("".join(d for d, _ in out).encode()).hexdigest()
    # the reference's own schedule() on every 1000th scenario
    sample = []
    for s in range(0, C4_SCENARIOS, 1000):
        stages, fleet = c4_instance(P, s)
        rep = S.schedule(stages, fleet)
        sample.append({"s": s, "runs": [[p, list(i)] for p, i in rep.runs], "makespan": rep.makespan,
                       "feasible": rep.feasible})
    res["c4"] = {"scenarios": C4_SCENARIOS, "chunk": C4_CHUNK, "n_batches": C4_NB, "samples_per_batch": C4_SPB,
                 "chunk_digests": [d for d, _ in out], "digest": top, "n_feasible": int(sum(f for _, f in out)),
                 "seconds": time.time() - t0, "reference_sample": sample}
    print("c4:", top, res["c4"]["n_feasible"], flush=True)
    save(res)


def save(res):
    OUT.write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")


def main(parts):
    oracle.build()
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    res["generator"] = {"python": sys.version, "threads": THREADS,
                        "note": "instances built by the reference package; see the module docstring"}
    table = {"c2": c2, "c2hi": c2hi, "c1": c1, "c3sched": c3sched, "c3rand": c3rand, "c5rand": c5rand, "c4": c4}
    for p in parts or list(table):
        table[p](res)
    save(res)


if __name__ == "__main__":
    main(sys.argv[1:])
