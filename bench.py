#!/usr/bin/env python3
"""Benchmark of the placement-cost / partition-search hot path.

Default workload (N=1 and scaling runs): BASELINE.json configs[1] — the
Llama-2-7B training workflow (34 layer cells) over a 32-device heterogeneous
fleet, EXHAUSTIVE split sweep: all 8,589,934,558 contiguous splits with run q
on worker q, each scored with the reference cost model (fits + compute +
crossing read, makespan) and reduced to the first strict minimum by
(makespan, rank).  One step = the full sweep of that fleet under each of 16
default-link settings (configs.C2_LINKS, the base 5 ms / 10 Gbit/s first):
16 x 8.59e9 candidates.  The 16 scenarios are sharded across the ranks (whole
scenarios per GPU, strong scaling; block-level parts of every scenario when
16 is not a multiple of the GPU count), plus one NCCL all-gather of the
per-rank winner records.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
       (multi-GPU: python -m torch.distributed.run --nproc-per-node N bench.py --gpus N)
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "candidate placements evaluated/sec (+ partition DPs solved/sec)"
UNIT = "candidates/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2"])
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary measurements")
    return ap.parse_args()


# ------------------------------------------------------------------ workload
def c2_instance():
    from paper_2309_01172_b200 import configs as CF
    stages = CF.model_stages("llama2-7b-layers")
    fleet = CF.load(CF.c2_fleet_doc(0))
    return stages, fleet


def c2_scenarios():
    """The C2 model and its fleet under every C2_LINKS default link."""
    from paper_2309_01172_b200 import configs as CF
    stages = CF.model_stages("llama2-7b-layers")
    return stages, [CF.load(CF.c2_fleet_doc(0, a, bw)) for a, bw in CF.C2_LINKS], list(CF.C2_LINKS)


def units_for(rank, world, n_scen):
    """(scenario, part, nparts) units of `rank`: whole scenarios when the
    batch divides evenly, else every scenario split into `world` parts."""
    if n_scen % world == 0:
        return [(s, 0, 1) for s in range(rank, n_scen, world)]
    return [(s, rank, world) for s in range(n_scen)]


def workload_config(total, links):
    return {"workload": "C2 llama2-7b (34 layer cells) x 32 heterogeneous workers, exhaustive split sweep under "
                        f"{len(links)} default-link settings per step",
            "candidates_per_step": total * len(links), "candidates_per_scenario": total, "scenarios": len(links),
            "default_links_s_gbps": [list(x) for x in links], "stages": 34, "workers": 32,
            "candidate_source": "generated on chip: splits grouped by (cut count, middle-cut position) as cross "
                                "products of left x right cut sets; each feasible candidate's makespan = "
                                "max(L, R) folded into the checksum, infeasible ones resolved per side element",
            "l2_policy": "no HBM-resident candidate stream; each scenario's side tables (134 MB) exceed L2 and are "
                         "rebuilt every step",
            "parallelism": "whole scenarios per GPU (block-level parts when the batch does not divide) + 1 NCCL "
                           "all-gather of 40-byte winner records"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50", "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except OSError:
            return None
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- b200 arm
def run_b200(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2309_01172_b200 import dist as D
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200.tensorize import build_host

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream()
    stages, fleets, links = c2_scenarios()
    S = len(fleets)
    n, p = len(stages), len(fleets[0].worker_ids())
    total = engine.splits_total(n, p)
    batch = engine.device_batch([build_host(stages, f, True) for f in fleets], device=dev)
    units = units_for(rank, world, S)

    def gather(out):
        """device records [units, 40] of every rank -> [world, units, 40]"""
        if world == 1:
            return out.view(1, len(units), -1)
        g = torch.empty(world * out.numel(), dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(g, out.reshape(-1))
        return g.view(world, len(units), -1)

    def merge(raw):
        per = [[] for _ in range(S)]
        for r in range(world):
            for i, (sc, _, _) in enumerate(units_for(r, world, S)):
                per[sc].append(raw[r, i])
        return [D.merge_records(np.stack(rows)) for rows in per]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the sweeps' kernels as one graph (tables resident in HBM).  Multi-GPU:
    # the winner all-gather follows each step and the host waits for it, so
    # NCCL's kernels never share the SMs with a running sweep
    kernels = engine.SweepGraph(batch, total, units=units, copy_inputs=False)
    for _ in range(max(args.warmup, 3)):
        kernels.launch()
        gather(kernels.out)
    barrier()
    clocks = ClockSampler(local_rank)
    if rank == 0:
        clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ev0.record(stream)
    for s in range(args.steps):
        kev[s][0].record(stream)
        kernels.launch()
        kev[s][1].record(stream)
        if world > 1:
            gather(kernels.out)
            stream.synchronize()
    ev1.record(stream)
    barrier()
    clk = clocks.stop() if rank == 0 else None
    ms = ev0.elapsed_time(ev1)
    kernel_ms = statistics.mean(a.elapsed_time(b) for a, b in kev)
    t = torch.tensor([ms, kernel_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kernel_ms = float(t[0]), float(t[1])
    res = merge(gather(kernels.out).cpu().numpy())

    # ---- e2e: the engine's serving form (engine.SweepGraph: one CUDA graph
    #      with the H2D copy of the scenario tables from pinned host memory,
    #      the sweeps' kernels and the D2H of the winner records), host
    #      synchronisation and the winners read every step
    sweep = engine.SweepGraph(batch, total, units=units)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pinned_out = torch.empty(world * len(units) * D.WINNER_BYTES, dtype=torch.uint8, pin_memory=True)
    e0.record(stream)
    for _ in range(args.steps):
        sweep.launch()
        if world > 1:
            pinned_out.copy_(gather(sweep.out).view(-1), non_blocking=True)
            stream.synchronize()
            merge(pinned_out.numpy().reshape(world, len(units), -1))
        else:
            sweep.read_all()
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te[0])
    e2e_d2h = (world if world > 1 else 1) * len(units) * D.WINNER_BYTES

    # the dominant kernel's own duration on every rank (its first unit): CUDA
    # events the library records around its launches, in a separate pass
    u0 = units[0]
    kb = kernels.unit_bufs[0]
    tab_ms, sweep_ms = engine.sweep_kernel_times(batch, total, steps=args.steps, bufs=kb, part=u0[1],
                                                 nparts=u0[2], index=u0[0])
    feas0 = kb.read()["n_feasible"]
    per_rank = torch.tensor([tab_ms, sweep_ms], dtype=torch.float64, device=dev)
    if world > 1:
        gathered = torch.empty(2 * world, dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(gathered, per_rank)
        per_rank = gathered
    per_rank = per_rank.view(-1, 2).cpu().tolist()
    extras = {}
    if rank == 0 and not args.no_extras and world == 1:
        extras = secondary_measurements(dev)
    if rank != 0:
        return None
    value = S * total * args.steps / (ms / 1e3)
    e2e_val = S * total * args.steps / (e2e_ms / 1e3)
    cross = extras.get("cross_peak_pairs_per_s")
    achieved = feas0 / (sweep_ms / 1e3) / 1e9      # one launch of the dominant kernel
    # theoretical ALU-pipe bound of the inner loop: 64 integer/select lane-ops
    # per clock per SM, 3 per candidate pair (FSEL, SEL, half of IADD3 + IADD3.X)
    alu_peak = None
    if clk and clk.get("sm_mhz"):
        alu_peak = torch.cuda.get_device_properties(dev).multi_processor_count * clk["sm_mhz"] * 1e6 * 64 / 3
    traffic = ncu_traffic("splits_sweep_kernel") or {}
    hbm_peak = _hbm_peak()[0]
    csum = 0
    for r in res:
        csum = (csum + r["checksum"]) & ((1 << 64) - 1)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(total, links),
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(batch.h2d_bytes),
                "d2h_bytes_per_step": int(e2e_d2h)},
        "gpu_launches": 5 * len(units) * args.steps,
        "roofline": {"bound": "issue", "achieved": achieved, "peak": (cross / 1e9) if cross else None,
                     "unit": "Gcand/s", "frac": (achieved / (cross / 1e9)) if cross else None,
                     "traffic": traffic.get("bytes"), "traffic_source": traffic.get("capture"),
                     "alu_peak_pairs_per_s": alu_peak, "frac_of_alu_peak": (achieved * 1e9 / alu_peak) if alu_peak else None,
                     "hbm_view": ({"achieved_gbs": traffic["bytes"] / (sweep_ms / 1e3) / 1e9, "peak_gbs": hbm_peak,
                                   "frac": traffic["bytes"] / (sweep_ms / 1e3) / 1e9 / hbm_peak,
                                   "note": "ncu DRAM bytes of one sweep / the kernel's duration: not memory bound"}
                                  if traffic.get("bytes") and hbm_peak else None),
                     "kernel": "splits_sweep_kernel", "kernel_ms": sweep_ms, "table_phase_ms": tab_ms,
                     "per_rank_table_sweep_ms": per_rank,
                     "step_kernels_ms": kernel_ms,
                     "algorithmic_work_per_candidate": "one fp64 max (DSETP + 64-bit select) and one 64-bit "
                                                       "checksum add per feasible candidate",
                     "note": "feasible candidates per second of one splits_sweep_kernel launch (rank 0's first "
                             "unit) vs dm_microbench_cross (the same inner loop alone, same grid and occupancy: "
                             "the ALU-pipe/issue bound); infeasible candidates are resolved per side element (an "
                             "unfit run), as the reference's `continue` skips them; table_phase_ms = T image + "
                             "side tables of that unit"},
        "winner": {"per_scenario": [[r["makespan"], r["rank"]] for r in res],
                   "n_feasible": sum(r["n_feasible"] for r in res), "n_evaluated": sum(r["n_evaluated"] for r in res),
                   "checksum_sum": csum},
    }
    if clk:
        line["clocks"] = clk
    line.update(extras)
    return line


_UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def ncu_traffic(kernel_substr, profile_glob="r1_prof_*_raw.csv"):
    """dram__bytes_read.sum + dram__bytes_write.sum of the newest committed
    `ncu --set full` capture (profiles/*_raw.csv) of a kernel, with the
    capture's duration, so callers can scale per launch / per candidate."""
    import csv
    best = None
    for f in sorted((ROOT / "profiles").glob(profile_glob), key=lambda x: x.stat().st_mtime):
        try:
            rows = list(csv.reader(open(f)))
            hdr, units, vals = rows[0], rows[1], rows[2]
            name = vals[hdr.index("Kernel Name")]
            if kernel_substr not in name:
                continue
            rd = float(vals[hdr.index("dram__bytes_read.sum")].replace(",", "")) * _UNITS[units[hdr.index("dram__bytes_read.sum")]]
            wr = float(vals[hdr.index("dram__bytes_write.sum")].replace(",", "")) * _UNITS[units[hdr.index("dram__bytes_write.sum")]]
            best = {"bytes": rd + wr, "capture": f.name, "kernel": name}
        except Exception:
            continue
    return best


def _hbm_peak():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _time_ms(fn, steps=5, warmup=3):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / steps


def mode_a_measure(dev, which):
    """Mode A scoring stream (owner vectors resident in HBM, > L2) with the
    fused arg-min; roofline = HBM bytes n*w + 9 per candidate."""
    import math
    import time as _t
    import torch
    from oracle import oracle
    from paper_2309_01172_b200 import configs as CF
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200.tensorize import build_host
    if which == "c2":
        stages, fleet = c2_instance()
        n, p = 34, 32
        N = 1 << 28
        total = engine.splits_total(n, p)
        k0 = total // 2 - N // 2
        own = engine.materialize(n, p, "splits", k0, N, device=dev)
        desc = f"C2 split ranks [{k0}, {k0 + N}) materialised as uint8 owner vectors ({N * n / 1e9:.1f} GB)"
    else:
        stages = CF.model_stages("gpt2-small")
        fleet = CF.load(CF.c1_fleet_doc(10.0, 1e-3))
        n, p = 26, 4
        total = engine.bruteforce_total(n, p)
        base = engine.materialize(n, p, "bruteforce", 0, total, device=dev)
        N = 1 << 27
        own = base.repeat(math.ceil(N / total), 1)[:N].contiguous()
        del base
        k0 = 0
        desc = (f"C1 (gpt2-small x 4 mixed GPUs, 10 Gbit/s, 1 ms) brute-force-order candidates, the 62,704 "
                f"population tiled to {N} uint8 owner vectors ({N * n / 1e9:.1f} GB)")
    host = build_host(stages, fleet, True)
    batch = engine.device_batch([host], device=dev)
    out = (torch.empty(N, dtype=torch.float64, device=dev), torch.empty(N, dtype=torch.uint8, device=dev))
    bufs = engine.WinnerBuffers(dev)
    ms = _time_ms(lambda: engine.eval_owner_argmin(batch, own, k0, bufs, out))
    win = bufs.read()
    res = {"config": desc, "candidates": N, "ms": ms, "value": N / (ms / 1e3), "unit": UNIT,
           "winner": {"makespan": win["makespan"], "rank": win["rank"], "n_feasible": win["n_feasible"],
                      "checksum": win["checksum"]}}
    if which == "c2":   # Mode A == Mode B on the same ranks (full-size property)
        res["matches_mode_b"] = engine.enum(batch, "splits", k0, k0 + N).read() == win
    peak, src = _hbm_peak()
    algo = N * (n * 1 + 9)
    achieved = algo / (ms / 1e3) / 1e9
    tr = ncu_traffic("eval_owner_stream_kernel", f"r1_prof_modea_{which}*_raw.csv") if which == "c1" else None
    res["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                       "traffic": (tr["bytes"] / (1 << 25) * N) if tr else None,
                       "traffic_note": (f"{tr['capture']}: DRAM read+write of a 2^25-candidate launch (same "
                                        "population), scaled per candidate to this launch") if tr else None,
                       "bytes_per_candidate": n + 9, "peak_source": src}
    inst = oracle.Instance(stages, fleet)
    sample = own[:20000].cpu().numpy().astype("int64")
    t0 = _t.perf_counter()
    for row in sample:
        inst.eval_owner(row)
    res["cpu_baseline_1core"] = 20000 / (_t.perf_counter() - t0)
    del own, out
    torch.cuda.empty_cache()
    return res


def dp_measure(dev):
    """Partition DPs solved/s: config C1's 32 x 32 link grid, one _subset_dp per fleet."""
    import time as _t
    from oracle import oracle
    from paper_2309_01172_b200 import configs as CF
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200.tensorize import build_host
    stages = CF.model_stages("gpt2-small")
    bws, alphas = CF.c1_link_grid()
    fleets = [CF.load(CF.c1_fleet_doc(bw, al)) for bw in bws for al in alphas]
    hosts = [build_host(stages, f, True) for f in fleets]
    batch = engine.device_batch(hosts, device=dev)
    ms = _time_ms(lambda: engine.subset_dp(batch, 26, 4))
    own, mk, found, _ = engine.subset_dp(batch, 26, 4)
    own = own.cpu().numpy()
    ok = True
    t0 = _t.perf_counter()
    for i in range(0, len(fleets), 64):
        o, _ = oracle.Instance(stages, fleets[i]).subset_dp()
        ok &= o is not None and own[i, :26].tolist() == o.tolist()
    cpu = 16 / (_t.perf_counter() - t0)
    return {"config": "C1 gpt2-small (26 stages) x 4 workers, 1024 link-grid fleets (bw logspace(-1,2,32) x "
                      "alpha linspace(0,10ms,32)), one _subset_dp each", "dps": len(fleets), "ms": ms,
            "value": len(fleets) / (ms / 1e3), "unit": "DPs/s", "oracle_spot_check": bool(ok),
            "cpu_baseline_1core": cpu}


def c4_measure(dev, n_scen=1 << 18):
    """schedule() solves/s over config C4 scenarios (proportional split + hill climb + epilogue)."""
    import time as _t
    from oracle import oracle
    from paper_2309_01172_b200 import batch as B
    from paper_2309_01172_b200 import engine
    sb = B.c4_batch(n_scen, seed=0, device=dev)

    def run():
        owner, _, _ = engine.prop_hill(sb, sb.n_max)
        return engine.epilogue(sb, sb.n_max, owner, 512, 4)
    ms = _time_ms(run, steps=3, warmup=3)
    owner, _, moves = engine.prop_hill(sb, sb.n_max)
    epi = engine.epilogue(sb, sb.n_max, owner, 512, 4).cpu().numpy()
    owner = owner.cpu().numpy()
    ok = True
    t0 = _t.perf_counter()
    for s in range(0, n_scen, n_scen // 16):
        st, fl = B.scenario_instance(sb, s)
        _, o = oracle.Instance(st, fl).schedule()
        ok &= owner[s, :len(st)].tolist() == o.tolist()
    cpu = 16 / (_t.perf_counter() - t0)
    feas = float((epi[:, 5] == 0).mean())
    return {"config": f"C4: {n_scen} scenarios, L~U{{32..80}}, h in {{2048,4096,5120,8192}}, p~U{{8..64}}, "
                      "GPU_TABLE mix, lambda~U[.3,1], alpha~U[0,10ms], bw~LogU[.1,10] Gbit/s",
            "schedules": n_scen, "ms": ms, "value": n_scen / (ms / 1e3), "unit": "schedules/s",
            "feasible_frac": feas, "mean_hill_moves": float(moves.float().mean()),
            "oracle_spot_check": bool(ok), "cpu_baseline_1core": cpu}


def random_measure(dev, which):
    """Random contiguous placements scored in-kernel (counter RNG):
    C5 = OPT-175B x 1024 workers with 10% churn (922 online), 10^9 candidates;
    C3 = Llama-2-70B x 256 workers with 32,640 randomised pairwise links."""
    import time as _t
    import numpy as np
    import torch
    from oracle import oracle
    from paper_2309_01172_b200 import configs as CF
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200 import rng as R
    from paper_2309_01172_b200.tensorize import build_host
    if which == "c5":
        stages = CF.model_stages("opt-175b")
        fleet = CF.load(CF.c5_fleet_doc(0))
        _, online_ids = CF.c5_churn(1024, 0.1, 0)
        N = 10 ** 9
        desc = "C5 OPT-175B (194 stages) x 1024 workers, 922 online after 10% churn, default 5 ms / 10 Gbit/s"
    else:
        stages = CF.model_stages("llama2-70b")
        fleet = CF.load(CF.c3_fleet_doc(0))
        online_ids = list(fleet.worker_ids())
        N = 1 << 28
        desc = "C3 Llama-2-70B (162 stages) x 256 workers, 32,640 randomised pairwise links (alpha U[0,20ms], bw LogU[.1,100])"
    host = build_host(stages, fleet, True)
    batch = engine.device_batch([host], device=dev)
    online = np.array([host.index_of[i] for i in online_ids], np.int32)
    on_d = torch.from_numpy(online).to(dev)
    bufs = engine.WinnerBuffers(dev)
    seed = 20260
    ms = _time_ms(lambda: engine.enum(batch, "random", 0, N, bufs, online=on_d, seed=seed), steps=3)
    win = bufs.read()
    inst = oracle.Instance(stages, fleet)
    t0 = _t.perf_counter()
    ref = inst.enum_random(online, seed, 0, 20000)
    cpu = 20000 / (_t.perf_counter() - t0)
    got = engine.enum(batch, "random", 0, 20000, online=on_d, seed=seed).read()
    return {"config": desc, "candidates": N, "ms": ms, "value": N / (ms / 1e3), "unit": UNIT,
            "candidate_distribution": "r ~ U{1..min(n, online)}, uniform (r-1)-subset of the cut positions "
                                      "(selection sampling), r distinct online peers (keyed Feistel permutation); "
                                      "paper_2309_01172_b200/rng.py",
            "feasible_frac": win["n_feasible"] / N,
            "winner": {"makespan": win["makespan"], "rank": win["rank"], "n_feasible": win["n_feasible"],
                       "checksum": win["checksum"]},
            "oracle_prefix_check": got == ref, "cpu_baseline_1core": cpu}


def dp_c4b_measure(dev, n_scen=4096):
    """Config C4b: layer-cell encoder chains (n = L + 2 <= 38) over p <= 8
    workers, the sizes where schedule() takes the exact subset DP."""
    import time as _t
    import numpy as np
    from oracle import oracle
    from paper_2309_01172_b200 import configs as CF
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200.tensorize import build_host
    rng = np.random.default_rng(7)
    models = {L: CF.encoder_stages(4096, L, 32000, 4, 1024, cells="layer") for L in range(24, 37)}
    insts, hosts = [], []
    for s_ in range(n_scen):
        L = int(rng.integers(24, 37))
        p = int(rng.integers(5, 9))
        peers = CF.hetero_peers(p, int(rng.integers(1 << 30)), lam=(0.3, 1.0))
        doc = CF.fleet_doc(peers, float(rng.uniform(0, 1e-2)), float(10 ** rng.uniform(-1, 1)))
        fl = CF.load(doc)
        st = models[L]
        assert len(st) ** 2 * p * 2 ** p <= 3_000_000
        insts.append((st, fl))
        hosts.append(build_host(st, fl, True))
    batch = engine.device_batch(hosts, device=dev)
    n_max = max(h.n for h in hosts)
    ms = _time_ms(lambda: engine.subset_dp(batch, n_max, 8), steps=3)
    own, mk, found, _ = engine.subset_dp(batch, n_max, 8)
    own = own.cpu().numpy()
    ok = True
    t0 = _t.perf_counter()
    for i in range(0, n_scen, n_scen // 8):
        o, _ = oracle.Instance(*insts[i]).subset_dp()
        ok &= (o is None and not int(found[i])) or (o is not None and own[i, :len(insts[i][0])].tolist() == o.tolist())
    cpu = 8 / (_t.perf_counter() - t0)
    return {"config": f"C4b: {n_scen} scenarios, layer-cell chains n = L+2 in [26, 38], p in [5, 8] "
                      "(n^2 p 2^p <= 3e6: the exact subset-DP path)", "dps": n_scen, "ms": ms,
            "value": n_scen / (ms / 1e3), "unit": "DPs/s", "oracle_spot_check": bool(ok), "cpu_baseline_1core": cpu}


def api_latency_measure(dev):
    """End-to-end latency of one public schedule() call (host objects in, a
    ScheduleReport out: tensorise, one H2D, DP kernel, report kernel, one D2H)
    on C1 and on C3, beside the reference's own schedule() (dagmesh from
    baseline/_ref, pure Python) on the same inputs in the same process."""
    import time as _t
    import torch
    from paper_2309_01172_b200 import configs as CF
    from paper_2309_01172_b200 import scheduling as S
    from paper_2309_01172_b200.refapi import dagmesh
    RS = dagmesh.scheduling
    out = {}
    for name, stages, fleet, reps in (
            ("c1", CF.model_stages("gpt2-small"), CF.load(CF.c1_fleet_doc(10.0, 1e-3)), 50),
            ("c3", CF.model_stages("llama2-70b"), CF.load(CF.c3_fleet_doc(0)), 10)):
        for _ in range(3):
            S.schedule(stages, fleet)
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            t0 = _t.perf_counter()
            rep = S.schedule(stages, fleet)
            times.append((_t.perf_counter() - t0) * 1e3)
        ref_times = []
        for _ in range(3 if name == "c1" else 1):
            t0 = _t.perf_counter()
            ref = RS.schedule(stages, fleet)
            ref_times.append((_t.perf_counter() - t0) * 1e3)
        out[name] = {"ms_per_call": statistics.median(times), "ms_min": min(times), "ms_max": max(times),
                     "calls": len(times), "reference_ms_per_call": statistics.median(ref_times),
                     "same_report": rep.runs == ref.runs and rep.makespan == ref.makespan and rep.trace == ref.trace,
                     "makespan": rep.makespan, "trace": list(rep.trace)}
    out["config"] = ("schedule() through the public API: C1 gpt2-small x 4 mixed GPUs (10 Gbit/s, 1 ms; exact subset "
                     "DP) and C3 llama2-70b x 256 workers with 32,640 pairwise links (proportional + hill climb); "
                     "reference = dagmesh.scheduling.schedule on the same objects")
    return out


def secondary_measurements(dev):
    """FP64 peak microbenchmark (roofline denominator), CPU baseline, and the
    secondary paths of the metric: Mode A streams (HBM roofline), DPs/s, schedules/s."""
    out = {}
    from paper_2309_01172_b200 import engine
    out["fp64_peak_ops_per_s"] = engine.fp64_peak()
    out["cross_peak_pairs_per_s"] = engine.cross_peak()
    out["cpu_baseline"] = cpu_baseline(threads=1, seconds=10.0)
    sec = {}
    for name, fn in (("mode_a_c1", lambda: mode_a_measure(dev, "c1")), ("mode_a_c2", lambda: mode_a_measure(dev, "c2")),
                     ("dp_c1_grid", lambda: dp_measure(dev)), ("schedule_c4", lambda: c4_measure(dev)),
                     ("random_c5", lambda: random_measure(dev, "c5")), ("random_c3", lambda: random_measure(dev, "c3")),
                     ("dp_c4b", lambda: dp_c4b_measure(dev)), ("schedule_api_latency_c1", lambda: api_latency_measure(dev))):
        try:
            sec[name] = fn()
        except Exception as exc:
            sec[name] = {"error": f"{type(exc).__name__}: {exc}"}
    out["secondary"] = sec
    return out


# ------------------------------------------------------------- CPU oracle
def cpu_baseline(threads=1, seconds=10.0):
    """Time the oracle (C restatement of brute_force_schedule's inner body,
    scheduling.py:264-272, in the identity-split order) on a bounded sample of
    the same population."""
    from oracle import oracle
    from paper_2309_01172_b200 import engine
    oracle.build()
    stages, fleet = c2_instance()
    inst = oracle.Instance(stages, fleet)
    total = engine.splits_total(inst.n, inst.p)
    # calibrate on a small sample from the middle of the population
    mid = total // 2
    t0 = time.perf_counter()
    inst.enum("splits", mid, mid + 20000)
    rate1 = 20000 / (time.perf_counter() - t0)
    per_thread = max(int(rate1 * seconds), 1000)
    from concurrent.futures import ThreadPoolExecutor
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda i: inst.enum("splits", mid + i * per_thread, mid + (i + 1) * per_thread), range(threads)))
    el = time.perf_counter() - t0
    return {"value": threads * per_thread / el, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{threads * per_thread} consecutive ranks from the middle of the C2 split population "
                      f"({el:.1f}s), oracle/dm_oracle.c or_enum mode 1"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    base = cpu_baseline(threads=threads, seconds=10.0)   # one ~10 s sample on every host core
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(8589934558, c2_scenarios()[2]),
            "cpu_baseline": {"value": base["value"], "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": base["sample"]},
            "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def main():
    args = _args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        line = run_b200(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
