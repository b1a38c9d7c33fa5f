"""Eq. 3 / Eq. 4 pipeline model and the batched link-grid sweep.

Mirrors pkg/src/dagmesh/pipeline.py:29-68 (profiles, fp_latency, bottleneck,
pipeline_time, throughput, asymptotic_throughput) and :197-248 (SweepRow,
SweepResult, sweep).  ``sweep`` is the hot-path version: every
(fleet x bandwidth x alpha) grid point becomes one scenario of a device batch,
solved by the batched kernels (pinned runs / subset DP / proportional + hill
climb) and scored by the fused epilogue kernel (dm_pipeline_epilogue), which
applies Eq. 3 with CPython's compensated sum and Eq. 4 in the reference's
rounding order.  The scalar helpers below operate on a handful of already
computed profile values (report formatting), exactly as the reference does.
"""

from __future__ import annotations

import csv
import itertools
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import engine, scheduling
from .refapi import DagmeshError, Link, SchedulingError, bandwidth_to_beta
from .tensorize import build_host


@dataclass(frozen=True)
class StageProfile:
    peer: str
    compute_s: float
    read_s: float


def profiles_from_report(report) -> list:
    return [StageProfile(row.peer, row.compute_s, row.read_s) for row in report.per_peer if row.stage_indices]


def fp_latency(profiles: Sequence[StageProfile]) -> float:
    """Eq. 3: one batch through every stage (pipeline.py:41-43)."""
    return sum(p.compute_s + p.read_s for p in profiles)


def bottleneck(profiles: Sequence[StageProfile]) -> float:
    """Slowest single compute or read (pipeline.py:46-50)."""
    if not profiles:
        raise SchedulingError("empty profile list")
    return max(max(p.compute_s, p.read_s) for p in profiles)


def pipeline_time(profiles: Sequence[StageProfile], n_batches: int) -> float:
    """Eq. 4 (pipeline.py:53-56)."""
    if n_batches < 1:
        raise SchedulingError(f"need at least one batch, got {n_batches}")
    return fp_latency(profiles) + (n_batches - 1) * bottleneck(profiles)


def throughput(profiles, n_batches: int, samples_per_batch: int) -> float:
    return n_batches * samples_per_batch / pipeline_time(profiles, n_batches)


def asymptotic_throughput(profiles, samples_per_batch: int) -> float:
    return samples_per_batch / bottleneck(profiles)


@dataclass(frozen=True)
class SweepRow:
    model: str
    fleet: str
    bandwidth_gbps: float
    alpha_ms: float
    n_batches: int
    latency_s: float
    pipe_time_s: float
    throughput: float


@dataclass
class SweepResult:
    rows: list = field(default_factory=list)
    infeasible: list = field(default_factory=list)

    def to_csv(self, path):
        with open(path, "w", newline="", encoding="utf-8") as fh:
            w = csv.writer(fh)
            w.writerow(["model", "fleet", "bandwidth_gbps", "alpha_ms", "n_b", "latency_s", "pipe_time_s",
                        "throughput"])
            for r in self.rows:
                w.writerow([r.model, r.fleet, f"{r.bandwidth_gbps:g}", f"{r.alpha_ms:g}", r.n_batches,
                            f"{r.latency_s:.9g}", f"{r.pipe_time_s:.9g}", f"{r.throughput:.9g}"])


def _contiguous_pins(pinned, n):
    """Owner vector (worker index per stage) when the pinned runs are
    contiguous, in stage order and cover every stage; else None."""
    owner = [-1] * n
    nxt = 0
    for k, run in enumerate(pinned):
        run = tuple(run)
        if not run:
            return None
        if run != tuple(range(nxt, nxt + len(run))):
            return None
        for i in run:
            owner[i] = k
        nxt += len(run)
    return owner if nxt == n else None


def sweep_stages(stages, name: str, samples_per_batch: int, fleets, bandwidth_gbps, alpha_s,
                 n_batches: int) -> SweepResult:
    """Batched sweep over pre-built stages (pipeline.py:228-248 semantics)."""
    stages = list(stages)
    n = len(stages)
    # the reference walks the grid in order and raises at the first point that
    # fails (bandwidth_to_beta / Link, schedule()'s input checks, then
    # pipeline_time's n_batches check on the first feasible point,
    # pipeline.py:235-245): errors are recorded per point and raised in that
    # order while the rows are emitted
    points, pending = [], None
    for fleet, bw, alpha in itertools.product(fleets, bandwidth_gbps, alpha_s):
        try:
            tuned = fleet.with_default_link(Link(alpha=alpha, beta=bandwidth_to_beta(bw)))
            workers = tuned.worker_ids()
            scheduling._check_inputs(stages, workers)
            if tuned.pinned_runs is not None and len(tuned.pinned_runs) > len(workers):
                raise scheduling.T.SchedulingError(f"{len(tuned.pinned_runs)} pinned runs but only "
                                                   f"{len(workers)} workers")
        except DagmeshError as exc:
            pending = exc
            break
        points.append((fleet, bw, alpha, tuned))
    result = SweepResult()
    if not points:
        if pending is not None:
            raise pending
        return result
    hosts = []
    kinds = []  # 'pin' | 'dp' | 'hill' | 'eval'
    owner0 = np.full((len(points), n), -1, dtype=np.int16)
    for s, (_, _, _, tuned) in enumerate(points):
        workers = tuned.worker_ids()
        p = len(workers)
        hosts.append(build_host(stages, tuned, True))
        if tuned.pinned_runs is not None:
            own = _contiguous_pins(tuned.pinned_runs, n)
            if own is None:
                kinds.append("eval")
            else:
                owner0[s] = own
                kinds.append("pin")
        elif n * n * p * (2 ** p) <= 3_000_000:
            kinds.append("dp")
        else:
            kinds.append("hill")
    import torch
    batch = engine.device_batch(hosts)
    dev = batch.dev_buf.device
    owner = torch.from_numpy(owner0).to(dev)
    dp_ok = np.ones(len(points), dtype=bool)
    dp_idx = [s for s, k in enumerate(kinds) if k == "dp"]
    hill_idx = [s for s, k in enumerate(kinds) if k == "hill"]
    if dp_idx:
        sub = engine.device_batch([hosts[s] for s in dp_idx])
        p_max = max(hosts[s].p for s in dp_idx)
        own_dp, _, found, _ = engine.subset_dp(sub, n, p_max)
        owner[dp_idx] = own_dp
        dp_ok[dp_idx] = found.cpu().numpy().astype(bool)
    if hill_idx:
        sub = engine.device_batch([hosts[s] for s in hill_idx])
        own_h, _, _ = engine.prop_hill(sub, n)
        owner[hill_idx] = own_h
    out = engine.epilogue(batch, n, owner, max(n_batches, 1), samples_per_batch).cpu().numpy()
    for s, (fleet, bw, alpha, tuned) in enumerate(points):
        kind = kinds[s]
        if kind == "eval" or (kind == "dp" and not dp_ok[s]) or int(out[s, 5]) != 0:
            report = scheduling.schedule(stages, tuned)   # reason string / irregular pins
            if not report.feasible:
                result.infeasible.append(f"{name} on {fleet.name} at {bw:g} Gbit/s, "
                                         f"alpha {alpha * 1e3:g} ms: {report.reason}")
                continue
            prof = profiles_from_report(report)
            result.rows.append(SweepRow(name, fleet.name, bw, alpha * 1e3, n_batches, fp_latency(prof),
                                        pipeline_time(prof, n_batches),
                                        throughput(prof, n_batches, samples_per_batch)))
            continue
        if n_batches < 1:                               # pipeline_time on the first feasible point (:53-55)
            raise SchedulingError(f"need at least one batch, got {n_batches}")
        result.rows.append(SweepRow(name, fleet.name, bw, alpha * 1e3, n_batches, float(out[s, 1]),
                                    float(out[s, 3]), float(out[s, 4])))
    if pending is not None:
        raise pending
    return result


def sweep(model, fleets, bandwidth_gbps, alpha_s, n_batches: int) -> SweepResult:
    """Schedule the model on each fleet across a link-quality grid
    (pipeline.py:228-248), batched on the GPU.  ``model`` is any object with
    ``name``, ``graph``, ``cells`` and ``samples_per_batch`` (stages from
    ``configs.stages_for``: encoder chains in closed form, other graphs
    through the reference's ``build_stages``), or an object exposing
    ``stages`` directly."""
    stages = getattr(model, "stages", None)
    if stages is None:
        from .configs import stages_for
        stages = stages_for(model.graph, model.cells)
    return sweep_stages(stages, model.name, model.samples_per_batch, fleets, bandwidth_gbps, alpha_s, n_batches)
