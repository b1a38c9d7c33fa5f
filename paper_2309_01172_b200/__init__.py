"""B200-native placement-cost evaluation and partition search for the
FusionAI / dagmesh planner (arXiv 2309.01172).

Public surface (mirrors the reference's ``dagmesh.scheduling`` and
``dagmesh.pipeline`` hot path):

    schedule, evaluate_runs, brute_force_schedule, verify_assignment,
    reschedule_on_failure                      -- scheduling.py mirror
    sweep, fp_latency, pipeline_time, ...      -- pipeline.py mirror
    search.*                                   -- batched engine APIs
    install()                                  -- drop-in for the reference package

All compute runs on the GPU through libdagmesh_b200.so (C ABI in
include/dagmesh_b200.h); there is no CPU fallback.
"""

from __future__ import annotations

from . import _lib, engine, opcost, pipeline, refapi, scheduling, tensorize
from ._lib import EngineError, EngineUnavailable
from .refapi import (GPU_TABLE, DagmeshError, Fleet, FleetError, Link, Peer, PeerLoad, Role,
                    ScheduleReport, SchedulingError, Stage, ZERO_LINK, bandwidth_to_beta, comm_time,
                    effective_speed, format_stage_run, load_fleet, parse_fleet, peer_sort_key)
from .pipeline import (StageProfile, SweepResult, SweepRow, asymptotic_throughput, bottleneck, fp_latency,
                       pipeline_time, profiles_from_report, sweep, sweep_stages, throughput)
from .scheduling import (brute_force_schedule, evaluate_runs, reschedule_on_failure, schedule,
                         verify_assignment)

__version__ = "0.1.0"

_INSTALLED: dict = {}


def install(dagmesh_module=None):
    """Make the reference package use this engine (drop-in).

    Rebinds ``dagmesh.scheduling.{schedule, evaluate_runs,
    brute_force_schedule, verify_assignment, reschedule_on_failure}``, the
    early-bound re-exports in ``dagmesh/__init__.py:12-25``,
    ``dagmesh.pipeline.sweep`` and ``dagmesh.hardware.{op_time, subgraph_time}``; reports are then built from the reference's
    own ``ScheduleReport``/``PeerLoad`` classes and errors are the
    reference's ``SchedulingError``/``FleetError``.  Every reference caller
    resolves these through the module attribute at call time (pipeline.py:237,
    cli.py:74,149, sim/loop.py:188,642), so the whole package runs on the GPU
    path.  Returns a callable that restores the originals."""
    if dagmesh_module is None:
        import dagmesh as dagmesh_module
    engine.warmup()
    ref_sched = dagmesh_module.scheduling
    ref_pipe = dagmesh_module.pipeline
    ref_err = dagmesh_module.errors
    saved = {}
    scheduling.T.ScheduleReport = ref_sched.ScheduleReport
    scheduling.T.PeerLoad = ref_sched.PeerLoad
    scheduling.T.SchedulingError = ref_err.SchedulingError
    scheduling.T.FleetError = ref_err.FleetError
    names = ("schedule", "evaluate_runs", "brute_force_schedule", "verify_assignment", "reschedule_on_failure")
    for name in names:
        saved[(ref_sched, name)] = getattr(ref_sched, name)
        setattr(ref_sched, name, getattr(scheduling, name))
        if hasattr(dagmesh_module, name):
            saved[(dagmesh_module, name)] = getattr(dagmesh_module, name)
            setattr(dagmesh_module, name, getattr(scheduling, name))

    def _sweep(model_, fleets, bandwidth_gbps, alpha_s, n_batches):
        from .configs import stages_for
        stages = stages_for(model_.graph, model_.cells)
        res = sweep_stages(stages, model_.name, model_.samples_per_batch, fleets, bandwidth_gbps, alpha_s,
                           n_batches)
        out = ref_pipe.SweepResult()
        out.rows = [ref_pipe.SweepRow(*[getattr(r, f) for f in SweepRow.__dataclass_fields__]) for r in res.rows]
        out.infeasible = list(res.infeasible)
        return out

    saved[(ref_pipe, "sweep")] = ref_pipe.sweep
    ref_pipe.sweep = _sweep
    ref_hw = dagmesh_module.hardware
    for name in ("op_time", "subgraph_time"):
        saved[(ref_hw, name)] = getattr(ref_hw, name)
        setattr(ref_hw, name, getattr(opcost, name))
        if hasattr(dagmesh_module, name):
            saved[(dagmesh_module, name)] = getattr(dagmesh_module, name)
            setattr(dagmesh_module, name, getattr(opcost, name))
    if hasattr(dagmesh_module, "sweep"):
        saved[(dagmesh_module, "sweep")] = dagmesh_module.sweep
        dagmesh_module.sweep = _sweep
    _INSTALLED.update(saved)

    def uninstall():
        for (mod, name), fn in saved.items():
            setattr(mod, name, fn)
        scheduling.T.ScheduleReport = refapi.ScheduleReport
        scheduling.T.PeerLoad = refapi.PeerLoad
        scheduling.T.SchedulingError = refapi.SchedulingError
        scheduling.T.FleetError = refapi.FleetError

    return uninstall
