"""Edge cases of the drop-in API compared with the reference's own functions
(dagmesh through paper_2309_01172_b200.refapi — the unmodified package from
baseline/_ref on the GPU box, or /root/reference here)."""

import math

import pytest

from gen import random_stages, uniform_fleet

pytestmark = pytest.mark.gpu


def _ref():
    from paper_2309_01172_b200.refapi import dagmesh
    return dagmesh


def test_int_peer_keys_like_reference(engine_ready):
    """Runs keyed by int peer ids: verify says 'unknown peer', costing
    str-converts (fleet.peer, hardware.py:122-126) — as the reference."""
    import numpy as np
    from paper_2309_01172_b200 import scheduling as S
    RS = _ref().scheduling
    rng = np.random.default_rng(3)
    stages = random_stages(rng, 6)
    fleet = uniform_fleet([1e9, 2e9, 3e9])
    runs = ((1, (0, 1, 2)), ("2", (3, 4, 5)))
    got, want = S.evaluate_runs(stages, fleet, runs), RS.evaluate_runs(stages, fleet, runs)
    assert got.reason == want.reason and got.feasible == want.feasible
    assert got.makespan == want.makespan and got.runs == want.runs
    from dataclasses import astuple
    assert [astuple(r) for r in got.per_peer] == [astuple(r) for r in want.per_peer]
    assert S.verify_assignment(stages, fleet, runs) == RS.verify_assignment(stages, fleet, runs)


def test_sweep_errors_where_reference_raises(engine_ready):
    """n_batches < 1 raises only on a feasible grid point (pipeline_time,
    pipeline.py:53-55); an all-infeasible grid returns its rows quietly."""
    from paper_2309_01172_b200 import pipeline as P
    dm = _ref()
    model = dm.pipeline.build_bert_large(2, 64)
    tiny = dm.hardware.parse_fleet({"name": "tiny", "peers": [{"id": "1", "tflops_tensor": 1.0, "gpu_gb": 0.001}]})
    for fn in (P.sweep, dm.pipeline.sweep):
        res = fn(model, [tiny], [1.0], [0.0], 0)
        assert not res.rows and len(res.infeasible) == 1
    ok = dm.hardware.parse_fleet({"name": "ok", "peers": [{"id": "1", "gpu": "h100"}, {"id": "2", "gpu": "h100"}]})
    for fn in (P.sweep, dm.pipeline.sweep):
        with pytest.raises(dm.errors.SchedulingError):
            fn(model, [tiny, ok], [1.0], [0.0], 0)
        with pytest.raises(dm.errors.FleetError):
            fn(model, [ok], [0.0], [0.0], 4)
    a, b = P.sweep(model, [tiny, ok], [1.0, 10.0], [0.0, 1e-3], 8), dm.pipeline.sweep(model, [tiny, ok], [1.0, 10.0],
                                                                                       [0.0, 1e-3], 8)
    assert a.infeasible == b.infeasible
    from dataclasses import astuple
    assert [astuple(r) for r in a.rows] == [astuple(r) for r in b.rows]


def test_schedule_report_kernel_infeasible_and_hill(engine_ready):
    """The fused schedule() path: DP with no feasible state (the reference
    scores (workers[0], all stages) and marks it infeasible) and the
    proportional + hill-climb path, against the reference's schedule()."""
    import numpy as np
    from paper_2309_01172_b200 import scheduling as S
    RS = _ref().scheduling
    rng = np.random.default_rng(11)
    stages = random_stages(rng, 8)
    starved = uniform_fleet([1e9, 2e9], gpu_gb=1e-6)
    for f in (starved, uniform_fleet([1e9] * 14, gpu_gb=64.0)):
        got, want = S.schedule(stages, f), RS.schedule(stages, f)
        assert got.runs == want.runs and got.reason == want.reason and got.trace == want.trace
        assert (got.makespan == want.makespan) or (math.isinf(got.makespan) and math.isinf(want.makespan))
