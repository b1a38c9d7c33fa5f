"""pytest plugin: run the REFERENCE package's own test suite with the B200
engine installed as its scheduling / pipeline backend.

    cd baseline/_ref_pkg
    PYTHONPATH=../_ref:../.. python -m pytest -p tools.ref_suite_plugin tests --ignore=tests/test_cli.py

(baseline/_ref holds the unmodified reference package installed with pip,
baseline/_ref_pkg a copy of its tests and data files; both are git-ignored
and travel to the GPU box.)  After install(), dagmesh.scheduling.schedule,
evaluate_runs, brute_force_schedule, verify_assignment,
reschedule_on_failure, dagmesh.pipeline.sweep and the dagmesh re-exports are
the engine's GPU implementations; the plugin records that they were called.
"""

import paper_2309_01172_b200 as engine
from paper_2309_01172_b200 import scheduling as eng_sched

CALLS = {"schedule": 0, "evaluate_runs": 0, "brute_force_schedule": 0}


def _counting(name, fn):
    def wrapper(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)
    wrapper.__wrapped__ = fn
    return wrapper


def pytest_configure(config):
    import dagmesh
    engine.install(dagmesh)
    for name in CALLS:
        f = _counting(name, getattr(dagmesh.scheduling, name))
        setattr(dagmesh.scheduling, name, f)
        if hasattr(dagmesh, name):
            setattr(dagmesh, name, f)
    # the engine's own internal calls (e.g. reschedule -> schedule) stay on the engine
    assert getattr(dagmesh.scheduling.schedule, "__wrapped__") is eng_sched.schedule


def pytest_terminal_summary(terminalreporter):
    terminalreporter.section("B200 engine backend")
    terminalreporter.write_line(f"engine calls from the reference suite: {CALLS}")
