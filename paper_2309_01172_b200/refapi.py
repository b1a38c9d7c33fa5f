"""The reference package's own data model.

The engine is a drop-in for the dagmesh planner's hot path, so it consumes and
returns dagmesh's types — ``Stage`` / ``ScheduleReport`` / ``PeerLoad``
(pkg/src/dagmesh/scheduling.py:29-105), ``Peer`` / ``Link`` / ``Fleet`` /
``parse_fleet`` / ``GPU_TABLE`` (hardware.py:30-144, 265-359), the error
classes (errors.py) and ``peer_sort_key`` (ir.py:343-345) — rather than
mirrors of them.  The package is imported from the interpreter's path, else
from the unmodified install in ``baseline/_ref`` next to this repository."""

from __future__ import annotations

import pathlib
import sys

try:
    import dagmesh  # noqa: F401
except ImportError:                                    # pragma: no cover - depends on the host
    _ref = pathlib.Path(__file__).resolve().parent.parent / "baseline" / "_ref"
    if not (_ref / "dagmesh").is_dir():
        raise ImportError("paper_2309_01172_b200 plugs into the dagmesh package: install it "
                          "(pip install /path/to/reference) or into baseline/_ref") from None
    sys.path.insert(0, str(_ref))
    import dagmesh  # noqa: F401

from dagmesh.errors import DagmeshError, FleetError, SchedulingError  # noqa: E402,F401
from dagmesh.hardware import (COMPUTE_COLUMNS, GPU_TABLE, ZERO_LINK, Fleet, GpuSpec, Link, Peer,  # noqa: E402,F401
                              Role, bandwidth_to_beta, comm_time, effective_speed, load_fleet, parse_fleet)
from dagmesh.ir import peer_sort_key  # noqa: E402,F401
from dagmesh.scheduling import PeerLoad, ScheduleReport, Stage, format_stage_run  # noqa: E402,F401
