"""Host-side data model mirroring the reference's scheduling types.

These are the types the drop-in path consumes and produces, with the
reference's names, fields, validation and error behaviour:

* ``Peer`` / ``Link`` / ``Fleet`` / ``comm_time`` / ``effective_speed`` /
  ``bandwidth_to_beta`` / ``parse_fleet`` — pkg/src/dagmesh/hardware.py:58-159,
  265-359 (fleet files under pkg/fleets load unchanged);
* ``Stage`` / ``PeerLoad`` / ``ScheduleReport`` / ``format_stage_run`` —
  pkg/src/dagmesh/scheduling.py:29-104;
* the error hierarchy — pkg/src/dagmesh/errors.py.

The engine itself only reads attributes (duck typing), so objects built by the
reference package work as inputs too; ``paper_2309_01172_b200.install()``
additionally makes the engine emit the reference's own report classes.
"""

from __future__ import annotations

import csv
import json
import math
from dataclasses import dataclass, field, replace
from enum import Enum
from typing import Sequence


# ---------------------------------------------------------------- errors
class DagmeshError(Exception):
    """Base error (errors.py:4)."""


class FleetError(DagmeshError):
    """Malformed fleet or invalid peer/link parameters (errors.py:16)."""


class SchedulingError(DagmeshError):
    """Unsatisfiable scheduling request (errors.py:20)."""


# ------------------------------------------------------------- peer ids
def peer_sort_key(peer_id):
    """Numeric ids by value first, then other ids lexicographically
    (ir.py:343-345)."""
    s = str(peer_id)
    return (0, int(s), "") if s.isdigit() else (1, 0, s)


# --------------------------------------------------------------- hardware
@dataclass(frozen=True)
class GpuSpec:
    tflops_fp32: float
    tflops_tensor: float
    memory_gb: float


# paper Table 1 peaks (hardware.py:36-42)
GPU_TABLE: dict[str, GpuSpec] = {
    "rtx4090": GpuSpec(82.58, 82.58, 24),
    "rtx4080": GpuSpec(48.74, 97.5, 16),
    "rtx3080": GpuSpec(29.77, 59.5, 10),
    "h100": GpuSpec(51.22, 756.0, 80),
    "a100": GpuSpec(19.49, 155.92, 80),
}
COMPUTE_COLUMNS = ("fp32", "tensor")


class Role(Enum):
    SUPERNODE = "supernode"
    ANTNODE = "antnode"


@dataclass(frozen=True)
class Peer:
    """A worker: peak rate, efficiency lambda, capacities (hardware.py:58-79)."""

    id: str
    role: Role = Role.ANTNODE
    peak_flops: float = 1e12
    lam: float = 1.0
    gpu_bytes: float = 8 * 2**30
    cpu_bytes: float = 16 * 2**30
    disk_bytes: float = 64 * 2**30
    write_bandwidth: float = math.inf

    def __post_init__(self):
        if self.peak_flops <= 0:
            raise FleetError(f"peer {self.id}: peak_flops must be positive")
        if not 0.0 < self.lam <= 1.0:
            raise FleetError(f"peer {self.id}: lambda must lie in (0, 1], got {self.lam}")
        if min(self.gpu_bytes, self.cpu_bytes, self.disk_bytes) < 0:
            raise FleetError(f"peer {self.id}: capacities must be nonnegative")
        if self.write_bandwidth <= 0:
            raise FleetError(f"peer {self.id}: write_bandwidth must be positive")


@dataclass(frozen=True)
class Link:
    """alpha seconds of latency plus beta seconds per byte (hardware.py:82-91)."""

    alpha: float = 0.0
    beta: float = 0.0

    def __post_init__(self):
        if self.alpha < 0 or self.beta < 0:
            raise FleetError("link alpha and beta must be nonnegative")


ZERO_LINK = Link(0.0, 0.0)


def bandwidth_to_beta(gbps: float) -> float:
    """Gbit/s to seconds per byte (hardware.py:97-100)."""
    if gbps <= 0:
        raise FleetError("bandwidth must be positive")
    return 8.0 / (gbps * 1e9)


@dataclass
class Fleet:
    """Peers, default link, pairwise overrides, backups (hardware.py:103-144).

    Mutable on purpose (the reference's tests assign ``pinned_runs`` after
    construction), so the engine re-tensorises it on every call."""

    peers: dict
    default_link: Link = ZERO_LINK
    links: dict = field(default_factory=dict)
    backup_pool: tuple = ()
    msg_ratio: float = 1.0
    pinned_runs: tuple | None = None
    name: str = "fleet"

    def __post_init__(self):
        for pid in self.backup_pool:
            if pid not in self.peers:
                raise FleetError(f"backup pool references unknown peer {pid!r}")
        if self.msg_ratio <= 0:
            raise FleetError("msg_ratio must be positive")

    def peer(self, pid) -> Peer:
        try:
            return self.peers[str(pid)]
        except KeyError:
            raise FleetError(f"unknown peer {pid!r}") from None

    def peer_ids(self) -> tuple:
        return tuple(sorted(self.peers, key=peer_sort_key))

    def worker_ids(self) -> tuple:
        held = set(self.backup_pool)
        return tuple(p for p in self.peer_ids() if p not in held)

    def link_between(self, a, b) -> Link:
        a, b = str(a), str(b)
        if a == b:
            return ZERO_LINK
        return self.links.get((a, b)) or self.links.get((b, a)) or self.default_link

    def with_default_link(self, link: Link) -> "Fleet":
        return replace(self, default_link=link, links={})


def comm_time(link: Link, message_bytes: float) -> float:
    """alpha + beta * M (hardware.py:147-150)."""
    if message_bytes < 0:
        raise FleetError("message size must be nonnegative")
    return link.alpha + link.beta * message_bytes


def effective_speed(peer) -> float:
    """peak * lambda (hardware.py:153-154)."""
    return peer.peak_flops * peer.lam


def _peer_entry(entry: dict, column: str) -> Peer:
    if "id" not in entry:
        raise FleetError(f"peer entry without id: {entry!r}")
    pid = str(entry["id"])
    spec = None
    if "gpu" in entry:
        key = str(entry["gpu"]).lower()
        if key not in GPU_TABLE:
            raise FleetError(f"peer {pid}: unknown gpu {entry['gpu']!r}")
        spec = GPU_TABLE[key]
    if column not in COMPUTE_COLUMNS:
        raise FleetError(f"compute column must be one of {COMPUTE_COLUMNS}")
    tkey = f"tflops_{column}"
    if tkey in entry:
        tflops = float(entry[tkey])
    elif spec is not None:
        tflops = getattr(spec, tkey)
    else:
        raise FleetError(f"peer {pid}: needs {tkey} or a gpu model")
    return Peer(id=pid, role=Role(str(entry.get("role", "antnode")).lower()),
                peak_flops=tflops * 1e12, lam=float(entry.get("lambda", 1.0)),
                gpu_bytes=float(entry.get("gpu_gb", spec.memory_gb if spec else 8.0)) * 2**30,
                cpu_bytes=float(entry.get("cpu_gb", 16.0)) * 2**30,
                disk_bytes=float(entry.get("disk_gb", 64.0)) * 2**30,
                write_bandwidth=float(entry.get("write_bandwidth_bytes_per_s", math.inf)))


def _link_entry(entry: dict) -> Link:
    alpha = float(entry.get("alpha_s", entry.get("default_alpha_s", 0.0)))
    if "beta_s_per_byte" in entry:
        beta = float(entry["beta_s_per_byte"])
    elif "bandwidth_gbps" in entry:
        beta = bandwidth_to_beta(float(entry["bandwidth_gbps"]))
    elif "default_beta_bytes_per_s" in entry:
        bps = float(entry["default_beta_bytes_per_s"])
        if bps <= 0:
            raise FleetError("default_beta_bytes_per_s must be positive")
        beta = 1.0 / bps
    else:
        beta = 0.0
    return Link(alpha, beta)


def parse_fleet(doc, compute_column: str = "tensor") -> Fleet:
    """Fleet file (JSON text or dict) to Fleet, schema of hardware.py:265-354."""
    if isinstance(doc, str):
        try:
            doc = json.loads(doc)
        except json.JSONDecodeError as exc:
            raise FleetError(f"fleet file is not valid JSON: {exc}") from exc
    if not isinstance(doc, dict) or not isinstance(doc.get("peers"), list):
        raise FleetError('fleet file must be an object with a "peers" list')
    peers: dict[str, Peer] = {}
    for entry in doc["peers"]:
        peer = _peer_entry(entry, compute_column)
        if peer.id in peers:
            raise FleetError(f"duplicate peer id {peer.id!r}")
        peers[peer.id] = peer
    links_doc = doc.get("links") or {}
    overrides = {}
    for entry in links_doc.get("overrides", []):
        a, b = str(entry["src"]), str(entry["dst"])
        for end in (a, b):
            if end not in peers:
                raise FleetError(f"link override references unknown peer {end!r}")
        overrides[(a, b)] = _link_entry(entry)
    pinned = doc.get("pinned_runs")
    if pinned is not None:  # 1-based in the file, 0-based in memory
        pinned = tuple(tuple(int(s) - 1 for s in run) for run in pinned)
    return Fleet(peers=peers, default_link=_link_entry(links_doc), links=overrides,
                 backup_pool=tuple(str(p) for p in doc.get("backup_pool", [])),
                 msg_ratio=float(doc.get("msg_ratio", 1.0)), pinned_runs=pinned,
                 name=str(doc.get("name", "fleet")))


def load_fleet(path, compute_column: str = "tensor") -> Fleet:
    with open(path, encoding="utf-8") as fh:
        return parse_fleet(fh.read(), compute_column)


# ------------------------------------------------------------- scheduling
Runs = tuple  # tuple[tuple[str, tuple[int, ...]], ...]


@dataclass(frozen=True)
class Stage:
    """One pipeline cell (scheduling.py:32-42)."""

    index: int
    label: str
    flops: float
    gpu_bytes: float
    cpu_bytes: float
    disk_bytes: float
    in_edges: tuple = ()


@dataclass(frozen=True)
class PeerLoad:
    peer: str
    stage_indices: tuple
    compute_s: float
    read_s: float
    load_s: float
    gpu_bytes: float
    cpu_bytes: float
    disk_bytes: float


def format_stage_run(indices: Sequence[int]) -> str:
    """1-based human form of a run: '', '3' or '2-25' (scheduling.py:99-104)."""
    if not indices:
        return ""
    lo, hi = min(indices) + 1, max(indices) + 1
    return str(lo) if lo == hi else f"{lo}-{hi}"


@dataclass(frozen=True)
class ScheduleReport:
    """Scored assignment (scheduling.py:57-96)."""

    stages: tuple
    runs: tuple
    per_peer: tuple
    makespan: float
    feasible: bool
    reason: str = ""
    include_comm: bool = True
    trace: tuple = ()

    @property
    def assignment(self) -> dict:
        return {s: peer for peer, idxs in self.runs for s in idxs}

    def load_of(self, peer: str):
        for row in self.per_peer:
            if row.peer == peer:
                return row
        raise SchedulingError(f"peer {peer!r} not in schedule")

    def to_csv(self, path):
        with open(path, "w", newline="", encoding="utf-8") as fh:
            w = csv.writer(fh)
            w.writerow(["peer_id", "stage_ids", "C_p_s", "R_p_s", "load_s", "gpu_bytes_used"])
            for row in self.per_peer:
                w.writerow([row.peer, format_stage_run(row.stage_indices),
                            f"{row.compute_s:.9g}", f"{row.read_s:.9g}",
                            f"{row.load_s:.9g}", int(row.gpu_bytes)])

    def summary_text(self) -> str:
        out = [f"stages: {len(self.stages)}",
               f"feasible: {self.feasible}" + (f" ({self.reason})" if self.reason else ""),
               f"makespan_s: {self.makespan:.9g}"]
        for row in self.per_peer:
            out.append(f"  peer {row.peer}: stages {format_stage_run(row.stage_indices)}"
                       f" load {row.load_s:.6g}s (C {row.compute_s:.6g}s"
                       f" R {row.read_s:.6g}s)")
        return "\n".join(out)
