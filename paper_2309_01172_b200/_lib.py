"""ctypes binding of the C ABI in include/dagmesh_b200.h.

The library is built in-tree (``paper_2309_01172_b200/libdagmesh_b200.so``,
see ``build.py``).  There is deliberately no fallback: if the library or a
CUDA device is missing, every engine call raises ``EngineUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import pathlib

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "libdagmesh_b200.so"

DM_OK = 0
DM_E_ARG, DM_E_CUDA, DM_E_UNKNOWN_PEER, DM_E_UNASSIGNED, DM_E_TOO_LARGE = -1, -2, -3, -4, -5

DM_V_OK, DM_V_TWO_RUNS, DM_V_UNKNOWN_PEER, DM_V_NOT_CONTIGUOUS = 0, 1, 2, 3
DM_V_ASSIGNED_TWICE, DM_V_GPU, DM_V_CPU, DM_V_DISK, DM_V_UNASSIGNED = 4, 5, 6, 7, 8

DM_F_FLOPS_EXACT, DM_F_BYTES_EXACT, DM_F_PAIR_LINKS = 1, 2, 4
DM_F_CHAIN, DM_F_BACKWARD, DM_F_INCLUDE_COMM = 8, 16, 32
DM_F_NP_FLOPS, DM_F_NP_COMM, DM_F_NP_BYTES = 64, 128, 256


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run (library not built, or no CUDA device)."""


class EngineError(RuntimeError):
    """A dm_* call returned a negative status."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"dm status {status}: {msg}")
        self.status = status


_P = C.c_void_p


class DmTables(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("p", C.c_int32), ("P", C.c_int32), ("n_edges", C.c_int32),
        ("flags", C.c_uint32), ("pad_", C.c_int32),
        ("def_alpha", C.c_double), ("def_beta", C.c_double),
        ("flops", _P), ("gpu", _P), ("cpu", _P), ("disk", _P),
        ("pre_flops", _P), ("pre_gpu", _P), ("pre_cpu", _P), ("pre_disk", _P),
        ("edge_ptr", _P), ("edge_src", _P), ("edge_m", _P),
        ("speed", _P), ("cap_gpu", _P), ("cap_cpu", _P), ("cap_disk", _P),
        ("link_alpha", _P), ("link_beta", _P), ("peer_np", _P),
    ]


DM_OPS_NP_LINKS = 1


class DmOps(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("flags", C.c_int32), ("flops", _P), ("mbytes", _P), ("arg_ptr", _P),
                ("arg_idx", _P), ("user_ptr", _P), ("user_idx", _P), ("write_np", _P)]


class DmWinner(C.Structure):
    _fields_ = [("makespan", C.c_double), ("rank", C.c_int64), ("n_evaluated", C.c_int64),
                ("n_feasible", C.c_int64), ("checksum", C.c_uint64)]


_SIGS = {
    "dm_abi_version": (C.c_int, []),
    "dm_last_error": (C.c_char_p, []),
    "dm_enum_scratch_bytes": (C.c_int64, []),
    "dm_eval_runs": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "dm_eval_owner": (C.c_int, [_P, C.c_int64, _P, C.c_int32, _P, _P, _P]),
    "dm_eval_owner_argmin": (C.c_int, [_P, C.c_int64, _P, C.c_int32, _P, _P, C.c_int64, _P, _P, _P]),
    "dm_argmin_scores": (C.c_int, [_P, _P, C.c_int64, C.c_int64, _P, _P, _P]),
    "dm_enum_bruteforce": (C.c_int, [_P, C.c_int64, C.c_int64, _P, _P, _P]),
    "dm_enum_splits": (C.c_int, [_P, C.c_int64, C.c_int64, _P, _P, _P]),
    "dm_enum_splits_part": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P]),
    "dm_splits_workspace_bytes": (C.c_int64, [_P]),
    "dm_enum_splits_ws": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P, C.c_int64, _P]),
    "dm_enum_splits_phase": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P, C.c_int64,
                                       C.c_int32, _P]),
    "dm_enum_random": (C.c_int, [_P, _P, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, _P, _P, _P]),
    "dm_finalize_winners": (C.c_int, [_P, C.c_int32, _P, _P]),
    "dm_subset_dp_scratch_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "dm_subset_dp": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P, _P]),
    "dm_prop_hill": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P]),
    "dm_prop_hill_epilogue": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, C.c_int64, C.c_int64, _P, _P]),
    "dm_pipeline_epilogue": (C.c_int, [_P, C.c_int32, C.c_int32, _P, C.c_int64, C.c_int64, _P, _P]),
    "dm_microbench_fp64": (C.c_int, [C.c_int64, _P, _P, _P]),
    "dm_microbench_cross": (C.c_int, [C.c_int64, _P, _P, _P]),
    "dm_microbench_alu": (C.c_int, [C.c_int64, _P, _P, _P]),
    "dm_sched_out_bytes": (C.c_int64, [C.c_int32]),
    "dm_eval_runs_ws_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "dm_eval_runs_ws": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "dm_schedule_report": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P]),
    "dm_sweep_timing": (C.c_int, [C.c_int32, _P, _P]),
    "dm_op_costs": (C.c_int, [_P, _P, _P, C.c_int32, _P, _P, _P, _P]),
    "dm_subgraph_times": (C.c_int, [C.c_int32, C.c_int32, _P, _P, C.c_int32, _P, _P, _P, _P]),
    "dm_materialize": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int64, _P, C.c_int32, _P]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(check_device: bool = True):
    """Load the engine library; raise EngineUnavailable when it cannot run."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise EngineUnavailable(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.dm_abi_version() != 1:
            raise EngineUnavailable("ABI version mismatch")
        _lib = lib
    if check_device:
        import torch
        if not torch.cuda.is_available():
            raise EngineUnavailable("no CUDA device: the B200 engine has no CPU fallback")
    return _lib


def check(status: int):
    if status != DM_OK:
        raise EngineError(status, (_lib.dm_last_error() or b"").decode(errors="replace"))


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def loaded_path() -> str | None:
    return str(LIB_PATH) if _lib is not None else None


def ptr(t) -> int:
    """data_ptr of a torch tensor (or 0 for None)."""
    return 0 if t is None else int(t.data_ptr())

