"""The C-ABI library loads without a GPU and exports exactly what
include/dagmesh_b200.h declares; struct layouts agree across the header, the
ctypes binding, the numpy record dtype and the oracle."""

import ctypes as C
import pathlib
import re

import numpy as np

from paper_2309_01172_b200 import _lib, tensorize

ROOT = pathlib.Path(__file__).resolve().parent.parent
HEADER = (ROOT / "include" / "dagmesh_b200.h").read_text()


def declared():
    return sorted(set(re.findall(r"^DM_API\s+[\w\s\*]+?\b(dm_\w+)\s*\(", HEADER, flags=re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "dm_eval_runs" in names and "dm_enum_splits" in names and "dm_subset_dp" in names
    assert len(names) >= 14


def test_library_exports_every_declared_symbol():
    lib = _lib.load(check_device=False)
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) == set(_lib.EXPORTED)
    assert lib.dm_abi_version() == 1


def test_struct_layouts_agree():
    from oracle import oracle
    assert C.sizeof(_lib.DmTables) == C.sizeof(oracle.Tables) == tensorize.TABLES_DTYPE.itemsize == 184
    for (a, _), (b, _) in zip(_lib.DmTables._fields_, oracle.Tables._fields_):
        assert a == b
        assert getattr(_lib.DmTables, a).offset == getattr(oracle.Tables, b).offset
        assert getattr(_lib.DmTables, a).offset == tensorize.TABLES_DTYPE.fields[a][1]
    assert C.sizeof(_lib.DmWinner) == 40
    assert C.sizeof(_lib.DmOps) == 64


def test_engine_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        return
    try:
        _lib.load(check_device=True)
    except _lib.EngineUnavailable as exc:
        assert "no CPU fallback" in str(exc)
    else:
        raise AssertionError("engine must refuse to run without a CUDA device")


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2309_01172_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f
