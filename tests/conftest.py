"""Shared test setup: the `gpu` marker, import paths, engine/oracle fixtures."""

import pathlib
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

REFERENCE_SRC = pathlib.Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine library")
    config.addinivalue_line("markers", "reference: needs the reference package at /root/reference (build container only)")


def pytest_collection_modifyitems(config, items):
    have_ref = REFERENCE_SRC.exists()
    skip_ref = pytest.mark.skip(reason="reference tree not present (GPU box)")
    for item in items:
        if "reference" in item.keywords and not have_ref:
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def engine_ready():
    """The CUDA engine; GPU tests fail loudly (no skip) when it cannot run."""
    from paper_2309_01172_b200 import _lib
    _lib.load(check_device=True)
    return True


@pytest.fixture(scope="session")
def dagmesh_ref():
    if not REFERENCE_SRC.exists():
        pytest.skip("reference tree not present")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import dagmesh
    return dagmesh
