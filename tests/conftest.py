import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")


def build_lib():
    """Build libgsp.so in-tree (loads _build.py by path: importing the package first
    would try to load the not-yet-built library, which fails loudly by design)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_gsp_build", os.path.join(ROOT, "paper_2402_03548_b200", "_build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


def pytest_sessionstart(session):
    # a fresh checkout has no libgsp.so; build it before any test imports the package
    # (a no-op when it is up to date)
    build_lib()


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden():
    return load_golden
