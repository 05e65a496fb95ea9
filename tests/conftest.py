import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "reference_counts.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_generators():
    with open(os.path.join(GOLDEN, "generators.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    import pyoracle
    pyoracle.build()
    return pyoracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference library itself (oracle/_ref), when it was built here."""
    import pyoracle
    if not os.path.exists(pyoracle.REF_SO):
        pytest.skip("oracle/_ref/libpospop_ref.so not built (needs /root/reference at build time)")
    return pyoracle.Reference()


@pytest.fixture(scope="session")
def pp():
    import paper_1911_02696_b200 as pp
    if not os.path.exists(pp.library_path()):
        import __graft_entry__
        __graft_entry__.build()
    return pp


@pytest.fixture
def tuning(pp):
    """Runs the test against the tuning build (libpospopcnt_b200_tuning.so):
    every measured kernel variant and the POSPOP_* tuning knobs, which the
    release library does not read.  Same kernel templates, so parity here is
    parity of the alternatives; the release build's own parity is every other
    test."""
    path = pp.library_path("tuning")
    if not os.path.exists(path):
        import __graft_entry__
        __graft_entry__.build()
    saved = pp._load()
    pp._lib = pp.load_library(path)
    try:
        yield pp._lib
    finally:
        pp._lib = saved
