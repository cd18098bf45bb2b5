import json
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def golden(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as f:
        return json.load(f)


def unhex(s):
    return float.fromhex(s)


@pytest.fixture(scope="session")
def port():
    from oracle import port as p
    return p


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r
    if not r.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return r


def _ref_available():
    from oracle import ref as r
    return r.available()


# tests that compare with the unmodified reference library (oracle/_ref)
requires_ref = pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built (needs /root/reference at build time)")
