"""Test configuration.

Markers
  gpu   needs a CUDA device (run on the B200 box: pytest -m gpu)

The CPU suite (pytest -m "not gpu") covers the oracles against the golden
fixtures, the host-side logic of the C ABI, the Python mirror of the
reference interface and the multi-process (gloo) sharding path.
"""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def pins():
    with open(os.path.join(GOLDEN, "pins.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def known_answers():
    with open(os.path.join(GOLDEN, "known_answers.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def restated():
    from oracle.oracle import Restated, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "_build", "liberato_oracle.so")):
        build(reference=False)
    return Restated()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference library, when it has been built (oracle/_ref)."""
    from oracle.oracle import REFERENCE_SO, Reference, build
    if not os.path.exists(REFERENCE_SO) and os.path.isdir("/root/reference/proj/src"):
        build(reference=True)
    if not os.path.exists(REFERENCE_SO):
        pytest.skip("reference library not built (oracle/_ref)")
    return Reference()


@pytest.fixture(scope="session")
def lib():
    from paper_1111_3297_b200 import _lib
    from paper_1111_3297_b200.build import build
    build()
    return _lib.load()


@pytest.fixture(scope="session")
def gpu_ctx():
    import paper_1111_3297_b200 as E
    if E.device_count() == 0:
        pytest.fail("no CUDA device: the gpu tests must run on the B200 box")
    return E.context(0)
