"""The INTEGRATION.md binding (tests/integration/gpu_binding.hpp) as a
compiled program: erato::run_sieve_gpu built against the unmodified reference
headers and library (oracle/_ref) and liberato_gpu.so.  On CPU it must build
and link; on the B200 it must equal the reference's own run_sieve on every sink
(NullSink, TableSink, PrimeCollectSink, FileSink, a user sink), in order."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "erato_binding_test")


@pytest.fixture(scope="module")
def binding(lib):
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "all", "binding"], check=True)
    if not os.path.exists(BIN):
        pytest.skip("binding test binary not built (needs /root/reference to compile)")
    return BIN


def test_binding_links(binding):
    r = subprocess.run([binding, "--link"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "linked" in r.stdout


@pytest.mark.gpu
def test_binding_equals_reference_run_sieve(binding):
    r = subprocess.run([binding], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "binding OK" in r.stdout
