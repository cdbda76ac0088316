"""The erato-gpu CLI against the reference CLI contract
(/root/reference/proj/tests/cli_smoke.sh, tools/erato.cpp:65-176)."""
import os
import subprocess
import tempfile

import pytest

from conftest import ROOT

CLI = os.path.join(ROOT, "paper_1111_3297_b200", "erato-gpu")


@pytest.fixture(scope="module")
def cli(lib):
    from paper_1111_3297_b200.build import build_cli
    if not os.path.exists(CLI):
        build_cli()
    return CLI


def run(cli, *args):
    return subprocess.run([cli, *args], capture_output=True, text=True, timeout=600)


def test_param_errors_exit_1(cli):
    r = run(cli, "sieve", "--log-seg", "9", "--first", "1", "--segments", "1")
    assert r.returncode == 1 and "L_OUT_OF_RANGE" in r.stderr            # cli_smoke.sh:15-16
    r = run(cli, "sieve", "--log-seg", "10", "--first", "0", "--segments", "1")
    assert r.returncode == 1 and "F_ZERO_OR_OVERLAP" in r.stderr         # cli_smoke.sh:17-18
    r = run(cli, "sieve")
    assert r.returncode == 1                                              # cli_smoke.sh:21-22
    r = run(cli, "sieve", "--first", "1", "--midpoint-exp", "7", "--segments", "4")
    assert r.returncode == 1
    r = run(cli, "bogus")
    assert r.returncode == 1


@pytest.mark.gpu
def test_cli_smoke_contract(cli):
    r = run(cli, "sieve", "--log-seg", "10", "--first", "2048", "--segments", "4", "--count-only")
    assert r.returncode == 0 and "primes    542" in r.stdout
    with tempfile.TemporaryDirectory() as d:
        r = run(cli, "sieve", "--log-seg", "10", "--first", "2048", "--segments", "4", "--out-dir", d)
        assert r.returncode == 0, r.stderr
        f = os.path.join(d, "erato_l10_f2048_n4.bits")
        assert os.path.getsize(f) == 512 and f in r.stdout
    r = run(cli, "verify", "--log-seg", "12", "--first", "4096", "--segments", "8")
    assert r.returncode == 0 and "PASS" in r.stdout
    r = run(cli, "sieve", "--log-seg", "4", "--first", "2048", "--segments", "4", "--count-only", "--test-mode")
    assert r.returncode == 0
    r = run(cli, "sieve", "--log-seg", "10", "--midpoint-exp", "7", "--segments", "4", "--count-only")
    assert r.returncode == 0
    r = run(cli, "sieve", "--log-seg", "17", "--first", "0", "--segments", "64", "--count-only", "--allow-overlap")
    assert r.returncode == 0 and "primes    1077871" in r.stdout
    with tempfile.TemporaryDirectory() as d:
        csv = os.path.join(d, "b.csv")
        r = run(cli, "bench", "--exps", "12,13", "--csv", csv, "--reps", "2")
        assert r.returncode == 0 and open(csv).read().startswith("e,seconds,l\n")


@pytest.mark.gpu
def test_cli_multi_gpu_shards(cli):
    """--devices: range shards driven by the C-ABI multi-GPU entry (here all on
    device 0, the 1-GPU box's test topology); count and file as one GPU."""
    r = run(cli, "sieve", "--log-seg", "20", "--first", "523776", "--segments", "1024", "--count-only",
            "--devices", "0,0")
    assert r.returncode == 0 and "primes    77449842" in r.stdout, r.stderr
    with tempfile.TemporaryDirectory() as d:
        r = run(cli, "sieve", "--log-seg", "10", "--first", "2048", "--segments", "4", "--out-dir", d,
                "--devices", "0,0,0")
        assert r.returncode == 0 and "primes    542" in r.stdout, r.stderr
        assert os.path.getsize(os.path.join(d, "erato_l10_f2048_n4.bits")) == 512
    r = run(cli, "sieve", "--log-seg", "20", "--first", "523776", "--segments", "1024", "--count-only",
            "--gpus", "1")
    assert r.returncode == 0 and "primes    77449842" in r.stdout
    r = run(cli, "sieve", "--log-seg", "20", "--first", "523776", "--segments", "16", "--count-only",
            "--devices", "0,99")
    assert r.returncode == 2 and "NO_DEVICE" in r.stderr
