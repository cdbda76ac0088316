"""The CPU oracles against the golden fixtures and the reference library.

oracle/erato_oracle.c is a restatement of the reference semantics; before it
is trusted as the checker it is pinned here against (a) the golden vectors
made from the unmodified reference (tests/golden/make_golden.py) and (b) the
reference library itself (oracle/_ref) on seeded instances.
"""
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN


def sha(t):
    return hashlib.sha256(np.ascontiguousarray(t).tobytes()).hexdigest()


def test_restated_smoke_pin(restated, pins):
    g = pins["configs"]["smoke"]
    t, c = restated.bit_table(g["l"], g["f"], g["n"])
    assert c == g["count"] == 542
    assert sha(t) == g["sha256"]


def test_restated_cfg1_f0_pin(restated, pins):
    g = pins["configs"]["cfg1"]
    t, c = restated.bit_table(g["l"], g["f"], g["n"], allow_overlap=True)
    assert c == g["count"] == 1077871  # pi(2^24): 1 counts instead of 2
    assert sha(t) == g["sha256"]


@pytest.mark.parametrize("k", range(0, 52, 1))
def test_restated_random_pins(restated, pins, k):
    rec = pins["random"][k % len(pins["random"])]
    t, c = restated.bit_table(rec["l"], rec["f"], rec["n"], test_mode=True,
                              allow_overlap=rec.get("allow_overlap", False))
    assert c == rec["count"]
    assert sha(t) == rec["sha256"]


def test_restated_small_tables(restated):
    z = np.load(os.path.join(GOLDEN, "small_tables.npz"))
    assert len(z.files) >= 4
    for name in z.files:
        l, f, n = (int(x[1:]) for x in name.split("_"))
        t, _ = restated.bit_table(l, f, n, test_mode=True)
        assert np.array_equal(t, z[name]), name


def test_restated_vs_reference_random(restated, reference):
    rng = np.random.default_rng(7)
    for _ in range(25):
        l = int(rng.integers(4, 15))
        n = int(rng.integers(1, 40))
        f = int(rng.integers(1, max(2, (1 << 33) >> (l + 1))))
        try:
            reference.validate(l, f, n, test_mode=True)
        except Exception:
            continue
        a, ca = restated.bit_table(l, f, n, test_mode=True)
        b, cb, _ = reference.run_sieve(l, f, n, test_mode=True)
        assert ca == cb and np.array_equal(a, b), (l, f, n)


def test_restated_f0_vs_reference_assembly(restated, reference):
    for (l, n) in [(10, 1), (10, 7), (12, 33), (4, 5)]:
        a, ca = restated.bit_table(l, 0, n, test_mode=True, allow_overlap=True)
        b, cb = reference.f0_table(l, n, test_mode=True)
        assert ca == cb and np.array_equal(a, b), (l, n)


def test_reference_brute_force_oracle_agrees(reference):
    # the reference's own oracle_bit_table vs its run_sieve (v <= 2^40)
    for (l, f, n) in [(10, 2048, 4), (12, 4096, 8), (10, 6, 1), (10, 5, 1)]:
        a = reference.oracle_bit_table(l, f, n)
        b, _, _ = reference.run_sieve(l, f, n)
        assert np.array_equal(a, b)


def test_known_answers_restated(restated, known_answers):
    for p, l, f, q in known_answers["first_offset"]:
        assert restated.first_offset(p, l, f) == q
    assert restated.first_offset(3, 4, 1) == 0 and restated.first_offset(7, 10, 3) == 4  # test_wheel.cpp:38-42
    for e, l, n, f in known_answers["params_from_midpoint"]:
        assert restated.params_from_midpoint(e, l, n) == f
    assert known_answers["params_from_midpoint"][0][3] == 238162  # test_params.cpp:128-138
    for x, r in known_answers["isqrt"]:
        assert restated.isqrt(x) == r
    l, f, n, u, v = known_answers["validate"][0]
    assert restated.validate(l, f, n) == (u, v) == (4194305, 4202496)  # test_params.cpp:21-27
    assert len(restated.simple_sieve(10 ** 6)) == known_answers["pi_1e6"] == 78498


def test_restated_rejects_like_reference(restated, known_answers):
    from oracle.oracle import OracleError
    for l, f, n, tm, name in known_answers["rejects"]:
        if name == "OK":
            restated.validate(l, f, n, test_mode=tm)
        else:
            with pytest.raises(OracleError) as ei:
                restated.validate(l, f, n, test_mode=tm)
            assert ei.value.name == name, (l, f, n, tm)


def test_pins_cover_all_configs(pins):
    for k in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        assert k in pins["configs"], k
    # SURVEY.md Appendix A
    assert pins["configs"]["cfg3"]["count"] == 77449842
    assert pins["configs"]["cfg4"]["count"] == 516358044
    assert pins["configs"]["cfg5"]["count"] == 1652382527
    assert pins["configs"]["cfg5"]["sha256"].startswith("1173a26c")
