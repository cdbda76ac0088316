"""The C ABI library on CPU: it loads, exports every symbol include/erato_gpu.h
declares, its host-side parameter logic matches the reference, and every
compute entry point refuses to run without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_functions():
    src = open(os.path.join(ROOT, "include", "erato_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(erato_gpu_\w+)\s*\(", src)))


def test_exports_every_header_symbol(lib):
    from paper_1111_3297_b200 import _lib
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTS)


def test_no_device_no_fallback(lib):
    import paper_1111_3297_b200 as E
    if E.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(E.Error) as ei:
        E.Context(0)
    assert ei.value.code == E.errc.no_device


def test_validate_matches_reference(lib, reference, known_answers):
    import paper_1111_3297_b200 as E
    for l, f, n, tm, name in known_answers["rejects"]:
        if name == "OK":
            E.validate_params(l, f, n, test_mode=tm)
        else:
            with pytest.raises(E.Error) as ei:
                E.validate_params(l, f, n, test_mode=tm)
            assert E.errc_name(ei.value.code) == name
            assert str(ei.value).startswith(name + ":")
    rng = np.random.default_rng(3)
    for _ in range(300):
        l = int(rng.integers(3, 32))
        n = int(rng.integers(0, 5000))
        f = int(rng.integers(0, 1 << 40)) >> int(rng.integers(0, 40))
        tm = bool(rng.integers(0, 2))
        try:
            ru = reference.validate(l, f, n, test_mode=tm)
            rerr = None
        except Exception as e:
            rerr = e.name
        try:
            p = E.validate_params(l, f, n, test_mode=tm)
            ours = (p.u, p.v)
            oerr = None
        except E.Error as e:
            oerr = E.errc_name(e.code)
        assert oerr == rerr, (l, f, n, tm)
        if rerr is None:
            assert ours == ru


def test_f0_rejected_by_default_accepted_with_overlap(lib):
    import paper_1111_3297_b200 as E
    with pytest.raises(E.Error) as ei:
        E.validate_params(10, 0, 1)
    assert ei.value.code == E.errc.f_zero_or_overlap  # cli_smoke.sh:17-18
    p = E.validate_params(17, 0, 64, allow_overlap=True)
    assert (p.u, p.v) == (1, 1 << 24)


def test_midpoint_isqrt_first_offset(lib, reference, known_answers):
    import paper_1111_3297_b200 as E
    for e, l, n, f in known_answers["params_from_midpoint"]:
        assert E.params_from_midpoint(e, l, n) == f
    with pytest.raises(E.Error):
        E.params_from_midpoint(20, 10, 4)
    for x, r in known_answers["isqrt"]:
        assert E.isqrt(x) == r
    rng = np.random.default_rng(11)
    for _ in range(2000):
        x = int(rng.integers(0, 1 << 63)) * 2 + int(rng.integers(0, 2))
        assert E.isqrt(x) == reference.isqrt(x)
    for p, l, f, q in known_answers["first_offset"]:
        assert E.first_offset(p, l, f) == q
    primes = reference.simple_sieve(200000)[1:]
    for _ in range(2000):
        p = int(primes[rng.integers(0, len(primes))])
        l = int(rng.integers(4, 31))
        f = int(rng.integers(0, 1 << 62)) >> l
        assert E.first_offset(p, l, f) == reference.first_offset(p, l, f)


def test_first_hit_host_twin_matches_wheel_align(lib, reference):
    """The device start-offset rule (cofactor wheel mod 30) lands on exactly the
    reference's wheel_align(first_offset) position (src/wheel.cpp:43-69)."""
    rng = np.random.default_rng(5)
    primes = [int(p) for p in reference.simple_sieve(1 << 20) if p > 5]
    for _ in range(3000):
        p = primes[int(rng.integers(0, len(primes)))]
        l = int(rng.integers(10, 23))
        f = int(rng.integers(1, 1 << 40))
        if (p << 4) > (1 << l) and False:
            continue
        q0 = reference.first_offset(p, l, f)
        qa, _ = reference.wheel_align(p, q0, l, f)
        off = C.c_uint64()
        cls = C.c_uint()
        assert lib.erato_gpu_first_hit(p, (f << (l + 1)) + 1, 2, C.byref(off), C.byref(cls)) == 0
        assert off.value == qa, (p, l, f)
        c = (2 * ((f << l) + off.value) + 1) // p  # the cofactor
        assert c % 30 == [1, 7, 11, 13, 17, 19, 23, 29][cls.value]


def test_table_filename_and_shard(lib):
    import paper_1111_3297_b200 as E
    p = E.validate_params(10, 2048, 4)
    assert E.table_filename(p) == "erato_l10_f2048_n4.bits"  # cli_smoke.sh:25-29
    buf = C.create_string_buffer(64)
    lib.erato_gpu_table_filename(22, (1 << 37) - 4096, 8192, buf, 64)
    assert buf.value.decode() == "erato_l22_f137438949376_n8192.bits"
    for n in (1, 7, 64, 8192, 10 ** 6 + 3):
        for world in (1, 2, 3, 4, 8):
            parts = [E.shard(100, n, r, world) for r in range(world)]
            assert parts[0][0] == 100
            assert sum(x[1] for x in parts) == n
            for a, b in zip(parts, parts[1:]):
                assert a[0] + a[1] == b[0]


def test_errc_names_match_reference_order(lib):
    import paper_1111_3297_b200 as E
    ref_order = ["L_OUT_OF_RANGE", "F_ZERO_OR_OVERLAP", "N_OUT_OF_RANGE", "OVERFLOW", "INDEX_OUT_OF_RANGE",
                 "NOT_ADMISSIBLE", "ALLOC_LIMIT", "LIMIT_TOO_LARGE", "RANGE_TOO_LARGE", "IO_ERROR"]
    for i, name in enumerate(ref_order):  # params.cpp:7-21
        assert lib.erato_gpu_errc_name(i + 1).decode() == name
        assert E.errc_name(E.errc(i)) == name


def test_header_flags_and_gpu_errc_match_python_mirror(lib):
    """The run flags and the GPU-only error codes of include/erato_gpu.h are
    the ones the Python mirror uses (ordinal + 1 on the ABI)."""
    import paper_1111_3297_b200 as E
    from paper_1111_3297_b200 import erato
    src = open(os.path.join(ROOT, "include", "erato_gpu.h")).read()
    flags = {m[0]: int(m[1], 16) for m in re.findall(r"#define (ERATO_GPU_\w+) (0x[0-9a-f]+)u", src)}
    assert flags["ERATO_GPU_TEST_MODE"] == erato.TEST_MODE
    assert flags["ERATO_GPU_ALLOW_OVERLAP"] == erato.ALLOW_OVERLAP
    assert flags["ERATO_GPU_CHECK_INVARIANTS"] == erato.CHECK_INVARIANTS
    codes = {m[0]: int(m[1]) for m in re.findall(r"(ERATO_GPU_E_\w+) = (\d+)", src)}
    for cname, py in [("ERATO_GPU_E_CUDA", E.errc.cuda_error), ("ERATO_GPU_E_NO_DEVICE", E.errc.no_device),
                      ("ERATO_GPU_E_INVALID_ARG", E.errc.invalid_argument),
                      ("ERATO_GPU_E_INVARIANT", E.errc.invariant)]:
        assert codes[cname] == int(py) + 1
        assert lib.erato_gpu_errc_name(codes[cname]).decode() == E.errc_name(py)


def test_wheel_deltas_walk_the_coprime_cofactors(lib):
    """erato_gpu_wheel_deltas: the large primes' wheel tables.  For every
    supported modulus the deltas walk exactly the odd residues coprime to M
    (the reference's wheel, src/wheel.cpp:10-34, is the M = 30 case with
    deltas {3,2,1,2,1,2,3,1}), sum to M/2 per turn and fit a nibble."""
    import ctypes as C
    from math import gcd
    assert lib.erato_gpu_wheel_deltas(77, None, 0) == 0
    for M, nres in ((30, 8), (210, 48), (2310, 480), (30030, 5760)):
        buf = (C.c_uint8 * nres)()
        assert lib.erato_gpu_wheel_deltas(M, buf, nres) == nres
        d = list(buf)
        assert sum(d) == M // 2 and max(d) <= 11 and min(d) >= 1
        r, seen = 1, []
        for x in d:
            seen.append(r)
            r += 2 * x
        assert r == 1 + M  # one full turn
        assert seen == [c for c in range(1, M, 2) if gcd(c, M) == 1]
    buf = (C.c_uint8 * 8)()
    lib.erato_gpu_wheel_deltas(30, buf, 8)
    assert list(buf) == [3, 2, 1, 2, 1, 2, 3, 1]  # wheel.cpp:27-30

