"""GPU parity: the sm_100a sieve (through the C ABI) against the reference.

Bar: bit-exact tables and counts.  Small and ragged cases are compared with
the reference's own run_sieve (oracle/_ref, the unmodified library) and with
the restated oracle; the five BASELINE configs with the golden pins (count +
sha256 of the whole table); full-size properties (shard concatenation,
Miller-Rabin spot checks, extract_primes) cover what the oracle cannot redo
in seconds.
"""
import hashlib
import os
import random
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def sha(t):
    return hashlib.sha256(np.ascontiguousarray(t).tobytes()).hexdigest()


def miller_rabin(n: int) -> bool:
    # deterministic for 64-bit (tests/support.hpp:28-54 bases)
    if n < 2:
        return False
    bases = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for p in bases:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in bases:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


SMALL = [(10, 2048, 4, False), (12, 4096, 8, False), (4, 2048, 4, True), (10, 6, 1, False), (10, 5, 1, False),
         (16, 3, 5, True), (13, 100, 300, True), (17, 9000, 64, False), (20, 523776, 16, False),
         (18, 1 << 30, 40, False), (12, 1 << 40, 1000, False), (16, 1 << 45, 200, False),
         (13, (1 << 46) + 12345, 3001, False), (20, 1 << 41, 600, False), (4, 1, 1, True), (5, 2, 7, True),
         (11, 7, 9, False), (14, 123456789, 17, False)]


@pytest.mark.parametrize("l,f,n,tm", SMALL)
def test_small_vs_reference(gpu_ctx, reference, l, f, n, tm):
    import paper_1111_3297_b200 as E
    p = E.validate_params(l, f, n, test_mode=tm)
    g, st = gpu_ctx.table(p)
    r, rc, _ = reference.run_sieve(l, f, n, test_mode=tm)
    assert st.prime_count == rc
    assert np.array_equal(g, r)


def test_random_pins(gpu_ctx, pins):
    import paper_1111_3297_b200 as E
    for rec in pins["random"]:
        p = E.validate_params(rec["l"], rec["f"], rec["n"], test_mode=True,
                              allow_overlap=rec.get("allow_overlap", False))
        g, st = gpu_ctx.table(p)
        assert st.prime_count == rec["count"], rec
        assert sha(g) == rec["sha256"], rec


def test_random_vs_reference_seeded(gpu_ctx, reference):
    import paper_1111_3297_b200 as E
    rng = random.Random(1002)  # acceptance.cpp:71 seed
    done = 0
    while done < 40:
        l = rng.randint(4, 20)
        n = rng.randint(1, 300)
        f = rng.randint(1, (1 << rng.randint(l + 2, 50)) >> (l + 1) or 1)
        try:
            p = E.validate_params(l, f, n, test_mode=True)
        except E.Error:
            continue
        if p.table_bytes() > 64 << 20:
            continue
        g, st = gpu_ctx.table(p)
        r, rc, _ = reference.run_sieve(l, f, n, test_mode=True)
        assert st.prime_count == rc and np.array_equal(g, r), (l, f, n)
        done += 1


@pytest.mark.parametrize("l,n", [(17, 64), (12, 50), (10, 1), (4, 3), (20, 64), (16, 40)])
def test_f0_overlap_convention(gpu_ctx, restated, reference, l, n):
    import paper_1111_3297_b200 as E
    p = E.validate_params(l, 0, n, test_mode=True, allow_overlap=True)
    g, st = gpu_ctx.table(p)
    o, oc = restated.bit_table(l, 0, n, test_mode=True, allow_overlap=True)
    r, rc = reference.f0_table(l, n, test_mode=True)
    assert st.prime_count == oc == rc
    assert np.array_equal(g, o) and np.array_equal(g, r)


def test_overlap_nonzero_f(gpu_ctx, restated):
    # u^2 <= v with f > 0 (rejected by the reference; p^2 convention here)
    import paper_1111_3297_b200 as E
    for (l, f, n) in [(10, 1, 2049), (12, 3, 5000), (8, 1, 100)]:
        p = E.validate_params(l, f, n, test_mode=True, allow_overlap=True)
        g, st = gpu_ctx.table(p)
        o, oc = restated.bit_table(l, f, n, test_mode=True, allow_overlap=True)
        assert st.prime_count == oc and np.array_equal(g, o)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_baseline_config_pins(gpu_ctx, pins, cfg):
    """All five BASELINE configs: count + sha256 of the whole table."""
    import paper_1111_3297_b200 as E
    rec = pins["configs"][cfg]
    p = E.validate_params(rec["l"], rec["f"], rec["n"], allow_overlap=rec["allow_overlap"])
    g, st = gpu_ctx.table(p)
    assert g.nbytes == rec["bytes"]
    assert st.prime_count == rec["count"]
    assert sha(g) == rec["sha256"]
    st2 = gpu_ctx.count(p)  # NullSink path agrees
    assert st2.prime_count == rec["count"]


def test_cfg5_shards_concatenate(gpu_ctx, pins):
    """Range sharding (the multi-GPU decomposition) is exact at full size: 8
    shard runs of cfg5, hashed in order, give the full-table pin."""
    import paper_1111_3297_b200 as E
    rec = pins["configs"]["cfg5"]
    h = hashlib.sha256()
    total = 0
    for r in range(8):
        fg, ng = E.shard(rec["f"], rec["n"], r, 8)
        g, st = gpu_ctx.table(E.validate_params(rec["l"], fg, ng))
        h.update(g.tobytes())
        total += st.prime_count
    assert total == rec["count"]
    assert h.hexdigest() == rec["sha256"]


def test_cfg5_miller_rabin_spot_checks(gpu_ctx, pins):
    import paper_1111_3297_b200 as E
    rec = pins["configs"]["cfg5"]
    fg, ng = E.shard(rec["f"], rec["n"], 3, 8)
    p = E.validate_params(rec["l"], fg, ng)
    g, _ = gpu_ctx.table(p)
    rng = np.random.default_rng(17)
    for j in rng.integers(0, p.table_bits(), 4000):
        j = int(j)
        bit = (int(g[j >> 3]) >> (j & 7)) & 1
        assert bit == (0 if miller_rabin(p.u + 2 * j) else 1), j


def test_extract_primes_and_collect_sink(gpu_ctx, reference):
    import paper_1111_3297_b200 as E
    p = E.validate_params(16, 1 << 20, 24)
    primes = gpu_ctx.extract_primes(p)
    sink = E.PrimeCollectSink()
    E.run_sieve(p, sink)
    assert np.array_equal(primes, sink.primes())
    _, rc, _ = reference.run_sieve(16, 1 << 20, 24)
    assert len(primes) == rc
    assert all(miller_rabin(int(x)) for x in primes[:: max(1, len(primes) // 300)])
    p0 = E.validate_params(12, 0, 8, allow_overlap=True)
    pr = gpu_ctx.extract_primes(p0)
    assert int(pr[0]) == 3 and 1 not in set(int(x) for x in pr[:4])


def test_run_sieve_sinks_match_reference(gpu_ctx, reference):
    import paper_1111_3297_b200 as E
    p = E.validate_params(12, 4096, 8)
    r, rc, _ = reference.run_sieve(12, 4096, 8)
    ts = E.TableSink()
    st = E.run_sieve(p, ts)
    assert st.prime_count == rc and np.array_equal(ts.bytes(), r)
    assert E.run_sieve(p, E.NullSink()).prime_count == rc

    class Collect(E.SegmentSink):
        def __init__(self):
            self.ts = []

        def on_segment(self, seg, t, params):
            self.ts.append((t, bytes(seg)))

    c = Collect()
    E.run_sieve(p, c)
    assert [t for t, _ in c.ts] == list(range(8))
    assert b"".join(b for _, b in c.ts) == r.tobytes()


def test_file_sink_matches_reference_file(gpu_ctx, reference):
    import paper_1111_3297_b200 as E
    with tempfile.TemporaryDirectory() as d1, tempfile.TemporaryDirectory() as d2:
        p = E.validate_params(10, 2048, 4)
        path = E.write_table(d1, p)
        rpath, _ = reference.write_table(d2, 10, 2048, 4)
        assert os.path.basename(path) == os.path.basename(rpath) == "erato_l10_f2048_n4.bits"
        assert os.path.getsize(path) == 512  # cli_smoke.sh:25-29
        assert open(path, "rb").read() == open(rpath, "rb").read()
        # byte0 bit0 = u = 4194305 = 5 * 838861 -> composite (test_driver.cpp:59-86)
        assert open(path, "rb").read()[0] & 1 == 1


def test_sharded_file_writes(gpu_ctx, reference):
    """Per-shard pwrite into one file (multi-GPU output) == the whole table."""
    import paper_1111_3297_b200 as E
    l, f, n = 16, 1 << 24, 37
    p = E.validate_params(l, f, n)
    with tempfile.TemporaryDirectory() as d:
        for r in (2, 0, 1):
            fg, ng = E.shard(f, n, r, 3)
            gpu_ctx.write_table(d, p, fg, ng)
        data = open(os.path.join(d, E.table_filename(p)), "rb").read()
    ref, _, _ = reference.run_sieve(l, f, n)
    assert data == ref.tobytes()


def test_edge_cases(gpu_ctx, reference, restated):
    import paper_1111_3297_b200 as E
    # v just below 2^64: l = 30, largest f
    l = 30
    f = (((1 << 64) - 1) >> (l + 1)) - 1  # largest valid f for n = 1
    p = E.validate_params(l, f, 1)
    assert p.v < 1 << 64 and p.v > (1 << 64) - (1 << 32)
    with pytest.raises(E.Error) as ei:
        E.validate_params(l, f + 1, 1)
    assert ei.value.code == E.errc.overflow
    with pytest.raises(E.Error) as ei:  # 2^32 base primes: over the reference's default cap
        gpu_ctx.count(p)
    assert ei.value.code == E.errc.alloc_limit
    gpu_ctx.set_max_base_pairs(1 << 28)
    st = gpu_ctx.count(p)
    assert 0 < st.prime_count < p.table_bits()
    f10 = (((1 << 64) - 1) >> 11) - 1
    pp = E.validate_params(10, f10, 1)
    g, _ = gpu_ctx.table(pp)
    rng = np.random.default_rng(1)
    for j in rng.integers(0, pp.table_bits(), 300):
        j = int(j)
        assert ((int(g[j >> 3]) >> (j & 7)) & 1) == (0 if miller_rabin(pp.u + 2 * j) else 1)
    gpu_ctx.set_max_base_pairs(1 << 27)
    # errors come back with the reference's codes
    with pytest.raises(E.Error) as ei:
        gpu_ctx.count(E.SieveParams(9, 1, 1, 0, 0))
    assert ei.value.code == E.errc.l_out_of_range
    with pytest.raises(E.Error) as ei:
        E.validate_params(10, 0, 1)
    assert ei.value.code == E.errc.f_zero_or_overlap


def test_repeat_runs_deterministic(gpu_ctx):
    import paper_1111_3297_b200 as E
    p = E.validate_params(21, (1 << 26) - 2048, 256)
    a, sa = gpu_ctx.table(p)
    b, sb = gpu_ctx.table(p)
    assert sa.prime_count == sb.prime_count and np.array_equal(a, b)


@pytest.mark.parametrize("l,f,n,overlap", [(20, 0, 4096, True), (20, 0, 3001, True), (13, 5000, 77, False),
                                            (20, (1 << 19) - 512, 1024, False), (16, 1 << 30, 9, False)])
def test_base_prime_count_fresh_context(restated, l, f, n, overlap):
    """The device base-prime list (odd primes <= isqrt(v)) is exact on a FRESH
    context, where [1, isqrt v] rarely ends on a byte boundary (a stale
    buffer from an earlier run must not hide an unwritten last byte)."""
    import math
    import paper_1111_3297_b200 as E
    p = E.validate_params(l, f, n, allow_overlap=overlap)
    ctx = E.Context(0)
    try:
        st = ctx.count(p)
    finally:
        ctx.close()
    r = math.isqrt(p.v)
    sieve = np.ones(r + 1, dtype=bool)
    sieve[:2] = False
    for i in range(2, math.isqrt(r) + 1):
        if sieve[i]:
            sieve[i * i::i] = False
    assert st.base_primes == int(sieve[3:].sum())


def test_medium_record_rebase_over_2p20_tiles(gpu_ctx):
    """Runs of more than 2^20 tiles re-base the medium-prime records every
    2^20 tiles (the per-tile fp32 quotient stays exact).  A count-only run of
    1,049,600 tiles must equal the sum of its two shards, neither of which
    re-bases."""
    import paper_1111_3297_b200 as E
    l, f, n = 30, 1 << 20, 1025  # T = 1025 * 2^30 bits = 1,049,600 tiles of 2^20
    whole = gpu_ctx.count(E.validate_params(l, f, n))
    assert whole.tiles > (1 << 20)
    a = gpu_ctx.count(E.validate_params(l, f, 512))
    b = gpu_ctx.count(E.validate_params(l, f + 512, n - 512))
    assert a.tiles < (1 << 20) and b.tiles < (1 << 20)
    assert whole.prime_count == a.prime_count + b.prime_count


@pytest.mark.parametrize("l,f,n", [(21, (1 << 26) - 2048, 300), (22, (1 << 37) - 4096, 400)])
def test_genbin_fallback_matches_split_scatter(gpu_ctx, l, f, n):
    """The k_gen + k_bin large-prime path (used when a wave has more than 256
    bins) gives the same table as the default k_scatter_ml/k_scatter_far path,
    with ML primes only (first case) and with far buckets (second)."""
    import paper_1111_3297_b200 as E
    p = E.validate_params(l, f, n)
    ref, sr = gpu_ctx.table(p)
    old = os.environ.get("ERATO_GPU_SCATTER")
    os.environ["ERATO_GPU_SCATTER"] = "genbin"
    try:
        got, sg = gpu_ctx.table(p)
    finally:
        if old is None:
            del os.environ["ERATO_GPU_SCATTER"]
        else:
            os.environ["ERATO_GPU_SCATTER"] = old
    assert sg.prime_count == sr.prime_count and np.array_equal(got, ref)


@pytest.mark.parametrize("l,f,n,mode", [(21, (1 << 26) - 2048, 512, None), (22, (1 << 37) - 4096, 256, None),
                                         (22, (1 << 37) - 4096, 256, "genbin"), (20, 1 << 21, 40, None)])
def test_large_prime_invariants_hold(gpu_ctx, l, f, n, mode):
    """ERATO_GPU_CHECK_INVARIANTS (validate_circle_invariants analog,
    src/kernels.cpp:103-179; acceptance.cpp:122-161 'each multiple exactly
    once'): far entries hit inside their bucket's wave, and the records the
    tiles consume equal the admissible multiples of the large primes."""
    import paper_1111_3297_b200 as E
    p = E.validate_params(l, f, n)
    old = os.environ.get("ERATO_GPU_SCATTER")
    if mode:
        os.environ["ERATO_GPU_SCATTER"] = mode
    try:
        st = gpu_ctx.count(p, check_invariants=True)
    finally:
        if mode:
            if old is None:
                del os.environ["ERATO_GPU_SCATTER"]
            else:
                os.environ["ERATO_GPU_SCATTER"] = old
    assert st.large_records > 0
    assert st.prime_count == gpu_ctx.count(p).prime_count


@pytest.mark.parametrize("inject,what", [("1", "admissible multiples"), ("2", "does not hit inside")])
def test_large_prime_invariants_catch_injected_faults(gpu_ctx, inject, what):
    """Fault injection (test_kernels.cpp:391-404 idea): dropping one far entry
    or corrupting its q must be reported as INVARIANT."""
    import paper_1111_3297_b200 as E
    p = E.validate_params(22, (1 << 37) - 4096, 256)
    os.environ["ERATO_GPU_TEST_INJECT"] = inject
    try:
        with pytest.raises(E.Error) as ei:
            gpu_ctx.count(p, check_invariants=True)
    finally:
        del os.environ["ERATO_GPU_TEST_INJECT"]
    assert ei.value.code == E.errc.invariant and what in str(ei.value)


@pytest.mark.parametrize("l,f,n", [(22, (1 << 37) - 4096, 300), (20, 523776, 333)])
def test_pinned_output_pipeline_matches(gpu_ctx, l, f, n):
    """sieve_to_host into pinned memory copies each wave's slice while the
    next waves run (output pipeline); the bytes equal the
    pageable path's single copy."""
    import torch
    import paper_1111_3297_b200 as E
    p = E.validate_params(l, f, n)
    ref, sr = gpu_ctx.table(p)
    pinned = torch.empty(p.table_bytes(), dtype=torch.uint8, pin_memory=True)
    got, sg = gpu_ctx.table(p, out=pinned.numpy())
    assert sg.prime_count == sr.prime_count and np.array_equal(got, ref)


def test_near_2p64_far_path_exact(gpu_ctx):
    """v just below 2^64 with the base-prime cap raised: base primes up to
    2^32 (far entries with D*p past 2^32, fp64 first hits near 2^64).  The
    large-prime invariants hold and 600 Miller-Rabin samples of the table
    agree bit for bit."""
    import paper_1111_3297_b200 as E
    l = 30
    f = (((1 << 64) - 1) >> (l + 1)) - 1
    p = E.validate_params(l, f, 1)
    gpu_ctx.set_max_base_pairs(1 << 28)
    try:
        st = gpu_ctx.count(p, check_invariants=True)
        g, st2 = gpu_ctx.table(p)
    finally:
        gpu_ctx.set_max_base_pairs(1 << 27)
    assert st.prime_count == st2.prime_count and st.large_records > 0
    rng = np.random.default_rng(7)
    for j in rng.integers(0, p.table_bits(), 600):
        j = int(j)
        assert ((int(g[j >> 3]) >> (j & 7)) & 1) == (0 if miller_rabin(p.u + 2 * j) else 1)


def test_random_large_geometries_invariants_and_mr(gpu_ctx):
    """Seeded random (l, f, n) over the whole range up to v < 2^64 (tile
    sizes, wave counts, ML/far splits and bucket rings all vary): the
    large-prime invariants hold and Miller-Rabin samples of every table agree."""
    import paper_1111_3297_b200 as E
    rng = random.Random(20261020)
    gpu_ctx.set_max_base_pairs(1 << 28)
    ran = 0
    try:
        for _ in range(12):
            l = rng.randint(12, 30)
            nmax = max(1, min(1 << 12, (1 << 31) >> l))  # tables of at most 2^31 bits
            n = rng.randint(1, nmax)
            fmax = (((1 << 64) - 1) >> (l + 1)) - n
            f = rng.randint(max(1, fmax >> rng.randint(0, 40)), fmax)
            try:
                p = E.validate_params(l, f, n)
            except E.Error:
                continue
            st = gpu_ctx.count(p, check_invariants=True)
            g, st2 = gpu_ctx.table(p)
            assert st.prime_count == st2.prime_count
            ran += 1
            for j in np.random.default_rng(l * 1000 + n).integers(0, p.table_bits(), 100):
                j = int(j)
                assert ((int(g[j >> 3]) >> (j & 7)) & 1) == (0 if miller_rabin(p.u + 2 * j) else 1), (l, f, n, j)
    finally:
        gpu_ctx.set_max_base_pairs(1 << 27)
    assert ran >= 10


@pytest.mark.parametrize("l,f,n", [(22, (1 << 37) - 4096, 300), (21, (1 << 26) - 2048, 300), (20, 1 << 21, 60)])
def test_mod210_record_skipping_matches_mod30(gpu_ctx, l, f, n):
    """(Legacy structures, ERATO_GPU_LARGE=legacy.)  Large primes may skip their multiples whose cofactor 7 divides (mod-210
    far entries / ML states; those numbers are marked by the pattern of 7).
    Every combination — both off (pure mod-30), default, both forced on —
    gives the same table, and the large-prime invariants (records consumed ==
    admissible multiples, counted coprime-210 where skipped) hold."""
    import paper_1111_3297_b200 as E
    p = E.validate_params(l, f, n)
    results = []
    for env in ({"ERATO_GPU_FAR7": "0", "ERATO_GPU_ML7": "0"}, {}, {"ERATO_GPU_ML7": "1"}):
        old = {k: os.environ.get(k) for k in ("ERATO_GPU_FAR7", "ERATO_GPU_ML7", "ERATO_GPU_LARGE")}
        os.environ.update(env)
        os.environ["ERATO_GPU_LARGE"] = "legacy"  # (the mod-30/210 states of the round-1/2 structures)
        try:
            st = gpu_ctx.count(p, check_invariants=True)
            t, _ = gpu_ctx.table(p)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        results.append((st.prime_count, sha(t), st.large_records))
    assert len({(c, h) for c, h, _ in results}) == 1
    if l >= 21:  # fewer records are consumed when multiples of 7 are skipped
        assert results[2][2] < results[0][2]


@pytest.mark.parametrize("l,f,n", [(22, (1 << 37) - 4096, 700), (21, (1 << 26) - 2048, 300), (20, 1 << 21, 60),
                                   (22, (1 << 37) - 4096, 37)])
def test_large_prime_path_variants_identical(gpu_ctx, l, f, n):
    """The default large-prime pipeline — table-driven mod-30030 wheel walks
    (k_ml_walk per wave, k_far_walk per window of waves) and one partition by
    tile per wave (k_wave_sort) — gives the same table as every other wheel
    modulus, as the legacy structures it replaced (mod-30/210 states, the
    sorting ML scatter, the per-wave far bucket ring), with a far class
    starting elsewhere, with one or many windows per run, and with the
    partition of a wave's far records early (default), beside or after its ML
    walk; the large-prime invariants hold on each, and a finer wheel makes
    fewer records."""
    import paper_1111_3297_b200 as E
    p = E.validate_params(l, f, n)
    keys = ("ERATO_GPU_LARGE", "ERATO_GPU_WHEEL", "ERATO_GPU_FAR_DIV", "ERATO_GPU_FAR_WINDOW", "ERATO_GPU_FAR7",
            "ERATO_GPU_ML7", "ERATO_GPU_EARLY_SORT", "ERATO_GPU_SORT_STREAM")
    results, records = [], {}
    for env in ({}, {"ERATO_GPU_WHEEL": "30"}, {"ERATO_GPU_WHEEL": "210"}, {"ERATO_GPU_WHEEL": "2310"},
                {"ERATO_GPU_LARGE": "legacy"}, {"ERATO_GPU_LARGE": "legacy", "ERATO_GPU_FAR7": "0", "ERATO_GPU_ML7": "0"},
                {"ERATO_GPU_FAR_DIV": "8", "ERATO_GPU_FAR_WINDOW": "2"}, {"ERATO_GPU_FAR_WINDOW": "1"},
                {"ERATO_GPU_EARLY_SORT": "0"}, {"ERATO_GPU_EARLY_SORT": "0", "ERATO_GPU_SORT_STREAM": "0"}):
        old = {k: os.environ.get(k) for k in keys}
        os.environ.update(env)
        try:
            st = gpu_ctx.count(p, check_invariants=True)
            t, _ = gpu_ctx.table(p)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        results.append((st.prime_count, sha(t)))
        if not env or "ERATO_GPU_WHEEL" in env:
            records[int(env.get("ERATO_GPU_WHEEL", "30030"))] = st.large_records
            assert st.wheel == int(env.get("ERATO_GPU_WHEEL", "30030"))
        assert st.far_records <= st.large_records
    assert len(set(results)) == 1, results
    if l >= 21:
        assert records[30030] < records[2310] < records[210] < records[30]


@pytest.mark.parametrize("l", [10, 13, 14])
def test_few_tiles_large_primes_vs_reference(gpu_ctx, reference, l):
    """Runs of 1..33 segments (a handful of small tiles per wave, one wave, a
    far window of one wave) whose base primes are far above the tile: the ML
    class may be empty (every large prime is a far prime), the far bucket tiny,
    the last wave ragged.  Tables and counts against the reference run_sieve,
    with the large-prime invariants on."""
    import paper_1111_3297_b200 as E
    for n in (1, 2, 3, 5, 8, 17, 33):
        for f in ((1 << 30) + 12345, 987654321):
            p = E.validate_params(l, f, n)
            t, st = gpu_ctx.table(p)
            rt, rc, _ = reference.run_sieve(l, f, n, table=True)
            assert st.prime_count == rc and np.array_equal(t, rt), (l, f, n)
            assert gpu_ctx.count(p, check_invariants=True).prime_count == rc


@pytest.mark.parametrize("limit", [4096, 92681, 1049087, 16777471, 1073741839])
def test_base_prime_list_equals_reference_simple_sieve(reference, limit):
    """The device base-prime list (odd primes <= isqrt(v) of cfg1..cfg5),
    element for element against the reference's simple_sieve
    (src/oracle.cpp:8-23, the list build_base uses, src/base.cpp:23)."""
    import paper_1111_3297_b200 as E
    got = E.erato.base_primes(limit)
    ref = reference.simple_sieve(limit)
    ref = ref[ref > 2]
    assert len(got) == len(ref) and np.array_equal(got, ref)
