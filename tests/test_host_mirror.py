"""The Python mirror of the reference interface (paper_1111_3297_b200.erato),
host-side parts only (no GPU): SieveParams geometry, index helpers, sinks."""
import numpy as np
import pytest


def test_sieveparams_geometry(lib):
    import paper_1111_3297_b200 as E
    p = E.validate_params(10, 2048, 4)
    assert (p.u, p.v) == (4194305, 4202496)
    assert p.segment_bits() == 1024 and p.table_bits() == 4096
    assert p.segment_bytes() == 128 and p.table_bytes() == 512
    assert p.first_index() == 2048 << 10
    # test_params.cpp:47-57
    assert E.index_to_number(p, 0) == 4194305
    assert E.number_to_index(p, 4194305 + 2 * 5) == 5
    with pytest.raises(E.Error):
        E.number_to_index(p, 4194306)
    with pytest.raises(E.Error):
        E.index_to_number(p, 4096)
    assert E.decompose_index(p, 3 * 1024 + 17) == (3, 17)


def test_prime_collect_sink_segment_logic(lib, restated):
    """PrimeCollectSink turns clear bits into u + 2j (driver.cpp:65-81); fed
    with oracle segments here, GPU segments in the gpu tests."""
    import paper_1111_3297_b200 as E
    p = E.validate_params(10, 6, 2)
    t, c = restated.bit_table(10, 6, 2)
    sink = E.PrimeCollectSink()
    for k in range(p.n):
        sink.on_segment(t[k * p.segment_bytes():(k + 1) * p.segment_bytes()], k, p)
    primes = sink.primes()
    assert len(primes) == c
    assert primes[0] == 12289  # test_driver.cpp:88-102: u = 12289 is prime
    assert all(all(int(x) % d for d in range(3, 200, 2) if d * d <= int(x)) for x in primes[:50])


def test_table_sink_concatenates(lib, restated):
    import paper_1111_3297_b200 as E
    p = E.validate_params(10, 2048, 4)
    t, _ = restated.bit_table(10, 2048, 4)
    sink = E.TableSink()
    for k in range(4):
        sink.on_segment(t[k * 128:(k + 1) * 128], k, p)
    assert np.array_equal(sink.bytes(), t)
