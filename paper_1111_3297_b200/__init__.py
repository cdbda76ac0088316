"""B200-native segmented odd-only sieve of Eratosthenes — drop-in for the
`run_sieve` path of the erato reference (arxiv 1111.3297, Járai & Vatai).

The compute lives in liberato_gpu.so (sm_100a CUDA behind the C ABI of
include/erato_gpu.h); this package is the host-side mirror of the reference
interface.  See DESIGN.md.
"""
from .erato import (  # noqa: F401
    ALLOW_OVERLAP, TEST_MODE, Context, Error, FileSink, MultiGPU, NullSink, PrimeCollectSink, RunOptions, RunStats,
    SegmentSink, SieveParams, TableSink, context, decompose_index, device_count, errc, errc_name,
    extract_primes, first_offset, index_to_number, isqrt, number_to_index, params_from_midpoint, run_sieve,
    shard, table_filename, validate_params, write_table,
)
