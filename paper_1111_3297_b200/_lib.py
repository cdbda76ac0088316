"""ctypes binding of the C ABI in include/erato_gpu.h (liberato_gpu.so, sm_100a).

The product path has no CPU fallback: if the in-tree extension is missing the
import fails loudly, and every compute entry point returns NO_DEVICE when no
CUDA device is visible.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("ERATO_GPU_SO") or os.path.join(_PKG, "liberato_gpu.so")

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)

# every symbol declared in include/erato_gpu.h
EXPORTS = (
    "erato_gpu_validate", "erato_gpu_f_from_midpoint", "erato_gpu_isqrt", "erato_gpu_first_offset",
    "erato_gpu_table_filename", "erato_gpu_errc_name", "erato_gpu_last_error", "erato_gpu_create",
    "erato_gpu_destroy", "erato_gpu_device_count", "erato_gpu_run", "erato_gpu_sieve_to_host",
    "erato_gpu_count", "erato_gpu_write_table", "erato_gpu_shard", "erato_gpu_extract_primes",
    "erato_gpu_first_hit", "erato_gpu_set_max_base_pairs", "erato_gpu_run_to_sink",
    "erato_gpu_multi_create", "erato_gpu_multi_destroy", "erato_gpu_multi_uses_nccl",
    "erato_gpu_multi_count", "erato_gpu_multi_write_table", "erato_gpu_base_primes", "erato_gpu_wheel_deltas",
)

COUNT_OVERFLOW = (1 << 64) - 1  # ERATO_GPU_COUNT_OVERFLOW

# int (*erato_gpu_sink_fn)(void* user, const uint8_t* bytes, uint64_t offset, uint64_t nbytes)
SINK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint8), C.c_uint64, C.c_uint64)


class Stats(C.Structure):
    _fields_ = [
        ("prime_count", C.c_uint64), ("segments", C.c_uint64),
        ("init_s", C.c_double), ("small_s", C.c_double), ("large_s", C.c_double),
        ("output_s", C.c_double), ("total_s", C.c_double),
        ("base_primes", C.c_uint64), ("tiles", C.c_uint64),
        ("log_tile", C.c_uint32), ("waves", C.c_uint32),
        ("kernel_launches", C.c_uint32), ("retries", C.c_uint32),
        ("gen_s", C.c_double), ("bin_s", C.c_double), ("large_records", C.c_uint64),
        ("masks_s", C.c_double), ("medium_primes", C.c_uint64), ("ml_primes", C.c_uint64),
        ("far_primes", C.c_uint64), ("skip7", C.c_uint32), ("wheel", C.c_uint32),
        ("far_records", C.c_uint64), ("walk_s", C.c_double), ("far_windows", C.c_uint32), ("reserved1", C.c_uint32),
    ]


_lib = None


def load(path: str = SO_PATH):
    """Load liberato_gpu.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not built: run `python -m paper_1111_3297_b200.build` "
            "(the sieve has no CPU fallback)")
    L = C.CDLL(path)
    L.erato_gpu_validate.restype = C.c_int
    L.erato_gpu_validate.argtypes = [C.c_uint, C.c_uint64, C.c_uint64, C.c_uint, u64p, u64p]
    L.erato_gpu_f_from_midpoint.restype = C.c_int
    L.erato_gpu_f_from_midpoint.argtypes = [C.c_uint, C.c_uint, C.c_uint64, C.c_uint, u64p]
    L.erato_gpu_isqrt.restype = C.c_uint64
    L.erato_gpu_isqrt.argtypes = [C.c_uint64]
    L.erato_gpu_first_offset.restype = C.c_uint32
    L.erato_gpu_first_offset.argtypes = [C.c_uint32, C.c_uint, C.c_uint64]
    L.erato_gpu_first_hit.restype = C.c_int
    L.erato_gpu_first_hit.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, u64p, C.POINTER(C.c_uint)]
    L.erato_gpu_table_filename.restype = C.c_size_t
    L.erato_gpu_table_filename.argtypes = [C.c_uint, C.c_uint64, C.c_uint64, C.c_char_p, C.c_size_t]
    L.erato_gpu_errc_name.restype = C.c_char_p
    L.erato_gpu_errc_name.argtypes = [C.c_int]
    L.erato_gpu_last_error.restype = C.c_char_p
    L.erato_gpu_last_error.argtypes = []
    L.erato_gpu_create.restype = C.c_int
    L.erato_gpu_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    L.erato_gpu_destroy.restype = None
    L.erato_gpu_destroy.argtypes = [C.c_void_p]
    L.erato_gpu_set_max_base_pairs.restype = C.c_int
    L.erato_gpu_set_max_base_pairs.argtypes = [C.c_void_p, C.c_uint64]
    L.erato_gpu_device_count.restype = C.c_int
    L.erato_gpu_device_count.argtypes = []
    L.erato_gpu_run.restype = C.c_int
    L.erato_gpu_run.argtypes = [C.c_void_p, C.c_uint, C.c_uint64, C.c_uint64, C.c_uint, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Stats)]
    L.erato_gpu_sieve_to_host.restype = C.c_int
    L.erato_gpu_sieve_to_host.argtypes = [C.c_void_p, C.c_uint, C.c_uint64, C.c_uint64, C.c_uint, u8p,
                                          C.c_size_t, C.POINTER(Stats)]
    L.erato_gpu_count.restype = C.c_int
    L.erato_gpu_count.argtypes = [C.c_void_p, C.c_uint, C.c_uint64, C.c_uint64, C.c_uint, u64p,
                                  C.POINTER(Stats)]
    L.erato_gpu_write_table.restype = C.c_int
    L.erato_gpu_write_table.argtypes = [C.c_void_p, C.c_char_p, C.c_uint, C.c_uint64, C.c_uint64,
                                        C.c_uint64, C.c_uint64, C.c_uint, C.c_char_p, C.c_size_t,
                                        C.POINTER(Stats)]
    L.erato_gpu_wheel_deltas.restype = C.c_size_t
    L.erato_gpu_wheel_deltas.argtypes = [C.c_uint32, u8p, C.c_size_t]
    L.erato_gpu_shard.restype = None
    L.erato_gpu_shard.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, u64p, u64p]
    L.erato_gpu_extract_primes.restype = C.c_int
    L.erato_gpu_extract_primes.argtypes = [C.c_void_p, C.c_uint, C.c_uint64, C.c_uint64, C.c_uint,
                                           u64p, C.c_uint64, u64p]
    L.erato_gpu_run_to_sink.restype = C.c_int
    L.erato_gpu_run_to_sink.argtypes = [C.c_void_p, C.c_uint, C.c_uint64, C.c_uint64, C.c_uint, SINK_FN,
                                        C.c_void_p, C.POINTER(Stats)]
    L.erato_gpu_multi_create.restype = C.c_int
    L.erato_gpu_multi_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]
    L.erato_gpu_multi_destroy.restype = None
    L.erato_gpu_multi_destroy.argtypes = [C.c_void_p]
    L.erato_gpu_multi_uses_nccl.restype = C.c_int
    L.erato_gpu_multi_uses_nccl.argtypes = [C.c_void_p]
    L.erato_gpu_multi_count.restype = C.c_int
    L.erato_gpu_multi_count.argtypes = [C.c_void_p, C.c_uint, C.c_uint64, C.c_uint64, C.c_uint, u64p,
                                        C.POINTER(Stats)]
    L.erato_gpu_multi_write_table.restype = C.c_int
    L.erato_gpu_multi_write_table.argtypes = [C.c_void_p, C.c_char_p, C.c_uint, C.c_uint64, C.c_uint64, C.c_uint,
                                              C.c_char_p, C.c_size_t, u64p, C.POINTER(Stats)]
    L.erato_gpu_base_primes.restype = C.c_int
    L.erato_gpu_base_primes.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint32), C.c_uint64, u64p]
    _lib = L
    return L
