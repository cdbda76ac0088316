"""ctypes front-end for the two CPU oracles — TEST INFRASTRUCTURE ONLY.

* ``Restated``  — oracle/_build/liberato_oracle.so, our plain-C restatement of
  the reference semantics (erato_oracle.c; each function cites the reference
  file:line it follows).
* ``Reference`` — oracle/_ref/liberato_ref.so, the UNMODIFIED reference library
  (/root/reference/proj/src/*.cpp compiled in place by oracle/Makefile) behind a
  small C shim (ref_shim.cpp).  Present in this container and, because the
  built .so travels with the repo snapshot, on the GPU box too.

Neither is ever called by the product path (paper_1111_3297_b200/).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_SO = os.path.join(HERE, "_build", "liberato_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "liberato_ref.so")

ERRC_NAMES = [
    "OK", "L_OUT_OF_RANGE", "F_ZERO_OR_OVERLAP", "N_OUT_OF_RANGE", "OVERFLOW",
    "INDEX_OUT_OF_RANGE", "NOT_ADMISSIBLE", "ALLOC_LIMIT", "LIMIT_TOO_LARGE",
    "RANGE_TOO_LARGE", "IO_ERROR",
]

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str = ""):
        self.code = code
        self.name = ERRC_NAMES[code] if 0 <= code < len(ERRC_NAMES) else f"E{code}"
        super().__init__(f"{self.name} {where}".strip())


def build(reference: bool = True) -> None:
    """Compile the restated oracle (always) and the reference (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if reference and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "all"], check=True)
        # the INTEGRATION.md binding test (needs liberato_gpu.so built first)
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_1111_3297_b200", "liberato_gpu.so")):
            subprocess.run(["make", "-s", "-C", HERE, "binding"], check=True)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class Restated:
    """Our plain-C restatement (erato_oracle.c)."""

    def __init__(self, path: str = RESTATED_SO):
        if not os.path.exists(path):
            build(reference=False)
        L = C.CDLL(path)
        L.eo_isqrt.restype = C.c_uint64
        L.eo_isqrt.argtypes = [C.c_uint64]
        L.eo_validate.restype = C.c_int
        L.eo_validate.argtypes = [C.c_uint, C.c_uint64, C.c_uint64, C.c_int, C.c_int, u64p, u64p]
        L.eo_params_from_midpoint.restype = C.c_int
        L.eo_params_from_midpoint.argtypes = [C.c_uint, C.c_uint, C.c_uint64, C.c_int, u64p]
        L.eo_first_offset.restype = C.c_uint32
        L.eo_first_offset.argtypes = [C.c_uint32, C.c_uint, C.c_uint64]
        L.eo_simple_sieve.restype = C.c_uint64
        L.eo_simple_sieve.argtypes = [C.c_uint64, u32p, C.c_uint64]
        L.eo_count_zeros.restype = C.c_uint64
        L.eo_count_zeros.argtypes = [u8p, C.c_uint64]
        L.eo_bit_table.restype = C.c_int
        L.eo_bit_table.argtypes = [C.c_uint, C.c_uint64, C.c_uint64, C.c_int, C.c_int, u8p, u64p]
        self.L = L

    def isqrt(self, x: int) -> int:
        return self.L.eo_isqrt(x)

    def validate(self, l, f, n, test_mode=False, allow_overlap=False):
        u, v = C.c_uint64(), C.c_uint64()
        rc = self.L.eo_validate(l, f, n, int(test_mode), int(allow_overlap), C.byref(u), C.byref(v))
        if rc:
            raise OracleError(rc, f"l={l} f={f} n={n}")
        return u.value, v.value

    def params_from_midpoint(self, e, l, n, test_mode=False) -> int:
        f = C.c_uint64()
        rc = self.L.eo_params_from_midpoint(e, l, n, int(test_mode), C.byref(f))
        if rc:
            raise OracleError(rc, f"e={e} l={l} n={n}")
        return f.value

    def first_offset(self, p, l, f) -> int:
        return self.L.eo_first_offset(p, l, f)

    def simple_sieve(self, limit: int) -> np.ndarray:
        cnt = self.L.eo_simple_sieve(limit, None, 0)
        out = np.zeros(max(cnt, 1), dtype=np.uint32)
        self.L.eo_simple_sieve(limit, _ptr(out, u32p), cnt)
        return out[:cnt]

    def bit_table(self, l, f, n, test_mode=False, allow_overlap=False):
        out = np.zeros((n << l) // 8, dtype=np.uint8)
        cnt = C.c_uint64()
        rc = self.L.eo_bit_table(l, f, n, int(test_mode), int(allow_overlap), _ptr(out, u8p), C.byref(cnt))
        if rc:
            raise OracleError(rc, f"l={l} f={f} n={n}")
        return out, cnt.value

    def count_zeros(self, table: np.ndarray, nbits: int) -> int:
        return self.L.eo_count_zeros(_ptr(table, u8p), nbits)


class Reference:
    """The unmodified reference library (oracle/_ref/liberato_ref.so)."""

    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(path)
        L.ref_validate_params.restype = C.c_int
        L.ref_validate_params.argtypes = [C.c_uint, C.c_uint64, C.c_uint64, C.c_int, u64p, u64p]
        L.ref_params_from_midpoint.restype = C.c_int
        L.ref_params_from_midpoint.argtypes = [C.c_uint, C.c_uint, C.c_uint64, C.c_int, u64p]
        L.ref_first_offset.restype = C.c_uint32
        L.ref_first_offset.argtypes = [C.c_uint32, C.c_uint, C.c_uint64]
        L.ref_wheel_align.restype = C.c_int
        L.ref_wheel_align.argtypes = [C.c_uint32, C.c_uint32, C.c_uint, C.c_uint64, u32p, C.POINTER(C.c_uint)]
        L.ref_isqrt.restype = C.c_uint64
        L.ref_isqrt.argtypes = [C.c_uint64]
        L.ref_simple_sieve.restype = C.c_uint64
        L.ref_simple_sieve.argtypes = [C.c_uint64, u32p, C.c_uint64]
        L.ref_run_sieve.restype = C.c_int
        L.ref_run_sieve.argtypes = [C.c_uint, C.c_uint64, C.c_uint64, C.c_int, u8p, u64p, C.POINTER(C.c_double)]
        L.ref_write_table.restype = C.c_int
        L.ref_write_table.argtypes = [C.c_char_p, C.c_uint, C.c_uint64, C.c_uint64, C.c_int, C.c_char_p, C.c_uint64, u64p]
        L.ref_oracle_bit_table.restype = C.c_int
        L.ref_oracle_bit_table.argtypes = [C.c_uint, C.c_uint64, C.c_uint64, C.c_int, u8p]
        L.ref_f0_table.restype = C.c_int
        L.ref_f0_table.argtypes = [C.c_uint, C.c_uint64, C.c_int, u8p, u64p]
        L.ref_extract_primes.restype = C.c_int
        L.ref_extract_primes.argtypes = [C.c_uint, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(u64p), u64p]
        L.ref_free_u64.restype = None
        L.ref_free_u64.argtypes = [u64p]
        L.ref_last_error.restype = C.c_char_p
        self.L = L

    def _chk(self, rc, where=""):
        if rc:
            raise OracleError(rc, (where + " " + self.L.ref_last_error().decode()).strip())

    def validate(self, l, f, n, test_mode=False):
        u, v = C.c_uint64(), C.c_uint64()
        self._chk(self.L.ref_validate_params(l, f, n, int(test_mode), C.byref(u), C.byref(v)))
        return u.value, v.value

    def params_from_midpoint(self, e, l, n, test_mode=False) -> int:
        f = C.c_uint64()
        self._chk(self.L.ref_params_from_midpoint(e, l, n, int(test_mode), C.byref(f)))
        return f.value

    def first_offset(self, p, l, f) -> int:
        return self.L.ref_first_offset(p, l, f)

    def wheel_align(self, p, q0, l, f):
        q, s = C.c_uint32(), C.c_uint()
        self.L.ref_wheel_align(p, q0, l, f, C.byref(q), C.byref(s))
        return q.value, s.value

    def isqrt(self, x):
        return self.L.ref_isqrt(x)

    def simple_sieve(self, limit: int) -> np.ndarray:
        cnt = self.L.ref_simple_sieve(limit, None, 0)
        out = np.zeros(max(cnt, 1), dtype=np.uint32)
        self.L.ref_simple_sieve(limit, _ptr(out, u32p), cnt)
        return out[:cnt]

    def run_sieve(self, l, f, n, test_mode=False, table=True):
        """reference run_sieve with TableSink (table=True) or NullSink; returns (table|None, count, phases)."""
        cnt = C.c_uint64()
        ph = (C.c_double * 5)()
        out = np.zeros((n << l) // 8, dtype=np.uint8) if table else None
        self._chk(self.L.ref_run_sieve(l, f, n, int(test_mode), _ptr(out, u8p) if table else None,
                                       C.byref(cnt), ph), f"l={l} f={f} n={n}")
        return out, cnt.value, list(ph)

    def write_table(self, out_dir, l, f, n, test_mode=False):
        buf = C.create_string_buffer(4096)
        cnt = C.c_uint64()
        self._chk(self.L.ref_write_table(out_dir.encode(), l, f, n, int(test_mode), buf, 4096, C.byref(cnt)))
        return buf.value.decode(), cnt.value

    def extract_primes(self, l, f, n, test_mode=False) -> np.ndarray:
        """run_sieve with the reference PrimeCollectSink (driver.cpp:53-57, :65-81)."""
        cnt = C.c_uint64()
        buf = u64p()
        self._chk(self.L.ref_extract_primes(l, f, n, int(test_mode), C.byref(buf), C.byref(cnt)))
        try:
            return np.ctypeslib.as_array(buf, shape=(max(cnt.value, 1),))[:cnt.value].copy()
        finally:
            self.L.ref_free_u64(buf)

    def oracle_bit_table(self, l, f, n, test_mode=False) -> np.ndarray:
        out = np.zeros((n << l) // 8, dtype=np.uint8)
        self._chk(self.L.ref_oracle_bit_table(l, f, n, int(test_mode), _ptr(out, u8p)))
        return out

    def f0_table(self, l, n, test_mode=False, table=True):
        cnt = C.c_uint64()
        out = np.zeros((n << l) // 8, dtype=np.uint8) if table else None
        self._chk(self.L.ref_f0_table(l, n, int(test_mode), _ptr(out, u8p) if table else None, C.byref(cnt)))
        return out, cnt.value
