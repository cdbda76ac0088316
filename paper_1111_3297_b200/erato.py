"""Host-side mirror of the reference erato API for the sieve path, on the GPU.

Same names, argument meaning and error behaviour as the reference library
(/root/reference/proj/include/erato/{params,driver}.hpp), so code written
against ``erato::run_sieve`` ports line by line:

    reference (C++)                               here (Python, GPU underneath)
    erato::validate_params(l, f, n, test)         validate_params(l, f, n, test_mode)
    erato::params_from_midpoint(e, l, n)          params_from_midpoint(e, l, n)
    erato::run_sieve(params, sink, opt)           run_sieve(params, sink, opt)
    NullSink / FileSink / TableSink / PrimeCollectSink   same classes
    erato::write_table(dir, params)               write_table(dir, params)
    erato::table_filename(params)                 table_filename(params)
    erato::extract_primes(seg, t, params)         extract_primes(params)  (whole run, on device)
    erato::Error / errc                           Error / errc

All compute goes through liberato_gpu.so (the C ABI in include/erato_gpu.h);
there is no CPU path.  Extension: ``allow_overlap=True`` accepts u^2 <= v
(incl. f = 0) with the SURVEY.md §8c convention (1 and primes stay 0); by
default f = 0 is rejected with F_ZERO_OR_OVERLAP exactly like the reference.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import tempfile
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _lib

TEST_MODE = 0x1
ALLOW_OVERLAP = 0x2
CHECK_INVARIANTS = 0x200  # device checks of the large-prime bookkeeping (erato_gpu.h)

kMinLogSeg = 10
kMinLogSegTest = 4
kMaxLogSeg = 30
kDefaultMaxBasePairs = 1 << 27


class errc(enum.IntEnum):
    """erato::errc (params.hpp:18-29), same ordinals."""
    l_out_of_range = 0
    f_zero_or_overlap = 1
    n_out_of_range = 2
    overflow = 3
    index_out_of_range = 4
    not_admissible = 5
    alloc_limit = 6
    limit_too_large = 7
    range_too_large = 8
    io_error = 9
    # GPU runtime errors (no reference counterpart)
    cuda_error = 63
    no_device = 64
    invalid_argument = 65
    invariant = 66


_ERRC_NAMES = {
    errc.l_out_of_range: "L_OUT_OF_RANGE", errc.f_zero_or_overlap: "F_ZERO_OR_OVERLAP",
    errc.n_out_of_range: "N_OUT_OF_RANGE", errc.overflow: "OVERFLOW",
    errc.index_out_of_range: "INDEX_OUT_OF_RANGE", errc.not_admissible: "NOT_ADMISSIBLE",
    errc.alloc_limit: "ALLOC_LIMIT", errc.limit_too_large: "LIMIT_TOO_LARGE",
    errc.range_too_large: "RANGE_TOO_LARGE", errc.io_error: "IO_ERROR",
    errc.cuda_error: "CUDA_ERROR", errc.no_device: "NO_DEVICE", errc.invalid_argument: "INVALID_ARGUMENT",
    errc.invariant: "INVARIANT",
}

PARAM_ERRORS = (errc.l_out_of_range, errc.f_zero_or_overlap, errc.n_out_of_range, errc.overflow,
                errc.index_out_of_range)


def errc_name(c: errc) -> str:
    return _ERRC_NAMES.get(errc(c), "UNKNOWN")


class Error(RuntimeError):
    """erato::Error (params.hpp:31-41): what() = "NAME: message"."""

    def __init__(self, code: errc, msg: str):
        self.code = errc(code)
        super().__init__(f"{errc_name(self.code)}: {msg}")

    def is_param_error(self) -> bool:
        return self.code in PARAM_ERRORS


def _check(rc: int) -> None:
    if rc:
        L = _lib.load()
        raw = L.erato_gpu_last_error().decode()
        msg = raw.split(": ", 1)[1] if ": " in raw else raw
        raise Error(errc(rc - 1), msg)


def _flags(test_mode: bool, allow_overlap: bool) -> int:
    return (TEST_MODE if test_mode else 0) | (ALLOW_OVERLAP if allow_overlap else 0)


@dataclass(frozen=True)
class SieveParams:
    """erato::SieveParams (params.hpp:43-56)."""
    l: int
    f: int
    n: int
    u: int
    v: int
    test_mode: bool = False
    allow_overlap: bool = False

    def segment_bits(self) -> int:
        return 1 << self.l

    def table_bits(self) -> int:
        return self.n << self.l

    def segment_bytes(self) -> int:
        return 1 << (self.l - 3)

    def table_bytes(self) -> int:
        return self.n << (self.l - 3)

    def first_index(self) -> int:
        return self.f << self.l

    @property
    def flags(self) -> int:
        return _flags(self.test_mode, self.allow_overlap)


def validate_params(l: int, f: int, n: int, test_mode: bool = False, allow_overlap: bool = False) -> SieveParams:
    """validate_params (src/params.cpp:23-44)."""
    L = _lib.load()
    u, v = C.c_uint64(), C.c_uint64()
    if not (0 <= l < 2**32 and 0 <= f < 2**64 and 0 <= n < 2**64):
        raise Error(errc.overflow, "argument out of 64-bit range")
    _check(L.erato_gpu_validate(l, f, n, _flags(test_mode, allow_overlap), C.byref(u), C.byref(v)))
    return SieveParams(l, f, n, u.value, v.value, test_mode, allow_overlap)


def params_from_midpoint(e: int, l: int, n: int, test_mode: bool = False) -> int:
    """params_from_midpoint (src/params.cpp:64-77), decimal 10^e."""
    L = _lib.load()
    f = C.c_uint64()
    _check(L.erato_gpu_f_from_midpoint(e, l, n, _flags(test_mode, False), C.byref(f)))
    return f.value


def isqrt(x: int) -> int:
    return _lib.load().erato_gpu_isqrt(x)


def first_offset(p: int, l: int, f: int) -> int:
    """Lemma 1 (src/wheel.cpp:43-47)."""
    return _lib.load().erato_gpu_first_offset(p, l, f)


def index_to_number(p: SieveParams, j: int) -> int:
    if not 0 <= j < p.table_bits():
        raise Error(errc.index_out_of_range, f"bit index {j}")
    return p.u + 2 * j


def number_to_index(p: SieveParams, value: int) -> int:
    if value % 2 == 0 or value < p.u or value > p.v:
        raise Error(errc.index_out_of_range, f"number {value}")
    return (value - p.u) // 2


def decompose_index(p: SieveParams, j: int):
    if not 0 <= j < p.table_bits():
        raise Error(errc.index_out_of_range, f"bit index {j}")
    return j >> p.l, j & (p.segment_bits() - 1)


def table_filename(params: SieveParams) -> str:
    """table_filename (src/driver.cpp:17-20)."""
    return f"erato_l{params.l}_f{params.f}_n{params.n}.bits"


def shard(f: int, n: int, rank: int, world: int):
    """Contiguous segment range of rank `rank`."""
    L = _lib.load()
    fo, no = C.c_uint64(), C.c_uint64()
    L.erato_gpu_shard(f, n, rank, world, C.byref(fo), C.byref(no))
    return fo.value, no.value


@dataclass
class RunStats:
    """RunStats (driver.hpp:24-32) plus GPU facts."""
    prime_count: int = 0
    segments: int = 0
    init_s: float = 0.0
    masks_s: float = 0.0
    medium_s: float = 0.0
    large_s: float = 0.0
    output_s: float = 0.0
    total_s: float = 0.0
    base_primes: int = 0
    tiles: int = 0
    log_tile: int = 0
    waves: int = 0
    kernel_launches: int = 0
    retries: int = 0
    gen_s: float = 0.0
    bin_s: float = 0.0
    large_records: int = 0
    medium_primes: int = 0
    ml_primes: int = 0
    far_primes: int = 0
    skip7: int = 0
    wheel: int = 0
    far_records: int = 0
    walk_s: float = 0.0
    far_windows: int = 0

    @classmethod
    def _from(cls, s: _lib.Stats) -> "RunStats":
        # masks_s: the pattern phase of the tile kernel (with PHASE_TIMING);
        # medium_s: the rest of the tile kernel (medium primes, hit records, count)
        return cls(prime_count=s.prime_count, segments=s.segments, init_s=s.init_s, masks_s=s.masks_s,
                   medium_s=max(0.0, s.small_s - s.masks_s),
                   large_s=s.large_s, output_s=s.output_s, total_s=s.total_s, base_primes=s.base_primes,
                   tiles=s.tiles, log_tile=s.log_tile, waves=s.waves, kernel_launches=s.kernel_launches,
                   retries=s.retries, gen_s=s.gen_s, bin_s=s.bin_s, large_records=s.large_records,
                   medium_primes=s.medium_primes, ml_primes=s.ml_primes, far_primes=s.far_primes,
                   skip7=s.skip7, wheel=s.wheel, far_records=s.far_records, walk_s=s.walk_s,
                   far_windows=s.far_windows)


@dataclass
class RunOptions:
    """RunOptions (driver.hpp:82-89).  `kernels` has no GPU counterpart (no
    multi-backend dispatch); max_base_pairs maps to the ALLOC_LIMIT check."""
    max_base_pairs: int = kDefaultMaxBasePairs
    device: int = 0


class Context:
    """One device context (erato_gpu_ctx): buffers are reused across runs."""

    def __init__(self, device: int = 0):
        L = _lib.load()
        h = C.c_void_p()
        _check(L.erato_gpu_create(device, C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self) -> None:
        if self._h:
            _lib.load().erato_gpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_max_base_pairs(self, n: int) -> None:
        """RunOptions::max_base_pairs (driver.hpp:84); default 2^27."""
        _check(_lib.load().erato_gpu_set_max_base_pairs(self._h, n))

    # ---- raw calls ------------------------------------------------------
    def count(self, params: SieveParams, check_invariants: bool = False) -> RunStats:
        """NullSink run; check_invariants adds the device checks of the
        large-prime path (validate_circle_invariants analog)."""
        st = _lib.Stats()
        cnt = C.c_uint64()
        flags = params.flags | (CHECK_INVARIANTS if check_invariants else 0)
        _check(_lib.load().erato_gpu_count(self._h, params.l, params.f, params.n, flags,
                                           C.byref(cnt), C.byref(st)))
        return RunStats._from(st)

    def table(self, params: SieveParams, out: Optional[np.ndarray] = None):
        nbytes = params.table_bytes()
        if out is None:
            out = np.empty(nbytes, dtype=np.uint8)
        assert out.nbytes >= nbytes and out.flags["C_CONTIGUOUS"]
        st = _lib.Stats()
        _check(_lib.load().erato_gpu_sieve_to_host(
            self._h, params.l, params.f, params.n, params.flags,
            out.ctypes.data_as(_lib.u8p), out.nbytes, C.byref(st)))
        return out[:nbytes], RunStats._from(st)

    def run_device(self, params: SieveParams, dev_table: int = 0, dev_count: int = 0, stream: int = 0,
                   sync: bool = True) -> RunStats:
        """Sieve into device memory (pointers as ints, e.g. torch data_ptr())."""
        st = _lib.Stats()
        _check(_lib.load().erato_gpu_run(self._h, params.l, params.f, params.n, params.flags,
                                         C.c_void_p(dev_table or None), C.c_void_p(dev_count or None),
                                         C.c_void_p(stream or None), 1 if sync else 0, C.byref(st)))
        return RunStats._from(st)

    def write_table(self, out_dir: str, params: SieveParams, part_f: Optional[int] = None,
                    part_n: Optional[int] = None):
        """FileSink run.  part_f/part_n: one shard of params (erato_gpu_shard),
        pwrite()n at its offset into the shared file; None = the whole table."""
        if part_f is None or part_n is None:
            part_f, part_n = params.f, params.n
        buf = C.create_string_buffer(4096)
        st = _lib.Stats()
        _check(_lib.load().erato_gpu_write_table(self._h, out_dir.encode(), params.l, params.f, params.n,
                                                 part_f, part_n, params.flags, buf, 4096, C.byref(st)))
        return buf.value.decode(), RunStats._from(st)

    def stream(self, params: SieveParams, fn) -> RunStats:
        """erato_gpu_run_to_sink: fn(view, offset) gets the table as ordered
        contiguous byte slices (numpy views valid only during the call)."""
        err = []

        def cb(_user, ptr, offset, nbytes):
            try:
                fn(np.ctypeslib.as_array(ptr, shape=(nbytes,)), offset)
                return 0
            except BaseException as e:  # noqa: BLE001 — re-raised below
                err.append(e)
                return 1

        cfn = _lib.SINK_FN(cb)
        st = _lib.Stats()
        rc = _lib.load().erato_gpu_run_to_sink(self._h, params.l, params.f, params.n, params.flags, cfn, None,
                                               C.byref(st))
        if err:
            raise err[0]
        _check(rc)
        return RunStats._from(st)

    def extract_primes(self, params: SieveParams, cap: Optional[int] = None) -> np.ndarray:
        """One sieve + device compaction; the first call (cap None) learns the
        count, the second only copies the cached list (erato_gpu_extract_primes)."""
        L = _lib.load()
        cnt = C.c_uint64()
        if cap is None:
            _check(L.erato_gpu_extract_primes(self._h, params.l, params.f, params.n, params.flags, None, 0,
                                              C.byref(cnt)))
            cap = cnt.value
        out = np.empty(max(cap, 1), dtype=np.uint64)
        _check(L.erato_gpu_extract_primes(self._h, params.l, params.f, params.n, params.flags,
                                          out.ctypes.data_as(_lib.u64p), cap, C.byref(cnt)))
        return out[:min(cap, cnt.value)]


def base_primes(limit: int, device: int = 0) -> np.ndarray:
    """The device base-prime list: odd primes <= limit, ascending (build_base's
    simple_sieve, src/base.cpp:19-53), as a run computes them."""
    ctx = context(device)
    L = _lib.load()
    cnt = C.c_uint64()
    _check(L.erato_gpu_base_primes(ctx.handle, limit, None, 0, C.byref(cnt)))
    out = np.empty(max(cnt.value, 1), dtype=np.uint32)
    _check(L.erato_gpu_base_primes(ctx.handle, limit, out.ctypes.data_as(C.POINTER(C.c_uint32)), cnt.value,
                                   C.byref(cnt)))
    return out[:cnt.value]


class MultiGPU:
    """erato_gpu_multi: contiguous range shards over several devices, one host
    thread each, counts summed by one ncclAllReduce."""

    def __init__(self, devices):
        devices = list(devices)
        L = _lib.load()
        h = C.c_void_p()
        arr = (C.c_int * len(devices))(*devices)
        _check(L.erato_gpu_multi_create(len(devices), arr, C.byref(h)))
        self._h = h
        self.devices = devices

    @property
    def uses_nccl(self) -> bool:
        return bool(_lib.load().erato_gpu_multi_uses_nccl(self._h))

    def close(self) -> None:
        if self._h:
            _lib.load().erato_gpu_multi_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def count(self, params: SieveParams) -> RunStats:
        st = _lib.Stats()
        cnt = C.c_uint64()
        _check(_lib.load().erato_gpu_multi_count(self._h, params.l, params.f, params.n, params.flags,
                                                 C.byref(cnt), C.byref(st)))
        return RunStats._from(st)

    def write_table(self, out_dir: str, params: SieveParams):
        buf = C.create_string_buffer(4096)
        st = _lib.Stats()
        cnt = C.c_uint64()
        _check(_lib.load().erato_gpu_multi_write_table(self._h, out_dir.encode(), params.l, params.f, params.n,
                                                       params.flags, buf, 4096, C.byref(cnt), C.byref(st)))
        return buf.value.decode(), RunStats._from(st)


_contexts: dict = {}


def context(device: int = 0) -> Context:
    if device not in _contexts:
        _contexts[device] = Context(device)
    return _contexts[device]


def device_count() -> int:
    return _lib.load().erato_gpu_device_count()


# ---- sinks (driver.hpp:34-80) -------------------------------------------
class SegmentSink:
    """on_segment(seg, t, params) is called in order t = 0..n-1 with a
    read-only numpy view of the segment's bytes (LSB-first); finish(params)
    at the end.  The view is valid only during the call."""

    def on_segment(self, seg: np.ndarray, t: int, params: SieveParams) -> None:
        raise NotImplementedError

    def finish(self, params: SieveParams) -> None:
        pass


class NullSink(SegmentSink):
    def on_segment(self, seg, t, params):
        pass


class TableSink(SegmentSink):
    def __init__(self):
        self._parts: List[np.ndarray] = []
        self._bytes: Optional[np.ndarray] = None

    def on_segment(self, seg, t, params):
        self._parts.append(np.array(seg, copy=True))

    def _set_all(self, table: np.ndarray) -> None:
        self._bytes = table

    def bytes(self) -> np.ndarray:
        if self._bytes is None:
            self._bytes = np.concatenate(self._parts) if self._parts else np.zeros(0, np.uint8)
        return self._bytes


class FileSink(SegmentSink):
    """Streams the table to dir/erato_l{l}_f{f}_n{n}.bits (driver.cpp:29-51)."""

    def __init__(self, dir: Optional[str], params: SieveParams):
        self.dir = dir if dir is not None else tempfile.gettempdir()
        os.makedirs(self.dir, exist_ok=True)
        self._path = os.path.join(self.dir, table_filename(params))
        self._fh = None

    def path(self) -> str:
        return self._path

    def on_segment(self, seg, t, params):
        if self._fh is None:
            try:
                self._fh = open(self._path, "wb")
            except OSError as e:
                raise Error(errc.io_error, f"cannot open {self._path}") from e
        self._fh.write(seg.tobytes())

    def finish(self, params):
        if self._fh is not None:
            self._fh.close()
            self._fh = None


class PrimeCollectSink(SegmentSink):
    def __init__(self):
        self._primes: List[np.ndarray] = []

    def on_segment(self, seg, t, params):
        base = params.u + 2 * (t << params.l)
        bits = np.unpackbits(seg, bitorder="little")
        idx = np.flatnonzero(bits == 0).astype(np.uint64)
        vals = np.uint64(base) + np.uint64(2) * idx
        if base == 1:
            vals = vals[vals != 1]
        self._primes.append(vals)

    def primes(self) -> np.ndarray:
        return np.concatenate(self._primes) if self._primes else np.zeros(0, np.uint64)


def run_sieve(params: SieveParams, sink: SegmentSink, opt: Optional[RunOptions] = None) -> RunStats:
    """run_sieve (src/driver.cpp:83-120) on the GPU.

    NullSink: count only (nothing but the count leaves the device).
    FileSink: the device table is written to the file by the C ABI.
    Other sinks: the table comes to host memory once and each segment view
    is handed to on_segment in order t = 0..n-1.
    """
    opt = opt or RunOptions()
    ctx = context(opt.device)
    ctx.set_max_base_pairs(opt.max_base_pairs)
    if isinstance(sink, NullSink):
        stats = ctx.count(params)
    elif isinstance(sink, FileSink):
        path, stats = ctx.write_table(sink.dir, params)
        sink._path = path
    elif isinstance(sink, TableSink):
        table, stats = ctx.table(params)
        sink._set_all(table)
    else:
        # any other sink: the table streams by (wave slices), re-cut into the
        # reference's segments, handed over in order t = 0..n-1
        sb = params.segment_bytes()
        carry = bytearray()
        nxt = [0]

        def on_slice(view, offset):
            carry.extend(view.tobytes())
            while len(carry) >= sb:
                seg = np.frombuffer(bytes(carry[:sb]), dtype=np.uint8)
                del carry[:sb]
                sink.on_segment(seg, nxt[0], params)
                nxt[0] += 1

        stats = ctx.stream(params, on_slice)
        if nxt[0] != params.n or carry:
            raise Error(errc.io_error, f"streamed {nxt[0]} of {params.n} segments")
    sink.finish(params)
    stats.segments = params.n
    return stats


def write_table(dir: str, params: SieveParams, opt: Optional[RunOptions] = None) -> str:
    """write_table (driver.hpp:98-99): sieve the whole run into dir."""
    sink = FileSink(dir, params)
    run_sieve(params, sink, opt)
    return sink.path()


def extract_primes(params: SieveParams, opt: Optional[RunOptions] = None) -> np.ndarray:
    """All primes of the run, ascending (extract_primes, driver.cpp:65-81), on the device."""
    opt = opt or RunOptions()
    return context(opt.device).extract_primes(params)
