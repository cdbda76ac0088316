// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product path).
//
// A C-ABI shim over the UNMODIFIED reference library (erato, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests, the golden-fixture generator and bench.py's reference arm call
// the reference's own run_sieve / validate_params / first_offset through ctypes.
//
// Reference interfaces wrapped (file:line under /root/reference/proj):
//   validate_params        src/params.cpp:23-44
//   params_from_midpoint   src/params.cpp:64-77
//   first_offset           src/wheel.cpp:43-47
//   wheel_align            src/wheel.cpp:60-69
//   simple_sieve           src/oracle.cpp:8-23
//   oracle_bit_table       src/oracle.cpp:25-46
//   run_sieve + TableSink/NullSink/FileSink   src/driver.cpp:83-120, :29-63
//   run_sieve + PrimeCollectSink (extract_primes)   src/driver.cpp:53-57, :65-81
#include <cstdint>
#include <cstring>
#include <string>

#include "erato/driver.hpp"
#include "erato/oracle.hpp"
#include "erato/params.hpp"
#include "erato/wheel.hpp"

namespace {

int code_of(const erato::Error& e) { return 1 + (int)e.code(); }

// phases: init, masks, medium, large, output (seconds)
void put_stats(const erato::RunStats& st, uint64_t* count, double* phases) {
  if (count) *count = st.prime_count;
  if (phases) {
    phases[0] = st.init_s;
    phases[1] = st.masks_s;
    phases[2] = st.medium_s;
    phases[3] = st.large_s;
    phases[4] = st.output_s;
  }
}

thread_local std::string g_last_error;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

const char* ref_errc_name(int code) {
  if (code <= 0) return "OK";
  return erato::errc_name((erato::errc)(code - 1));
}

int ref_validate_params(unsigned l, uint64_t f, uint64_t n, int test_mode, uint64_t* u,
                        uint64_t* v) {
  try {
    auto p = erato::validate_params(l, f, n, test_mode != 0);
    if (u) *u = p.u;
    if (v) *v = p.v;
    return 0;
  } catch (const erato::Error& e) {
    g_last_error = e.what();
    return code_of(e);
  }
}

int ref_params_from_midpoint(unsigned e, unsigned l, uint64_t n, int test_mode, uint64_t* f) {
  try {
    *f = erato::params_from_midpoint(e, l, n, test_mode != 0);
    return 0;
  } catch (const erato::Error& ex) {
    g_last_error = ex.what();
    return code_of(ex);
  }
}

uint32_t ref_first_offset(uint32_t p, unsigned l, uint64_t f) {
  return erato::first_offset(p, l, f);
}

int ref_wheel_align(uint32_t p, uint32_t q0, unsigned l, uint64_t f, uint32_t* q, unsigned* s) {
  auto a = erato::wheel_align(p, q0, l, f);
  *q = a.q;
  *s = a.s;
  return 0;
}

uint64_t ref_isqrt(uint64_t x) { return erato::isqrt(x); }

// Writes up to cap primes <= limit; returns the total count.
uint64_t ref_simple_sieve(uint64_t limit, uint32_t* out, uint64_t cap) {
  auto v = erato::oracle::simple_sieve(limit);
  const uint64_t m = v.size() < cap ? v.size() : cap;
  if (out && m) std::memcpy(out, v.data(), m * sizeof(uint32_t));
  return v.size();
}

// The production path: run_sieve with a TableSink (out != NULL, out must hold
// n*2^(l-3) bytes) or a NullSink (out == NULL).
int ref_run_sieve(unsigned l, uint64_t f, uint64_t n, int test_mode, uint8_t* out,
                  uint64_t* count, double* phases) {
  try {
    const auto params = erato::validate_params(l, f, n, test_mode != 0);
    erato::RunStats st;
    if (out) {
      erato::TableSink sink;
      st = erato::run_sieve(params, sink);
      std::memcpy(out, sink.bytes().data(), sink.bytes().size());
    } else {
      erato::NullSink sink;
      st = erato::run_sieve(params, sink);
    }
    put_stats(st, count, phases);
    return 0;
  } catch (const erato::Error& e) {
    g_last_error = e.what();
    return code_of(e);
  }
}

// FileSink run (write_table); path_out receives the file path.
int ref_write_table(const char* dir, unsigned l, uint64_t f, uint64_t n, int test_mode,
                    char* path_out, uint64_t cap, uint64_t* count) {
  try {
    const auto params = erato::validate_params(l, f, n, test_mode != 0);
    erato::FileSink sink(dir, params);
    auto st = erato::run_sieve(params, sink);
    put_stats(st, count, nullptr);
    std::snprintf(path_out, cap, "%s", sink.path().c_str());
    return 0;
  } catch (const erato::Error& e) {
    g_last_error = e.what();
    return code_of(e);
  }
}

// PrimeCollectSink run (driver.hpp:62-69, driver.cpp:53-57 / :65-81): the
// ascending primes of the run in a new[] buffer (*out, free with
// ref_free_u64), *count = their number.
int ref_extract_primes(unsigned l, uint64_t f, uint64_t n, int test_mode, uint64_t** out, uint64_t* count) {
  try {
    const auto params = erato::validate_params(l, f, n, test_mode != 0);
    erato::PrimeCollectSink sink;
    erato::run_sieve(params, sink);
    const auto& v = sink.primes();
    *out = new uint64_t[v.size() ? v.size() : 1];
    if (!v.empty()) std::memcpy(*out, v.data(), v.size() * sizeof(uint64_t));
    *count = v.size();
    return 0;
  } catch (const erato::Error& e) {
    g_last_error = e.what();
    return code_of(e);
  }
}

void ref_free_u64(uint64_t* p) { delete[] p; }

// The reference's brute-force oracle (v <= 2^40).
int ref_oracle_bit_table(unsigned l, uint64_t f, uint64_t n, int test_mode, uint8_t* out) {
  try {
    const auto params = erato::validate_params(l, f, n, test_mode != 0);
    auto t = erato::oracle::oracle_bit_table(params);
    std::memcpy(out, t.bytes.data(), t.bytes.size());
    return 0;
  } catch (const erato::Error& e) {
    g_last_error = e.what();
    return code_of(e);
  }
}

// f = 0 tables, assembled from reference pieces (SURVEY.md §8c convention:
// bit j = 1 iff 2j+1 is composite; 1 and the base primes stay 0):
// segment 0 (numbers 1..2^(l+1)) from simple_sieve, segments 1..n-1 from
// run_sieve(l, 1, n-1).  out may be NULL (count only).
int ref_f0_table(unsigned l, uint64_t n, int test_mode, uint8_t* out, uint64_t* count) {
  try {
    const uint64_t segbits = uint64_t{1} << l;
    const uint64_t segbytes = segbits / 8;
    auto primes = erato::oracle::simple_sieve(uint64_t{2} << l);
    // segment 0: all bits composite except primes and 1
    std::string seg0(segbytes, '\xff');
    seg0[0] &= (char)~1;  // number 1
    uint64_t zeros = 1;
    for (uint32_t p : primes) {
      if (p == 2) continue;
      const uint64_t j = (p - 1) / 2;
      seg0[j >> 3] &= (char)~(1u << (j & 7));
      ++zeros;
    }
    if (out) std::memcpy(out, seg0.data(), segbytes);
    uint64_t rest = 0;
    if (n > 1) {
      const auto params = erato::validate_params(l, 1, n - 1, test_mode != 0);
      erato::RunStats st;
      if (out) {
        erato::TableSink sink;
        st = erato::run_sieve(params, sink);
        std::memcpy(out + segbytes, sink.bytes().data(), sink.bytes().size());
      } else {
        erato::NullSink sink;
        st = erato::run_sieve(params, sink);
      }
      rest = st.prime_count;
    }
    if (count) *count = zeros + rest;
    return 0;
  } catch (const erato::Error& e) {
    g_last_error = e.what();
    return code_of(e);
  }
}

}  // extern "C"
