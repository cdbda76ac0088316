/* erato_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker; never linked
 * into, loaded by, or called from the product path).
 *
 * Plain-C restatement of the reference's sieve semantics for the hot path
 * `run_sieve` (/root/reference/proj/src/driver.cpp:83-120).  Every function
 * cites the reference code it restates.  Parity of this restatement is pinned
 * against the reference itself (oracle/_ref, built by oracle/Makefile from the
 * reference sources) and against the golden vectors in tests/golden/.
 *
 * Output contract (/root/reference/proj/include/erato/driver.hpp:6-8):
 *   bit j of the table = bit (j mod 8) of byte floor(j/8) (LSB first);
 *   1 = the odd number 2(f*2^l + j) + 1 is composite, 0 = prime.
 *
 * Extension (the f = 0 convention): when the interval overlaps
 * its own base primes (u^2 <= v, which the reference rejects with
 * F_ZERO_OR_OVERLAP), multiples are marked from max(u, p^2), so 1 and every
 * prime stay 0 and the zero-bit count is pi(v) (1 replaces 2).  For
 * non-overlapping intervals the p^2 floor never changes the table: a multiple
 * p*c < p^2 has the smaller factor c, whose prime factors also sieve it.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* error codes = 1 + ordinal of erato::errc (/root/reference/proj/include/erato/params.hpp:18-29) */
enum {
  EO_OK = 0,
  EO_L_OUT_OF_RANGE = 1,
  EO_F_ZERO_OR_OVERLAP = 2,
  EO_N_OUT_OF_RANGE = 3,
  EO_OVERFLOW = 4,
  EO_INDEX_OUT_OF_RANGE = 5,
  EO_NOT_ADMISSIBLE = 6,
  EO_ALLOC_LIMIT = 7,
  EO_LIMIT_TOO_LARGE = 8,
  EO_RANGE_TOO_LARGE = 9,
  EO_IO_ERROR = 10,
};

/* isqrt: /root/reference/proj/src/params.cpp:79-85 */
uint64_t eo_isqrt(uint64_t x) {
  uint64_t r = (uint64_t)sqrt((double)x);
  if (r > UINT32_MAX) r = UINT32_MAX;
  while (r > 0 && (unsigned __int128)r * r > x) --r;
  while ((unsigned __int128)(r + 1) * (r + 1) <= x) ++r;
  return r;
}

/* validate_params: /root/reference/proj/src/params.cpp:23-44.
 * allow_overlap != 0 admits u^2 <= v (incl. f = 0) under the p^2 convention. */
int eo_validate(unsigned l, uint64_t f, uint64_t n, int test_mode, int allow_overlap,
                uint64_t* u, uint64_t* v) {
  const unsigned lmin = test_mode ? 4 : 10;
  if (l < lmin || l > 30) return EO_L_OUT_OF_RANGE;
  if (n == 0) return EO_N_OUT_OF_RANGE;
  if (f > UINT64_MAX - n || (f + n) > (UINT64_MAX >> (l + 1))) return EO_OVERFLOW;
  const uint64_t uu = (f << (l + 1)) + 1, vv = (f + n) << (l + 1);
  if (!allow_overlap && (unsigned __int128)uu * uu <= vv) return EO_F_ZERO_OR_OVERLAP;
  if (u) *u = uu;
  if (v) *v = vv;
  return EO_OK;
}

/* params_from_midpoint: /root/reference/proj/src/params.cpp:64-77 (decimal 10^e) */
int eo_params_from_midpoint(unsigned e, unsigned l, uint64_t n, int test_mode, uint64_t* f) {
  if (e > 19) return EO_OVERFLOW;
  uint64_t pow10 = 1;
  for (unsigned i = 0; i < e; ++i) pow10 *= 10;
  if (l > 30) return EO_L_OUT_OF_RANGE;
  const uint64_t mid = pow10 >> (l + 1);
  if (mid <= n / 2) return EO_F_ZERO_OR_OVERLAP;
  const uint64_t ff = mid - n / 2;
  const int rc = eo_validate(l, ff, n, test_mode, 0, 0, 0);
  if (rc) return rc;
  *f = ff;
  return EO_OK;
}

/* first_offset (Lemma 1): /root/reference/proj/src/wheel.cpp:43-47,
 * /root/reference/PAPER.md:194-215.  Unique q in [0,p) with p | 2(f*2^l+q)+1. */
uint32_t eo_first_offset(uint32_t p, unsigned l, uint64_t f) {
  const uint64_t r = ((f % p) << (l + 1)) % p;
  return (uint32_t)(r % 2 == 0 ? (p - r - 1) / 2 : (2 * (uint64_t)p - r - 1) / 2);
}

/* simple_sieve: /root/reference/proj/src/oracle.cpp:8-23 — byte per number.
 * Writes up to cap primes <= limit to out; returns the number of primes. */
uint64_t eo_simple_sieve(uint64_t limit, uint32_t* out, uint64_t cap) {
  if (limit < 2) return 0;
  if (limit > ((uint64_t)1 << 32)) return 0;
  uint8_t* comp = (uint8_t*)calloc(limit + 1, 1);
  if (!comp) return 0;
  for (uint64_t i = 2; i * i <= limit; ++i)
    if (!comp[i])
      for (uint64_t j = i * i; j <= limit; j += i) comp[j] = 1;
  uint64_t cnt = 0;
  for (uint64_t i = 2; i <= limit; ++i)
    if (!comp[i]) {
      if (out && cnt < cap) out[cnt] = (uint32_t)i;
      ++cnt;
    }
  free(comp);
  return cnt;
}

/* Zero bits among the first nbits of a byte table (count_zeros semantics,
 * /root/reference/proj/src/simd.cpp:18-25). */
uint64_t eo_count_zeros(const uint8_t* t, uint64_t nbits) {
  uint64_t ones = 0;
  const uint64_t nbytes = nbits / 8;
  const uint64_t* w = (const uint64_t*)t;
  uint64_t i = 0;
  for (; i + 8 <= nbytes; i += 8) ones += (uint64_t)__builtin_popcountll(w[i / 8]);
  for (; i < nbytes; ++i) ones += (uint64_t)__builtin_popcount(t[i]);
  return nbits - ones;
}

/* The bit table by direct stepping per prime — restates oracle_bit_table
 * (/root/reference/proj/src/oracle.cpp:25-46) without its v <= 2^40 limit,
 * plus the p^2 floor of the overlap convention.  out: n*2^(l-3) bytes. */
int eo_bit_table(unsigned l, uint64_t f, uint64_t n, int test_mode, int allow_overlap,
                 uint8_t* out, uint64_t* count) {
  uint64_t u, v;
  int rc = eo_validate(l, f, n, test_mode, allow_overlap, &u, &v);
  if (rc) return rc;
  const uint64_t nbits = n << l;
  memset(out, 0, nbits / 8);
  const uint64_t lim = eo_isqrt(v);
  uint64_t np = eo_simple_sieve(lim, 0, 0);
  uint32_t* primes = (uint32_t*)malloc((np ? np : 1) * sizeof(uint32_t));
  if (!primes) return EO_ALLOC_LIMIT;
  eo_simple_sieve(lim, primes, np);
  for (uint64_t i = 0; i < np; ++i) {
    const uint64_t p = primes[i];
    if (p == 2) continue;
    /* first odd multiple c*p >= max(u, p^2) */
    uint64_t c = (u + p - 1) / p;
    if (c < p) c = p;
    if (c % 2 == 0) ++c;
    if ((unsigned __int128)c * p > v) continue;
    for (uint64_t m = c * p;; m += 2 * p) {
      const uint64_t j = (m - u) / 2;
      out[j >> 3] |= (uint8_t)(1u << (j & 7));
      if (m > v - 2 * p) break;
    }
  }
  free(primes);
  if (count) *count = eo_count_zeros(out, nbits);
  return EO_OK;
}
