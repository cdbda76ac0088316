// erato_gpu.cu — host orchestration + C ABI (include/erato_gpu.h).
//
// Replaces run_sieve (/root/reference/proj/src/driver.cpp:83-120) and its
// sinks.  Per run:
//   init  (base.cpp:19-89 analog, all on the device)
//     1. odd primes < 2^16 and pattern tables (cached per context)
//     2. sieve [1, isqrt(v)] with the tile kernel -> bitmap -> sorted u32
//        prime list (popcount + scan compaction)
//     3. one host sync: prime count, class boundaries, largest prime
//     4. large primes: first hits (fp64 quotient estimate + exact u64
//        remainder) -> ML array + far wave buckets
//   waves (the reference's per-segment loop, driver.cpp:93-117)
//     for each wave of W tiles: k_scatter_ml + k_scatter_far (large primes
//     -> per-tile hit records, far entries re-bucketed) then k_tile
//     (patterns, medium primes, hits, popcount, 128-bit write-out)
//   count: device u64 (NullSink: only it leaves the device).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/erato_gpu.h"
#include "sieve_kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = std::string(erato_gpu_errc_name(code)) + ": " + msg;
  return code;
}

#define CUDA_TRY(x)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      return fail(ERATO_GPU_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));      \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

uint64_t isqrt_u64(uint64_t x) {
  uint64_t r = (uint64_t)std::sqrt((double)x);
  if (r > UINT32_MAX) r = UINT32_MAX;
  while (r > 0 && (unsigned __int128)r * r > x) --r;
  while ((unsigned __int128)(r + 1) * (r + 1) <= x) ++r;
  return r;
}

// Rosser–Schoenfeld: pi(x) < 1.25506 x / ln x for x > 1
uint64_t pi_upper(uint64_t x) {
  if (x < 17) return 8;
  return (uint64_t)(1.25506 * (double)x / std::log((double)x)) + 16;
}

constexpr uint32_t kBaseLogTile = 20;  // tile size for the sieve of [1, sqrt(v)]
constexpr uint32_t kGenBlocksPerSm = 2;
constexpr uint64_t kFewLarge = 2048;  // at most this many primes > S are sieved as medium primes

}  // namespace

struct erato_gpu_ctx {
  int device = 0;
  int nsm = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t xstream = nullptr;               // D2H copies of finished waves (sieve_to_host)
  cudaEvent_t xev = nullptr, xjoin = nullptr;   // wave done / copies done
  // cached per context
  DevBuf sp, spm, ptab;  // small primes < 2^16, their base-sieve records, pattern tables
  std::vector<uint32_t> h_sp;
  // grow-only run buffers
  DevBuf base_bits, primes, med, ml, buckets, bcount, hits, hitcnt, blk_cnt, blk_off, scal, table, outbuf;
  DevBuf recs, rcount, frecs, fslot, fcount;  // k_gen -> k_bin per-warp regions
  double hcap_scale = 1.0, bcap_scale = 1.0;
  uint64_t max_base_pairs = uint64_t{1} << 27;  // base.hpp:87
  cudaEvent_t ev[4] = {};
  std::vector<cudaEvent_t> phase_ev;  // pairs, grown on demand
};

extern "C" {

const char* erato_gpu_errc_name(int code) {
  switch (code) {
    case ERATO_GPU_OK: return "OK";
    case ERATO_GPU_L_OUT_OF_RANGE: return "L_OUT_OF_RANGE";
    case ERATO_GPU_F_ZERO_OR_OVERLAP: return "F_ZERO_OR_OVERLAP";
    case ERATO_GPU_N_OUT_OF_RANGE: return "N_OUT_OF_RANGE";
    case ERATO_GPU_OVERFLOW: return "OVERFLOW";
    case ERATO_GPU_INDEX_OUT_OF_RANGE: return "INDEX_OUT_OF_RANGE";
    case ERATO_GPU_NOT_ADMISSIBLE: return "NOT_ADMISSIBLE";
    case ERATO_GPU_ALLOC_LIMIT: return "ALLOC_LIMIT";
    case ERATO_GPU_LIMIT_TOO_LARGE: return "LIMIT_TOO_LARGE";
    case ERATO_GPU_RANGE_TOO_LARGE: return "RANGE_TOO_LARGE";
    case ERATO_GPU_IO_ERROR: return "IO_ERROR";
    case ERATO_GPU_E_CUDA: return "CUDA_ERROR";
    case ERATO_GPU_E_NO_DEVICE: return "NO_DEVICE";
    case ERATO_GPU_E_INVALID_ARG: return "INVALID_ARGUMENT";
    case ERATO_GPU_E_INVARIANT: return "INVARIANT";
  }
  return "UNKNOWN";
}

const char* erato_gpu_last_error(void) { return g_err.c_str(); }

uint64_t erato_gpu_isqrt(uint64_t x) { return isqrt_u64(x); }

// validate_params, /root/reference/proj/src/params.cpp:23-44
int erato_gpu_validate(unsigned l, uint64_t f, uint64_t n, unsigned flags, uint64_t* u, uint64_t* v) {
  const unsigned lmin = (flags & ERATO_GPU_TEST_MODE) ? 4 : 10;
  if (l < lmin || l > 30)
    return fail(ERATO_GPU_L_OUT_OF_RANGE,
                "l=" + std::to_string(l) + " outside [" + std::to_string(lmin) + ", 30]");
  if (n == 0) return fail(ERATO_GPU_N_OUT_OF_RANGE, "n must be >= 1");
  if (f > UINT64_MAX - n || (f + n) > (UINT64_MAX >> (l + 1)))
    return fail(ERATO_GPU_OVERFLOW, "v = (f+n)*2^(l+1) exceeds 2^64");
  const uint64_t uu = (f << (l + 1)) + 1, vv = (f + n) << (l + 1);
  if (!(flags & ERATO_GPU_ALLOW_OVERLAP) && (unsigned __int128)uu * uu <= vv)
    return fail(ERATO_GPU_F_ZERO_OR_OVERLAP,
                "interval overlaps its own base primes (need u^2 > v); f=" + std::to_string(f));
  if (u) *u = uu;
  if (v) *v = vv;
  return 0;
}

// params_from_midpoint, /root/reference/proj/src/params.cpp:64-77
int erato_gpu_f_from_midpoint(unsigned e, unsigned l, uint64_t n, unsigned flags, uint64_t* f) {
  if (e > 19) return fail(ERATO_GPU_OVERFLOW, "10^" + std::to_string(e) + " exceeds 2^64");
  uint64_t pow10 = 1;
  for (unsigned i = 0; i < e; ++i) pow10 *= 10;
  if (l > 30) return fail(ERATO_GPU_L_OUT_OF_RANGE, "l=" + std::to_string(l));
  const uint64_t mid = pow10 >> (l + 1);
  if (mid <= n / 2)
    return fail(ERATO_GPU_F_ZERO_OR_OVERLAP,
                "midpoint 10^" + std::to_string(e) + " below half the interval");
  const uint64_t ff = mid - n / 2;
  const int rc = erato_gpu_validate(l, ff, n, flags & ERATO_GPU_TEST_MODE, nullptr, nullptr);
  if (rc) return rc;
  *f = ff;
  return 0;
}

// first_offset, /root/reference/proj/src/wheel.cpp:43-47
uint32_t erato_gpu_first_offset(uint32_t p, unsigned l, uint64_t f) {
  const uint64_t r = ((f % p) << (l + 1)) % p;
  return (uint32_t)(r % 2 == 0 ? (p - r - 1) / 2 : (2 * (uint64_t)p - r - 1) / 2);
}

// host twin of eg::first_hit (same arithmetic, 128-bit quotient)
int erato_gpu_first_hit(uint32_t p, uint64_t x, uint64_t cmin, uint64_t* offset, unsigned* wheel_class) {
  static const uint8_t adv[30] = {1, 0, 5, 4, 3, 2, 1, 0, 3, 2, 1, 0, 1, 0, 3, 2, 1, 0, 1, 0, 3, 2, 1, 0, 5, 4, 3, 2, 1, 0};
  static const uint8_t cls[30] = {255, 0, 255, 255, 255, 255, 255, 1, 255, 255, 255, 2, 255, 3, 255,
                                  255, 255, 4, 255, 5, 255, 255, 255, 6, 255, 255, 255, 255, 255, 7};
  if (p < 7 || p % 2 == 0 || p % 3 == 0 || p % 5 == 0 || x % 2 == 0)
    return fail(ERATO_GPU_E_INVALID_ARG, "first_hit needs p coprime to 30, p >= 7, x odd");
  uint64_t c = x / p, r = x % p;
  uint64_t d = 0;
  if (r) {
    ++c;
    d = p - r;
  }
  if (c < cmin) {
    d += (cmin - c) * (uint64_t)p;
    c = cmin;
  }
  const unsigned cm = (unsigned)(c % 30), a = adv[cm];
  d += (uint64_t)a * p;
  if (offset) *offset = d >> 1;
  if (wheel_class) *wheel_class = cls[cm + a];
  return 0;
}

// table_filename, /root/reference/proj/src/driver.cpp:17-20
size_t erato_gpu_table_filename(unsigned l, uint64_t f, uint64_t n, char* out, size_t cap) {
  const std::string s = "erato_l" + std::to_string(l) + "_f" + std::to_string(f) + "_n" +
                        std::to_string(n) + ".bits";
  if (out && cap) std::snprintf(out, cap, "%s", s.c_str());
  return s.size() + 1;
}

void erato_gpu_shard(uint64_t f, uint64_t n, int rank, int world, uint64_t* f_out, uint64_t* n_out) {
  if (world < 1) world = 1;
  const unsigned __int128 b = (unsigned __int128)n * (unsigned)rank / (unsigned)world;
  const unsigned __int128 e = (unsigned __int128)n * (unsigned)(rank + 1) / (unsigned)world;
  *f_out = f + (uint64_t)b;
  *n_out = (uint64_t)(e - b);
}

int erato_gpu_set_max_base_pairs(erato_gpu_ctx* c, uint64_t max_pairs) {
  if (!c) return fail(ERATO_GPU_E_INVALID_ARG, "ctx is NULL");
  c->max_base_pairs = max_pairs;
  return 0;
}

int erato_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int erato_gpu_create(int device, erato_gpu_ctx** out) {
  if (!out) return fail(ERATO_GPU_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (erato_gpu_device_count() == 0) return fail(ERATO_GPU_E_NO_DEVICE, "no CUDA device visible");
  if (device < 0) CUDA_TRY(cudaGetDevice(&device));
  CUDA_TRY(cudaSetDevice(device));
  auto* c = new erato_gpu_ctx();
  c->device = device;
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  c->nsm = prop.multiProcessorCount;
  CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->xstream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&c->xev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->xjoin, cudaEventDisableTiming));
  for (auto& e : c->ev) CUDA_TRY(cudaEventCreate(&e));
  for (auto kt : {eg::k_tile<false, false>, eg::k_tile<true, false>, eg::k_tile<false, true>, eg::k_tile<true, true>})
    CUDA_TRY(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(eg::kPatWords * 4 + (1u << kBaseLogTile) / 8 + eg::kMaxWarpPrimes * 8 +
                                        eg::kTileWarps * eg::kHitChunk * 4)));
  CUDA_TRY(cudaFuncSetAttribute(eg::k_bin, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(eg::BinSmem)));
  CUDA_TRY(cudaFuncSetAttribute(eg::k_scatter_ml, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(eg::MlSmem)));
  CUDA_TRY(cudaFuncSetAttribute(eg::k_scatter_far, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(eg::FarSmem)));
  // cached tables: small primes < 2^16 and the pattern windows
  CUDA_TRY(c->sp.ensure(8192 * 4));
  CUDA_TRY(c->spm.ensure((8192 + eg::kMedPad) * 16));
  CUDA_TRY(c->ptab.ensure(eg::kPatWords * 4));
  CUDA_TRY(c->scal.ensure(64 * 8));
  eg::k_build_patterns<<<(eg::kPatWords + 255) / 256, 256, 0, c->stream>>>(c->ptab.as<uint32_t>());
  eg::k_small_primes<<<1, 1024, 0, c->stream>>>(c->sp.as<uint32_t>(), c->scal.as<uint32_t>());
  uint32_t nsp = 0;
  CUDA_TRY(cudaMemcpyAsync(&nsp, c->scal.p, 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  // base-sieve records: g0 = 0 (x0 = 1), tiles of 2^kBaseLogTile bits
  eg::k_med_records<<<(nsp + 255) / 256, 256, 0, c->stream>>>(c->sp.as<uint32_t>(), nsp, 1, kBaseLogTile,
                                                              c->spm.as<uint4>());
  c->h_sp.resize(nsp);
  CUDA_TRY(cudaMemcpyAsync(c->h_sp.data(), c->sp.p, nsp * 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaGetLastError());
  *out = c;
  return 0;
}

void erato_gpu_destroy(erato_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (DevBuf* b : {&c->sp, &c->spm, &c->ptab, &c->base_bits, &c->primes, &c->med, &c->ml, &c->buckets,
                    &c->bcount, &c->hits, &c->hitcnt, &c->blk_cnt, &c->blk_off, &c->scal, &c->table,
                    &c->outbuf, &c->recs, &c->rcount, &c->frecs, &c->fslot, &c->fcount})
    b->release();
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->phase_ev) cudaEventDestroy(e);
  if (c->xev) cudaEventDestroy(c->xev);
  if (c->xjoin) cudaEventDestroy(c->xjoin);
  if (c->xstream) cudaStreamDestroy(c->xstream);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

}  // extern "C"

namespace {

// Launch the tile kernel over `ntiles` tiles starting at `tile0`.
// p2: multiples from p^2 on (overlap runs, base sieve).
void launch_tiles(cudaStream_t st, const eg::TileArgs& a, uint32_t ntiles, bool p2) {
  const size_t smem = eg::kPatWords * 4 + ((size_t)1 << a.log_s) / 8 + (size_t)((a.nmed_warp + 1) & ~1u) * 8 +
                      (a.hits ? (size_t)eg::kTileWarps * eg::kHitChunk * 4 : 0);
  if (a.hits) {
    if (p2) eg::k_tile<true, true><<<ntiles, eg::kTileThreads, smem, st>>>(a);
    else eg::k_tile<false, true><<<ntiles, eg::kTileThreads, smem, st>>>(a);
  } else {
    if (p2) eg::k_tile<true, false><<<ntiles, eg::kTileThreads, smem, st>>>(a);
    else eg::k_tile<false, false><<<ntiles, eg::kTileThreads, smem, st>>>(a);
  }
}

// Split of the group-per-prime medium primes (indices [0, nwarp) of the
// medium list, ascending p): counts for 32-lane (p < S/256) and 16-lane
// (p < S/128) groups, from the list indices of those bounds.
void group_split(eg::TileArgs& ta, uint64_t i256, uint64_t i128) {
  ta.nmed_g32 = (uint32_t)std::min<uint64_t>(i256, ta.nmed_warp);
  ta.nmed_g16 = (uint32_t)std::min<uint64_t>(std::max(i128, i256), ta.nmed_warp) - ta.nmed_g32;
}

// Sorted list of the zero bits of bits[0..nbits) at indices >= lo, as base + 2*j.
template <class T>
int compact_zeros(erato_gpu_ctx* c, cudaStream_t st, const uint32_t* bits, uint64_t nbits, uint64_t lo,
                  uint64_t base, T* out, uint64_t cap, uint64_t* d_total) {
  const uint64_t nwords = (nbits + 31) / 32;
  const uint64_t nblk = (nwords + eg::kCompactWords - 1) / eg::kCompactWords;
  if (nblk == 0) {
    CUDA_TRY(cudaMemsetAsync(d_total, 0, 8, st));
    return 0;
  }
  if (nblk > (1u << 26)) return fail(ERATO_GPU_RANGE_TOO_LARGE, "compaction too large");
  CUDA_TRY(c->blk_cnt.ensure(nblk * 4));
  CUDA_TRY(c->blk_off.ensure(nblk * 8));
  eg::k_count_zeros_blocks<<<(unsigned)nblk, 1024, 0, st>>>(bits, nbits, lo, c->blk_cnt.as<uint32_t>());
  eg::k_scan_counts<<<1, 1024, 0, st>>>(c->blk_cnt.as<uint32_t>(), (uint32_t)nblk, c->blk_off.as<uint64_t>(),
                                        d_total);
  eg::k_write_zeros<T><<<(unsigned)nblk, 1024, 0, st>>>(bits, nbits, lo, c->blk_off.as<uint64_t>(), base, out,
                                                        cap);
  return 0;
}

struct Plan {
  unsigned l;
  uint64_t f, n, u, v, T, g0;
  uint32_t log_s, S, W, WS;
  uint32_t MW;  // ML window: waves walked per ML scatter launch (ML primes: S < p <= MW*WS)
  uint64_t ntiles, nwaves;
  bool overlap;
};

}  // namespace

namespace {
// host_dst (pinned, optional): each wave's finished slice of dev_table is
// copied to host_dst on a side stream while the next waves run.
int run_impl(erato_gpu_ctx* c, unsigned l, uint64_t f, uint64_t n, unsigned flags, void* dev_table,
             uint64_t* dev_count, void* stream_v, int sync, erato_gpu_stats* stats, uint8_t* host_dst) {
  if (!c) return fail(ERATO_GPU_E_INVALID_ARG, "ctx is NULL");
  Plan P{};
  int rc = erato_gpu_validate(l, f, n, flags, &P.u, &P.v);
  if (rc) return rc;
  if (dev_table && ((uintptr_t)dev_table & 15))
    return fail(ERATO_GPU_E_INVALID_ARG, "dev_table must be 16-byte aligned");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = stream_v ? (cudaStream_t)stream_v : c->stream;
  P.l = l;
  P.f = f;
  P.n = n;
  P.T = n << l;
  P.g0 = f << l;
  P.overlap = (unsigned __int128)P.u * P.u <= P.v;
  // tile size: 2^20 bits unless the run is too small to fill the GPU
  {
    uint32_t ls = 20;
    while (ls > 13 && (P.T >> ls) < (uint64_t)2 * c->nsm) --ls;
    P.log_s = ls;
    P.S = 1u << ls;
  }
  P.ntiles = (P.T + P.S - 1) >> P.log_s;
  {
    int occ = 1;
    const size_t smem = eg::kPatWords * 4 + (size_t)P.S / 8 + eg::kMaxWarpPrimes * 8 + eg::kTileWarps * eg::kHitChunk * 4;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, eg::k_tile<false, true>, eg::kTileThreads, smem));
    if (occ < 1) occ = 1;
    uint64_t W = (uint64_t)c->nsm * occ;
    W = std::min<uint64_t>(W, eg::kMaxWaveTiles);

    // ML states / far entries keep positions in 29 bits.  A stored position
    // is below 3p <= 3*W*S (first hit: (c*p - x)/2 with c*p - x < 6p; next
    // hit after a wave: pos + D*p - W*S with pos < W*S, D <= 3), so
    // 3*W*S < 2^29 (W <= 170 at S = 2^20: one tile per SM on a B200).
    W = std::min<uint64_t>(W, (((uint64_t)1 << 29) - 1) / (3ull * P.S));
    W = std::min<uint64_t>(W, P.ntiles);
    P.W = (uint32_t)std::max<uint64_t>(W, 1);
  }
  P.WS = P.W * P.S;
  P.nwaves = (P.ntiles + P.W - 1) / P.W;
  P.MW = 1;  // (an ML walk over 2 waves per launch measured 2 ms slower at cfg5)

  uint32_t launches = 0;
  for (int attempt = 0;; ++attempt) {
    const uint64_t vroot = isqrt_u64(P.v);
    CUDA_TRY(cudaEventRecord(c->ev[0], st));
    // ---------------- 1-2. base primes <= sqrt(v) ----------------
    uint64_t nbase_bits = (vroot + 1) / 2;  // odd numbers 1..vroot
    const uint64_t prime_cap = pi_upper(vroot) + 64;
    CUDA_TRY(c->primes.ensure(prime_cap * 4));
    // [0] total primes, [8..15] bounds + largest prime, [16] count, [17] overflow,
    // [18] hit records consumed, [19] expected records, [20] base-sieve count, [21] bad far entry
    uint64_t* d_scal = c->scal.as<uint64_t>();
    CUDA_TRY(cudaMemsetAsync(d_scal + 18, 0, 16, st));
    CUDA_TRY(cudaMemsetAsync(d_scal + 21, 0, 8, st));
    if (nbase_bits > 1) {
      const uint64_t words = ((nbase_bits + ((1u << kBaseLogTile) - 1)) >> kBaseLogTile) << (kBaseLogTile - 5);
      CUDA_TRY(c->base_bits.ensure(words * 4));
      const uint64_t rr = isqrt_u64(vroot);
      // small primes in (61, rr]
      const auto b61 = std::upper_bound(c->h_sp.begin(), c->h_sp.end(), 61u) - c->h_sp.begin();
      const auto brr = std::upper_bound(c->h_sp.begin(), c->h_sp.end(), (uint32_t)std::min<uint64_t>(rr, 65535)) -
                       c->h_sp.begin();
      eg::TileArgs ta{};
      ta.g0 = 0;
      ta.tbits = nbase_bits;
      ta.tile0 = 0;
      ta.log_s = kBaseLogTile;
      ta.med = c->spm.as<uint4>() + b61;
      ta.nmed = brr > b61 ? (uint32_t)(brr - b61) : 0;
      {
        auto idx_below = [&](uint32_t x) {  // medium-list index of the first prime >= x
          const int64_t i = std::lower_bound(c->h_sp.begin(), c->h_sp.end(), x) - c->h_sp.begin();
          return (uint64_t)std::max<int64_t>(i - b61, 0);
        };
        ta.nmed_warp = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(idx_below((1u << kBaseLogTile) / 64), ta.nmed),
                                                    eg::kMaxWarpPrimes);
        group_split(ta, idx_below((1u << kBaseLogTile) / 256), idx_below((1u << kBaseLogTile) / 128));
      }
      ta.ptab = c->ptab.as<uint32_t>();
      ta.table = c->base_bits.as<uint32_t>();
      ta.count = reinterpret_cast<unsigned long long*>(d_scal + 20);
      const uint64_t bt = (nbase_bits + (1u << kBaseLogTile) - 1) >> kBaseLogTile;
      launch_tiles(st, ta, (uint32_t)bt, true);
      ++launches;
      rc = compact_zeros<uint32_t>(c, st, c->base_bits.as<uint32_t>(), nbase_bits, 1, 1, c->primes.as<uint32_t>(),
                                   prime_cap, d_scal + 0);
      if (rc) return rc;
      launches += 3;
    } else {
      CUDA_TRY(cudaMemsetAsync(d_scal, 0, 8, st));
    }
    // ---------------- 3. class boundaries (one host sync) ----------------
    // index of the first prime above 61, S/64, S, MW*WS, max(WS/8, S), S/256, S/128
    uint64_t thr[7] = {61, (uint64_t)P.S / 64, P.S, (uint64_t)P.MW * P.WS, std::max<uint64_t>(P.WS / 8, P.S),
                       (uint64_t)P.S / 256, (uint64_t)P.S / 128};
    CUDA_TRY(cudaMemcpyAsync(d_scal + 24, thr, sizeof(thr), cudaMemcpyHostToDevice, st));
    eg::k_bounds<<<1, 32, 0, st>>>(c->primes.as<uint32_t>(), d_scal + 0, d_scal + 24, 7, d_scal + 8);
    ++launches;
    uint64_t hb[16];  // [15] = largest base prime
    CUDA_TRY(cudaMemcpyAsync(hb, d_scal, sizeof(hb), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const uint64_t nprimes = hb[0];
    if (nprimes > c->max_base_pairs)
      return fail(ERATO_GPU_ALLOC_LIMIT, std::to_string(nprimes) + " base primes exceed cap " +
                                              std::to_string(c->max_base_pairs));
    const uint32_t pmax = (uint32_t)hb[15];
    // A handful of primes just above the tile size (cfg3: 37) are cheaper as
    // medium primes (a per-tile start offset each) than through the scatter,
    // whose per-wave cost is mostly fixed.
    const bool few_large = nprimes - hb[10] <= kFewLarge && pmax < (1u << 24);
    const uint64_t i61 = hb[8], iwarp = std::max(hb[9], hb[8]);
    const uint64_t iS = few_large ? nprimes : hb[10], iWS = std::max(hb[11], iS);
    const uint64_t idense = std::max(hb[12], iS);

    // ---------------- 4. medium constants + large-prime structures ----------------
    const uint64_t nmed = iS - i61, nml = iWS - iS, nfar = nprimes - iWS;
    CUDA_TRY(c->med.ensure((nmed + eg::kMedPad) * 16));  // padded: the tile kernel prefetches past the end
    if (nmed)
      eg::k_med_records<<<(unsigned)((nmed + 255) / 256), 256, 0, st>>>(c->primes.as<uint32_t>() + i61, (uint32_t)nmed,
                                                                         2 * P.g0 + 1, P.log_s, c->med.as<uint4>());
    ++launches;
    const bool have_large = nml + nfar > 0;
    uint32_t ring = 1, bcap = 1, hcap = 4, rcap = 1, fcap = 1;
    if (have_large) {
      const double lnP = std::log((double)std::max<uint32_t>(pmax, 3));
      const double sum_recip = std::max(0.0, std::log(lnP / std::log((double)P.S))) + 0.02;  // sum 1/p, S<p<=P
      const double eh = (double)P.S * (8.0 / 15.0) * sum_recip;
      hcap = (uint32_t)std::min<double>(((eh * 1.10 + 4096) * c->hcap_scale), (double)P.S * 4);
      hcap = (hcap + 3) & ~3u;
      CUDA_TRY(c->ml.ensure(std::max<uint64_t>(nml, 1) * 8));
      // the lists of the MW waves of an ML window, + trash of the split scatter
      CUDA_TRY(c->hits.ensure(((uint64_t)P.MW * P.W * hcap + eg::kScTrash) * 4));
      CUDA_TRY(c->hitcnt.ensure((uint64_t)P.MW * P.W * 4));
      CUDA_TRY(cudaMemsetAsync(c->hitcnt.p, 0, (uint64_t)P.MW * P.W * 4, st));
      if (nfar) {
        ring = (uint32_t)std::min<uint64_t>(4ull * pmax / P.WS + 3, P.nwaves + 2);
        if (ring > (uint32_t)eg::kMaxRing) return fail(ERATO_GPU_RANGE_TOO_LARGE, "far bucket ring exceeds 256 waves");
        const double sr_far = std::max(0.0, std::log(lnP / std::log((double)P.MW * P.WS))) + 0.01;
        const double eb = (double)P.WS * (8.0 / 15.0) * sr_far;
        bcap = (uint32_t)std::min<double>((eb * 1.10 + 8192) * c->bcap_scale, (double)nfar + 64);
      }
      CUDA_TRY(c->buckets.ensure(((uint64_t)ring * bcap + eg::kScTrash) * 8));
      {
        const uint64_t gen_warps = (uint64_t)c->nsm * kGenBlocksPerSm * (eg::kGenThreads / 32);
        const double per_wave = eh * P.W;  // records per wave
        rcap = (uint32_t)std::min<double>((per_wave / gen_warps * 1.3 + 2048) * c->hcap_scale, 1u << 30);
        rcap = (rcap + 31) & ~31u;
        fcap = nfar ? (uint32_t)std::min<double>(((double)bcap / gen_warps * 1.3 + 512) * c->bcap_scale, 1u << 30) : 1;
        CUDA_TRY(c->recs.ensure(gen_warps * rcap * 4));
        CUDA_TRY(c->rcount.ensure(gen_warps * 4));
        CUDA_TRY(c->frecs.ensure(gen_warps * fcap * 8));
        CUDA_TRY(c->fslot.ensure(gen_warps * fcap));
        CUDA_TRY(c->fcount.ensure(gen_warps * 4));
      }
      CUDA_TRY(c->bcount.ensure((uint64_t)ring * 4 + 4));
      CUDA_TRY(cudaMemsetAsync(c->bcount.p, 0, (uint64_t)ring * 4 + 4, st));
      CUDA_TRY(cudaMemsetAsync(d_scal + 17, 0, 8, st));  // overflow flag
      eg::SetupArgs sa{};
      sa.primes = c->primes.as<uint32_t>();
      sa.i0 = iS;
      sa.i_ml_end = iWS;
      sa.i_end = nprimes;
      sa.x0 = 2 * P.g0 + 1;
      sa.ml = c->ml.as<uint2>();
      sa.far_buckets = c->buckets.as<uint64_t>();
      sa.far_bcount = c->bcount.as<uint32_t>();
      sa.ring = ring;
      sa.bcap = bcap;
      sa.nwaves = P.nwaves;
      sa.WS = P.WS;
      sa.inv_ws = 1.0 / (double)P.WS;
      sa.overflow = reinterpret_cast<int*>(d_scal + 17);
      if (const char* inj = std::getenv("ERATO_GPU_TEST_INJECT")) sa.inject = std::atoi(inj);  // tests only
      const uint64_t nl = nprimes - iS;
      eg::k_setup_large<<<(unsigned)((nl + eg::kSetupThreads - 1) / eg::kSetupThreads), eg::kSetupThreads, 0, st>>>(sa);
      ++launches;
      if (flags & ERATO_GPU_CHECK_INVARIANTS) {
        // expected hit records: admissible multiples of the large primes in the tiles
        const unsigned __int128 x_hi = (unsigned __int128)P.u + 2 * (unsigned __int128)(P.ntiles << P.log_s) - 2;
        const uint64_t xh = x_hi > UINT64_MAX ? UINT64_MAX : (uint64_t)x_hi;
        eg::k_expected_records<<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(
            c->primes.as<uint32_t>(), iS, nprimes, P.u, xh, reinterpret_cast<unsigned long long*>(d_scal + 19));
        ++launches;
      }
    } else {
      CUDA_TRY(cudaMemsetAsync(d_scal + 17, 0, 8, st));
    }
    CUDA_TRY(cudaEventRecord(c->ev[1], st));

    // ---------------- 5. waves ----------------
    unsigned long long* d_count = reinterpret_cast<unsigned long long*>(d_scal + 16);
    CUDA_TRY(cudaMemsetAsync(d_count, 0, 8, st));
    eg::TileArgs ta{};
    ta.g0 = P.g0;
    ta.tbits = P.T;
    ta.log_s = P.log_s;
    ta.med = c->med.as<uint4>();
    ta.nmed = (uint32_t)nmed;
    ta.nmed_warp = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(iwarp - i61, nmed), eg::kMaxWarpPrimes);
    group_split(ta, std::max(hb[13], i61) - i61, std::max(hb[14], i61) - i61);
    ta.ptab = c->ptab.as<uint32_t>();
    ta.hits = have_large ? c->hits.as<uint32_t>() : nullptr;
    ta.hitcnt = c->hitcnt.as<uint32_t>();
    ta.hcap = hcap;
    ta.table = static_cast<uint32_t*>(dev_table);
    ta.count = d_count;
    ta.tbase = 0;
    const uint32_t gen_blocks = (uint32_t)c->nsm * kGenBlocksPerSm;
    const uint32_t gen_warps = gen_blocks * (eg::kGenThreads / 32);
    const uint32_t bin_blocks = std::max<uint32_t>((uint32_t)c->nsm * 2, (gen_warps + eg::kMaxRegionsPerCta - 1) / eg::kMaxRegionsPerCta);
    eg::GenArgs ga{};
    eg::BinArgs ba{};
    if (have_large) {
      ga.ml = c->ml.as<uint2>();
      ga.nml = (uint32_t)nml;
      ga.noct = (uint32_t)std::min<uint64_t>(idense - iS, nml);
      ga.bcap = bcap;
      ga.ring = ring;
      ga.nwaves = P.nwaves;
      ga.WS = P.WS;
      ga.log_s = P.log_s;
      ga.recs = c->recs.as<uint32_t>();
      ga.rcount = c->rcount.as<uint32_t>();
      ga.rcap = rcap;
      ga.frecs = c->frecs.as<uint64_t>();
      ga.fslot = c->fslot.as<uint8_t>();
      ga.fcount = c->fcount.as<uint32_t>();
      ga.fcap = fcap;
      ga.overflow = reinterpret_cast<int*>(d_scal + 17);
      ba.recs = ga.recs;
      ba.rcount = ga.rcount;
      ba.rcap = rcap;
      ba.nregions = gen_warps;
      ba.frecs = nfar ? ga.frecs : nullptr;
      ba.fslot = ga.fslot;
      ba.fcount = ga.fcount;
      ba.fcap = fcap;
      ba.log_s = P.log_s;
      ba.hits = c->hits.as<uint32_t>();
      ba.hitcnt = c->hitcnt.as<uint32_t>();
      ba.hcap = hcap;
      ba.far_buckets = c->buckets.as<uint64_t>();
      ba.far_bcount = c->bcount.as<uint32_t>();
      ba.ring = ring;
      ba.bcap = bcap;
      ba.overflow = ga.overflow;
    }
    // large-prime path: k_scatter_ml + k_scatter_far (default), or k_gen +
    // k_bin (ERATO_GPU_SCATTER=genbin, or when a wave has more than 256 tiles
    // or ring slots, or 32-bit list offsets do not fit)
    const char* sc_env = std::getenv("ERATO_GPU_SCATTER");
    const bool sortable = ring <= (uint32_t)eg::kScBins && (uint64_t)P.MW * P.W <= (uint64_t)eg::kScBins;
    const bool idx32 = (uint64_t)P.MW * P.W * hcap + eg::kScTrash < (1ull << 32) &&
                       (uint64_t)ring * bcap + eg::kScTrash < (1ull << 32);
    const bool split = sortable && idx32 && !(sc_env && std::strcmp(sc_env, "genbin") == 0);
    eg::ScatterArgs sca{};
    uint32_t ml_blocks = c->nsm, far_blocks = c->nsm;
    if (split) {
      int occ = 1;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, eg::k_scatter_ml, eg::kMlWarps * 32,
                                                             sizeof(eg::MlSmem)));
      // no more CTAs than units of work (small runs: a handful of ML primes)
      const uint64_t ml_units = (nml + 31) / 32;
      ml_blocks = (uint32_t)std::min<uint64_t>((uint64_t)c->nsm * (uint32_t)std::max(occ, 1),
                                               std::max<uint64_t>(1, (ml_units + eg::kMlWarps - 1) / eg::kMlWarps));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, eg::k_scatter_far, eg::kFarWarps * 32,
                                                             sizeof(eg::FarSmem)));
      const uint64_t far_units = (std::min<uint64_t>(nfar, bcap) + 31) / 32;  // bucket size bound
      far_blocks = (uint32_t)std::min<uint64_t>((uint64_t)c->nsm * (uint32_t)std::max(occ, 1),
                                                std::max<uint64_t>(1, (far_units + eg::kFarWarps - 1) / eg::kFarWarps));
    }
    if (have_large) {
      sca.ml = ga.ml;
      sca.nml = ga.nml;
      sca.far_buckets = c->buckets.as<uint64_t>();
      sca.far_bcount = c->bcount.as<uint32_t>();
      sca.bcap = bcap;
      sca.ring = ring;
      sca.nwaves = P.nwaves;
      sca.WS = P.WS;
      sca.log_s = P.log_s;
      sca.inv_ws_f = 1.0f / (float)P.WS;
      sca.hits = c->hits.as<uint32_t>();
      sca.hitcnt = c->hitcnt.as<uint32_t>();
      sca.hcap = hcap;
      sca.overflow = ga.overflow;
    }
    const bool timing = (flags & ERATO_GPU_PHASE_TIMING) != 0;
    const size_t nev = timing ? (size_t)P.nwaves * 5 + 8 : 0;
    while (c->phase_ev.size() < nev) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      c->phase_ev.push_back(e);
    }
    size_t evi = 0;
    std::vector<std::pair<size_t, bool>> ev_pairs;  // (first event index, is_scatter)
    for (uint64_t w = 0; w < P.nwaves; ++w) {
      const uint64_t tile0 = w * P.W;
      const uint32_t ntw = (uint32_t)std::min<uint64_t>(P.W, P.ntiles - tile0);
      if (have_large) {
        ga.wave = w;
        ga.ntiles_w = ntw;
        ba.ntiles_w = ntw;
        const uint32_t slot = nfar ? (uint32_t)(w % ring) : 0;
        ga.far_in = nfar ? c->buckets.as<uint64_t>() + (uint64_t)slot * bcap : nullptr;
        ga.far_in_count = c->bcount.as<uint32_t>() + slot;
        if (timing) CUDA_TRY(cudaEventRecord(c->phase_ev[evi], st));
        // this wave's hit lists inside the ML window's lists
        const uint32_t wi = (uint32_t)(w % P.MW);
        uint32_t* const hits_w = c->hits.as<uint32_t>() + (uint64_t)wi * P.W * hcap;
        uint32_t* const hitcnt_w = c->hitcnt.as<uint32_t>() + (uint64_t)wi * P.W;
        ta.hits = hits_w;
        ta.hitcnt = hitcnt_w;
        if (split) {
          if (nml && wi == 0) {  // ML walk over the window's tiles, state re-based by the window span
            eg::ScatterArgs m = sca;
            m.ntiles_w = (uint32_t)std::min<uint64_t>((uint64_t)P.MW * P.W, P.ntiles - tile0);
            m.WS = P.MW * P.WS;
            m.hits = c->hits.as<uint32_t>();
            m.hitcnt = c->hitcnt.as<uint32_t>();
            eg::k_scatter_ml<<<ml_blocks, eg::kMlWarps * 32, sizeof(eg::MlSmem), st>>>(m);
            launches += 1;
          }
          if (timing) CUDA_TRY(cudaEventRecord(c->phase_ev[evi + 1], st));
          if (nfar) {
            sca.wave = w;
            sca.wslot = slot;
            sca.ntiles_w = ntw;
            sca.far_in = ga.far_in;
            sca.far_in_count = ga.far_in_count;
            sca.hits = hits_w;
            sca.hitcnt = hitcnt_w;
            eg::k_scatter_far<<<far_blocks, eg::kFarWarps * 32, sizeof(eg::FarSmem), st>>>(sca);
            launches += 1;
          }
        } else {
          // k_gen walks the ML primes wave by wave (any ML bound works)
          ba.hits = hits_w;
          ba.hitcnt = hitcnt_w;
          eg::k_gen<<<gen_blocks, eg::kGenThreads, 0, st>>>(ga);
          if (timing) CUDA_TRY(cudaEventRecord(c->phase_ev[evi + 1], st));
          eg::k_bin<<<bin_blocks, eg::kBinThreads, sizeof(eg::BinSmem), st>>>(ba);
          launches += 2;
        }
        if (timing) {
          CUDA_TRY(cudaEventRecord(c->phase_ev[evi + 2], st));
          ev_pairs.push_back({evi, true});
          evi += 3;
        }
        ta.reset_bucket_count = nfar ? c->bcount.as<uint32_t>() + slot : nullptr;
        if (flags & ERATO_GPU_CHECK_INVARIANTS) {
          eg::k_check_wave<<<(unsigned)c->nsm, 256, 0, st>>>(
              hitcnt_w, ntw, hcap, nfar ? ga.far_in : nullptr, ga.far_in_count, bcap, P.WS,
              reinterpret_cast<unsigned long long*>(d_scal + 18), reinterpret_cast<int*>(d_scal + 21));
          ++launches;
        }
      }
      ta.tile0 = tile0;
      if (tile0 + ntw - ta.tbase > eg::kMaxChunkTiles && nmed) {
        // new chunk: medium records for tile indices relative to tile0 (< 2^22)
        ta.tbase = tile0;
        eg::k_med_records<<<(unsigned)((nmed + 255) / 256), 256, 0, st>>>(
            c->primes.as<uint32_t>() + i61, (uint32_t)nmed, 2 * (P.g0 + (tile0 << P.log_s)) + 1, P.log_s,
            c->med.as<uint4>());
        ++launches;
      }
      if (timing) CUDA_TRY(cudaEventRecord(c->phase_ev[evi], st));
      launch_tiles(st, ta, ntw, P.overlap);
      if (host_dst && dev_table) {  // output pipeline: this wave's bytes go to the host now
        const uint64_t b0 = (tile0 << P.log_s) / 8, b1 = std::min<uint64_t>((tile0 + ntw) << P.log_s, P.T) / 8;
        CUDA_TRY(cudaEventRecord(c->xev, st));
        CUDA_TRY(cudaStreamWaitEvent(c->xstream, c->xev, 0));
        CUDA_TRY(cudaMemcpyAsync(host_dst + b0, static_cast<uint8_t*>(dev_table) + b0, b1 - b0,
                                 cudaMemcpyDeviceToHost, c->xstream));
      }
      if (timing) {
        CUDA_TRY(cudaEventRecord(c->phase_ev[evi + 1], st));
        ev_pairs.push_back({evi, false});
        evi += 2;
      }
      ++launches;
    }
    if (host_dst && dev_table) {  // join the copies
      CUDA_TRY(cudaEventRecord(c->xjoin, c->xstream));
      CUDA_TRY(cudaStreamWaitEvent(st, c->xjoin, 0));
    }
    CUDA_TRY(cudaGetLastError());
    if (dev_count) CUDA_TRY(cudaMemcpyAsync(dev_count, d_count, 8, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaEventRecord(c->ev[2], st));
    if (!sync) {
      if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->segments = n;
        stats->base_primes = nprimes;
        stats->tiles = P.ntiles;
        stats->log_tile = P.log_s;
        stats->waves = (uint32_t)P.nwaves;
        stats->kernel_launches = launches;
      }
      return 0;  // overflow cannot be checked without a sync; capacities are generous
    }
    uint64_t res[6];  // d_scal[16..21]
    CUDA_TRY(cudaMemcpyAsync(res, d_scal + 16, sizeof(res), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if ((int)res[1] != 0) {
      if (attempt >= 4) return fail(ERATO_GPU_ALLOC_LIMIT, "bucket capacity overflow persists");
      c->hcap_scale *= 2.0;
      c->bcap_scale *= 2.0;
      if (stats) stats->retries = attempt + 1;
      continue;
    }
    if ((flags & ERATO_GPU_CHECK_INVARIANTS) && have_large) {
      if (res[5])
        return fail(ERATO_GPU_E_INVARIANT, "a far bucket entry does not hit inside the wave of its bucket");
      if (res[2] != res[3])
        return fail(ERATO_GPU_E_INVARIANT, "large-prime hit records " + std::to_string(res[2]) + " != " +
                                               std::to_string(res[3]) + " admissible multiples in the tiles");
    }
    if (stats) {
      float t_init = 0, t_tot = 0;
      cudaEventElapsedTime(&t_init, c->ev[0], c->ev[1]);
      cudaEventElapsedTime(&t_tot, c->ev[0], c->ev[2]);
      const uint32_t retries = stats->retries;
      std::memset(stats, 0, sizeof(*stats));
      stats->retries = retries;
      stats->prime_count = res[0];
      stats->large_records = res[2];  // (counted with ERATO_GPU_CHECK_INVARIANTS)
      stats->segments = n;
      stats->init_s = t_init * 1e-3;
      stats->small_s = (t_tot - t_init) * 1e-3;
      if (timing) {
        double ts = 0, tl = 0, tg = 0, tb = 0;
        for (const auto& pr : ev_pairs) {
          float ms = 0, ms2 = 0;
          cudaEventElapsedTime(&ms, c->phase_ev[pr.first], c->phase_ev[pr.first + 1]);
          if (pr.second) {
            cudaEventElapsedTime(&ms2, c->phase_ev[pr.first + 1], c->phase_ev[pr.first + 2]);
            tg += ms;
            tb += ms2;
            tl += ms + ms2;
          } else {
            ts += ms;
          }
        }
        stats->gen_s = tg * 1e-3;
        stats->bin_s = tb * 1e-3;
        stats->small_s = ts * 1e-3;
        stats->large_s = tl * 1e-3;
      }
      stats->total_s = t_tot * 1e-3;
      stats->base_primes = nprimes;
      stats->tiles = P.ntiles;
      stats->log_tile = P.log_s;
      stats->waves = (uint32_t)P.nwaves;
      stats->kernel_launches = launches;
    }
    return 0;
  }
}

}  // namespace

extern "C" int erato_gpu_run(erato_gpu_ctx* c, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                             void* dev_table, uint64_t* dev_count, void* stream_v, int sync,
                             erato_gpu_stats* stats) {
  return run_impl(c, l, f, n, flags, dev_table, dev_count, stream_v, sync, stats, nullptr);
}

extern "C" int erato_gpu_count(erato_gpu_ctx* c, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                               uint64_t* count, erato_gpu_stats* stats) {
  erato_gpu_stats local{};
  erato_gpu_stats* s = stats ? stats : &local;
  std::memset(s, 0, sizeof(*s));
  const int rc = erato_gpu_run(c, l, f, n, flags, nullptr, nullptr, nullptr, 1, s);
  if (rc) return rc;
  if (count) *count = s->prime_count;
  return 0;
}

extern "C" int erato_gpu_sieve_to_host(erato_gpu_ctx* c, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                                       uint8_t* dst, size_t dst_cap, erato_gpu_stats* stats) {
  if (!c || !dst) return fail(ERATO_GPU_E_INVALID_ARG, "NULL argument");
  int rc = erato_gpu_validate(l, f, n, flags, nullptr, nullptr);
  if (rc) return rc;
  const uint64_t bytes = (n << l) / 8;
  if (dst_cap < bytes) return fail(ERATO_GPU_E_INVALID_ARG, "dst_cap < table bytes");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(c->table.ensure((bytes + 15) & ~15ull));
  erato_gpu_stats local{};
  erato_gpu_stats* s = stats ? stats : &local;
  std::memset(s, 0, sizeof(*s));
  // pinned destination: copy each wave's slice while the next waves run
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  rc = run_impl(c, l, f, n, flags, c->table.p, nullptr, nullptr, 1, s, pinned ? dst : nullptr);
  if (rc) return rc;
  if (pinned) return 0;  // (output_s stays 0: the copies overlapped the sieve)
  CUDA_TRY(cudaEventRecord(c->ev[0], c->stream));
  CUDA_TRY(cudaMemcpyAsync(dst, c->table.p, bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaEventRecord(c->ev[3], c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev[0], c->ev[3]);
  s->output_s = ms * 1e-3;
  return 0;
}

extern "C" int erato_gpu_write_table(erato_gpu_ctx* c, const char* out_dir, unsigned l, uint64_t f, uint64_t n,
                                     uint64_t part_f, uint64_t part_n, unsigned flags, char* path_out,
                                     size_t path_cap, erato_gpu_stats* stats) {
  if (!c || !out_dir) return fail(ERATO_GPU_E_INVALID_ARG, "NULL argument");
  int rc = erato_gpu_validate(l, f, n, flags, nullptr, nullptr);
  if (rc) return rc;
  if (part_n == 0) {
    part_f = f;
    part_n = n;
  }
  if (part_f < f || part_f + part_n > f + n) return fail(ERATO_GPU_E_INVALID_ARG, "part outside (f, n)");
  // FileSink: create_directories + exact name (driver.cpp:29-36)
  std::string dir(out_dir);
  for (size_t i = 1; i <= dir.size(); ++i)
    if (i == dir.size() || dir[i] == '/') ::mkdir(dir.substr(0, i).c_str(), 0777);
  char name[128];
  erato_gpu_table_filename(l, f, n, name, sizeof(name));
  const std::string path = dir + (dir.empty() || dir.back() == '/' ? "" : "/") + name;
  const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT, 0644);
  if (fd < 0) return fail(ERATO_GPU_IO_ERROR, "cannot open " + path);
  const uint64_t total_bytes = (n << l) / 8;
  if (part_f == f && part_n == n) {
    if (::ftruncate(fd, (off_t)total_bytes) != 0) {
      ::close(fd);
      return fail(ERATO_GPU_IO_ERROR, "truncate failed for " + path);
    }
  }
  const uint64_t bytes = (part_n << l) / 8;
  const uint64_t off = ((part_f - f) << l) / 8;
  std::vector<uint8_t> host;
  uint8_t* pinned = nullptr;
  if (cudaMallocHost(&pinned, bytes ? bytes : 1) != cudaSuccess) {
    cudaGetLastError();
    pinned = nullptr;
    host.resize(bytes);
  }
  uint8_t* dst = pinned ? pinned : host.data();
  rc = erato_gpu_sieve_to_host(c, l, part_f, part_n, flags, dst, bytes, stats);
  if (rc) {
    if (pinned) cudaFreeHost(pinned);
    ::close(fd);
    return rc;
  }
  uint64_t done = 0;
  while (done < bytes) {
    const ssize_t w = ::pwrite(fd, dst + done, (size_t)std::min<uint64_t>(bytes - done, 1ull << 30), (off_t)(off + done));
    if (w <= 0) {
      if (pinned) cudaFreeHost(pinned);
      ::close(fd);
      return fail(ERATO_GPU_IO_ERROR, "short write to " + path);
    }
    done += (uint64_t)w;
  }
  if (pinned) cudaFreeHost(pinned);
  if (::close(fd) != 0) return fail(ERATO_GPU_IO_ERROR, "close failed for " + path);
  if (path_out && path_cap) std::snprintf(path_out, path_cap, "%s", path.c_str());
  return 0;
}

extern "C" int erato_gpu_extract_primes(erato_gpu_ctx* c, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                                        uint64_t* dst, uint64_t cap, uint64_t* count) {
  if (!c) return fail(ERATO_GPU_E_INVALID_ARG, "ctx is NULL");
  uint64_t u = 0, v = 0;
  int rc = erato_gpu_validate(l, f, n, flags, &u, &v);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  const uint64_t T = n << l;
  CUDA_TRY(c->table.ensure(((T / 8) + 15) & ~15ull));
  erato_gpu_stats s{};
  rc = erato_gpu_run(c, l, f, n, flags, c->table.p, nullptr, nullptr, 1, &s);
  if (rc) return rc;
  // the number 1 (bit 0 of an f = 0 run) is a clear bit but not a prime
  const uint64_t lo = (u == 1) ? 1 : 0;
  const uint64_t np = s.prime_count - lo;
  CUDA_TRY(c->outbuf.ensure(std::max<uint64_t>(np, 1) * 8));
  uint64_t* d_total = c->scal.as<uint64_t>() + 40;
  // extract_primes (driver.cpp:65-81): clear bits -> u + 2j
  rc = compact_zeros<uint64_t>(c, c->stream, c->table.as<uint32_t>(), T, lo, u, c->outbuf.as<uint64_t>(), np, d_total);
  if (rc) return rc;
  const uint64_t m = std::min(np, cap);
  if (dst && m) CUDA_TRY(cudaMemcpyAsync(dst, c->outbuf.p, m * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (count) *count = np;
  return 0;
}
