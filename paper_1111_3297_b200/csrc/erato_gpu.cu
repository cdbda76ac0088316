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
//        remainder), advanced to the first cofactor on the mod-30030 wheel
//        -> ML states / far states (next hit + wheel index)
//   waves (the reference's per-segment loop, driver.cpp:93-117)
//     per window of K waves: k_far_walk (far primes -> per-wave record buckets)
//     for each wave of W tiles: k_ml_walk (ML primes -> per-tile hit records),
//     k_wave_sort (the wave's far records -> per-tile hit records), then k_tile
//     (patterns, medium primes, hits, popcount, 128-bit write-out)
//   count: device u64 (NullSink: only it leaves the device).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
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

bool wheel_residues(uint32_t M, std::vector<uint32_t>& res, std::vector<uint16_t>* rank);
uint32_t wheel_delta(const std::vector<uint32_t>& res, uint32_t M, size_t i);

constexpr uint32_t kBaseLogTile = 20;  // tile size for the sieve of [1, sqrt(v)]
constexpr uint32_t kGenBlocksPerSm = 2;
constexpr uint64_t kFewLarge = 2048;  // at most this many primes > S are sieved as medium primes
constexpr int kOutSlots = 4;          // streaming output: wave slices in flight (device and pinned host)

}  // namespace

struct erato_gpu_ctx {
  int device = 0;
  int nsm = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t xstream = nullptr;               // D2H copies of finished waves (sieve_to_host)
  cudaEvent_t xev = nullptr, xjoin = nullptr;   // wave done / copies done
  // k_wave_sort runs beside k_ml_walk on a side stream (both only append to the hit lists)
  cudaStream_t sstream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_sorted = nullptr;
  // early partition (ERATO_GPU_EARLY_SORT): wave w+1's far records are partitioned while wave w runs
  cudaEvent_t ev_walk = nullptr, ev_tile[2] = {}, ev_sort[2] = {};
  // cached per context
  DevBuf sp, spm, ptab;  // small primes < 2^16, their base-sieve records, pattern tables
  std::vector<uint32_t> h_sp;
  // grow-only run buffers
  DevBuf base_bits, primes, med, ml, buckets, bcount, hits, hitcnt, blk_cnt, blk_off, scal, table, outbuf;
  DevBuf recs, rcount, frecs, fslot, fcount;  // k_gen -> k_bin per-warp regions
  DevBuf fst, wbuf, wcnt;                     // windowed far path: prime states, per-wave record buckets
  DevBuf mlst;                                // wheel mode: ML states (pos | idx << 32)
  DevBuf wdelta, wrank;                       // wheel tables of the large primes (cached per modulus)
  uint32_t wheel_M = 0, wheel_nres = 0;
  size_t mem_free0 = 0;                       // free device memory when the context was created
  double hcap_scale = 1.0, bcap_scale = 1.0;
  uint64_t max_base_pairs = uint64_t{1} << 27;  // base.hpp:87
  cudaEvent_t ev[4] = {};
  std::vector<cudaEvent_t> phase_ev;  // pairs, grown on demand
  // streaming output (run_to_sink, sieve_to_host, write_table): a ring of
  // kOutSlots wave slices on the device and in pinned host memory, so no
  // call needs the whole table in HBM or in host memory
  DevBuf slices;
  uint8_t* hslots = nullptr;
  size_t hslots_cap = 0;
  uint64_t* hflags = nullptr;  // pinned [kOutSlots]: overflow flag as of each slot's wave
  cudaEvent_t ev_copy[kOutSlots] = {};
  // extract_primes: the last compaction, reused by a follow-up call with the same key
  uint64_t xp_key[4] = {~0ull, ~0ull, ~0ull, ~0ull};
  uint64_t xp_count = 0;
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

size_t erato_gpu_wheel_deltas(uint32_t M, uint8_t* delta, size_t cap) {
  std::vector<uint32_t> res;
  if (!wheel_residues(M, res, nullptr)) return 0;
  for (size_t i = 0; i < res.size() && i < cap && delta; ++i) delta[i] = (uint8_t)wheel_delta(res, M, i);
  return res.size();
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

namespace {
int create_impl(erato_gpu_ctx* c) {
  const int device = c->device;
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  c->nsm = prop.multiProcessorCount;
  {
    size_t mem_total = 0;
    CUDA_TRY(cudaMemGetInfo(&c->mem_free0, &mem_total));
  }
  CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->xstream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&c->xev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->xjoin, cudaEventDisableTiming));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->sstream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_sorted, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_walk, cudaEventDisableTiming));
  for (int k = 0; k < 2; ++k) {
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_tile[k], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_sort[k], cudaEventDisableTiming));
  }

  for (auto& e : c->ev) CUDA_TRY(cudaEventCreate(&e));
  for (auto& e : c->ev_copy) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CUDA_TRY(cudaMallocHost(&c->hflags, kOutSlots * sizeof(uint64_t)));
  if (const char* e = std::getenv("ERATO_GPU_TEST_CAP_SCALE")) {  // tests only: force capacity overflows
    const double v = std::atof(e);
    if (v > 0) c->hcap_scale = c->bcap_scale = v;
  }
  for (auto kt : {eg::k_tile<false, false>, eg::k_tile<true, false>, eg::k_tile<false, true>, eg::k_tile<true, true>})
    CUDA_TRY(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(eg::kPatWords * 4 + (1u << kBaseLogTile) / 8 + eg::kMaxWarpPrimes * 8 +
                                        eg::kTileWarps * eg::kHitChunk * 4)));
  CUDA_TRY(cudaFuncSetAttribute(eg::k_bin, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(eg::BinSmem)));
  for (auto km : {eg::k_scatter_ml<false>, eg::k_scatter_ml<true>})
    CUDA_TRY(cudaFuncSetAttribute(km, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(eg::MlSmem)));
  for (auto kf : {eg::k_scatter_far<false>, eg::k_scatter_far<true>})
    CUDA_TRY(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(eg::FarSmem)));
  CUDA_TRY(cudaFuncSetAttribute(eg::k_far_walk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(eg::WkSmem) + 16 + eg::kWheelMaxBytes)));
  CUDA_TRY(cudaFuncSetAttribute(eg::k_ml_walk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(eg::MlSmem) + 16 + eg::kWheelMaxBytes)));
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
  return 0;
}
}  // namespace

int erato_gpu_create(int device, erato_gpu_ctx** out) {
  if (!out) return fail(ERATO_GPU_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (erato_gpu_device_count() == 0) return fail(ERATO_GPU_E_NO_DEVICE, "no CUDA device visible");
  if (device < 0) CUDA_TRY(cudaGetDevice(&device));
  auto* c = new erato_gpu_ctx();
  c->device = device;
  const int rc = create_impl(c);
  if (rc) {  // release whatever was created before the failure
    const std::string msg = g_err;
    erato_gpu_destroy(c);
    g_err = msg;
    return rc;
  }
  *out = c;
  return 0;
}

void erato_gpu_destroy(erato_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->xstream) cudaStreamSynchronize(c->xstream);
  if (c->sstream) cudaStreamSynchronize(c->sstream);
  for (DevBuf* b : {&c->sp, &c->spm, &c->ptab, &c->base_bits, &c->primes, &c->med, &c->ml, &c->buckets,
                    &c->bcount, &c->hits, &c->hitcnt, &c->blk_cnt, &c->blk_off, &c->scal, &c->table,
                    &c->outbuf, &c->recs, &c->rcount, &c->frecs, &c->fslot, &c->fcount, &c->slices, &c->fst,
                    &c->wbuf, &c->wcnt, &c->mlst, &c->wdelta, &c->wrank})
    b->release();
  if (c->hslots) cudaFreeHost(c->hslots);
  if (c->hflags) cudaFreeHost(c->hflags);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev_copy)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->phase_ev) cudaEventDestroy(e);
  if (c->xev) cudaEventDestroy(c->xev);
  if (c->xjoin) cudaEventDestroy(c->xjoin);
  if (c->xstream) cudaStreamDestroy(c->xstream);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_sorted) cudaEventDestroy(c->ev_sorted);
  if (c->ev_walk) cudaEventDestroy(c->ev_walk);
  for (int k = 0; k < 2; ++k) {
    if (c->ev_tile[k]) cudaEventDestroy(c->ev_tile[k]);
    if (c->ev_sort[k]) cudaEventDestroy(c->ev_sort[k]);
  }
  if (c->sstream) cudaStreamDestroy(c->sstream);

  if (c->stream) cudaStreamDestroy(c->stream);
  cudaGetLastError();
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

// build_base's simple_sieve(isqrt v) (src/base.cpp:19-53, src/oracle.cpp:8-23) on
// the device: the odd numbers 1..vroot sieved by the tile kernel (multiples
// from p^2), then a popcount-scan compaction into c->primes (ascending u32);
// the count lands in scal[0].
int base_primes(erato_gpu_ctx* c, cudaStream_t st, uint64_t vroot, uint32_t& launches) {
  uint64_t* d_scal = c->scal.as<uint64_t>();
  const uint64_t nbase_bits = (vroot + 1) / 2;  // odd numbers 1..vroot
  const uint64_t prime_cap = pi_upper(vroot) + 64;
  CUDA_TRY(c->primes.ensure(prime_cap * 4));
  if (nbase_bits <= 1) {
    CUDA_TRY(cudaMemsetAsync(d_scal, 0, 8, st));
    return 0;
  }
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
  const int rc = compact_zeros<uint32_t>(c, st, c->base_bits.as<uint32_t>(), nbase_bits, 1, 1,
                                         c->primes.as<uint32_t>(), prime_cap, d_scal + 0);
  if (rc) return rc;
  launches += 3;
  return 0;
}

// Wheel tables of the large primes for modulus M (30, 210, 2310 or 30030):
// delta[i] = half the gap from the i-th residue coprime to M to the next one
// (wrapping), rank[r] = index of residue r (0xffff if not coprime).  Cached.
// residues coprime to M (odd, ascending) and their ranks; false for an unsupported modulus
bool wheel_residues(uint32_t M, std::vector<uint32_t>& res, std::vector<uint16_t>* rank) {
  if (M != 30 && M != 210 && M != 2310 && M != 30030) return false;
  res.clear();
  if (rank) rank->assign(M, 0xffff);
  for (uint32_t r = 1; r < M; r += 2)
    if (r % 3 && r % 5 && (M % 7 || r % 7) && (M % 11 || r % 11) && (M % 13 || r % 13)) {
      if (rank) (*rank)[r] = (uint16_t)res.size();
      res.push_back(r);
    }
  return true;
}
uint32_t wheel_delta(const std::vector<uint32_t>& res, uint32_t M, size_t i) {  // half gap to the next residue (<= 11)
  return ((i + 1 < res.size() ? res[i + 1] : res[0] + M) - res[i]) / 2;
}

int ensure_wheel(erato_gpu_ctx* c, cudaStream_t st, uint32_t M) {
  if (c->wheel_M == M) return 0;
  std::vector<uint32_t> res;
  std::vector<uint16_t> rank;
  if (!wheel_residues(M, res, &rank) || res.size() > eg::kWheelMaxRes || res.size() % 8)
    return fail(ERATO_GPU_E_INVALID_ARG, "wheel modulus");
  std::vector<uint32_t> delta(res.size() / 8 + 1, 0);  // 8 nibbles per word + the wrap-around word
  for (size_t i = 0; i < res.size(); ++i) delta[i / 8] |= wheel_delta(res, M, i) << (4 * (i % 8));
  delta.back() = delta[0];
  // for a cofactor residue c coprime to 30: the first wheel residue >= c (index | half the gap << 16)
  std::vector<uint32_t> next(M, 0xffffffffu);
  for (uint32_t cm = 1; cm < M; cm += 2) {
    if (cm % 3 == 0 || cm % 5 == 0) continue;
    uint32_t c = cm;
    while (rank[c % M] == 0xffff) c += 2;
    next[cm] = rank[c % M] | (((c - cm) / 2) << 16);
  }
  CUDA_TRY(c->wdelta.ensure(eg::kWheelMaxBytes));
  CUDA_TRY(c->wrank.ensure((size_t)30030 * 4));
  CUDA_TRY(cudaMemcpyAsync(c->wdelta.p, delta.data(), delta.size() * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->wrank.p, next.data(), next.size() * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));  // (the host vectors go out of scope)
  c->wheel_M = M;
  c->wheel_nres = (uint32_t)res.size();
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

__global__ void k_finish(const unsigned long long* __restrict__ count, const uint64_t* __restrict__ overflow,
                         uint64_t* __restrict__ out) {
  *out = *overflow ? ERATO_GPU_COUNT_OVERFLOW : (uint64_t)*count;
}

// Streaming output of finished waves (the FileSink / TableSink analog that
// never holds the whole table): wave w's tiles write device slice w % K; the
// slice goes D2H on the copy stream while the next waves sieve, either
// straight into a pinned whole-table destination (host_dst) or into pinned
// slot w % K, which a writer thread hands to fn in order.  A wave is handed
// over only if the overflow flag, copied with it, is clear; after a
// capacity retry the waves already delivered (delivered bytes) are skipped,
// so fn sees every byte exactly once, in order.
struct OutSpec {
  uint8_t* host_dst = nullptr;
  erato_gpu_sink_fn fn = nullptr;
  void* user = nullptr;
  uint64_t delivered = 0;  // bytes handed to fn so far (survives retries)
};

struct WaveJob {
  uint32_t slot;
  uint64_t b0, nbytes;
};

struct Writer {
  erato_gpu_ctx* c = nullptr;
  OutSpec* out = nullptr;
  size_t slice_bytes = 0;
  std::mutex m;
  std::condition_variable cv;
  std::deque<WaveJob> q;
  bool closing = false;
  uint64_t consumed = 0;  // waves taken off the queue and finished with
  int err = 0;            // first failure (ERATO_GPU_IO_ERROR / E_CUDA)
  bool overflow = false;  // a wave arrived with the overflow flag set
  std::string msg;
  std::thread th;

  ~Writer() { finish(); }  // early error returns of run_impl still join the thread
  void start() {
    th = std::thread([this] { loop(); });
  }
  void push(const WaveJob& j) {
    std::lock_guard<std::mutex> g(m);
    q.push_back(j);
    cv.notify_all();
  }
  // block until at least `waves` waves are consumed; false if the run must stop
  bool wait_consumed(uint64_t waves) {
    std::unique_lock<std::mutex> g(m);
    cv.wait(g, [&] { return consumed >= waves || err || overflow; });
    return !(err || overflow);
  }
  void finish() {
    {
      std::lock_guard<std::mutex> g(m);
      closing = true;
      cv.notify_all();
    }
    if (th.joinable()) th.join();
  }
  void loop() {
    cudaSetDevice(c->device);
    for (;;) {
      WaveJob j;
      {
        std::unique_lock<std::mutex> g(m);
        cv.wait(g, [&] { return !q.empty() || closing; });
        if (q.empty()) return;
        j = q.front();
        q.pop_front();
      }
      int e = 0;
      bool ovf = false;
      std::string why;
      const bool stop = err || overflow;
      if (!stop) {
        const cudaError_t ce = cudaEventSynchronize(c->ev_copy[j.slot]);
        if (ce != cudaSuccess) {
          e = ERATO_GPU_E_CUDA;
          why = std::string("copy of a finished wave: ") + cudaGetErrorString(ce);
        } else if (c->hflags[j.slot]) {
          ovf = true;
        } else if (j.b0 + j.nbytes > out->delivered) {
          const uint64_t skip = out->delivered > j.b0 ? out->delivered - j.b0 : 0;
          const uint8_t* src = c->hslots + (size_t)j.slot * slice_bytes + skip;
          if (out->fn(out->user, src, j.b0 + skip, j.nbytes - skip) != 0) {
            e = ERATO_GPU_IO_ERROR;
            why = "sink rejected bytes at offset " + std::to_string(j.b0 + skip);
          } else {
            out->delivered = j.b0 + j.nbytes;
          }
        }
      }
      std::lock_guard<std::mutex> g(m);
      if (e && !err) {
        err = e;
        msg = why;
      }
      if (ovf) overflow = true;
      ++consumed;
      cv.notify_all();
    }
  }
};

int run_impl(erato_gpu_ctx* c, unsigned l, uint64_t f, uint64_t n, unsigned flags, void* dev_table,
             uint64_t* dev_count, void* stream_v, int sync, erato_gpu_stats* stats, OutSpec* out) {
  if (!c) return fail(ERATO_GPU_E_INVALID_ARG, "ctx is NULL");
  if (!sync && (flags & ERATO_GPU_CHECK_INVARIANTS))
    return fail(ERATO_GPU_E_INVALID_ARG, "ERATO_GPU_CHECK_INVARIANTS needs sync = 1 (the checks are read on the host)");
  if (out && (dev_table || !sync)) return fail(ERATO_GPU_E_INVALID_ARG, "streaming output is synchronous and owns the table");
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
  // Large primes, default ("wheel") path: table-driven wheel walks — ML primes
  // per wave (k_ml_walk), far primes per window of waves (k_far_walk) with one
  // partition by tile per wave (k_wave_sort).  ERATO_GPU_LARGE=legacy selects
  // the round-1/2 structures instead (mod-30/210 states, k_scatter_ml, the far
  // bucket ring k_scatter_far, or k_gen/k_bin with ERATO_GPU_SCATTER=genbin).
  // In wheel mode the far class starts at WS / far_div.
  const char* sc_env0 = std::getenv("ERATO_GPU_SCATTER");
  const char* lg_env = std::getenv("ERATO_GPU_LARGE");
  const bool win = !(lg_env && std::strcmp(lg_env, "legacy") == 0) && !(sc_env0 && std::strcmp(sc_env0, "genbin") == 0) &&
                   P.W <= (uint32_t)eg::kScBins;
  uint32_t wheel_M = 30030;
  if (const char* e = std::getenv("ERATO_GPU_WHEEL")) wheel_M = (uint32_t)std::atoi(e);
  if (wheel_M != 30 && wheel_M != 210 && wheel_M != 2310 && wheel_M != 30030)
    return fail(ERATO_GPU_E_INVALID_ARG, "ERATO_GPU_WHEEL must be 30, 210, 2310 or 30030");
  const uint32_t wmask = (wheel_M % 7 == 0 ? 1u : 0u) | (wheel_M % 11 == 0 ? 2u : 0u) | (wheel_M % 13 == 0 ? 4u : 0u);
  const double wdens = (8.0 / 15.0) * ((wmask & 1) ? 6.0 / 7.0 : 1.0) * ((wmask & 2) ? 10.0 / 11.0 : 1.0) *
                       ((wmask & 4) ? 12.0 / 13.0 : 1.0);  // records per odd multiple
  if (win) {
    rc = ensure_wheel(c, st, wheel_M);
    if (rc) return rc;
  }
  // (cfg5, same-box A/B: far_div 1 / 2 / 4 / 8 = 54.1 / 51.4 / 49.9 / 50.1 ms — an ML prime above WS/4 hits a
  // wave less than twice, and the per-wave walk pays a state round trip and 2-3 mostly idle steps for it)
  uint32_t far_div = 4;
  if (const char* e = std::getenv("ERATO_GPU_FAR_DIV")) far_div = (uint32_t)std::max(1, std::atoi(e));
  uint32_t kwin_max = 128;
  if (const char* e = std::getenv("ERATO_GPU_FAR_WINDOW")) kwin_max = (uint32_t)std::max(1, std::atoi(e));
  kwin_max = std::min<uint32_t>(kwin_max, eg::kScBins);

  // Early partition (default; ERATO_GPU_EARLY_SORT=0: the wave's own partition beside its ML walk): wave
  // w+1's far records are split by tile on the side stream while wave w's ML walk and tiles run, into a
  // second set of hit lists (cfg5 45.6 -> 44.9 ms; with a 16 KB smaller k_tile and 256-thread partition
  // CTAs that fit beside a tile CTA: 48.3 ms)
  const char* es_env = std::getenv("ERATO_GPU_EARLY_SORT");
  const bool early_req = win && !(flags & (ERATO_GPU_PHASE_TIMING | ERATO_GPU_CHECK_INVARIANTS)) &&
                         !(es_env && std::strcmp(es_env, "0") == 0);
  uint32_t launches = 0;
  for (int attempt = 0;; ++attempt) {
    const uint64_t vroot = isqrt_u64(P.v);
    CUDA_TRY(cudaEventRecord(c->ev[0], st));
    // ---------------- 1-2. base primes <= sqrt(v) ----------------
    // [0] total primes, [8..15] bounds + largest prime, [16] count, [17] overflow,
    // [18] hit records consumed, [19] expected records, [20] base-sieve count, [21] bad far entry,
    // [22] pattern-phase ns (PHASE_TIMING), [24..30] class thresholds, [40] compaction total
    uint64_t* d_scal = c->scal.as<uint64_t>();
    CUDA_TRY(cudaMemsetAsync(d_scal + 18, 0, 16, st));
    CUDA_TRY(cudaMemsetAsync(d_scal + 21, 0, 8, st));
    CUDA_TRY(cudaMemsetAsync(d_scal + 23, 0, 8, st));  // [23] far records (CHECK_INVARIANTS)
    rc = base_primes(c, st, vroot, launches);
    if (rc) return rc;
    // ---------------- 3. class boundaries (one host sync) ----------------
    // index of the first prime above 61, S/64, S, MW*WS, max(WS/8, S), S/256, S/128
    const uint64_t p_ml = win ? std::max<uint64_t>(P.WS / far_div, P.S) : (uint64_t)P.MW * P.WS;  // largest ML prime
    uint64_t thr[7] = {61, (uint64_t)P.S / 64, P.S, p_ml, std::max<uint64_t>(P.WS / 8, P.S),
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
    uint32_t kwin = 1, wcap = 4, wmagic = 0;  // window mode: waves per window, records per wave bucket
    bool split = false, far7 = false, ml7 = false;
    if (have_large) {
      const double lnP = std::log((double)std::max<uint32_t>(pmax, 3));
      const double sum_recip = std::max(0.0, std::log(lnP / std::log((double)P.S))) + 0.02;  // sum 1/p, S<p<=P
      const double eh = (double)P.S * (8.0 / 15.0) * sum_recip;
      hcap = (uint32_t)std::min<double>(((eh * 1.10 + 4096) * c->hcap_scale), (double)P.S * 4);
      hcap = (hcap + 3) & ~3u;
      CUDA_TRY(c->ml.ensure(std::max<uint64_t>(nml, 1) * 8));
      if (win) CUDA_TRY(c->mlst.ensure(std::max<uint64_t>(nml, 1) * 8));
      // the lists of the MW waves of an ML window, + trash of the split scatter
      const uint32_t nlists = early_req ? 2 : P.MW;
      CUDA_TRY(c->hits.ensure(((uint64_t)nlists * P.W * hcap + eg::kScTrash) * 4));
      CUDA_TRY(c->hitcnt.ensure((uint64_t)nlists * P.W * 4));
      CUDA_TRY(cudaMemsetAsync(c->hitcnt.p, 0, (uint64_t)nlists * P.W * 4, st));
      if (nfar && win) {
        const double sr_far = std::max(0.0, std::log(lnP / std::log((double)p_ml))) + 0.01;
        const double ew = (double)P.WS * wdens * sr_far;  // records per wave
        wcap = (uint32_t)std::min<double>((ew * 1.10 + 8192) * c->bcap_scale, 1u << 30);
        wcap = (wcap + 3) & ~3u;
        const uint64_t nwin = (P.nwaves + kwin_max - 1) / kwin_max;
        kwin = (uint32_t)((P.nwaves + nwin - 1) / nwin);
        // (the window's record buckets: at most 6 GiB and a quarter of the device memory that is free now)
        // (free memory as of the context's creation: cudaMemGetInfo costs milliseconds, not per run)
        uint64_t wmax = 6ull << 30;
        if (const char* e = std::getenv("ERATO_GPU_FAR_BUDGET_GB")) wmax = (uint64_t)std::max(1, std::atoi(e)) << 30;
        const uint64_t wbudget = std::min<uint64_t>(wmax, std::max<uint64_t>(c->mem_free0 / 4, 64ull << 20));
        while (kwin > 1 && ((uint64_t)kwin * wcap + eg::kScTrash >= (1ull << 32) || (uint64_t)kwin * wcap * 4 > wbudget))
          kwin = (kwin + 1) / 2;
        wmagic = (uint32_t)((1ull << 32) / P.W) + 1;  // umulhi(t, wmagic) = t / W for t * W < 2^32
        CUDA_TRY(c->fst.ensure(nfar * 8));
        CUDA_TRY(c->wbuf.ensure(((uint64_t)kwin * wcap + eg::kScTrash) * 4));
        CUDA_TRY(c->wcnt.ensure((uint64_t)eg::kScBins * 4));
      } else if (nfar) {
        // an entry's next hit lies at most 3p (mod 30) or 5p (mod 210: two wheel steps) ahead
        ring = (uint32_t)std::min<uint64_t>(6ull * pmax / P.WS + 3, P.nwaves + 2);
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
      // large-prime path: k_scatter_ml + k_scatter_far (default), or k_gen +
      // k_bin (ERATO_GPU_SCATTER=genbin, or when a wave has more than 256 tiles
      // or ring slots, or 32-bit list offsets do not fit)
      const char* sc_env = std::getenv("ERATO_GPU_SCATTER");
      const bool sortable = ring <= (uint32_t)eg::kScBins && (uint64_t)P.MW * P.W <= (uint64_t)eg::kScBins;
      const bool idx32 = (uint64_t)P.MW * P.W * hcap + eg::kScTrash < (1ull << 32) &&
                         (uint64_t)ring * bcap + eg::kScTrash < (1ull << 32);
      split = sortable && idx32 && !(sc_env && std::strcmp(sc_env, "genbin") == 0);
      // far primes skip cofactors divisible by 7 (mod-210 entries) when p < 2^31 and q < 2^28 fit
      const char* f7_env = std::getenv("ERATO_GPU_FAR7");
      far7 = split && !win && nfar && pmax < (1u << 31) && P.WS <= (1u << 28) &&
             !(f7_env && std::strcmp(f7_env, "0") == 0);
      // ML primes too (p < 2^28 and next-hit offsets < 6p < 2^30 need WS <= 170 * 2^20), when they all
      // hit a wave >= ~4 times (p <= WS/8: cfg4 -7% ML time); with primes up to WS (cfg5) the extra
      // data-dependent step in the walk costs more than the skipped records save (+13% measured)
      const char* m7_env = std::getenv("ERATO_GPU_ML7");
      ml7 = split && !win && nml && P.MW == 1 && P.WS <= 170u * (1u << 20) &&
            (m7_env ? std::strcmp(m7_env, "1") == 0 : idense >= iWS);
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
      sa.far7 = far7 ? 1 : 0;
      sa.ml7 = ml7 ? 1 : 0;
      if (win) {
        sa.fst = c->fst.as<uint64_t>();
        sa.mlst = c->mlst.as<uint64_t>();
        sa.wnext = c->wrank.as<uint32_t>();
        sa.wM = wheel_M;
        sa.wR32 = (uint32_t)((1ull << 32) % wheel_M);
        sa.wmask = wmask;
      }
      const uint64_t nl = nprimes - iS;
      eg::k_setup_large<<<(unsigned)((nl + eg::kSetupThreads - 1) / eg::kSetupThreads), eg::kSetupThreads, 0, st>>>(sa);
      ++launches;
      if (flags & ERATO_GPU_CHECK_INVARIANTS) {
        // expected hit records: admissible multiples of the large primes in the tiles
        const unsigned __int128 x_hi = (unsigned __int128)P.u + 2 * (unsigned __int128)(P.ntiles << P.log_s) - 2;
        const uint64_t xh = x_hi > UINT64_MAX ? UINT64_MAX : (uint64_t)x_hi;
        eg::k_expected_records<<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(
            c->primes.as<uint32_t>(), iS, nprimes, P.u, xh, reinterpret_cast<unsigned long long*>(d_scal + 19),
            win ? iS : (ml7 ? iS : (far7 ? iWS : nprimes)), win ? nprimes : (far7 ? nprimes : iWS), win ? wmask : 1u);
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
    // streaming output: K wave slices on the device (+ pinned slots for a sink)
    const uint64_t slice_bytes = std::min<uint64_t>((uint64_t)P.W << P.log_s, P.T) / 8;
    Writer wr;
    if (out) {
      CUDA_TRY(c->slices.ensure(((slice_bytes + 15) & ~15ull) * kOutSlots));
      if (out->fn && c->hslots_cap < slice_bytes * kOutSlots) {
        if (c->hslots) cudaFreeHost(c->hslots);
        c->hslots = nullptr;
        c->hslots_cap = 0;
        CUDA_TRY(cudaMallocHost(&c->hslots, slice_bytes * kOutSlots));
        c->hslots_cap = slice_bytes * kOutSlots;
      }
      if (out->fn) {
        wr.c = c;
        wr.out = out;
        wr.slice_bytes = slice_bytes;
        wr.start();
      }
    }
    auto stop_writer = [&]() {
      if (out && out->fn) wr.finish();
    };
    ta.count = d_count;
    ta.tbase = 0;
    const bool timing = (flags & ERATO_GPU_PHASE_TIMING) != 0;
    if (timing) {
      CUDA_TRY(cudaMemsetAsync(d_scal + 22, 0, 8, st));
      ta.phase_ns = reinterpret_cast<unsigned long long*>(d_scal + 22);
    }
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
    int sa_inject = 0;
    if (const char* inj = std::getenv("ERATO_GPU_TEST_INJECT")) sa_inject = std::atoi(inj);  // tests only
    eg::ScatterArgs sca{};
    uint32_t ml_blocks = c->nsm, far_blocks = c->nsm, walk_blocks = c->nsm;
    const bool winfar = win && nfar > 0;
    const bool wml = win && nml > 0;  // wheel-mode ML walk (k_ml_walk)
    // the wave's far-record partition beside the ML walk (not with per-launch timing events)
    const char* cs_env = std::getenv("ERATO_GPU_SORT_STREAM");
    const bool conc_sort = !timing && !(cs_env && std::strcmp(cs_env, "0") == 0);
    int ml_ctas = 0;  // ML-walk CTAs per SM (0: as many as fit)
    if (const char* e = std::getenv("ERATO_GPU_ML_CTAS")) ml_ctas = std::atoi(e);
    const size_t wsm_ml = ((sizeof(eg::MlSmem) + 15) & ~size_t{15}) + c->wheel_nres / 2 + 4;
    const size_t wsm_far = ((sizeof(eg::WkSmem) + 15) & ~size_t{15}) + c->wheel_nres / 2 + 4;
    eg::Wheel wheel{c->wdelta.as<uint32_t>(), c->wheel_nres};
    uint32_t mlw_blocks = c->nsm;
    eg::MlWalkArgs mwa{};
    eg::FarWalkArgs fwa{};
    eg::WaveSortArgs wsa{};
    wsa.log_s = P.log_s;
    wsa.hcap = hcap;
    wsa.overflow = reinterpret_cast<int*>(d_scal + 17);
    if (wml) {
      int occ = 1;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, eg::k_ml_walk, eg::kMlWarps * 32, wsm_ml));
      const uint64_t units = (nml + 31) / 32;
      if (ml_ctas > 0) occ = std::min(occ, ml_ctas);
      int over = 1;  // CTAs per resident slot (more, shorter CTAs: the hardware scheduler evens out the tail)
      if (const char* e = std::getenv("ERATO_GPU_ML_OVER")) over = std::max(1, std::atoi(e));
      mlw_blocks = (uint32_t)std::min<uint64_t>((uint64_t)c->nsm * (uint32_t)std::max(occ, 1) * over,
                                                std::max<uint64_t>(1, (units + eg::kMlWarps - 1) / eg::kMlWarps));
      mwa.primes = c->primes.as<uint32_t>() + iS;
      mwa.st = c->mlst.as<uint64_t>();
      mwa.nml = (uint32_t)nml;
      mwa.wheel = wheel;
    }
    if (winfar) {
      int occ = 1;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, eg::k_far_walk, eg::kWkWarps * 32, wsm_far));
      const uint64_t units = (nfar + 31) / 32;
      int wover = 16;  // (cfg5: 1 / 2 / 4 / 8 / 16 CTAs per resident slot = 8.87 / 8.74 / 8.60 / 8.44 / 8.35 ms of far walk)
      if (const char* e = std::getenv("ERATO_GPU_WALK_OVER")) wover = std::max(1, std::atoi(e));
      walk_blocks = (uint32_t)std::min<uint64_t>((uint64_t)c->nsm * (uint32_t)std::max(occ, 1) * wover,
                                                 std::max<uint64_t>(1, (units + eg::kWkWarps - 1) / eg::kWkWarps));
      fwa.primes = c->primes.as<uint32_t>() + iWS;
      fwa.st = c->fst.as<uint64_t>();
      fwa.nfar = (uint32_t)nfar;
      fwa.span = (uint64_t)kwin * P.WS;
      fwa.WS = P.WS;
      fwa.log_s = P.log_s;
      fwa.magic = wmagic;
      fwa.wbuf = c->wbuf.as<uint32_t>();
      fwa.wcnt = c->wcnt.as<uint32_t>();
      fwa.wcap = wcap;
      fwa.trash_at = kwin * wcap;
      fwa.overflow = reinterpret_cast<int*>(d_scal + 17);
      fwa.wheel = wheel;
    }
    if (split) {
      int occ = 1;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, eg::k_scatter_ml<false>, eg::kMlWarps * 32,
                                                             sizeof(eg::MlSmem)));
      // no more CTAs than units of work (small runs: a handful of ML primes)
      const uint64_t ml_units = (nml + 31) / 32;
      ml_blocks = (uint32_t)std::min<uint64_t>((uint64_t)c->nsm * (uint32_t)std::max(occ, 1),
                                               std::max<uint64_t>(1, (ml_units + eg::kMlWarps - 1) / eg::kMlWarps));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, eg::k_scatter_far<false>, eg::kFarWarps * 32,
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
    const size_t nev = timing ? (size_t)P.nwaves * 7 + 8 : 0;
    while (c->phase_ev.size() < nev) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      c->phase_ev.push_back(e);
    }
    size_t evi = 0;
    std::vector<std::pair<size_t, bool>> ev_pairs;  // (first event index, is_scatter)
    std::vector<size_t> walk_ev;                    // first event index of each k_far_walk launch
    for (uint64_t w = 0; w < P.nwaves; ++w) {
      const uint64_t tile0 = w * P.W;
      const uint32_t ntw = (uint32_t)std::min<uint64_t>(P.W, P.ntiles - tile0);
      if (have_large) {
        ga.wave = w;
        ga.ntiles_w = ntw;
        ba.ntiles_w = ntw;
        const uint32_t slot = nfar ? (uint32_t)(w % ring) : 0;
        ga.far_in = (nfar && !winfar) ? c->buckets.as<uint64_t>() + (uint64_t)slot * bcap : nullptr;
        ga.far_in_count = c->bcount.as<uint32_t>() + slot;
        if (timing) CUDA_TRY(cudaEventRecord(c->phase_ev[evi], st));
        // this wave's hit lists inside the ML window's lists
        const bool early = early_req && winfar && wml;
        const uint32_t wi = early ? (uint32_t)(w & 1) : (uint32_t)(w % P.MW);
        uint32_t* const hits_w = c->hits.as<uint32_t>() + (uint64_t)wi * P.W * hcap;
        uint32_t* const hitcnt_w = c->hitcnt.as<uint32_t>() + (uint64_t)wi * P.W;
        ta.hits = hits_w;
        ta.hitcnt = hitcnt_w;
        cudaStream_t sst = st;  // stream of the wave's far-record partition
        if (split && early) {
          // wave x's far records -> the hit lists x & 1, on the side stream, as soon as those lists' last
          // tiles (wave x - 2) are done and the window's walk has filled the bucket
          auto issue_sort = [&](uint64_t x) -> int {
            const uint32_t bx = (uint32_t)(x & 1), xl = (uint32_t)(x % kwin);
            cudaStream_t ss = c->sstream;
            CUDA_TRY(cudaStreamWaitEvent(ss, x >= 2 ? c->ev_tile[bx] : c->ev_fork, 0));
            if (xl == 0) CUDA_TRY(cudaStreamWaitEvent(ss, c->ev_walk, 0));
            wsa.in[0] = c->wbuf.as<uint32_t>() + (uint64_t)xl * wcap;
            wsa.in_count[0] = c->wcnt.as<uint32_t>() + xl;
            wsa.cap[0] = wcap;
            wsa.nb = (uint32_t)std::min<uint64_t>(P.W, P.ntiles - x * P.W);
            wsa.hits = c->hits.as<uint32_t>() + (uint64_t)bx * P.W * hcap;
            wsa.hitcnt = c->hitcnt.as<uint32_t>() + (uint64_t)bx * P.W;
            eg::k_wave_sort<<<dim3((wcap + eg::kWsChunk - 1) / eg::kWsChunk, 1), eg::kWsThreads, 0, ss>>>(wsa);
            CUDA_TRY(cudaEventRecord(c->ev_sort[bx], ss));
            launches += 1;
            return 0;
          };
          if (w == 0) CUDA_TRY(cudaEventRecord(c->ev_fork, st));
          if ((uint32_t)(w % kwin) == 0) {  // a new window: walk the far primes through its waves
            const uint64_t tiles_left = P.ntiles - tile0;
            fwa.nbins = (uint32_t)std::min<uint64_t>(kwin, P.nwaves - w);
            fwa.lim = std::min<uint64_t>((uint64_t)kwin * P.W, tiles_left) << P.log_s;
            CUDA_TRY(cudaMemsetAsync(c->wcnt.p, 0, (uint64_t)eg::kScBins * 4, st));
            eg::k_far_walk<<<walk_blocks, eg::kWkWarps * 32, wsm_far, st>>>(fwa);
            launches += 1;
            CUDA_TRY(cudaEventRecord(c->ev_walk, st));
            rc = issue_sort(w);
            if (rc) return rc;
          }
          mwa.sc = sca;
          mwa.sc.ntiles_w = ntw;
          mwa.sc.hits = hits_w;
          mwa.sc.hitcnt = hitcnt_w;
          eg::k_ml_walk<<<mlw_blocks, eg::kMlWarps * 32, wsm_ml, st>>>(mwa);
          launches += 1;
          if (w + 1 < P.nwaves && (uint32_t)((w + 1) % kwin) != 0) {
            rc = issue_sort(w + 1);
            if (rc) return rc;
          }
          CUDA_TRY(cudaStreamWaitEvent(st, c->ev_sort[wi], 0));
        } else if (split) {
          if (winfar && (uint32_t)(w % kwin) == 0) {  // a new window: walk the far primes through its waves
            const uint64_t tiles_left = P.ntiles - tile0;
            fwa.nbins = (uint32_t)std::min<uint64_t>(kwin, P.nwaves - w);
            fwa.lim = std::min<uint64_t>((uint64_t)kwin * P.W, tiles_left) << P.log_s;
            CUDA_TRY(cudaMemsetAsync(c->wcnt.p, 0, (uint64_t)eg::kScBins * 4, sst));
            if (timing) CUDA_TRY(cudaEventRecord(c->phase_ev[nev - 2 * walk_ev.size() - 1], st));
            eg::k_far_walk<<<walk_blocks, eg::kWkWarps * 32, wsm_far, sst>>>(fwa);
            if (timing) {
              CUDA_TRY(cudaEventRecord(c->phase_ev[nev - 2 * walk_ev.size() - 2], st));
              walk_ev.push_back(nev - 2 * walk_ev.size() - 1);
            }
            launches += 1;
            if (w == 0 && sa_inject == 2) eg::k_inject_wrec<<<1, 1, 0, sst>>>(fwa.wbuf, fwa.wcnt);  // tests only
            if (timing) CUDA_TRY(cudaEventRecord(c->phase_ev[evi], st));  // (the wave's ML interval starts here)
          }
          // k_wave_sort runs beside k_ml_walk on the side stream: both only append to the hit lists
          if (conc_sort && winfar && wml) {
            sst = c->sstream;
            CUDA_TRY(cudaEventRecord(c->ev_fork, st));
            CUDA_TRY(cudaStreamWaitEvent(sst, c->ev_fork, 0));
          }
          if (wml) {
            mwa.sc = sca;
            mwa.sc.ntiles_w = ntw;
            mwa.sc.hits = hits_w;
            mwa.sc.hitcnt = hitcnt_w;
            eg::k_ml_walk<<<mlw_blocks, eg::kMlWarps * 32, wsm_ml, st>>>(mwa);
            launches += 1;
          } else if (nml && wi == 0) {  // ML walk over the window's tiles, state re-based by the window span
            eg::ScatterArgs m = sca;
            m.ntiles_w = (uint32_t)std::min<uint64_t>((uint64_t)P.MW * P.W, P.ntiles - tile0);
            m.WS = P.MW * P.WS;
            m.hits = c->hits.as<uint32_t>();
            m.hitcnt = c->hitcnt.as<uint32_t>();
            if (ml7) eg::k_scatter_ml<true><<<ml_blocks, eg::kMlWarps * 32, sizeof(eg::MlSmem), st>>>(m);
            else eg::k_scatter_ml<false><<<ml_blocks, eg::kMlWarps * 32, sizeof(eg::MlSmem), st>>>(m);
            launches += 1;
          }
          if (timing) CUDA_TRY(cudaEventRecord(c->phase_ev[evi + 1], st));
          uint32_t nseg = 0, max_cap = 0;  // record segments k_wave_sort partitions by tile
          if (winfar) {
            const uint32_t wl = (uint32_t)(w % kwin);
            const uint32_t* in = c->wbuf.as<uint32_t>() + (uint64_t)wl * wcap;
            const uint32_t* in_count = c->wcnt.as<uint32_t>() + wl;
            if (flags & ERATO_GPU_CHECK_INVARIANTS) {
              eg::k_check_wrecs<<<(unsigned)c->nsm, 256, 0, sst>>>(in, in_count, wcap, ntw << P.log_s,
                                                                  reinterpret_cast<int*>(d_scal + 21),
                                                                  reinterpret_cast<unsigned long long*>(d_scal + 23));
              ++launches;
            }
            wsa.in[nseg] = in;
            wsa.in_count[nseg] = in_count;
            wsa.cap[nseg] = wcap;
            ++nseg;
            max_cap = std::max(max_cap, wcap);
          } else if (nfar) {
            sca.wave = w;
            sca.wslot = slot;
            sca.ntiles_w = ntw;
            sca.far_in = ga.far_in;
            sca.far_in_count = ga.far_in_count;
            sca.hits = hits_w;
            sca.hitcnt = hitcnt_w;
            if (far7) eg::k_scatter_far<true><<<far_blocks, eg::kFarWarps * 32, sizeof(eg::FarSmem), st>>>(sca);
            else eg::k_scatter_far<false><<<far_blocks, eg::kFarWarps * 32, sizeof(eg::FarSmem), st>>>(sca);
            launches += 1;
          }
          if (nseg) {  // one chunk per CTA; CTAs past a segment's count exit
            wsa.nb = ntw;
            wsa.hits = hits_w;
            wsa.hitcnt = hitcnt_w;
            const uint32_t chunks = (max_cap + eg::kWsChunk - 1) / eg::kWsChunk;
            eg::k_wave_sort<<<dim3(chunks, nseg), eg::kWsThreads, 0, sst>>>(wsa);
            launches += 1;
          }
          if (sst != st) {  // join before the tiles
            CUDA_TRY(cudaEventRecord(c->ev_sorted, sst));
            CUDA_TRY(cudaStreamWaitEvent(st, c->ev_sorted, 0));
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
        ta.reset_bucket_count = (nfar && !winfar) ? c->bcount.as<uint32_t>() + slot : nullptr;
        if (flags & ERATO_GPU_CHECK_INVARIANTS) {
          eg::k_check_wave<<<(unsigned)c->nsm, 256, 0, st>>>(
              hitcnt_w, ntw, hcap, (nfar && !winfar) ? ga.far_in : nullptr, ga.far_in_count, bcap, P.WS,
              reinterpret_cast<unsigned long long*>(d_scal + 18), reinterpret_cast<int*>(d_scal + 21), far7 ? 1 : 0);
          ++launches;
        }
      }
      ta.tile0 = tile0;
      const uint32_t oslot = (uint32_t)(w % kOutSlots);
      if (out) {  // this wave's tiles go to slice oslot once its previous wave has left it
        if (out->fn && w >= kOutSlots && !wr.wait_consumed(w - kOutSlots + 1)) break;
        if (w >= kOutSlots) CUDA_TRY(cudaStreamWaitEvent(st, c->ev_copy[oslot], 0));
        ta.table = reinterpret_cast<uint32_t*>(c->slices.as<uint8_t>() + (size_t)oslot * ((slice_bytes + 15) & ~15ull));
        ta.out_tile0 = tile0;
      }
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
      if (have_large && early_req && winfar && nml) CUDA_TRY(cudaEventRecord(c->ev_tile[w & 1], st));
      if (out) {  // output pipeline: this wave's bytes go to the host now
        const uint64_t b0 = (tile0 << P.log_s) / 8, b1 = std::min<uint64_t>((tile0 + ntw) << P.log_s, P.T) / 8;
        CUDA_TRY(cudaEventRecord(c->xev, st));
        CUDA_TRY(cudaStreamWaitEvent(c->xstream, c->xev, 0));
        uint8_t* dst = out->fn ? c->hslots + (size_t)oslot * slice_bytes : out->host_dst + b0;
        CUDA_TRY(cudaMemcpyAsync(dst, ta.table, b1 - b0, cudaMemcpyDeviceToHost, c->xstream));
        if (out->fn)
          CUDA_TRY(cudaMemcpyAsync(c->hflags + oslot, d_scal + 17, 8, cudaMemcpyDeviceToHost, c->xstream));
        CUDA_TRY(cudaEventRecord(c->ev_copy[oslot], c->xstream));
        if (out->fn) wr.push(WaveJob{oslot, b0, b1 - b0});
      }
      if (timing) {
        CUDA_TRY(cudaEventRecord(c->phase_ev[evi + 1], st));
        ev_pairs.push_back({evi, false});
        evi += 2;
      }
      ++launches;
    }
    if (early_req) {  // join the side stream (a partition may be pending after an early exit of the loop)
      CUDA_TRY(cudaEventRecord(c->ev_sorted, c->sstream));
      CUDA_TRY(cudaStreamWaitEvent(st, c->ev_sorted, 0));
    }
    if (out) {  // join the copies
      CUDA_TRY(cudaEventRecord(c->xjoin, c->xstream));
      CUDA_TRY(cudaStreamWaitEvent(st, c->xjoin, 0));
    }
    CUDA_TRY(cudaGetLastError());
    // the caller's count, or ERATO_GPU_COUNT_OVERFLOW if a capacity overflowed
    // (visible on the device without a host sync when sync = 0)
    if (dev_count) k_finish<<<1, 1, 0, st>>>(d_count, d_scal + 17, dev_count);
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
    uint64_t res[8];  // d_scal[16..23]
    CUDA_TRY(cudaMemcpyAsync(res, d_scal + 16, sizeof(res), cudaMemcpyDeviceToHost, st));
    const cudaError_t se = cudaStreamSynchronize(st);
    stop_writer();
    if (se != cudaSuccess) return fail(ERATO_GPU_E_CUDA, std::string("run: ") + cudaGetErrorString(se));
    if (out && out->fn && wr.err) return fail(wr.err, wr.msg);
    if (out && out->fn && !wr.overflow && out->delivered != P.T / 8 && !res[1])
      return fail(ERATO_GPU_E_CUDA, "streaming output incomplete");
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
        stats->masks_s = (double)res[6] * 1e-9;
        double tw = 0;
        for (const size_t e0 : walk_ev) {
          float ms = 0;
          cudaEventElapsedTime(&ms, c->phase_ev[e0], c->phase_ev[e0 - 1]);
          tw += ms;
        }
        stats->walk_s = tw * 1e-3;
        tb += tw;  // (the walks run before their window's first wave interval)
        tl += tw;
        stats->bin_s = tb * 1e-3;
        stats->small_s = ts * 1e-3;
        stats->large_s = tl * 1e-3;
      }
      stats->total_s = t_tot * 1e-3;
      stats->medium_primes = nmed;
      stats->ml_primes = nml;
      stats->far_primes = nfar;
      stats->skip7 = win ? ((wmask & 1) ? 3u : 0u) : (far7 ? 1u : 0u) | (ml7 ? 2u : 0u);
      stats->wheel = win && have_large ? wheel_M : 0;
      stats->far_records = res[7];
      stats->far_windows = (win && nfar) ? (uint32_t)((P.nwaves + kwin - 1) / kwin) : 0;
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

extern "C" int erato_gpu_run_to_sink(erato_gpu_ctx* c, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                                     erato_gpu_sink_fn fn, void* user, erato_gpu_stats* stats) {
  if (!c || !fn) return fail(ERATO_GPU_E_INVALID_ARG, "NULL argument");
  erato_gpu_stats local{};
  erato_gpu_stats* s = stats ? stats : &local;
  std::memset(s, 0, sizeof(*s));
  OutSpec o;
  o.fn = fn;
  o.user = user;
  return run_impl(c, l, f, n, flags, nullptr, nullptr, nullptr, 1, s, &o);
}

namespace {
struct HostCopy {
  uint8_t* dst;
};
int host_copy_fn(void* user, const uint8_t* bytes, uint64_t offset, uint64_t nbytes) {
  std::memcpy(static_cast<HostCopy*>(user)->dst + offset, bytes, nbytes);
  return 0;
}
}  // namespace

extern "C" int erato_gpu_sieve_to_host(erato_gpu_ctx* c, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                                       uint8_t* dst, size_t dst_cap, erato_gpu_stats* stats) {
  if (!c || !dst) return fail(ERATO_GPU_E_INVALID_ARG, "NULL argument");
  int rc = erato_gpu_validate(l, f, n, flags, nullptr, nullptr);
  if (rc) return rc;
  const uint64_t bytes = (n << l) / 8;
  if (dst_cap < bytes) return fail(ERATO_GPU_E_INVALID_ARG, "dst_cap < table bytes");
  CUDA_TRY(cudaSetDevice(c->device));
  erato_gpu_stats local{};
  erato_gpu_stats* s = stats ? stats : &local;
  std::memset(s, 0, sizeof(*s));
  // pinned destination: each wave's slice is copied straight into it while
  // the next waves run; pageable: through the pinned slots
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  OutSpec o;
  HostCopy hc{dst};
  if (pinned) {
    o.host_dst = dst;
  } else {
    o.fn = host_copy_fn;
    o.user = &hc;
  }
  return run_impl(c, l, f, n, flags, nullptr, nullptr, nullptr, 1, s, &o);
}

namespace {
struct FileOut {
  int fd;
  uint64_t base;  // byte offset of this shard in the file
};
int pwrite_fn(void* user, const uint8_t* bytes, uint64_t offset, uint64_t nbytes) {
  auto* fo = static_cast<FileOut*>(user);
  uint64_t done = 0;
  while (done < nbytes) {
    const ssize_t w = ::pwrite(fo->fd, bytes + done, (size_t)std::min<uint64_t>(nbytes - done, 1ull << 30),
                               (off_t)(fo->base + offset + done));
    if (w <= 0) return 1;
    done += (uint64_t)w;
  }
  return 0;
}

// FileSink: create_directories + exact name (driver.cpp:17-36)
std::string table_path(const char* out_dir, unsigned l, uint64_t f, uint64_t n) {
  std::string dir(out_dir);
  for (size_t i = 1; i <= dir.size(); ++i)
    if (i == dir.size() || dir[i] == '/') ::mkdir(dir.substr(0, i).c_str(), 0777);
  char name[128];
  erato_gpu_table_filename(l, f, n, name, sizeof(name));
  return dir + (dir.empty() || dir.back() == '/' ? "" : "/") + name;
}

// Stream the shard (part_f, part_n) of (l, f, n) into fd at its byte offset.
int write_shard(erato_gpu_ctx* c, int fd, unsigned l, uint64_t f, uint64_t part_f, uint64_t part_n,
                unsigned flags, erato_gpu_stats* stats) {
  FileOut fo{fd, ((part_f - f) << l) / 8};
  return erato_gpu_run_to_sink(c, l, part_f, part_n, flags, pwrite_fn, &fo, stats);
}
}  // namespace

extern "C" int erato_gpu_write_table(erato_gpu_ctx* c, const char* out_dir, unsigned l, uint64_t f, uint64_t n,
                                     uint64_t part_f, uint64_t part_n, unsigned flags, char* path_out,
                                     size_t path_cap, erato_gpu_stats* stats) {
  if (!c || !out_dir) return fail(ERATO_GPU_E_INVALID_ARG, "NULL argument");
  int rc = erato_gpu_validate(l, f, n, flags, nullptr, nullptr);
  if (rc) return rc;
  if (part_f < f || part_n > n || part_f - f > n - part_n) return fail(ERATO_GPU_E_INVALID_ARG, "part outside (f, n)");
  const std::string path = table_path(out_dir, l, f, n);
  const uint64_t total_bytes = (n << l) / 8;
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (part_f == f && part_n == n) {
    // whole table: stream into a temporary file, rename on success (a failed
    // run never leaves a table at the reference name)
    const std::string tmp = path + ".tmp." + std::to_string(::getpid());
    const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) return fail(ERATO_GPU_IO_ERROR, "cannot open " + tmp);
    rc = write_shard(c, fd, l, f, f, n, flags, stats);
    if (!rc && ::ftruncate(fd, (off_t)total_bytes) != 0) rc = fail(ERATO_GPU_IO_ERROR, "truncate failed for " + tmp);
    if (::close(fd) != 0 && !rc) rc = fail(ERATO_GPU_IO_ERROR, "close failed for " + tmp);
    if (!rc && ::rename(tmp.c_str(), path.c_str()) != 0) rc = fail(ERATO_GPU_IO_ERROR, "rename to " + path + " failed");
    if (rc) {
      ::unlink(tmp.c_str());
      return rc;
    }
  } else {
    // one shard of a multi-GPU run: pwrite at its offset into the shared file
    // (part_n == 0: an empty shard, nothing to sieve)
    const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT, 0644);
    if (fd < 0) return fail(ERATO_GPU_IO_ERROR, "cannot open " + path);
    if (::ftruncate(fd, (off_t)total_bytes) != 0) {  // idempotent across shards
      ::close(fd);
      return fail(ERATO_GPU_IO_ERROR, "truncate failed for " + path);
    }
    if (part_n) rc = write_shard(c, fd, l, f, part_f, part_n, flags, stats);
    if (::close(fd) != 0 && !rc) rc = fail(ERATO_GPU_IO_ERROR, "close failed for " + path);
    if (rc) return rc;
  }
  if (stats) stats->segments = part_n;
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
  const uint64_t key[4] = {l, f, n, flags};
  if (!std::equal(key, key + 4, c->xp_key)) {
    // sieve + compaction once; a follow-up call with the same (l, f, n, flags)
    // (e.g. the first to learn the count, the second with a buffer) only copies
    std::fill(c->xp_key, c->xp_key + 4, ~0ull);
    const uint64_t T = n << l;
    CUDA_TRY(c->table.ensure(((T / 8) + 15) & ~15ull));
    erato_gpu_stats s{};
    rc = erato_gpu_run(c, l, f, n, flags, c->table.p, nullptr, nullptr, 1, &s);
    if (rc) return rc;
    // the number 1 (bit 0 of an f = 0 run) is a clear bit but not a prime
    const uint64_t lo = (u == 1) ? 1 : 0;
    const uint64_t np0 = s.prime_count - lo;
    CUDA_TRY(c->outbuf.ensure(std::max<uint64_t>(np0, 1) * 8));
    uint64_t* d_total = c->scal.as<uint64_t>() + 40;
    // extract_primes (driver.cpp:65-81): clear bits -> u + 2j
    rc = compact_zeros<uint64_t>(c, c->stream, c->table.as<uint32_t>(), T, lo, u, c->outbuf.as<uint64_t>(), np0,
                                 d_total);
    if (rc) return rc;
    uint64_t written = 0;
    CUDA_TRY(cudaMemcpyAsync(&written, d_total, 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (written != np0)
      return fail(ERATO_GPU_E_INVARIANT, "compaction wrote " + std::to_string(written) + " primes, count says " +
                                             std::to_string(np0));
    c->xp_count = np0;
    std::copy(key, key + 4, c->xp_key);
  }
  const uint64_t np = c->xp_count;
  const uint64_t m = std::min(np, cap);
  if (dst && m) CUDA_TRY(cudaMemcpyAsync(dst, c->outbuf.p, m * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (count) *count = np;
  return 0;
}

// ---------------------------------------------------------------------------
// Multi-GPU run_sieve: contiguous range shards, one host
// thread per shard driving its device, and one collective — the sum of the
// per-shard counts, ncclAllReduce(uint64, sum) over NVLink between the
// devices' count words.  NCCL is loaded at run time (libnccl.so.2): the
// library has no link-time NCCL dependency, and a process that already
// loaded torch's NCCL shares it.
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((h = ::dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      api.why = std::string("cannot load libnccl.so.2: ") + ::dlerror();
      return;
    }
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(::dlsym(h, "ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(::dlsym(h, "ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(::dlsym(h, "ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(::dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(::dlsym(h, "ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(::dlsym(h, "ncclGetErrorString"));
    api.ok = api.CommInitAll && api.CommDestroy && api.AllReduce && api.GroupStart && api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a needed symbol";
  });
  return api;
}

}  // namespace

struct erato_gpu_multi {
  int num = 0;
  std::vector<int> devices;
  std::vector<erato_gpu_ctx*> ctx;
  std::vector<uint64_t*> dcount;  // one count word per shard, on its device
  std::vector<ncclComm_t> comms;  // empty: devices repeat (test topology), counts summed on the host
};

extern "C" void erato_gpu_multi_destroy(erato_gpu_multi* m) {
  if (!m) return;
  if (!m->comms.empty() && nccl().ok)
    for (auto cm : m->comms) nccl().CommDestroy(cm);
  for (int g = 0; g < (int)m->ctx.size(); ++g) {
    if (m->dcount[g]) {
      cudaSetDevice(m->devices[g]);
      cudaFree(m->dcount[g]);
    }
    erato_gpu_destroy(m->ctx[g]);
  }
  cudaGetLastError();
  delete m;
}

extern "C" int erato_gpu_multi_create(int num_gpus, const int* devices, erato_gpu_multi** out) {
  if (!out) return fail(ERATO_GPU_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  const int ndev = erato_gpu_device_count();
  if (ndev == 0) return fail(ERATO_GPU_E_NO_DEVICE, "no CUDA device visible");
  if (num_gpus < 1 || num_gpus > 4096) return fail(ERATO_GPU_E_INVALID_ARG, "num_gpus out of range");
  auto* m = new erato_gpu_multi();
  m->num = num_gpus;
  for (int g = 0; g < num_gpus; ++g) {
    const int d = devices ? devices[g] : g;
    if (d < 0 || d >= ndev) {
      erato_gpu_multi_destroy(m);
      return fail(ERATO_GPU_E_NO_DEVICE, "device " + std::to_string(d) + " not visible (" + std::to_string(ndev) +
                                             " devices)");
    }
    m->devices.push_back(d);
  }
  m->ctx.assign(num_gpus, nullptr);
  m->dcount.assign(num_gpus, nullptr);
  for (int g = 0; g < num_gpus; ++g) {
    int rc = erato_gpu_create(m->devices[g], &m->ctx[g]);
    if (!rc && cudaSetDevice(m->devices[g]) == cudaSuccess &&
        cudaMalloc(reinterpret_cast<void**>(&m->dcount[g]), 8) != cudaSuccess)
      rc = fail(ERATO_GPU_E_CUDA, "count word allocation failed");
    if (rc) {
      const std::string msg = g_err;
      erato_gpu_multi_destroy(m);
      g_err = msg;
      return rc;
    }
  }
  std::vector<int> sorted = m->devices;
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  if (distinct) {  // NCCL communicators over the devices (one process, one comm per device)
    const NcclApi& api = nccl();
    if (!api.ok) {
      erato_gpu_multi_destroy(m);
      return fail(ERATO_GPU_E_CUDA, "NCCL unavailable: " + api.why);
    }
    m->comms.assign(num_gpus, nullptr);
    const ncclResult_t r = api.CommInitAll(m->comms.data(), num_gpus, m->devices.data());
    if (r != ncclSuccess) {
      m->comms.clear();
      erato_gpu_multi_destroy(m);
      return fail(ERATO_GPU_E_CUDA, std::string("ncclCommInitAll: ") + api.GetErrorString(r));
    }
  }
  *out = m;
  return 0;
}

extern "C" int erato_gpu_multi_uses_nccl(const erato_gpu_multi* m) { return m && !m->comms.empty() ? 1 : 0; }

namespace {
// One shard per device thread: count-only (fd < 0) or streamed into fd.
int multi_run(erato_gpu_multi* m, int fd, unsigned l, uint64_t f, uint64_t n, unsigned flags, uint64_t* count,
              erato_gpu_stats* stats) {
  int rc = erato_gpu_validate(l, f, n, flags, nullptr, nullptr);
  if (rc) return rc;
  const int G = m->num;
  std::vector<int> rcs(G, 0);
  std::vector<std::string> errs(G);
  std::vector<erato_gpu_stats> st(G);
  std::vector<uint64_t> parts(G, 0);
  std::vector<std::thread> th;
  for (int g = 0; g < G; ++g) {
    th.emplace_back([&, g] {
      uint64_t fg = 0, ng = 0;
      erato_gpu_shard(f, n, g, G, &fg, &ng);
      std::memset(&st[g], 0, sizeof(st[g]));
      int r = 0;
      erato_gpu_ctx* c = m->ctx[g];
      if (cudaSetDevice(c->device) != cudaSuccess) r = fail(ERATO_GPU_E_CUDA, "cudaSetDevice");
      if (!r && ng == 0) {  // empty shard (more devices than segments): count 0, still joins the reduction
        r = cudaMemsetAsync(m->dcount[g], 0, 8, c->stream) == cudaSuccess ? 0 : fail(ERATO_GPU_E_CUDA, "memset");
      } else if (!r && fd < 0) {
        r = erato_gpu_run(c, l, fg, ng, flags, nullptr, m->dcount[g], nullptr, 1, &st[g]);
      } else if (!r) {
        r = write_shard(c, fd, l, f, fg, ng, flags, &st[g]);
        if (!r && cudaMemcpyAsync(m->dcount[g], &st[g].prime_count, 8, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
          r = fail(ERATO_GPU_E_CUDA, "count upload");
      }
      if (!r && cudaStreamSynchronize(c->stream) != cudaSuccess) r = fail(ERATO_GPU_E_CUDA, "shard sync");
      parts[g] = st[g].prime_count;
      rcs[g] = r;
      if (r) errs[g] = g_err;
    });
  }
  for (auto& t : th) t.join();
  for (int g = 0; g < G; ++g)
    if (rcs[g]) {
      g_err = errs[g];
      return rcs[g];
    }
  uint64_t total = 0;
  if (!m->comms.empty()) {
    // the one collective: sum of the shards' device count words over NVLink
    const NcclApi& api = nccl();
    ncclResult_t r = api.GroupStart();
    for (int g = 0; g < G && r == ncclSuccess; ++g) {
      cudaSetDevice(m->devices[g]);
      r = api.AllReduce(m->dcount[g], m->dcount[g], 1, ncclUint64, ncclSum, m->comms[g], m->ctx[g]->stream);
    }
    const ncclResult_t r2 = api.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
      return fail(ERATO_GPU_E_CUDA, std::string("ncclAllReduce: ") + api.GetErrorString(r != ncclSuccess ? r : r2));
    std::vector<uint64_t> red(G, 0);
    for (int g = 0; g < G; ++g) {
      CUDA_TRY(cudaSetDevice(m->devices[g]));
      CUDA_TRY(cudaMemcpyAsync(&red[g], m->dcount[g], 8, cudaMemcpyDeviceToHost, m->ctx[g]->stream));
      CUDA_TRY(cudaStreamSynchronize(m->ctx[g]->stream));
    }
    total = red[0];
    for (int g = 1; g < G; ++g)
      if (red[g] != total) return fail(ERATO_GPU_E_INVARIANT, "all-reduced counts differ across devices");
  } else {
    for (int g = 0; g < G; ++g) total += parts[g];
  }
  uint64_t check = 0;
  for (int g = 0; g < G; ++g) check += parts[g];
  if (check != total) return fail(ERATO_GPU_E_INVARIANT, "all-reduced count differs from the sum of the shards");
  if (count) *count = total;
  if (stats) {  // device times: max over shards (the shards run concurrently)
    std::memset(stats, 0, sizeof(*stats));
    stats->prime_count = total;
    stats->segments = n;
    for (int g = 0; g < G; ++g) {
      stats->init_s = std::max(stats->init_s, st[g].init_s);
      stats->small_s = std::max(stats->small_s, st[g].small_s);
      stats->large_s = std::max(stats->large_s, st[g].large_s);
      stats->total_s = std::max(stats->total_s, st[g].total_s);
      stats->base_primes = std::max(stats->base_primes, st[g].base_primes);
      stats->tiles += st[g].tiles;
      stats->waves = std::max(stats->waves, st[g].waves);
      stats->kernel_launches += st[g].kernel_launches;
      stats->retries += st[g].retries;
      stats->log_tile = std::max(stats->log_tile, st[g].log_tile);
    }
  }
  return 0;
}
}  // namespace

extern "C" int erato_gpu_multi_count(erato_gpu_multi* m, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                                     uint64_t* count, erato_gpu_stats* stats) {
  if (!m) return fail(ERATO_GPU_E_INVALID_ARG, "multi is NULL");
  return multi_run(m, -1, l, f, n, flags, count, stats);
}

extern "C" int erato_gpu_multi_write_table(erato_gpu_multi* m, const char* out_dir, unsigned l, uint64_t f,
                                           uint64_t n, unsigned flags, char* path_out, size_t path_cap,
                                           uint64_t* count, erato_gpu_stats* stats) {
  if (!m || !out_dir) return fail(ERATO_GPU_E_INVALID_ARG, "NULL argument");
  int rc = erato_gpu_validate(l, f, n, flags, nullptr, nullptr);
  if (rc) return rc;
  const std::string path = table_path(out_dir, l, f, n);
  const std::string tmp = path + ".tmp." + std::to_string(::getpid());
  const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return fail(ERATO_GPU_IO_ERROR, "cannot open " + tmp);
  rc = ::ftruncate(fd, (off_t)((n << l) / 8)) == 0 ? 0 : fail(ERATO_GPU_IO_ERROR, "truncate failed for " + tmp);
  if (!rc) rc = multi_run(m, fd, l, f, n, flags, count, stats);  // shards pwrite concurrently
  if (::close(fd) != 0 && !rc) rc = fail(ERATO_GPU_IO_ERROR, "close failed for " + tmp);
  if (!rc && ::rename(tmp.c_str(), path.c_str()) != 0) rc = fail(ERATO_GPU_IO_ERROR, "rename to " + path + " failed");
  if (rc) {
    ::unlink(tmp.c_str());
    return rc;
  }
  if (path_out && path_cap) std::snprintf(path_out, path_cap, "%s", path.c_str());
  return 0;
}

// The device base-prime list of a run (the odd primes <= limit, ascending):
// build_base / simple_sieve(isqrt v) (src/base.cpp:19-53) as run_impl computes it.
extern "C" int erato_gpu_base_primes(erato_gpu_ctx* c, uint64_t limit, uint32_t* dst, uint64_t cap, uint64_t* count) {
  if (!c) return fail(ERATO_GPU_E_INVALID_ARG, "ctx is NULL");
  if (limit > UINT32_MAX) return fail(ERATO_GPU_E_INVALID_ARG, "limit above 2^32");
  CUDA_TRY(cudaSetDevice(c->device));
  uint32_t launches = 0;
  const int rc = base_primes(c, c->stream, limit, launches);
  if (rc) return rc;
  uint64_t n = 0;
  CUDA_TRY(cudaMemcpyAsync(&n, c->scal.p, 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const uint64_t m = std::min(n, cap);
  if (dst && m) CUDA_TRY(cudaMemcpy(dst, c->primes.p, m * 4, cudaMemcpyDeviceToHost));
  if (count) *count = n;
  return 0;
}
