// sieve_kernels.cuh — sm_100a device code of the segmented odd-only sieve.
//
// Geometry (reference: /root/reference/proj/include/erato/params.hpp:1-9):
// global odd index i stands for the number 2i+1; table bit j of a run
// (l, f, n) is global index f*2^l + j.  The GPU does not process the
// reference's 2^l-bit segments one after another; it processes TILES of
// S = 2^log_s bits (S is decoupled from l — the output is position
// independent), many tiles at once, one CTA per tile, with
// the tile resident in shared memory.
//
// Prime classes (GPU split; the reference's split is base.cpp:11-17):
//   small   p <= 61        periodic word patterns (masks.cpp:9-50 idea)
//   medium  61 < p <= S    shared-memory atomicOr marking inside the tile,
//                          start offset recomputed per tile from 32-bit
//                          residues (k_med_records), mod-30 wheel over the
//                          cofactor (wheel.cpp:10-69 idea: 8 of 15 odd
//                          cofactors)
//   ML      S < p <= W*S/4 walked once per wave (k_ml_walk) into per-tile
//                          hit records; a table-driven mod-30030 wheel over the
//                          cofactor (the reference's wheel three primes further)
//   far     p > W*S/4      walked once per window of K waves (k_far_walk) into
//                          the record bucket of the wave of each hit — the
//                          paper's bucket of the segment of the next hit
//                          (large_kernel.hpp, Lemma 2) filled K waves
//                          ahead — and split by tile per wave (k_wave_sort)
//   (k_scatter_ml / k_scatter_far / k_gen / k_bin: the round-1/2 structures,
//   ERATO_GPU_LARGE=legacy and the fallback for waves of more than 256 tiles)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// EG_CHECK: device-side bounds checks, compiled in with -DEG_DEBUG (debug
// builds only; compute-sanitizer is unavailable on the GPU pool).
#ifdef EG_DEBUG
#include <cstdio>
#define EG_CHECK(cond, ...)                                            \
  do {                                                                 \
    if (!(cond)) {                                                     \
      printf("EG_CHECK failed %s:%d: %s | ", __FILE__, __LINE__, #cond); \
      printf(__VA_ARGS__);                                             \
      printf("\n");                                                    \
      __trap();                                                        \
    }                                                                  \
  } while (0)
#else
#define EG_CHECK(cond, ...) \
  do {                      \
  } while (0)
#endif

#ifndef EG_PLACE_UNROLL
#define EG_PLACE_UNROLL 2
#endif
#ifndef EG_WRITE_UNROLL
#define EG_WRITE_UNROLL 2
#endif

namespace eg {
constexpr int kPlaceUnroll = EG_PLACE_UNROLL, kWriteUnroll = EG_WRITE_UNROLL;

constexpr uint32_t kFull = 0xffffffffu;

// 32-bit shared-memory address of a generic pointer into shared memory
// (volatile: computed once, not rematerialised inside hot loops).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  uint32_t r;
  asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(r) : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------
// mod-30 wheel over odd cofactors c of p*c.  Admissible residues (coprime to
// 30): R = {1,7,11,13,17,19,23,29}; class s <-> R[s].  In index space the
// step from class s to s+1 is D[s]*p with D = {3,2,1,2,1,2,3,1} — the
// reference's wheel deltas (src/wheel.cpp:27-30).
__device__ __forceinline__ uint32_t wheel_D(uint32_t s) { return (0x13212123u >> (s << 2)) & 15u; }

// adv[r]: smallest a >= 0 with r+a admissible; cls[r]: class of admissible r.
__constant__ uint8_t c_adv[30] = {1, 0, 5, 4, 3, 2, 1, 0, 3, 2, 1, 0, 1, 0, 3,
                                  2, 1, 0, 1, 0, 3, 2, 1, 0, 5, 4, 3, 2, 1, 0};
__constant__ uint8_t c_cls[30] = {255, 0,   255, 255, 255, 255, 255, 1,   255, 255,
                                  255, 2,   255, 3,   255, 255, 255, 4,   255, 5,
                                  255, 255, 255, 6,   255, 255, 255, 255, 255, 7};
// cum[s][t] = sum_{i<t} D[(s+i)&7]
__constant__ uint8_t c_cum[8][8] = {
    {0, 3, 5, 6, 8, 9, 11, 14}, {0, 2, 3, 5, 6, 8, 11, 12}, {0, 1, 3, 4, 6, 9, 10, 13},
    {0, 2, 3, 5, 8, 9, 12, 14}, {0, 1, 3, 6, 7, 10, 12, 13}, {0, 2, 5, 6, 9, 11, 12, 14},
    {0, 3, 4, 7, 9, 10, 12, 13}, {0, 1, 4, 6, 7, 9, 10, 12}};

__device__ __forceinline__ uint32_t mod30_u64(uint64_t c) {
  const uint32_t hi = (uint32_t)(c >> 32), lo = (uint32_t)c;
  return ((hi % 30u) * 16u + lo % 30u) % 30u;  // 2^32 = 16 (mod 30)
}

// First wheel-admissible multiple p*c >= x with c >= cmin, for odd x = 2g+1
// (g = global odd index of the tile start).  Returns its index offset from g,
// (c*p - x)/2, and the wheel class s of c.  Restates Lemma 1 / first_offset
// (src/wheel.cpp:43-47) plus wheel_align (src/wheel.cpp:60-69) for 64-bit
// starts: floor(x/p) from an fp64 estimate (off by at most one), then the
// exact remainder in wrap-around u64 arithmetic.
__device__ __forceinline__ uint64_t first_hit(uint32_t p, uint64_t x, uint64_t cmin, uint32_t& s,
                                              uint64_t* cof = nullptr) {
  uint64_t c = __double2ull_rz(__dmul_rz(__ull2double_rz(x), __drcp_rn((double)p)));
  int64_t r = (int64_t)(x - c * p);  // true remainder, in (-p, 2p)
  if (r < 0) {
    r += p;
    --c;
  } else if (r >= (int64_t)p) {
    r -= p;
    ++c;
  }
  uint64_t d = 0;  // c*p - x after rounding c up
  if (r) {
    ++c;
    d = p - (uint64_t)r;
  }
  if (c < cmin) {
    d += (cmin - c) * (uint64_t)p;
    c = cmin;
  }
  const uint32_t cm = mod30_u64(c);
  const uint32_t a = c_adv[cm];
  s = c_cls[cm + a];
  d += (uint64_t)a * p;
  if (cof) *cof = c + a;  // the cofactor of the returned hit
  return d >> 1;
}

// Far entries (u64).  Mod-30 format: p | (q | s << 29) << 32.  Mod-210 format
// (FAR7, when every far prime is < 2^31 and a wave spans <= 2^28 bits): the
// entry also carries the cofactor mod 7, and a far prime skips its multiples
// whose cofactor is divisible by 7 (those are marked by the pattern of 7):
//   bits 0..29 (p-1)/2 | bits 30..57 q | bits 58..60 s | bits 61..63 c mod 7 (1..6)
__device__ __forceinline__ uint64_t far7_pack(uint32_t p, uint32_t q, uint32_t s, uint32_t c7) {
  return (uint64_t)(p >> 1) | ((uint64_t)q << 30) | ((uint64_t)(s & 7) << 58) | ((uint64_t)c7 << 61);
}
// ML states (uint2).  Mod-30: {p | s << 29, pos}.  Mod-210 (ML7, when a wave
// spans at most 170 * 2^20 bits, so p < 2^28 and pos < 6p < 2^30):
//   x = p | s << 28 | (c7 & 1) << 31,   y = pos | (c7 >> 1) << 30.
__device__ __forceinline__ uint2 ml7_pack(uint32_t p, uint32_t pos, uint32_t s, uint32_t c7) {
  return make_uint2(p | ((s & 7) << 28) | ((c7 & 1) << 31), pos | ((c7 >> 1) << 30));
}
__device__ __forceinline__ uint32_t far_q(uint64_t e, bool far7) {
  return far7 ? (uint32_t)(e >> 30) & 0xfffffffu : (uint32_t)(e >> 32) & 0x1fffffffu;
}

// ---------------------------------------------------------------------------
// Small-prime patterns.  Eight groups of primes 3..61 with product moduli M;
// table entry c of group k is the 32-bit window of the group's composite
// pattern starting at pattern phase 32c mod M (gcd(32, M) = 1, so one word
// step = one entry step).  Bit b of entry c is set iff (32c+b) = (p-1)/2
// (mod p) for a p of the group (masks.hpp:4-12).
constexpr int kNumGroups = 8;
constexpr uint32_t kPatPad = 96;        // wrap-around entries per group (4 windows 32 apart)
constexpr uint32_t kPatWords = 11008;  // sum of (M + 96), rounded to a multiple of 4
__constant__ uint32_t c_gmod[kNumGroups] = {105, 143, 323, 667, 1147, 1763, 2491, 3599};
__constant__ uint32_t c_goff[kNumGroups] = {0, 201, 440, 859, 1622, 2865, 4724, 7311};  // M + 96 each
__constant__ uint32_t c_ginv32[kNumGroups] = {23, 76, 212, 271, 466, 1157, 1012, 1912};
// the same as compile-time constants for unrolled loops (modulo by a
// constant: multiply-high sequences instead of a division subroutine)
__host__ __device__ constexpr uint32_t gmod(int k) {
  return k == 0 ? 105 : k == 1 ? 143 : k == 2 ? 323 : k == 3 ? 667 : k == 4 ? 1147 : k == 5 ? 1763 : k == 6 ? 2491 : 3599;
}
__host__ __device__ constexpr uint32_t goff(int k) {
  return k == 0 ? 0 : k == 1 ? 201 : k == 2 ? 440 : k == 3 ? 859 : k == 4 ? 1622 : k == 5 ? 2865 : k == 6 ? 4724 : 7311;
}
__host__ __device__ constexpr uint32_t ginv32(int k) {
  return k == 0 ? 23 : k == 1 ? 76 : k == 2 ? 212 : k == 3 ? 271 : k == 4 ? 466 : k == 5 ? 1157 : k == 6 ? 1012 : 1912;
}
__constant__ uint8_t c_gprimes[kNumGroups][3] = {{3, 5, 7},   {11, 13, 0}, {17, 19, 0}, {23, 29, 0},
                                                 {31, 37, 0}, {41, 43, 0}, {47, 53, 0}, {59, 61, 0}};
__constant__ uint8_t c_small17[17] = {3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61};

__global__ void k_build_patterns(uint32_t* __restrict__ ptab) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kPatWords) return;
  int k = kNumGroups - 1;
  while (k > 0 && i < c_goff[k]) --k;
  const uint32_t M = c_gmod[k];
  uint32_t c = i - c_goff[k];
  if (c >= M + kPatPad) {  // alignment padding after the last group
    ptab[i] = 0;
    return;
  }
  if (c >= M) c -= M;  // wrap-around entries
  uint32_t w = 0;
  for (uint32_t b = 0; b < 32; ++b) {
    const uint32_t x = (32u * c + b) % M;
    for (int j = 0; j < 3; ++j) {
      const uint32_t p = c_gprimes[k][j];
      if (p && x % p == (p - 1) / 2) w |= 1u << b;
    }
  }
  ptab[i] = w;
}

// ---------------------------------------------------------------------------
// Medium-prime record, one per prime per chunk of tiles (16 B, read by
// every tile), M = 30p (one wheel period of cofactors):
//   x    p                          (p < 2^24)
//   y    R0  = x_0 mod M            (x_0 = first odd number of the chunk)
//   z    rho = (2*S) mod M          (residue step per tile)
//   w    float rho / M
// Tile t of the chunk starts at x_t = x_0 + 2*S*t with R_t = x_t mod M =
// (R0 + t*rho) mod M (fp32 quotient estimate, 32-bit wrap-around remainder,
// t < 2^20).  The first multiple c*p >= x_t has c = 30k + ceil(R_t/p), so
// c' = ceil(R_t/p) in [0, 30] alone gives the first wheel-admissible
// cofactor (table combo[c']) and its offset (c'+adv)*p - R_t: Lemma 1
// (first_offset, src/wheel.cpp:43-47) and wheel_align (src/wheel.cpp:60-69)
// per (prime, tile) without 64-bit division.
constexpr uint32_t kMaxChunkTiles = 1u << 20;
constexpr uint32_t kMedPad = 4096;  // records past the end the tile kernel may prefetch (up to three items of 1024)

__global__ void k_med_records(const uint32_t* __restrict__ primes, uint32_t n, uint64_t x0, uint32_t log_s,
                              uint4* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t p = primes[i];
  const uint32_t M = 30u * p;
  const uint32_t rho = (uint32_t)(((uint64_t)2 << log_s) % M);
  out[i] = make_uint4(p, (uint32_t)(x0 % M), rho, __float_as_uint((float)((double)rho / (double)M)));
}

// combo[cm] = adv | cls << 3 ; cum4[s] = nibbles cum[s][0..7]
__device__ __forceinline__ uint32_t nib(uint32_t packed, uint32_t k) { return (packed >> (k << 2)) & 15u; }

struct TileArgs {
  uint64_t g0;     // global odd index of table bit 0 (= f << l)
  uint64_t tbits;  // table bits T of this run (shard)
  uint64_t tile0;  // first tile of this launch
  uint64_t tbase;  // first tile of the chunk the medium records were made for
  uint32_t log_s;
  const uint4* med;      // medium-prime records (61 < p <= S), ascending p
  uint32_t nmed;
  uint32_t nmed_warp;    // the first nmed_warp medium primes (p < S/64) are marked group-per-prime:
  uint32_t nmed_g32, nmed_g16;  // the first nmed_g32 by 32 lanes (p < S/256), the next nmed_g16 by 16
  const uint32_t* ptab;  // kPatWords pattern words (global)
  const uint32_t* hits;  // [gridDim.x][hcap] hit offsets (large primes), may be null
  uint32_t* hitcnt;      // [gridDim.x], zeroed after use
  uint32_t hcap;
  uint32_t* table;               // output words (nullable: count only); tile t writes at
  uint64_t out_tile0;            //   table + (t - out_tile0) * S/32 (a wave slice when streaming)
  unsigned long long* count;     // zero-bit accumulator
  uint32_t* reset_bucket_count;  // far bucket slot consumed this wave (nullable)
  unsigned long long* phase_ns;  // nullable: CTA 0 adds its pattern-phase time (masks_s)
};

#ifndef EG_ITEM_UNROLL2
#define EG_ITEM_UNROLL2 1  // lane-per-prime items two per trip (cfg5 k_tile 21.0 -> 20.1 ms; cfg2-4 unchanged)
#endif
#ifndef EG_EVERY_NUM
#define EG_EVERY_NUM 1  // hit-chunk cadence: one chunk per (items / (chunks + 1)) * NUM / DEN medium items
#endif
#ifndef EG_EVERY_DEN
#define EG_EVERY_DEN 1
#endif
constexpr int kTileThreads = 1024;
constexpr uint32_t kMaxWarpPrimes = 2048;  // medium primes below S/64 (pi(16384) = 1900 at S = 2^20)
#ifndef EG_HIT_CHUNK
#define EG_HIT_CHUNK 256
#endif
constexpr uint32_t kHitChunk = EG_HIT_CHUNK;  // hit records per warp chunk (1 KB of shared staging per warp): 256 or 128
static_assert(kHitChunk == 256 || kHitChunk == 128, "one or two uint4 per lane");
constexpr int kTileWarps = kTileThreads / 32;

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void mark(uint32_t* tile, uint32_t q) { atomicOr(&tile[q >> 5], 1u << (q & 31)); }
// the same on a 32-bit shared address (the tile sits at the start of the
// dynamic shared memory): SHF + LOP3 + SHF.L.W + ATOMS [R + UR] per mark
__device__ __forceinline__ void mark_a(uint32_t tile_a, uint32_t q) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(tile_a + ((q >> 5) << 2)), "r"(1u << (q & 31)) : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" : : "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" : : : "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" : : : "memory"); }

// First wheel-admissible multiple of a medium prime in tile t of the chunk
// (see k_med_records): index offset from the tile start (may be >= S) and
// the cofactor class s.  P2: multiples from p^2 on (overlap runs and the
// base sieve, where the primes themselves lie inside the interval).
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t lds_u8c(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

template <bool P2>
__device__ __forceinline__ uint32_t med_first(const uint4 rec, uint32_t t, float tf, uint64_t x_t, uint32_t combo_a,
                                              uint32_t& p, uint32_t& s) {
  p = rec.x;
  const uint32_t M = 30u * p;
  // floor(t*rho/M) or one less (t < 2^20: |fp32 error| < 0.1), so the
  // 32-bit wrap-around remainder lies in [0, 2M)
  const uint32_t qe = __float2uint_rz(__fmaf_rn(tf, __uint_as_float(rec.w), -0.5f));
  uint32_t R = rec.y + (t * rec.z - qe * M);  // R_t in [0, 3M)
  R -= R >= M ? M : 0;
  R -= R >= M ? M : 0;
  EG_CHECK(R < M, "med_first R=%u M=%u p=%u t=%u qe=%u rec=(%u,%u,%u,%08x)", R, M, p, t, qe, rec.x, rec.y, rec.z, rec.w);
  uint32_t c = __float2uint_ru(__uint2float_rz(R) * rcp_approx(__uint2float_rn(p)));  // ceil(R/p) +- 1
  int32_t e = (int32_t)(c * p - R);
  const bool lo = e < 0;
  c += lo ? 1u : 0u;
  e += lo ? (int32_t)p : 0;
  const bool hi = e >= (int32_t)p;
  c -= hi ? 1u : 0u;
  e -= hi ? (int32_t)p : 0;
  EG_CHECK(c <= 30 && e >= 0 && e < (int32_t)p, "med_first c=%u e=%d p=%u R=%u", c, e, p, R);
  const uint32_t cb = lds_u8c(combo_a + c);
  uint32_t d = (uint32_t)e + (cb & 7u) * p;  // c_adm * p - x_t
  s = cb >> 3;
  if (P2 && x_t + d < (uint64_t)p * p) {  // cofactor p: p^2 (admissible, class of p mod 30)
    const uint64_t dd = (uint64_t)p * p - x_t;
    d = dd < (1u << 30) ? (uint32_t)dd : (1u << 30);
    s = lds_u8c(combo_a + 32 + p % 30u);
  }
  return d >> 1;
}

// P2: multiples from p^2 (overlap runs, base sieve); HITS: large-prime hit
// lists to mark (a.hits != null).
template <bool P2, bool HITS>
__global__ void __launch_bounds__(kTileThreads, 1) k_tile(const TileArgs a) {
  extern __shared__ uint4 smem4[];
  uint32_t* const tile = reinterpret_cast<uint32_t*>(smem4);  // first: mark addresses need no base add
  uint32_t* const pat = tile + ((1u << a.log_s) >> 5);
  uint2* const s_wq = reinterpret_cast<uint2*>(pat + kPatWords);  // [nmed_warp] (q0, p | s<<29)
  uint4* const s_hits = reinterpret_cast<uint4*>(s_wq + ((a.nmed_warp + 1) & ~1u));  // [warps][kHitChunk/4] if hits
  __shared__ unsigned long long s_red[kTileWarps];
  __shared__ uint8_t s_combo[64];  // [c'] = adv | cls << 3 (c' = 0..30); [32 + r] = cls of r
  __shared__ uint32_t s_cum[8];

  const uint32_t tid = threadIdx.x, bd = kTileThreads, lane = tid & 31, warp = tid >> 5;  // (always launched with kTileThreads)
  const uint32_t log_s = a.log_s;
  const uint32_t S = 1u << log_s, nw = S >> 5;
  const uint64_t t64 = a.tile0 + blockIdx.x;
  const uint64_t tstart = t64 << log_s;
  const uint64_t g = a.g0 + tstart;
  uint64_t t_start = 0;
  if (a.phase_ns && blockIdx.x == 0 && tid == 0) t_start = globaltimer();

  {  // stage pattern tables and the wheel tables
    const uint4* src = reinterpret_cast<const uint4*>(a.ptab);
    uint4* const pat4 = reinterpret_cast<uint4*>(pat);
    for (uint32_t i = tid; i < kPatWords / 4; i += bd) pat4[i] = src[i];
    if (tid < 31) {
      const uint32_t r = tid % 30u;
      s_combo[tid] = (uint8_t)(c_adv[r] | (c_cls[r + c_adv[r]] << 3));
    } else if (tid >= 32 && tid < 62) {
      s_combo[tid] = c_cls[tid - 32];
    }
    if (tid < 8) {
      uint32_t v = 0;
      for (int k = 0; k < 8; ++k) v |= (uint32_t)c_cum[tid][k] << (4 * k);
      s_cum[tid] = v;
    }
  }
  __syncthreads();

  const uint64_t x_t = 2 * g + 1;
  const uint32_t t = (uint32_t)(t64 - a.tbase);  // tile index within the chunk (< 2^20)
  const float tf = __uint2float_rz(t);
  const uint32_t combo_a = smem_addr(s_combo);
  const uint32_t tile_a = smem_addr(tile);
  // 0. start offsets of the group-marked medium primes (p < S/64), lane-
  // parallel into shared memory (no barrier of its own: phase 1's covers it)
  for (uint32_t i = tid; i < a.nmed_warp; i += bd) {
    uint32_t p, s;
    const uint32_t q0 = med_first<P2>(a.med[i], t, tf, x_t, combo_a, p, s);
    s_wq[i] = make_uint2(q0, p | (s << 29));
  }

  // 1. small primes: OR of the 8 group windows.  Lane l of a warp builds
  // words l, l+32, l+64, l+96 of the warp's 128-word block: one phase
  // update per 4 words, conflict-free loads (each group table is padded by
  // 96 entries, so the 4 windows never wrap).
  {
    constexpr uint32_t kBlock = 128, kStride = kTileWarps * kBlock;
    uint32_t cur[kNumGroups], stp[kNumGroups];
#pragma unroll
    for (int k = 0; k < kNumGroups; ++k) {
      const uint32_t M = gmod(k);
      const uint32_t cg = (uint32_t)((g % M) * ginv32(k) % M);
      cur[k] = (cg + warp * kBlock + lane) % M;
      stp[k] = kStride % M;
    }
    for (uint32_t w = warp * kBlock + lane; w < nw; w += kStride) {
      uint32_t v0 = 0, v1 = 0, v2 = 0, v3 = 0;
#pragma unroll
      for (int k = 0; k < kNumGroups; ++k) {
        const uint32_t* src = pat + goff(k) + cur[k];
        v0 |= src[0];
        v1 |= src[32];
        v2 |= src[64];
        v3 |= src[96];
        cur[k] += stp[k];
        if (cur[k] >= gmod(k)) cur[k] -= gmod(k);
      }
      tile[w] = v0;
      tile[w + 32] = v1;
      tile[w + 64] = v2;
      tile[w + 96] = v3;
    }
  }
  __syncthreads();
  if (a.phase_ns && blockIdx.x == 0 && tid == 0) atomicAdd(a.phase_ns, (unsigned long long)(globaltimer() - t_start));
  // the patterns also hit the primes 3..61 themselves: clear them if inside
  if (tid < 17) {
    const uint64_t idx = (c_small17[tid] - 1) / 2;
    if (idx >= g && idx < g + S) {
      const uint32_t q = (uint32_t)(idx - g);
      atomicAnd(&tile[q >> 5], ~(1u << (q & 31)));
    }
  }

  // 2. medium primes
  {
    // 2a. group-per-prime (p < S/64): start offsets were computed
    // lane-parallel into shared memory (above); a group of G lanes takes one prime, lane j
    // marking wheel class (s+j)&7 of period j>>3 (step G/8 wheel periods):
    // G = 32 for p < S/256, 16 below S/128, 8 below S/64 — every lane makes
    // at least ~4 marks.
    const uint32_t n32 = a.nmed_g32, n16 = a.nmed_g16, i16 = (n16 + 1) >> 1;
    const uint32_t nitems = n32 + i16 + (a.nmed_warp - n32 - n16 + 3) / 4;
    // 3. large primes: this tile's hit records, in chunks of kHitChunk per
    // warp, fetched by cp.async into the warp's shared staging while the
    // warp marks medium primes (the DRAM reads overlap the shared-atomic
    // work instead of forming a phase of their own); every lane marks the
    // 8 records it copied itself.
    const uint32_t hcnt = HITS ? min(a.hitcnt[blockIdx.x], a.hcap) : 0;
    const uint32_t nch = (hcnt + kHitChunk - 1) / kHitChunk;
    const uint32_t* const hl = HITS ? a.hits + (uint64_t)blockIdx.x * a.hcap : nullptr;
    const uint32_t hst_a = smem_addr(s_hits + warp * (kHitChunk / 4) + lane);
    uint32_t ch = warp;  // next chunk of this warp (chunks warp, warp + 32, ...)
    bool pend = false;
    auto issue = [&]() {
      if (HITS && ch < nch) {
        const uint32_t* src = hl + ch * kHitChunk + 4 * lane;
        cp_async16(hst_a, src);
        if (kHitChunk == 256) cp_async16(hst_a + 512, src + 128);
        cp_async_commit();
        pend = true;
      }
    };
    auto consume = [&]() {
      if constexpr (HITS) {
        if (!pend) return;
        cp_async_wait_all();
        const uint4 v0 = s_hits[warp * (kHitChunk / 4) + lane];
        const uint4 v1 = kHitChunk == 256 ? s_hits[warp * (kHitChunk / 4) + 32 + lane] : make_uint4(0, 0, 0, 0);
        const uint32_t i0 = ch * kHitChunk + 4 * lane, i1 = kHitChunk == 256 ? i0 + 128 : hcnt;
        EG_CHECK(i0 >= hcnt || (v0.x < S && (i0 + 3 >= hcnt || v0.w < S)), "hit record beyond the tile %u %u", v0.x, v0.w);
        EG_CHECK(i1 >= hcnt || (v1.x < S && (i1 + 3 >= hcnt || v1.w < S)), "hit record beyond the tile %u %u", v1.x, v1.w);
        if (kHitChunk == 256 ? i1 + 3 < hcnt : i0 + 3 < hcnt) {
          mark_a(tile_a, v0.x); mark_a(tile_a, v0.y); mark_a(tile_a, v0.z); mark_a(tile_a, v0.w);
          if (kHitChunk == 256) {
            mark_a(tile_a, v1.x); mark_a(tile_a, v1.y); mark_a(tile_a, v1.z); mark_a(tile_a, v1.w);
          }
        } else {
          if (i0 < hcnt) mark_a(tile_a, v0.x);
          if (i0 + 1 < hcnt) mark_a(tile_a, v0.y);
          if (i0 + 2 < hcnt) mark_a(tile_a, v0.z);
          if (i0 + 3 < hcnt) mark_a(tile_a, v0.w);
          if (i1 < hcnt) mark_a(tile_a, v1.x);
          if (i1 + 1 < hcnt) mark_a(tile_a, v1.y);
          if (i1 + 2 < hcnt) mark_a(tile_a, v1.z);
          if (i1 + 3 < hcnt) mark_a(tile_a, v1.w);
        }
        __syncwarp();  // every lane has read its staging before it is refilled
        pend = false;
        ch += kTileWarps;
        issue();
      }
    };
    issue();
    // one chunk per `every` medium items of this warp
#ifndef EG_HITS_GROUPW
#define EG_HITS_GROUPW 0  // weight (in quarters) of a group-marked item in the hit-chunk cadence (a lane-per-prime item = 4): the
                          // records are consumed between the ALU-heavy lane-per-prime items only (cfg5 0 / 2 / 4 / 8: 45.58 / 45.81 / 45.82 / 45.91 ms)
#endif
    const uint32_t my_items = (nitems * EG_HITS_GROUPW / 4 + (a.nmed - a.nmed_warp + 31) / 32 + kTileWarps - 1) / kTileWarps;
    const uint32_t my_chunks = (nch + kTileWarps - 1) / kTileWarps;
    const uint32_t every = my_chunks ? max(1u, my_items * EG_EVERY_NUM / ((my_chunks + 1) * EG_EVERY_DEN)) : 0xffffffffu;
    uint32_t since = 0;
    // static round-robin (no barrier follows: the lane-per-prime phase
    // absorbs the imbalance)
    for (uint32_t item = warp; item < nitems; item += kTileWarps) {
      uint32_t idx, j, lim, shp;  // prime, lane in group, end of the group's class, log2(G/8)
      if (item < n32) {
        idx = item;
        j = lane;
        lim = n32;
        shp = 2;
      } else if (item < n32 + i16) {
        idx = n32 + 2 * (item - n32) + (lane >> 4);
        j = lane & 15;
        lim = n32 + n16;
        shp = 1;
      } else {
        idx = n32 + n16 + 4 * (item - n32 - i16) + (lane >> 3);
        j = lane & 7;
        lim = a.nmed_warp;
        shp = 0;
      }
      const uint2 w = s_wq[idx < lim ? idx : 0];
      const uint32_t p = w.y & 0x1fffffffu, s = w.y >> 29;
      uint32_t q = idx < lim ? w.x + p * (nib(s_cum[s], j & 7) + 15u * (j >> 3)) : S;
      const uint32_t step = (15u * p) << shp;
      for (; q + 3 * step < S; q += 4 * step) {
        mark_a(tile_a, q);
        mark_a(tile_a, q + step);
        mark_a(tile_a, q + 2 * step);
        mark_a(tile_a, q + 3 * step);
      }
      for (; q < S; q += step) mark_a(tile_a, q);
      if (HITS && EG_HITS_GROUPW && (since += EG_HITS_GROUPW) >= 4 * every) {
        since = 0;
        consume();
      }
    }
    since = 0;
    // 2b. lane-per-prime (S/64 <= p): whole wheel periods unrolled for
    // p <= S/8, a plain wheel walk for the few-mark primes above
    const uint32_t nlane = a.nmed - a.nmed_warp;
    const uint32_t nitem = (nlane + 31) / 32;
    // the record array is padded (kMedPad): next item's record in flight
    const uint4* rp = a.med + a.nmed_warp + warp * 32 + lane;
#if EG_ITEM_UNROLL2
    auto process = [&](const uint4 cur, const uint32_t item) {
      const bool valid = item * 32 + lane < nlane;
      if (valid) {
        uint32_t p, s;
        uint32_t q = med_first<P2>(cur, t, tf, x_t, combo_a, p, s);
#ifndef EG_TWO_HIT
#define EG_TWO_HIT 1
#endif
        if (EG_TWO_HIT && (p << 1) > S) {  // p > S/2: hits are > S/2 apart, at most two in the tile
          if (q < S) {
            mark_a(tile_a, q);
            q += wheel_D(s) * p;
            if (q < S) mark_a(tile_a, q);
          }
        } else if ((p << 3) > S) {
          uint32_t dd = __funnelshift_r(0x13212123u, 0x13212123u, 4 * s);  // low nibble = wheel_D(s)
          while (q < S) {
            mark_a(tile_a, q);
            q += (dd & 15u) * p;
            dd = __funnelshift_r(dd, dd, 4);
          }
        } else {
          const uint32_t cp = s_cum[s];
          const uint32_t o1 = p * nib(cp, 1), o2 = p * nib(cp, 2), o3 = p * nib(cp, 3), o4 = p * nib(cp, 4),
                         o5 = p * nib(cp, 5), o6 = p * nib(cp, 6), o7 = p * nib(cp, 7);
          const uint32_t per = 15u * p;
          for (; q + o7 < S; q += per) {
            mark_a(tile_a, q);
            mark_a(tile_a, q + o1);
            mark_a(tile_a, q + o2);
            mark_a(tile_a, q + o3);
            mark_a(tile_a, q + o4);
            mark_a(tile_a, q + o5);
            mark_a(tile_a, q + o6);
            mark_a(tile_a, q + o7);
          }
          // last partial period: a short wheel walk from class s
          uint32_t dd = __funnelshift_r(0x13212123u, 0x13212123u, 4 * s);
          while (q < S) {
            mark_a(tile_a, q);
            q += (dd & 15u) * p;
            dd = __funnelshift_r(dd, dd, 4);
          }
        }
      }
      if (HITS && (since += 4) >= 4 * every) {
        since = 0;
        consume();
      }
    };
    // two items per trip, their records in two register sets (no copies), the next two in flight
    uint4 rA = *rp, rB = rp[kTileWarps * 32];
    for (uint32_t item = warp; item < nitem; item += 2 * kTileWarps) {
      rp += 2 * kTileWarps * 32;
      const uint4 cA = rA, cB = rB;
      rA = rp[0];
      rB = rp[kTileWarps * 32];
      process(cA, item);
      if (item + kTileWarps < nitem) process(cB, item + kTileWarps);
    }
#else
    uint4 rec = *rp;
    for (uint32_t item = warp; item < nitem; item += kTileWarps) {
      const uint4 cur = rec;
      const bool valid = item * 32 + lane < nlane;
      rp += kTileWarps * 32;
      rec = *rp;
      if (valid) {
        uint32_t p, s;
        uint32_t q = med_first<P2>(cur, t, tf, x_t, combo_a, p, s);
#ifndef EG_TWO_HIT
#define EG_TWO_HIT 1
#endif
        if (EG_TWO_HIT && (p << 1) > S) {  // p > S/2: hits are > S/2 apart, at most two in the tile
          if (q < S) {
            mark_a(tile_a, q);
            q += wheel_D(s) * p;
            if (q < S) mark_a(tile_a, q);
          }
        } else if ((p << 3) > S) {
          uint32_t dd = __funnelshift_r(0x13212123u, 0x13212123u, 4 * s);  // low nibble = wheel_D(s)
          while (q < S) {
            mark_a(tile_a, q);
            q += (dd & 15u) * p;
            dd = __funnelshift_r(dd, dd, 4);
          }
        } else {
          const uint32_t cp = s_cum[s];
          const uint32_t o1 = p * nib(cp, 1), o2 = p * nib(cp, 2), o3 = p * nib(cp, 3), o4 = p * nib(cp, 4),
                         o5 = p * nib(cp, 5), o6 = p * nib(cp, 6), o7 = p * nib(cp, 7);
          const uint32_t per = 15u * p;
          for (; q + o7 < S; q += per) {
            mark_a(tile_a, q);
            mark_a(tile_a, q + o1);
            mark_a(tile_a, q + o2);
            mark_a(tile_a, q + o3);
            mark_a(tile_a, q + o4);
            mark_a(tile_a, q + o5);
            mark_a(tile_a, q + o6);
            mark_a(tile_a, q + o7);
          }
          // last partial period: a short wheel walk from class s
          uint32_t dd = __funnelshift_r(0x13212123u, 0x13212123u, 4 * s);
          while (q < S) {
            mark_a(tile_a, q);
            q += (dd & 15u) * p;
            dd = __funnelshift_r(dd, dd, 4);
          }
        }
      }
      if (HITS && (since += 4) >= 4 * every) {
        since = 0;
        consume();
      }
    }
#endif
    while (HITS && pend) consume();  // this warp's remaining hit chunks
  }
  __syncthreads();
  if (tid == 0) {
    if (HITS) a.hitcnt[blockIdx.x] = 0;
    if (blockIdx.x == 0 && a.reset_bucket_count) *a.reset_bucket_count = 0;
  }

  // 4. popcount + write-out (count_zeros simd.cpp:18-25, segment_to_bytes
  // driver.cpp:22-27: LSB-first bytes == little-endian words)
  const uint64_t rem = a.tbits - tstart;
  const uint32_t valid = rem < S ? (uint32_t)rem : S;  // multiple of 16 except in the base sieve
  const uint32_t vbytes = (valid + 7) >> 3;  // the base sieve table may end inside a byte
  unsigned long long ones = 0;
  uint32_t* out = a.table ? a.table + (((t64 - a.out_tile0) << log_s) >> 5) : nullptr;
  for (uint32_t w4 = tid; w4 < (nw >> 2); w4 += bd) {
    const uint32_t w0 = w4 << 2;
    if (w0 * 32 >= valid) break;
    uint4 v = smem4[w4];
    if ((w0 + 4) * 32 > valid) {  // partial quad at the end of the run
      uint32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t lo = (w0 + k) * 32;
        if (lo >= valid) e[k] = 0;
        else if (valid - lo < 32) e[k] &= (1u << (valid - lo)) - 1;
      }
      v = make_uint4(e[0], e[1], e[2], e[3]);
      if (out) {
        uint8_t* ob = reinterpret_cast<uint8_t*>(out + w0);
        for (uint32_t b = 0; b < 16 && w0 * 4 + b < vbytes; ++b) ob[b] = (uint8_t)(e[b >> 2] >> (8 * (b & 3)));
      }
    } else if (out) {
      __stcs(reinterpret_cast<uint4*>(out + w0), v);
    }
    ones += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
  }
  for (int o = 16; o; o >>= 1) ones += __shfl_xor_sync(kFull, ones, o);
  if (lane == 0) s_red[warp] = ones;
  __syncthreads();
  if (warp == 0) {
    unsigned long long tsum = lane < (bd >> 5) ? s_red[lane] : 0;
    for (int o = 16; o; o >>= 1) tsum += __shfl_xor_sync(kFull, tsum, o);
    if (lane == 0) atomicAdd(a.count, (unsigned long long)valid - tsum);
  }
}

// ---------------------------------------------------------------------------
// Large primes (p > S), per wave of W tiles (WS = W*S bits).  The paper's
// bucket sort (large_kernel.hpp: an entry lands in the bucket of the segment
// it next hits, the segment consumes the bucket, the entry advances and
// re-buckets) rebuilt for ~148 tiles in flight, in two kernels per wave:
//
//  k_gen  walks every large prime with a hit in the wave — ML primes
//         (S < p <= WS: state u32 pos | s << 29, visited every wave) and the
//         wave's far bucket (p > WS, u64 entries p | (q | s<<29) << 32) —
//         and appends one record per wheel-admissible multiple (its position
//         in the wave) to a per-warp region of a global buffer, 32 lanes at a
//         time (ballot/popc compaction: coalesced stores, no atomics).  Far
//         entries leave re-bucketed into per-warp regions tagged with the
//         ring slot of the wave of their next hit (Lemma 2).
//         Control flow is warp-uniform (loops run while any lane has work).
//  k_bin  counting-sorts the records by tile (and the re-bucketed far entries
//         by ring slot) in shared memory, chunk by chunk, and flushes each
//         tile's run with coalesced stores into that tile's hit list; one
//         global atomicAdd per (chunk, tile) reserves the run.
//
// ML primes with p <= WS/8 are walked by 8 lanes (lane j of an octet: wheel
// class (s+j)&7, step 15p), the others one per lane.
struct GenArgs {
  uint2* ml;             // ML primes, ascending: {p | s << 29, pos}
  uint32_t nml, noct;    // the first noct ML primes are walked by octets
  const uint64_t* far_in;  // far bucket of this wave
  const uint32_t* far_in_count;
  uint32_t bcap, ring;
  uint64_t wave, nwaves;
  uint32_t WS;        // wave span in bits
  uint32_t ntiles_w;  // tiles in this wave (records beyond are dropped)
  uint32_t log_s;
  uint32_t* recs;     // [nwarps][rcap] records (position in the wave)
  uint32_t* rcount;   // [nwarps]
  uint32_t rcap;
  uint64_t* frecs;    // [nwarps][fcap] re-bucketed far entries
  uint8_t* fslot;     // [nwarps][fcap] their ring slot
  uint32_t* fcount;   // [nwarps]
  uint32_t fcap;
  int* overflow;
};

constexpr int kGenThreads = 512;

struct WarpOut {
  uint32_t* rec;
  uint32_t n, cap;
  uint64_t* frec;
  uint8_t* fsl;
  uint32_t fn, fcap;
};

// append the valid lanes' records (warp-uniform call)
__device__ __forceinline__ void wappend(WarpOut& o, bool valid, uint32_t rec) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t m = __ballot_sync(kFull, valid);
  const uint32_t k = o.n + __popc(m & ((1u << lane) - 1));
  if (valid && k < o.cap) o.rec[k] = rec;
  o.n += __popc(m);
}

__global__ void __launch_bounds__(kGenThreads) k_gen(const GenArgs a) {
  __shared__ uint32_t s_cum[8];
  if (threadIdx.x < 8) {
    uint32_t v = 0;
    for (int k = 0; k < 8; ++k) v |= (uint32_t)c_cum[threadIdx.x][k] << (4 * k);
    s_cum[threadIdx.x] = v;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t)blockIdx.x * (kGenThreads / 32) + (threadIdx.x >> 5);
  const uint64_t nw = (uint64_t)gridDim.x * (kGenThreads / 32);
  const uint32_t WS = a.WS;
  const uint32_t lim = a.ntiles_w << a.log_s;  // positions past the last tile of the wave are dropped
  WarpOut o{a.recs + gw * a.rcap, 0, a.rcap, a.frecs + gw * a.fcap, a.fslot + gw * a.fcap, 0, a.fcap};

  // octets: 4 primes per warp-step (next step's data prefetched)
  const uint64_t uo = (a.noct + 3) / 4;
  {
    const uint32_t j = lane & 7;
    uint64_t u = gw;
    uint32_t pn = 0, stn = 0;
    if (u < uo && u * 4 + (lane >> 3) < a.noct) {
      const uint2 e = a.ml[u * 4 + (lane >> 3)];
      pn = e.x;
      stn = e.y;
    }
    for (; u < uo; u += nw) {
      const uint64_t i = u * 4 + (lane >> 3);
      const bool ok = i < a.noct;
      const uint32_t p = pn & 0x1fffffffu, st = stn, cls = pn >> 29;
      const uint64_t inx = (u + nw) * 4 + (lane >> 3);
      if (u + nw < uo && inx < a.noct) {
        const uint2 e = a.ml[inx];
        pn = e.x;
        stn = e.y;
      }
      const uint32_t s0 = cls;
      uint32_t pos = ok ? st + p * nib(s_cum[s0], j) : WS;
      const uint32_t step = 15u * p;
      while (__any_sync(kFull, pos < WS)) {
        const bool v = pos < WS;
        wappend(o, v && pos < lim, pos);
        if (v) pos += step;
      }
      // next hit of the prime = smallest exit of its 8 class progressions
      const uint32_t ex = pos - WS;
      uint32_t m = ex;
      m = min(m, __shfl_xor_sync(kFull, m, 1));
      m = min(m, __shfl_xor_sync(kFull, m, 2));
      m = min(m, __shfl_xor_sync(kFull, m, 4));
      const uint32_t bal = (__ballot_sync(kFull, ex == m) >> (lane & ~7u)) & 0xffu;
      if (ok && j == 0) a.ml[i] = make_uint2(p | (((s0 + __ffs(bal) - 1) & 7) << 29), m);
    }
  }
  // single ML primes: one per lane (next step's data prefetched)
  const uint64_t us = (a.nml - a.noct + 31) / 32;
  {
    uint64_t u = gw;
    uint32_t pn = 0, stn = 0;
    if (u < us && a.noct + u * 32 + lane < a.nml) {
      const uint2 e = a.ml[a.noct + u * 32 + lane];
      pn = e.x;
      stn = e.y;
    }
    for (; u < us; u += nw) {
      const uint64_t i = a.noct + u * 32 + lane;
      const bool ok = i < a.nml;
      const uint32_t p = pn & 0x1fffffffu, st = stn, cls = pn >> 29;
      const uint64_t inx = a.noct + (u + nw) * 32 + lane;
      if (u + nw < us && inx < a.nml) {
        const uint2 e = a.ml[inx];
        pn = e.x;
        stn = e.y;
      }
      uint32_t pos = ok ? st : WS;
      uint32_t s = cls;
      while (__any_sync(kFull, pos < WS)) {
        const bool v = pos < WS;
        wappend(o, v && pos < lim, pos);
        if (v) {
          pos += wheel_D(s) * p;
          s = (s + 1) & 7;
        }
      }
      if (ok) a.ml[i] = make_uint2(p | (s << 29), pos - WS);
    }
  }
  // far: exactly one hit in this wave, then re-bucket
  const uint32_t nfar = a.far_in ? min(*a.far_in_count, a.bcap) : 0;
  const uint64_t uf = (nfar + 31) / 32;
  for (uint64_t u = gw; u < uf; u += nw) {
    const uint64_t i = u * 32 + lane;
    const bool ok = i < nfar;
    const uint64_t e = ok ? a.far_in[i] : 0;
    const uint32_t p = (uint32_t)e;
    const uint32_t q = (uint32_t)(e >> 32) & 0x1fffffffu, s = (uint32_t)(e >> 61);
    wappend(o, ok && q < lim, q);
    bool keep = false;
    uint32_t slot = 0;
    uint64_t ne = 0;
    if (ok) {
      const uint64_t q2 = (uint64_t)q + (uint64_t)wheel_D(s) * p;
      const uint64_t d = q2 / WS;
      const uint64_t tgt = a.wave + d;
      if (tgt < a.nwaves) {
        keep = true;
        slot = (uint32_t)(tgt % a.ring);
        ne = (uint64_t)p | ((uint64_t)((uint32_t)(q2 - d * WS) | (((s + 1) & 7) << 29)) << 32);
      }
    }
    const uint32_t m = __ballot_sync(kFull, keep);
    const uint32_t k = o.fn + __popc(m & ((1u << lane) - 1));
    if (keep && k < o.fcap) {
      o.frec[k] = ne;
      o.fsl[k] = (uint8_t)slot;
    }
    o.fn += __popc(m);
  }
  // pad the record region to a multiple of 4 records (k_bin loads uint4);
  // the sentinel's tile index is above every wave's tile count
  const uint32_t nv = min(o.n, o.cap), n4 = min((nv + 3) & ~3u, o.cap);
  if (lane < n4 - nv) o.rec[nv + lane] = 0xffffffffu;
  if (lane == 0) {
    a.rcount[gw] = n4;
    a.fcount[gw] = min(o.fn, o.fcap);
    if (o.n > o.cap || o.fn > o.fcap) atomicExch(a.overflow, 1);
  }
}

struct BinArgs {
  const uint32_t* recs;
  const uint32_t* rcount;
  uint32_t rcap, nregions;
  const uint64_t* frecs;  // nullable: no far entries
  const uint8_t* fslot;
  const uint32_t* fcount;
  uint32_t fcap;
  uint32_t ntiles_w, log_s;
  uint32_t* hits;    // [ntiles_w][hcap]
  uint32_t* hitcnt;  // [ntiles_w]
  uint32_t hcap;
  uint64_t* far_buckets;  // [ring][bcap]
  uint32_t* far_bcount;
  uint32_t ring, bcap;
  int* overflow;
};

constexpr int kBinThreads = 512;
constexpr int kBinPer = 16;                          // records per thread per chunk
constexpr int kBinChunk = kBinThreads * kBinPer;     // 8192 records
constexpr int kFarPer = 8;
constexpr int kFarChunk = kBinThreads * kFarPer;     // 4096 far entries
constexpr int kMaxWaveTiles = 256;
constexpr int kMaxRing = 256;
constexpr int kMaxRegionsPerCta = 64;

struct BinSmem {
  union {
    struct {
      uint32_t a[kBinChunk];  // chunk as loaded
      uint32_t b[kBinChunk];  // chunk sorted by tile
    } r;
    struct {
      uint64_t a[kFarChunk];
      uint64_t b[kFarChunk];
      uint8_t ka[kFarChunk];
      uint8_t kb[kFarChunk];
    } f;
  } u;
  uint32_t cnt[kMaxRing + 1];  // [nb]: spill bucket of the sentinels
  uint32_t off[kMaxRing + 1];
  uint32_t base[kMaxRing + 1];
  uint32_t pre[kMaxRegionsPerCta + 1];  // prefix of the CTA's region counts
  uint32_t total;
};

__device__ __forceinline__ uint32_t warp_excl_scan(const uint32_t* cnt, uint32_t* off, uint32_t n) {
  // one warp scans n counters; returns the total
  const uint32_t lane = threadIdx.x & 31;
  uint32_t run = 0;
  for (uint32_t t0 = 0; t0 < n; t0 += 32) {
    const uint32_t t = t0 + lane;
    const uint32_t c = t < n ? cnt[t] : 0;
    uint32_t x = c;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (t < n) off[t] = run + x - c;
    run += __shfl_sync(kFull, x, 31);
  }
  return run;
}

// index of the region holding stream position i (pre[] ascending, nr regions)
__device__ __forceinline__ uint32_t region_of(const uint32_t* pre, uint32_t nr, uint32_t i) {
  uint32_t lo = 0, hi = nr;  // pre[lo] <= i < pre[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (pre[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Counting sort of sm.u.r.a[0..n) (n % 4 == 0; sentinels have key >> shift
// >= nb and land in the spill bucket nb, after the real records) by
// key >> shift into sm.u.r.b, then one coalesced run per bucket to
// dst[bucket * cap + reserved ...].
__device__ void bin_sort_flush(BinSmem& sm, uint32_t n, uint32_t shift, uint32_t nb, uint32_t vmask, uint32_t* dst,
                               uint32_t* gcnt, uint32_t cap, int* overflow) {
  const uint32_t tid = threadIdx.x;
  const uint4* a4 = reinterpret_cast<const uint4*>(sm.u.r.a);
  const uint32_t n4 = n >> 2;
  for (uint32_t i = tid; i < n4; i += blockDim.x) {
    const uint4 k = a4[i];
    atomicAdd(&sm.cnt[min(k.x >> shift, nb)], 1u);
    atomicAdd(&sm.cnt[min(k.y >> shift, nb)], 1u);
    atomicAdd(&sm.cnt[min(k.z >> shift, nb)], 1u);
    atomicAdd(&sm.cnt[min(k.w >> shift, nb)], 1u);
  }
  __syncthreads();
  if (tid < 32) {
    const uint32_t tot = warp_excl_scan(sm.cnt, sm.off, nb + 1);  // off[nb] = real total
    if (tid == 0) sm.total = sm.off[nb];
    (void)tot;
  }
  uint32_t resv = 0, rc = 0;
  if (tid >= 32 && tid < 32 + nb) {  // reservation in flight during the placement
    rc = sm.cnt[tid - 32];
    if (rc) resv = atomicAdd(&gcnt[tid - 32], rc);
  }
  __syncthreads();
  for (uint32_t t = tid; t <= nb; t += blockDim.x) sm.cnt[t] = 0;
  __syncthreads();
  for (uint32_t i = tid; i < n4; i += blockDim.x) {
    const uint4 k = a4[i];
    const uint32_t t0 = min(k.x >> shift, nb), t1 = min(k.y >> shift, nb), t2 = min(k.z >> shift, nb),
                   t3 = min(k.w >> shift, nb);
    const uint32_t s0 = sm.off[t0] + atomicAdd(&sm.cnt[t0], 1u);
    const uint32_t s1 = sm.off[t1] + atomicAdd(&sm.cnt[t1], 1u);
    const uint32_t s2 = sm.off[t2] + atomicAdd(&sm.cnt[t2], 1u);
    const uint32_t s3 = sm.off[t3] + atomicAdd(&sm.cnt[t3], 1u);
    sm.u.r.b[s0] = k.x;
    sm.u.r.b[s1] = k.y;
    sm.u.r.b[s2] = k.z;
    sm.u.r.b[s3] = k.w;
  }
  if (tid >= 32 && tid < 32 + nb) {
    sm.base[tid - 32] = resv;
    if (rc && resv + rc > cap) atomicExch(overflow, 1);
  }
  __syncthreads();
  for (uint32_t t = tid; t <= nb; t += blockDim.x) sm.cnt[t] = 0;
  const uint32_t total = sm.total;
  for (uint32_t i = tid; i < total; i += blockDim.x) {
    const uint32_t key = sm.u.r.b[i];
    const uint32_t t = key >> shift;
    EG_CHECK(t < nb && i >= sm.off[t], "bin t=%u nb=%u i=%u off=%u", t, nb, i, sm.off[t]);
    const uint32_t slot = sm.base[t] + (i - sm.off[t]);
    if (slot < cap) dst[(uint64_t)t * cap + slot] = key & vmask;
  }
  __syncthreads();
}

// same for far entries keyed by their ring slot
__device__ void bin_sort_flush_far(BinSmem& sm, uint32_t n, uint32_t nb, uint64_t* dst, uint32_t* gcnt, uint32_t cap,
                                   int* overflow) {
  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i < n; i += blockDim.x) atomicAdd(&sm.cnt[sm.u.f.ka[i]], 1u);
  __syncthreads();
  if (tid < 32) {
    const uint32_t tot = warp_excl_scan(sm.cnt, sm.off, nb);
    if (tid == 0) sm.total = tot;
  }
  uint32_t resv = 0, rc = 0;
  if (tid >= 32 && tid < 32 + nb) {
    rc = sm.cnt[tid - 32];
    if (rc) resv = atomicAdd(&gcnt[tid - 32], rc);
  }
  __syncthreads();
  for (uint32_t t = tid; t < nb; t += blockDim.x) sm.cnt[t] = 0;
  __syncthreads();
  for (uint32_t i = tid; i < n; i += blockDim.x) {
    const uint32_t t = sm.u.f.ka[i];
    const uint32_t k = sm.off[t] + atomicAdd(&sm.cnt[t], 1u);
    sm.u.f.b[k] = sm.u.f.a[i];
    sm.u.f.kb[k] = (uint8_t)t;
  }
  if (tid >= 32 && tid < 32 + nb) {
    sm.base[tid - 32] = resv;
    if (rc && resv + rc > cap) atomicExch(overflow, 1);
  }
  __syncthreads();
  for (uint32_t t = tid; t < nb; t += blockDim.x) sm.cnt[t] = 0;
  for (uint32_t i = tid; i < n; i += blockDim.x) {
    const uint32_t t = sm.u.f.kb[i];
    const uint32_t slot = sm.base[t] + (i - sm.off[t]);
    if (slot < cap) dst[(uint64_t)t * cap + slot] = sm.u.f.b[i];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kBinThreads) k_bin(const BinArgs a) {
  extern __shared__ uint4 smem_raw[];
  BinSmem& sm = *reinterpret_cast<BinSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  // this CTA's contiguous block of k_gen regions
  const uint32_t per = (a.nregions + gridDim.x - 1) / gridDim.x;
  const uint32_t rb = min(a.nregions, blockIdx.x * per), re = min(a.nregions, rb + per);
  const uint32_t nr = re - rb;
  EG_CHECK(nr <= kMaxRegionsPerCta, "regions per CTA %u", nr);
  for (uint32_t t = tid; t < kMaxRing; t += blockDim.x) sm.cnt[t] = 0;
  // ---- hit records: the CTA's regions as one stream, 8192-record chunks ----
  if (tid < 32) {
    uint32_t run = 0;
    for (uint32_t r0 = 0; r0 < nr; r0 += 32) {
      const uint32_t r = r0 + tid;
      const uint32_t c = r < nr ? a.rcount[rb + r] : 0;
      uint32_t x = c;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (tid >= o) x += y;
      }
      if (r < nr) sm.pre[r] = run + x - c;
      run += __shfl_sync(kFull, x, 31);
    }
    if (tid == 0) sm.pre[nr] = run;
  }
  __syncthreads();
  const uint32_t ntot = sm.pre[nr];  // multiple of 4: every region is padded
  const uint32_t smask = (1u << a.log_s) - 1;
  constexpr int kPer4 = kBinPer / 4;
  uint4 reg[kPer4];
  auto load_chunk = [&](uint32_t c0) {
    // uint4 units c0/4 + tid + k*512 grow with k: one search, then forward walks
    const uint32_t i0 = c0 + 4 * tid;
    uint32_t r = i0 < ntot ? region_of(sm.pre, nr, i0) : 0;
#pragma unroll
    for (int k = 0; k < kPer4; ++k) {
      const uint32_t i = i0 + 4 * k * kBinThreads;
      if (i < ntot) {
        while (sm.pre[r + 1] <= i) ++r;
        reg[k] = *reinterpret_cast<const uint4*>(a.recs + (uint64_t)(rb + r) * a.rcap + (i - sm.pre[r]));
      }
    }
  };
  if (ntot) load_chunk(0);
  for (uint32_t c0 = 0; c0 < ntot; c0 += kBinChunk) {
    const uint32_t n = min((uint32_t)kBinChunk, ntot - c0);
    uint4* a4 = reinterpret_cast<uint4*>(sm.u.r.a);
#pragma unroll
    for (int k = 0; k < kPer4; ++k)
      if (4 * (tid + k * kBinThreads) < n) a4[tid + k * kBinThreads] = reg[k];
    __syncthreads();
    if (c0 + kBinChunk < ntot) load_chunk(c0 + kBinChunk);  // next chunk in flight
    bin_sort_flush(sm, n, a.log_s, a.ntiles_w, smask, a.hits, a.hitcnt, a.hcap, a.overflow);
  }
  // ---- re-bucketed far entries, sorted by ring slot ----
  if (a.frecs) {
    if (tid < 32) {
      uint32_t run = 0;
      for (uint32_t r0 = 0; r0 < nr; r0 += 32) {
        const uint32_t r = r0 + tid;
        const uint32_t c = r < nr ? a.fcount[rb + r] : 0;
        uint32_t x = c;
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, o);
          if (tid >= o) x += y;
        }
        if (r < nr) sm.pre[r] = run + x - c;
        run += __shfl_sync(kFull, x, 31);
      }
      if (tid == 0) sm.pre[nr] = run;
    }
    __syncthreads();
    const uint32_t ftot = sm.pre[nr];
    for (uint32_t c0 = 0; c0 < ftot; c0 += kFarChunk) {
      const uint32_t n = min((uint32_t)kFarChunk, ftot - c0);
      uint32_t r = c0 + tid < ftot ? region_of(sm.pre, nr, c0 + tid) : 0;
#pragma unroll
      for (int k = 0; k < kFarPer; ++k) {
        const uint32_t i = c0 + tid + k * kBinThreads;
        if (i < ftot) {
          while (sm.pre[r + 1] <= i) ++r;
          const uint64_t src = (uint64_t)(rb + r) * a.fcap + (i - sm.pre[r]);
          sm.u.f.a[i - c0] = a.frecs[src];
          sm.u.f.ka[i - c0] = a.fslot[src];
        }
      }
      __syncthreads();
      bin_sort_flush_far(sm, n, a.ring, a.far_buckets, a.far_bcount, a.bcap, a.overflow);
    }
  }
}

// ---------------------------------------------------------------------------
// Large-prime scatter (default path), two kernels per wave:
//  k_scatter_ml   walks the ML primes (S < p <= WS), one lane per prime,
//                 resumable per step: a warp walks until its staging area is
//                 full, not until its primes are done;
//  k_scatter_far  takes the wave's far bucket (p > WS): exactly one hit in
//                 the wave, then the entry moves to the bucket of the wave of
//                 its next hit, k or k+1 waves ahead (Lemma 2,
//                 the paper's in-place bucket sort,
//                 large_kernel.hpp:61-213, as a ring of per-wave buckets).
// Every hit becomes one u32 record (its position in the wave).  A warp stages
// one record per lane per step in shared memory at [step][lane] (no ballot
// compaction: an idle lane stores a sentinel), with its rank among this
// round's records of the same tile — the value of the shared tile counter
// the lane bumps when it emits.  When a warp's area is full the CTA runs a
// round: a scan of the tile counts and one global atomicAdd per non-empty
// tile reserving a run in that tile's hit list; records are placed in tile
// order at off[tile] + rank (no atomics) and written as coalesced runs.
// Re-bucketed far entries (8 B) go from staging straight to
// bucket[reserved + rank].
struct ScatterArgs {
  uint2* ml;  // ML primes, ascending: {p | s << 29, pos} (pos = next hit from the current window start)
  uint32_t nml;
  const uint64_t* far_in;  // far bucket of this wave: p | (q | s << 29) << 32
  const uint32_t* far_in_count;
  uint64_t* far_buckets;  // [ring][bcap] + trash
  uint32_t* far_bcount;
  uint32_t bcap, ring, wslot;  // wslot = wave % ring
  uint64_t wave, nwaves;
  uint32_t WS, ntiles_w, log_s;
  float inv_ws_f;  // 1 / WS
  uint32_t* hits;    // [ntiles_w][hcap] + trash
  uint32_t* hitcnt;  // [ntiles_w]
  uint32_t hcap;
  int* overflow;
};

constexpr int kScBins = 256;            // >= tiles per ML window and >= ring slots
constexpr uint32_t kNoRec = 0xffffffffu;  // staged-slot sentinel (idle lane)
constexpr uint8_t kNoSlot = 0xff;

template <int NW, int SL, bool FAR>
struct ScSmem {
  static constexpr int R = SL * 32;  // staged records per warp
  static constexpr int FR = FAR ? R : 1;
  uint32_t reg[NW * R];   // warp w, step k, lane j at [w*R + k*32 + j]
  uint16_t rank[NW * R];  // rank among this round's records of the same tile
  uint32_t srt[NW * R];   // this round's records sorted by tile
  uint64_t freg[NW * FR];
  uint16_t frank[NW * FR];
  uint8_t fslot[NW * FR];
  // cnt: per-round counts (bumped at emission; [kScBins + lane] = sinks of
  // idle lanes, one per lane: no same-address conflicts); off: their
  // exclusive scan; gofs[t] = global index of sorted slot 0 of tile t
  // (t*cap + reserved - off)
  uint32_t cnt[kScBins + 32], off[kScBins], gofs[kScBins];
  uint32_t fcnt[FAR ? kScBins + 32 : 1], fgofs[FAR ? kScBins : 1];
  uint32_t total;
  static_assert(NW * R < 65536, "ranks are 16-bit");
};

// Shared-memory helpers for the emission loops (32-bit shared addresses).
// r = atomicAdd(cnt, 1) and the record store (unconditional: idle lanes
// count into their sink and stage the sentinel).  The rank r is stored one
// step later (st_rank), so the atomic's latency overlaps the next step.
__device__ __forceinline__ uint32_t stage_rec(uint32_t cnt_addr, uint32_t reg_addr, uint32_t val) {
  uint32_t r;
  asm volatile(
      "atom.shared.add.u32 %0, [%1], 1;\n\t"
      "st.shared.u32 [%2], %3;"
      : "=r"(r)
      : "r"(cnt_addr), "r"(reg_addr), "r"(val)
      : "memory");
  return r;
}
__device__ __forceinline__ uint32_t stage_far(uint32_t cnt_addr, uint32_t ent_addr, uint32_t slot_addr, uint64_t ent,
                                              uint32_t slot) {
  uint32_t r;
  asm volatile(
      "atom.shared.add.u32 %0, [%1], 1;\n\t"
      "st.shared.u64 [%2], %4;\n\t"
      "st.shared.u8 [%3], %5;"
      : "=r"(r)
      : "r"(cnt_addr), "r"(ent_addr), "r"(slot_addr), "l"(ent), "r"(slot)
      : "memory");
  return r;
}
__device__ __forceinline__ void st_rank(uint32_t addr, uint32_t r) {
  asm volatile("st.shared.u16 [%0], %1;" : : "r"(addr), "r"(r) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" : : "r"(addr), "r"(v) : "memory");
}
// if (key != kNoRec) *addr = key
__device__ __forceinline__ void sts_if_rec(uint32_t addr, uint32_t key) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %1, -1; @q st.shared.u32 [%0], %1; }" : : "r"(addr), "r"(key)
               : "memory");
}

// COMPACT: the warp's staging holds n real records (no sentinels).
template <int NW, int SL, bool FAR, bool COMPACT = false>
__device__ __forceinline__ void sc_flush(ScSmem<NW, SL, FAR>& sm, const ScatterArgs& a, uint32_t n) {
  using Sm = ScSmem<NW, SL, FAR>;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t NT = NW * 32;
  const uint32_t nb = a.ntiles_w, ring = FAR ? a.ring : 0;
  if (tid < 32) {
    const uint32_t tot = warp_excl_scan(sm.cnt, sm.off, nb);
    if (tid == 0) sm.total = tot;
  } else {
    for (uint32_t b = tid - 32; b < nb + ring; b += NT - 32) {
      if (b < nb) {
        const uint32_t c = sm.cnt[b];
        if (c) {
          const uint32_t r = atomicAdd(&a.hitcnt[b], c);
          const bool over = r + c > a.hcap;
          if (over) atomicExch(a.overflow, 1);
          sm.gofs[b] = over ? nb * a.hcap : b * a.hcap + r;
        }
      } else if constexpr (FAR) {
        const uint32_t t = b - nb, c = sm.fcnt[t];
        if (c) {
          sm.fcnt[t] = 0;  // nobody counts again before the next barrier
          const uint32_t r = atomicAdd(&a.far_bcount[t], c);
          const bool over = r + c > a.bcap;
          if (over) atomicExch(a.overflow, 1);
          sm.fgofs[t] = over ? a.ring * a.bcap : t * a.bcap + r;
        }
      }
    }
  }
  __syncthreads();
  const uint32_t shift = a.log_s, smask = (1u << shift) - 1;
  const uint32_t off_a = smem_addr(sm.off), srt_a = smem_addr(sm.srt), gofs_a = smem_addr(sm.gofs);
  {
    // placement in tile order (sentinels of idle lanes are skipped)
    const uint32_t rg_a = smem_addr(sm.reg + warp * Sm::R), rk_a = smem_addr(sm.rank + warp * Sm::R);
#pragma unroll kPlaceUnroll
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t key = lds_u32(rg_a + 4 * i);
      if constexpr (COMPACT) {
        const uint32_t o = lds_u32(off_a + 4 * (key >> shift));
        sts_u32(srt_a + 4 * (o + lds_u16(rk_a + 2 * i)), key);
      } else {
        const uint32_t o = lds_u32(off_a + 4 * min(key >> shift, (uint32_t)kScBins - 1));  // sentinels: any bin
        sts_if_rec(srt_a + 4 * (o + lds_u16(rk_a + 2 * i)), key);
      }
    }
  }
  if constexpr (FAR) {
    const uint32_t base = warp * Sm::FR;
    const uint32_t fs_a = smem_addr(sm.fslot + base), fr_a = smem_addr(sm.frank + base),
                   fe_a = smem_addr(sm.freg + base), fg_a = smem_addr(sm.fgofs);
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t t = lds_u8(fs_a + i);
      EG_CHECK(t == kNoSlot || (t < a.ring && lds_u32(fg_a + 4 * t) + lds_u16(fr_a + 2 * i) < a.ring * a.bcap + NW * Sm::R),
               "far bucket index out of range slot=%u", t);
      if (t != kNoSlot) a.far_buckets[lds_u32(fg_a + 4 * t) + lds_u16(fr_a + 2 * i)] = lds_u64(fe_a + 8 * i);
    }
  }
  for (uint32_t b = tid; b < nb; b += NT) {
    if (sm.cnt[b]) sm.gofs[b] -= sm.off[b];
    sm.cnt[b] = 0;
  }  // (the sinks are never read: their counts may wrap)
  __syncthreads();
  const uint32_t total = sm.total;
#pragma unroll kWriteUnroll
  for (uint32_t i = tid; i < total; i += NT) {
    const uint32_t key = lds_u32(srt_a + 4 * i);
    EG_CHECK((key >> shift) < nb && lds_u32(gofs_a + 4 * (key >> shift)) + i < nb * a.hcap + NW * Sm::R,
             "hit list index out of range key=%u", key);
    a.hits[lds_u32(gofs_a + 4 * (key >> shift)) + i] = key & smask;
  }
  // off/gofs/srt are rewritten only after the next round's first barrier
}

#ifndef EG_ML_WARPS
#define EG_ML_WARPS 8
#endif
#ifndef EG_ML_STEPS
#define EG_ML_STEPS 12
#endif
#ifndef EG_FAR_WARPS
#define EG_FAR_WARPS 8
#endif
#ifndef EG_FAR_STEPS
#define EG_FAR_STEPS 6
#endif
#ifndef EG_ML_PF
#define EG_ML_PF 1
#endif
#ifndef EG_ML_COMPACT
#define EG_ML_COMPACT 1
#endif
constexpr int kMlWarps = EG_ML_WARPS, kMlSteps = EG_ML_STEPS, kMlPf = EG_ML_PF;
#ifndef EG_FAR_PF
#define EG_FAR_PF 2
#endif
constexpr int kFarWarps = EG_FAR_WARPS, kFarSteps = EG_FAR_STEPS, kFarPf = EG_FAR_PF;
using MlSmem = ScSmem<kMlWarps, kMlSteps, false>;
using FarSmem = ScSmem<kFarWarps, kFarSteps, true>;
// records / entries one round may send to the trash area
constexpr uint32_t kScTrash0 = (uint32_t)(MlSmem::R * kMlWarps > FarSmem::R * kFarWarps ? MlSmem::R * kMlWarps
                                                                                        : FarSmem::R * kFarWarps);
constexpr uint32_t kScTrash = kScTrash0 > 8192 ? kScTrash0 : 8192;  // (>= a k_far_walk round and a k_wave_sort chunk)

__device__ __forceinline__ uint32_t rotr4(uint32_t x) { return __funnelshift_r(x, x, 4); }

template <bool ML7>
__device__ __forceinline__ void scatter_ml(const ScatterArgs& a, uint32_t blk, uint32_t nblk, MlSmem& sm) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t t = tid; t < kScBins; t += blockDim.x) sm.cnt[t] = 0;
  __syncthreads();
  const uint32_t WS = a.WS, shift = a.log_s;
  // walk bound: the wave end, or the end of the last tile in the last wave
  // (the state written back after the last wave is never read)
  const uint32_t B = a.ntiles_w << a.log_s;
  const uint32_t nw = nblk * kMlWarps;
  const uint32_t nu = (a.nml + 31) / 32;
  const uint32_t reg_a = smem_addr(sm.reg + warp * MlSmem::R + lane);
  const uint32_t rank_a = smem_addr(sm.rank + warp * MlSmem::R + lane);
  const uint32_t cnt_a = smem_addr(sm.cnt), sink_a = cnt_a + 4 * (kScBins + lane);
#ifndef EG_BOUS
#define EG_BOUS 1
#endif
  // unit order of a warp: row k of nw units, alternately from the left and
  // from the right (primes ascend, so hits per unit descend: pairing a dense
  // unit of one row with a sparse one of the next evens out the warps' work)
  const uint32_t gw0 = blk * kMlWarps + warp;
  uint32_t urow = 0;
  auto unit_at = [&](uint32_t k) -> uint32_t {
    return k * nw + ((EG_BOUS && EG_ML_COMPACT && (k & 1)) ? nw - 1 - gw0 : gw0);
  };
  uint32_t u = gw0;
  uint32_t idx = u * 32 + lane;
  bool ok = u < nu && idx < a.nml;
  uint2 e0 = ok ? a.ml[idx] : make_uint2(0, 0);
  uint32_t p, pos, s, c7 = 0;
  auto decode = [&](uint2 e) {
    if (ML7) {
      p = e.x & 0x0fffffffu;
      s = (e.x >> 28) & 7;
      c7 = (e.x >> 31) | ((e.y >> 30) << 1);
      pos = ok ? e.y & 0x3fffffffu : B;
    } else {
      p = e.x & 0x1fffffffu;
      s = e.x >> 29;
      pos = ok ? e.y : B;
    }
  };
  decode(e0);
  uint32_t dd = __funnelshift_r(0x13212123u, 0x13212123u, 4 * s);  // low nibble = wheel_D(s)
  // the next kMlPf units' primes and states are in flight (a sparse unit
  // takes only a few steps, far less than a DRAM round trip)
  auto load = [&](uint32_t uu) -> uint2 {
    const uint32_t j = uu * 32 + lane;
    return (uu < nu && j < a.nml) ? a.ml[j] : make_uint2(0, 0);
  };
  uint2 pf[kMlPf];
#pragma unroll
  for (int k = 0; k < kMlPf; ++k) pf[k] = load(unit_at(k + 1));
  bool live = u < nu;  // warp-uniform
#if EG_ML_COMPACT
  // Compacted emission: a step's records go to consecutive staging slots
  // (ballot + popc), so a round holds R real records per warp whatever the
  // share of idle lanes, and the placement / write passes and the per-round
  // scan, reservations and barriers are paid per record, not per lane slot.
  uint32_t ltm;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltm));
  const uint32_t regw_a = smem_addr(sm.reg + warp * MlSmem::R), rankw_a = smem_addr(sm.rank + warp * MlSmem::R);
  for (;;) {
    uint32_t kb = 0;  // staged records of this warp (warp-uniform)
    while (live && kb <= (uint32_t)MlSmem::R - 32) {
      const bool v = pos < B;
      const uint32_t m = __ballot_sync(kFull, v);
      if (!m) {
        if (ok) a.ml[idx] = ML7 ? ml7_pack(p, pos - WS, s, c7) : make_uint2(p | ((s & 7) << 29), pos - WS);
        ++urow;
        u = unit_at(urow);
        if (u >= nu) {
          live = false;
          break;
        }
        idx = u * 32 + lane;
        ok = idx < a.nml;
        decode(pf[0]);
        dd = __funnelshift_r(0x13212123u, 0x13212123u, 4 * s);
#pragma unroll
        for (int k = 0; k + 1 < kMlPf; ++k) pf[k] = pf[k + 1];
        pf[kMlPf - 1] = load(unit_at(urow + kMlPf));
        continue;
      }
      const uint32_t slot = kb + __popc(m & ltm);
      kb += __popc(m);
      if (v) {
        uint32_t r;
        asm volatile(
            "atom.shared.add.u32 %0, [%1], 1;\n\t"
            "st.shared.u32 [%2], %3;"
            : "=r"(r)
            : "r"(cnt_a + ((pos >> shift) << 2)), "r"(regw_a + (slot << 2)), "r"(pos)
            : "memory");
        const uint32_t D = dd & 15u;
        pos += D * p;
        dd = rotr4(dd);
        ++s;
        if (ML7) {  // the next admissible cofactor may be divisible by 7: then take the one after
          c7 += 2 * D;
          c7 -= c7 >= 7 ? 7 : 0;
          if (c7 == 0) {
            const uint32_t D2 = dd & 15u;
            pos += D2 * p;
            dd = rotr4(dd);
            ++s;
            c7 = 2 * D2;
          }
          EG_CHECK(c7 >= 1 && c7 <= 6 && pos < (1u << 30) + WS, "ML c7=%u pos=%u p=%u", c7, pos, p);
        }
        st_rank(rankw_a + (slot << 1), r);
      }
    }
    const int more = __syncthreads_or(live);
    sc_flush<kMlWarps, kMlSteps, false, true>(sm, a, kb);
    if (!more) break;
  }
  (void)reg_a;
  (void)rank_a;
  (void)sink_a;
#else
  for (;;) {
    bool rk_pend = false;  // the last staged rank is stored one step late
    uint32_t rk_addr = 0, rk_val = 0;
    uint32_t k = 0;  // staged steps (warp-uniform)
    while (live && k < (uint32_t)kMlSteps) {
      const bool v = pos < B;
      if (!__any_sync(kFull, v)) {
        if (ok) a.ml[idx] = ML7 ? ml7_pack(p, pos - WS, s, c7) : make_uint2(p | ((s & 7) << 29), pos - WS);
        u += nw;
        if (u >= nu) {
          live = false;
          break;
        }
        idx = u * 32 + lane;
        ok = idx < a.nml;
        decode(pf[0]);
        dd = __funnelshift_r(0x13212123u, 0x13212123u, 4 * s);
#pragma unroll
        for (int k = 0; k + 1 < kMlPf; ++k) pf[k] = pf[k + 1];
        pf[kMlPf - 1] = load(u + kMlPf * nw);
        continue;
      }
      const uint32_t r = stage_rec(v ? cnt_a + ((pos >> shift) << 2) : sink_a, reg_a + (k << 7), v ? pos : kNoRec);
      if (rk_pend) st_rank(rk_addr, rk_val);
      rk_pend = true;
      rk_addr = rank_a + (k << 6);
      rk_val = r;
      ++k;
      if (v) {
        const uint32_t D = dd & 15u;
        pos += D * p;
        dd = rotr4(dd);
        ++s;
        if (ML7) {  // the next admissible cofactor may be divisible by 7: then take the one after
          c7 += 2 * D;
          c7 -= c7 >= 7 ? 7 : 0;
          if (c7 == 0) {
            const uint32_t D2 = dd & 15u;
            pos += D2 * p;
            dd = rotr4(dd);
            ++s;
            c7 = 2 * D2;
          }
          EG_CHECK(c7 >= 1 && c7 <= 6 && pos < (1u << 30) + WS, "ML c7=%u pos=%u p=%u", c7, pos, p);
        }
      }
    }
    if (rk_pend) st_rank(rk_addr, rk_val);
    k *= 32;
    const int more = __syncthreads_or(live);
    sc_flush(sm, a, k);
    if (!more) break;
  }
#endif
}

template <bool FAR7>
__device__ __forceinline__ void scatter_far(const ScatterArgs& a, uint32_t blk, uint32_t nblk, FarSmem& sm) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t t = tid; t < kScBins; t += blockDim.x) {
    sm.cnt[t] = 0;
    sm.fcnt[t] = 0;
  }
  __syncthreads();
  const uint32_t WS = a.WS, ring = a.ring, shift = a.log_s;
  const uint32_t lim = a.ntiles_w << a.log_s;
  const uint32_t nfar = min(*a.far_in_count, a.bcap);
  const uint32_t nw = nblk * kFarWarps;
  const uint32_t nu = (nfar + 31) / 32;
  const uint32_t left = (uint32_t)min(a.nwaves - a.wave, (uint64_t)0xffffffffu);  // waves from this one to the end
  const uint32_t wofs = warp * FarSmem::R + lane;
  const uint32_t reg_a = smem_addr(sm.reg + warp * FarSmem::R + lane), rank_a = smem_addr(sm.rank + warp * FarSmem::R + lane);
  const uint32_t ent_a = smem_addr(sm.freg + wofs), slot_a = smem_addr(sm.fslot + wofs),
                 frank_a = smem_addr(sm.frank + wofs);
  const uint32_t cnt_a = smem_addr(sm.cnt), sink_a = cnt_a + 4 * (kScBins + lane);
  const uint32_t fcnt_a = smem_addr(sm.fcnt), fsink_a = fcnt_a + 4 * (kScBins + lane);
  uint32_t u = blk * kFarWarps + warp;
  // the entries of the next kFarPf units are in flight (loads issued early)
  auto load = [&](uint32_t uu) -> uint64_t {
    const uint32_t j = uu * 32 + lane;
    return (uu < nu && j < nfar) ? a.far_in[j] : 0;
  };
  uint64_t pfe[kFarPf];  // entries of the next kFarPf units in flight
#pragma unroll
  for (int j = 0; j < kFarPf; ++j) pfe[j] = load(u + j * nw);
  uint32_t rk1 = 0, rk2 = 0;  // ranks of the last step, stored one step late
  for (;;) {
    uint32_t k = 0;  // staged steps (warp-uniform)
    for (; u < nu && k < (uint32_t)kFarSteps; ++k) {
      const uint32_t i = u * 32 + lane;
      const bool ok = i < nfar;
      const uint64_t e = pfe[0];
#pragma unroll
      for (int j = 0; j + 1 < kFarPf; ++j) pfe[j] = pfe[j + 1];
      pfe[kFarPf - 1] = load(u + kFarPf * nw);
      u += nw;
      uint32_t p, q, s, c7 = 0;
      if (FAR7) {
        p = 2 * ((uint32_t)e & 0x3fffffffu) + 1;
        q = (uint32_t)(e >> 30) & 0xfffffffu;
        s = (uint32_t)(e >> 58) & 7;
        c7 = (uint32_t)(e >> 61);
      } else {
        p = (uint32_t)e;
        q = (uint32_t)(e >> 32) & 0x1fffffffu;
        s = (uint32_t)(e >> 61);
      }
      const bool emit = ok && q < lim;
      const uint32_t r1 = stage_rec(emit ? cnt_a + ((q >> shift) << 2) : sink_a, reg_a + (k << 7), emit ? q : kNoRec);
      if (k) {  // ranks of the previous step
        st_rank(rank_a + ((k - 1) << 6), rk1);
        st_rank(frank_a + ((k - 1) << 6), rk2);
      }
      rk1 = r1;
      // next hit q + D*p lies d waves ahead (Lemma 2): fp32 estimate of d,
      // then the exact remainder in 32-bit wrap-around arithmetic
      uint32_t D = wheel_D(s), s1 = s + 1;
      if (FAR7) {  // the next admissible cofactor may be divisible by 7: then take the one after
        c7 += 2 * D;
        c7 -= c7 >= 7 ? 7 : 0;
        if (c7 == 0) {
          const uint32_t D2 = wheel_D(s1 & 7);
          D += D2;
          c7 = 2 * D2;
          ++s1;
        }
      }
      // (q + D*p < 2^29 + 5*2^32: the fp32 estimate is off by at most one wave)
      uint32_t d = __float2uint_rz(__fmaf_rn((float)D, (float)p, (float)q) * a.inv_ws_f);
      int32_t r = (int32_t)(q + D * p - d * WS);
      const bool lo = r < 0;
      r += lo ? (int32_t)WS : 0;
      d -= lo ? 1u : 0u;
      const bool hi = r >= (int32_t)WS;
      r -= hi ? (int32_t)WS : 0;
      d += hi ? 1u : 0u;
      EG_CHECK(!ok || (uint32_t)r < WS, "far next-hit remainder r=%d WS=%u p=%u q=%u", r, WS, p, q);
      EG_CHECK(!FAR7 || !ok || (c7 >= 1 && c7 <= 6), "far c7=%u p=%u", c7, p);
      const bool keep = ok && d < left;
      uint32_t slot = a.wslot + d;
      if (slot >= ring) slot -= ring;
      const uint64_t ne = FAR7 ? far7_pack(p, (uint32_t)r, s1, c7)
                               : (uint64_t)p | ((uint64_t)((uint32_t)r | ((s1 & 7) << 29)) << 32);
      rk2 = stage_far(keep ? fcnt_a + (slot << 2) : fsink_a, ent_a + (k << 8), slot_a + (k << 5), ne,
                      keep ? slot : kNoSlot);
    }
    if (k) {
      st_rank(rank_a + ((k - 1) << 6), rk1);
      st_rank(frank_a + ((k - 1) << 6), rk2);
    }
    const int more = __syncthreads_or(u < nu);
    sc_flush(sm, a, k * 32);
    if (!more) break;
  }
}

#ifndef EG_ML_MINB
#define EG_ML_MINB 0
#endif
template <bool ML7>
#if EG_ML_MINB
__global__ void __launch_bounds__(kMlWarps * 32, EG_ML_MINB) k_scatter_ml(const ScatterArgs a) {
#else
__global__ void __launch_bounds__(kMlWarps * 32) k_scatter_ml(const ScatterArgs a) {
#endif
  extern __shared__ uint4 smem_raw[];
  scatter_ml<ML7>(a, blockIdx.x, gridDim.x, *reinterpret_cast<MlSmem*>(smem_raw));
}
#ifndef EG_FAR_MINB
#define EG_FAR_MINB 6  // 40 registers: 6 CTAs per SM (the shared-memory limit); 48 measured 3% slower
#endif
template <bool FAR7>
__global__ void __launch_bounds__(kFarWarps * 32, EG_FAR_MINB) k_scatter_far(const ScatterArgs a) {
  extern __shared__ uint4 smem_raw[];
  scatter_far<FAR7>(a, blockIdx.x, gridDim.x, *reinterpret_cast<FarSmem*>(smem_raw));
}

// ---------------------------------------------------------------------------
// Wheel tables of the large primes (default path).  A large prime p marks only
// the multiples c*p whose cofactor c is coprime to the wheel modulus
// M = 30, 210, 2310 or 30030 (default): every other multiple is divisible by a
// prime <= 13 and set by the small-prime patterns anyway.  This is the
// reference's wheel (src/wheel.cpp:10-34: residues coprime to 30, deltas
// {3,2,1,2,1,2,3,1}) taken three primes further — 5760 residues of 30030,
// 28 % fewer records than mod 30.  A prime's state is its next hit and the
// index of that hit's cofactor in the residue list; delta[idx] (half the gap to
// the next coprime residue, <= 11) * p is the step to the next hit.  The
// deltas are packed 8 nibbles to a word (+ one wrap-around word); a walking
// lane keeps the next 8 deltas in a register, so a step costs the reference
// wheel's shift-and-mask (delta = dd & 15, dd >>= 4, ++idx), and a warp
// reloads its lanes' windows together every 8th step (warp-uniform, two
// shared-memory words and a funnel shift per lane).
constexpr uint32_t kWheelMaxRes = 5760;
constexpr uint32_t kWheelMaxBytes = kWheelMaxRes / 2 + 4;
struct Wheel {
  const uint32_t* delta8;  // [nres / 8 + 1] nibble i of word w = delta[(8w + i) mod nres]
  uint32_t nres;
};
__device__ __forceinline__ void stage_wheel(uint32_t* dst, const Wheel& w) {
  for (uint32_t i = threadIdx.x; i <= w.nres / 8; i += blockDim.x) dst[i] = w.delta8[i];
}
// the 8 deltas from index wi on (wi < nres + 8 is wrapped first)
__device__ __forceinline__ uint32_t wheel_window(uint32_t wd_a, uint32_t nres, uint32_t& wi) {
  wi -= wi >= nres ? nres : 0;
  EG_CHECK(wi < nres, "wheel index %u of %u", wi, nres);
  const uint32_t a = wd_a + ((wi >> 3) << 2);
  return __funnelshift_r(lds_u32(a), lds_u32(a + 4), (wi & 7) << 2);
}

// ML primes (S < p <= P_ml), wheel mode: the per-wave walk of k_scatter_ml with
// the state split in two arrays — the prime list itself (read only) and
// u64 states pos | idx << 32 — compacted emission, and the round's counting
// sort by tile (sc_flush).
struct MlWalkArgs {
  ScatterArgs sc;         // WS, ntiles_w, log_s, hits, hitcnt, hcap, overflow
  const uint32_t* primes; // the ML primes (ascending)
  uint64_t* st;           // per ML prime: pos | idx << 32
  uint32_t nml;
  Wheel wheel;
};

__global__ void __launch_bounds__(kMlWarps * 32) k_ml_walk(const MlWalkArgs a) {
  extern __shared__ uint4 smem_raw[];
  MlSmem& sm = *reinterpret_cast<MlSmem*>(smem_raw);
  uint32_t* const s_wd = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(smem_raw) + ((sizeof(MlSmem) + 15) & ~size_t{15}));
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t t = tid; t < kScBins; t += blockDim.x) sm.cnt[t] = 0;
  stage_wheel(s_wd, a.wheel);
  __syncthreads();
  const uint32_t WS = a.sc.WS, shift = a.sc.log_s, nres = a.wheel.nres;
  const uint32_t B = a.sc.ntiles_w << a.sc.log_s;  // walk bound (the end of the last tile in the last wave)
  const uint32_t nw = gridDim.x * kMlWarps;
  const uint32_t nu = (a.nml + 31) / 32;
  const uint32_t cnt_a = smem_addr(sm.cnt), wd_a = smem_addr(s_wd);
  const uint32_t regw_a = smem_addr(sm.reg + warp * MlSmem::R), rankw_a = smem_addr(sm.rank + warp * MlSmem::R);
  uint32_t ltm;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltm));
  const uint32_t gw0 = blockIdx.x * kMlWarps + warp;
  uint32_t urow = 0;
  auto unit_at = [&](uint32_t k) -> uint32_t { return k * nw + ((EG_BOUS && (k & 1)) ? nw - 1 - gw0 : gw0); };
  uint32_t u = gw0;
  uint32_t idx = u * 32 + lane;
  bool ok = u < nu && idx < a.nml;
  uint32_t p = ok ? a.primes[idx] : 0;
  uint64_t e = ok ? a.st[idx] : 0;
  uint32_t pos = ok ? (uint32_t)e : B, wi = (uint32_t)(e >> 32);
  uint32_t dd = wheel_window(wd_a, nres, wi);
  uint32_t since = 0;  // steps of this warp since its lanes loaded their delta windows
  // the next unit's primes and states are in flight
  uint32_t pn = 0;
  uint64_t en = 0;
  auto prefetch = [&](uint32_t uu) {
    const uint32_t j = uu * 32 + lane;
    if (uu < nu && j < a.nml) {
      pn = a.primes[j];
      en = a.st[j];
    }
  };
  prefetch(unit_at(1));
  bool live = u < nu;  // warp-uniform
  for (;;) {
    uint32_t kb = 0;  // staged records of this warp (warp-uniform)
    while (live && kb <= (uint32_t)MlSmem::R - 32) {
      const bool v = pos < B;
      const uint32_t m = __ballot_sync(kFull, v);
      if (!m) {
        if (ok) a.st[idx] = (uint64_t)(pos - WS) | ((uint64_t)(wi >= nres ? wi - nres : wi) << 32);
        ++urow;
        u = unit_at(urow);
        if (u >= nu) {
          live = false;
          break;
        }
        idx = u * 32 + lane;
        ok = idx < a.nml;
        p = pn;
        pos = ok ? (uint32_t)en : B;
        wi = (uint32_t)(en >> 32);
        dd = wheel_window(wd_a, nres, wi);
        since = 0;
        prefetch(unit_at(urow + 1));
        continue;
      }
      if (since == 8) {  // (warp-uniform) every lane has used at most 8 deltas of its window
        dd = wheel_window(wd_a, nres, wi);
        since = 0;
      }
      ++since;
      const uint32_t slot = kb + __popc(m & ltm);
      kb += __popc(m);
      if (v) {
        uint32_t r;
        asm volatile(
            "atom.shared.add.u32 %0, [%1], 1;\n\t"
            "st.shared.u32 [%2], %3;"
            : "=r"(r)
            : "r"(cnt_a + ((pos >> shift) << 2)), "r"(regw_a + (slot << 2)), "r"(pos)
            : "memory");
        pos += (dd & 15u) * p;
        dd >>= 4;
        ++wi;
        EG_CHECK(pos < 16u * WS, "ML walk pos=%u p=%u", pos, p);
        st_rank(rankw_a + (slot << 1), r);
      }
    }
    const int more = __syncthreads_or(live);
    sc_flush<kMlWarps, kMlSteps, false, true>(sm, a.sc, kb);
    if (!more) break;
  }
}

// ---------------------------------------------------------------------------
// Windowed far path (default for p > P_ml): the far primes' hits are routed in
// two counting-sort levels instead of moving an 8-byte entry from wave bucket
// to wave bucket at every hit (k_scatter_far).
//  k_far_walk  once per WINDOW of K waves: walks every far prime through the
//              window (state = next hit relative to the window start, wheel
//              class, cofactor mod 7; 8 B read + written per window, not per
//              hit) and emits one u32 record per hit — its offset inside its
//              wave — into the record bucket of that wave: the paper's bucket
//              of the segment of the next hit (large_kernel.hpp:61-213), with
//              the bucket filled for K waves ahead in one pass.  Staging,
//              shared-memory counting sort by wave and coalesced runs as in
//              the ML scatter; emission is compacted (ballot + popc).
//  k_wave_sort once per wave: partitions the wave's record bucket by tile into
//              the tiles' hit lists (dense: every lane holds a record).
struct FarWalkArgs {
  const uint32_t* primes;  // the far primes (ascending)
  uint64_t* st;            // per far prime: pos (40 bits) | idx << 40
  uint32_t nfar;
  uint64_t lim;   // valid bits of this window (walk bound)
  uint64_t span;  // K * WS: the state is re-based by this after the window
  uint32_t WS, log_s, magic;  // wave of tile t in the window = umulhi(t, magic)
  uint32_t nbins;             // waves of this window
  uint32_t* wbuf;             // [K][wcap] + trash
  uint32_t* wcnt;             // [K]
  uint32_t wcap, trash_at;    // trash_at = K * wcap
  int* overflow;
  Wheel wheel;
};

// test-only fault (ERATO_GPU_TEST_INJECT=2): a record outside its wave
__global__ void k_inject_wrec(uint32_t* wbuf, const uint32_t* wcnt) {
  if (*wcnt) wbuf[0] |= 0x80000000u;
}

constexpr uint64_t kFarPosMask = (1ull << 40) - 1;
__device__ __forceinline__ uint64_t farw_pack(uint64_t pos, uint32_t idx) {
  return (pos & kFarPosMask) | ((uint64_t)idx << 40);
}

#ifndef EG_WK_WARPS
#define EG_WK_WARPS 8
#endif
#ifndef EG_WK_STEPS
#define EG_WK_STEPS 12
#endif
constexpr int kWkWarps = EG_WK_WARPS, kWkSteps = EG_WK_STEPS;

struct WkSmem {
  static constexpr int R = kWkSteps * 32;  // staged records per warp
  uint32_t val[kWkWarps * R];
  uint32_t rb[kWkWarps * R];  // rank among the round's records of the same wave | wave << 16
  uint32_t srt[kWkWarps * R];
  uint8_t sbin[kWkWarps * R];
  uint32_t cnt[kScBins], off[kScBins], gofs[kScBins];
  uint32_t total;
  static_assert(kWkWarps * R < 65536, "ranks are 16-bit");
};

// Exclusive scan of cnt[0..nb) into off by warp 0 while the other warps
// reserve c slots per non-empty bin in gcnt[b].  The atomics' results stay in
// registers (rsv) until reserve_finish, after the placement, so their latency
// overlaps the scan and the placement; a thread holds at most two bins.
struct Resv {
  uint32_t c0, c1, r0, r1;  // counts and reserved starts of bins tid - 32 and tid - 32 + (NT - 32)
};
template <int NW>
__device__ __forceinline__ void scan_reserve(const uint32_t* cnt, uint32_t* off, uint32_t* total, uint32_t nb,
                                             uint32_t* gcnt, Resv& rsv) {
  static_assert(kScBins <= 2 * (NW * 32 - 32), "two reservations per thread");
  const uint32_t tid = threadIdx.x, b0 = tid - 32, b1 = b0 + (NW * 32 - 32);
  rsv.c0 = rsv.c1 = rsv.r0 = rsv.r1 = 0;
  if (tid < 32) {
    const uint32_t tot = warp_excl_scan(cnt, off, nb);
    if (tid == 0) *total = tot;
  } else {
    if (b0 < nb) {
      rsv.c0 = cnt[b0];
      if (rsv.c0) rsv.r0 = atomicAdd(&gcnt[b0], rsv.c0);
    }
    if (b1 < nb) {
      rsv.c1 = cnt[b1];
      if (rsv.c1) rsv.r1 = atomicAdd(&gcnt[b1], rsv.c1);
    }
  }
}
// gofs[b] = global index of sorted slot 0 of bin b
template <int NW>
__device__ __forceinline__ void reserve_finish(const Resv& rsv, const uint32_t* off, uint32_t* gofs, uint32_t cap,
                                               uint32_t trash_at, int* overflow) {
  const uint32_t b0 = threadIdx.x - 32, b1 = b0 + (NW * 32 - 32);
  if (rsv.c0) {
    const bool over = rsv.r0 + rsv.c0 > cap;
    if (over) atomicExch(overflow, 1);
    gofs[b0] = (over ? trash_at : b0 * cap + rsv.r0) - off[b0];
  }
  if (rsv.c1) {
    const bool over = rsv.r1 + rsv.c1 > cap;
    if (over) atomicExch(overflow, 1);
    gofs[b1] = (over ? trash_at : b1 * cap + rsv.r1) - off[b1];
  }
}

__global__ void __launch_bounds__(kWkWarps * 32) k_far_walk(const FarWalkArgs a) {
  extern __shared__ uint4 smem_raw[];
  WkSmem& sm = *reinterpret_cast<WkSmem*>(smem_raw);
  uint32_t* const s_wd = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(smem_raw) + ((sizeof(WkSmem) + 15) & ~size_t{15}));
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t NT = kWkWarps * 32;
  for (uint32_t t = tid; t < kScBins; t += NT) sm.cnt[t] = 0;
  stage_wheel(s_wd, a.wheel);
  __syncthreads();
  const uint32_t WS = a.WS, shift = a.log_s, magic = a.magic, nres = a.wheel.nres, wd_a = smem_addr(s_wd);
  const uint64_t lim = a.lim, span = a.span;
  const uint32_t nw = gridDim.x * kWkWarps;
  const uint32_t nu = (a.nfar + 31) / 32;
  uint32_t ltm;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltm));
  const uint32_t val_a = smem_addr(sm.val + warp * WkSmem::R), rb_a = smem_addr(sm.rb + warp * WkSmem::R),
                 cnt_a = smem_addr(sm.cnt);
  const uint32_t gw0 = blockIdx.x * kWkWarps + warp;
  uint32_t urow = 0;
  auto unit_at = [&](uint32_t k) -> uint32_t { return k * nw + ((EG_BOUS && (k & 1)) ? nw - 1 - gw0 : gw0); };
  uint32_t u = gw0;
  uint32_t idx = u * 32 + lane;
  bool ok = u < nu && idx < a.nfar;
  uint32_t p = ok ? a.primes[idx] : 0;
  uint64_t e = ok ? a.st[idx] : 0;
  uint64_t pos;
  uint32_t wi, dd, since = 0;  // since: steps of this warp since its lanes loaded their delta windows
  auto decode = [&]() {
    pos = ok ? (e & kFarPosMask) : lim;
    wi = (uint32_t)(e >> 40);
    dd = wheel_window(wd_a, nres, wi);
    since = 0;
  };
  decode();
  // the next unit's prime and state are in flight
  uint32_t pn = 0;
  uint64_t en = 0;
  auto prefetch = [&](uint32_t uu) {
    const uint32_t j = uu * 32 + lane;
    if (uu < nu && j < a.nfar) {
      pn = a.primes[j];
      en = a.st[j];
    }
  };
  prefetch(unit_at(1));
  bool live = u < nu;  // warp-uniform
  for (;;) {
    uint32_t kb = 0;  // staged records of this warp (warp-uniform)
    while (live && kb <= (uint32_t)WkSmem::R - 32) {
      const bool v = pos < lim;
      const uint32_t m = __ballot_sync(kFull, v);
      if (!m) {
        if (ok) a.st[idx] = farw_pack(pos - span, wi >= nres ? wi - nres : wi);
        ++urow;
        u = unit_at(urow);
        if (u >= nu) {
          live = false;
          break;
        }
        idx = u * 32 + lane;
        ok = idx < a.nfar;
        p = pn;
        e = en;
        decode();
        prefetch(unit_at(urow + 1));
        continue;
      }
      if (since == 8) {  // (warp-uniform) every lane has used at most 8 deltas of its window
        dd = wheel_window(wd_a, nres, wi);
        since = 0;
      }
      ++since;
      const uint32_t slot = kb + __popc(m & ltm);
      kb += __popc(m);
      if (v) {
        const uint32_t tile = (uint32_t)(pos >> shift);
        const uint32_t wv = __umulhi(tile, magic);
        const uint32_t off = (uint32_t)pos - wv * WS;
        EG_CHECK(wv < a.nbins && off < WS, "far walk wave=%u nbins=%u off=%u", wv, a.nbins, off);
        uint32_t r;
        asm volatile(
            "atom.shared.add.u32 %0, [%1], 1;\n\t"
            "st.shared.u32 [%2], %3;"
            : "=r"(r)
            : "r"(cnt_a + (wv << 2)), "r"(val_a + (slot << 2)), "r"(off)
            : "memory");
        pos += (uint64_t)(dd & 15u) * p;
        dd >>= 4;
        ++wi;
        sts_u32(rb_a + (slot << 2), r | (wv << 16));
      }
    }
    const int more = __syncthreads_or(live);
    // ---- round: sort this round's records by wave, coalesced runs out ----
    Resv rsv;
    scan_reserve<kWkWarps>(sm.cnt, sm.off, &sm.total, a.nbins, a.wcnt, rsv);
    __syncthreads();
    {
      const uint32_t off_a = smem_addr(sm.off), srt_a = smem_addr(sm.srt), sbin_a = smem_addr(sm.sbin);
#pragma unroll 2
      for (uint32_t i = lane; i < kb; i += 32) {
        const uint32_t rb = lds_u32(rb_a + 4 * i), b = rb >> 16;
        const uint32_t k = lds_u32(off_a + 4 * b) + (rb & 0xffffu);
        sts_u32(srt_a + 4 * k, lds_u32(val_a + 4 * i));
        asm volatile("st.shared.u8 [%0], %1;" : : "r"(sbin_a + k), "r"(b) : "memory");
      }
    }
    reserve_finish<kWkWarps>(rsv, sm.off, sm.gofs, a.wcap, a.trash_at, a.overflow);
    for (uint32_t b = tid; b < a.nbins; b += NT) sm.cnt[b] = 0;
    __syncthreads();
    const uint32_t total = sm.total;
    for (uint32_t i = tid; i < total; i += NT) a.wbuf[sm.gofs[sm.sbin[i]] + i] = sm.srt[i];
    // off/gofs/srt are rewritten only after the next round's first barrier
    if (!more) break;
  }
}

// Partition of one wave's far records by tile into the tiles' hit lists.
constexpr int kWsSegs = 9;  // record segments one launch sorts: the far bucket of the wave + the ML sub-buckets
struct WaveSortArgs {
  const uint32_t* in[kWsSegs];        // record segments (offsets inside the wave), blockIdx.y picks one
  const uint32_t* in_count[kWsSegs];
  uint32_t cap[kWsSegs];
  uint32_t nb, log_s;        // tiles of this wave
  uint32_t* hits;            // [nb][hcap] + trash
  uint32_t* hitcnt;          // [nb]
  uint32_t hcap;
  int* overflow;
};
#ifndef EG_WS_THREADS
#define EG_WS_THREADS 512
#endif
#ifndef EG_WS_PER
#define EG_WS_PER 8
#endif
constexpr int kWsThreads = EG_WS_THREADS, kWsPer = EG_WS_PER, kWsChunk = kWsThreads * kWsPer;
struct WsSmem {
  uint32_t srt[kWsChunk];
  uint32_t cnt[kScBins], off[kScBins], gofs[kScBins];
  uint32_t total;
};

// One chunk of kWsChunk records per CTA (the grid covers the bucket's
// capacity; CTAs past the count exit).  The kernel is latency-bound, so the
// scan runs on all warps (32 bins each, a warp sums the lower groups itself).
__global__ void __launch_bounds__(kWsThreads) k_wave_sort(const WaveSortArgs a) {
  __shared__ WsSmem sm;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = min(*a.in_count[blockIdx.y], a.cap[blockIdx.y]);
  const uint32_t c0 = blockIdx.x * kWsChunk;
  if (c0 >= n) return;
  const uint32_t* const in = a.in[blockIdx.y];
  const uint32_t nb = a.nb, shift = a.log_s, smask = (1u << shift) - 1;
  const uint32_t cnt_a = smem_addr(sm.cnt), off_a = smem_addr(sm.off), srt_a = smem_addr(sm.srt),
                 gofs_a = smem_addr(sm.gofs);
  constexpr int K4 = kWsPer / 4;
  uint32_t key[kWsPer], rk[kWsPer];
#pragma unroll
  for (int k = 0; k < K4; ++k) {
    const uint32_t i = c0 + 4 * (tid + k * kWsThreads);
    uint4 v = make_uint4(kNoRec, kNoRec, kNoRec, kNoRec);
    if (i + 3 < n) {
      v = __ldcs(reinterpret_cast<const uint4*>(in + i));
    } else {
      if (i < n) v.x = in[i];
      if (i + 1 < n) v.y = in[i + 1];
      if (i + 2 < n) v.z = in[i + 2];
    }
    key[4 * k] = v.x;
    key[4 * k + 1] = v.y;
    key[4 * k + 2] = v.z;
    key[4 * k + 3] = v.w;
  }
  for (uint32_t t = tid; t < kScBins; t += kWsThreads) sm.cnt[t] = 0;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kWsPer; ++k) {
    const uint32_t t = key[k] >> shift;
    rk[k] = 0;
    if (t < nb) {  // (sentinels and corrupted records are dropped)
      asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(rk[k]) : "r"(cnt_a + (t << 2)) : "memory");
    }
  }
  __syncthreads();
  // scan of the tile counts: warp w takes bins 32w.. (nb <= 256 = 8 groups of
  // the 16 warps) and sums the lower groups itself; the bin's thread reserves
  // the run in the tile's hit list — the atomic's result is first needed
  // after the placement, so its latency overlaps it
  const uint32_t b = tid;  // bin of this thread (warps 0..7)
  uint32_t c = 0, r = 0, ofs = 0;
  if (warp * 32 < nb) {
    c = b < nb ? sm.cnt[b] : 0;
    uint32_t low = 0;
    for (uint32_t j = 0; j < warp; ++j) low += sm.cnt[j * 32 + lane];
    if (c) r = atomicAdd(&a.hitcnt[b], c);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) low += __shfl_xor_sync(kFull, low, o);
    ofs = low + x - c;
    if (b < nb) {
      sm.off[b] = ofs;
      if (b == nb - 1) sm.total = ofs + c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kWsPer; ++k) {
    const uint32_t t = key[k] >> shift;
    if (t < nb) sts_u32(srt_a + 4 * (lds_u32(off_a + 4 * t) + rk[k]), key[k]);
  }
  if (c) {
    const bool over = r + c > a.hcap;
    if (over) atomicExch(a.overflow, 1);
    sm.gofs[b] = (over ? nb * a.hcap : b * a.hcap + r) - ofs;  // global index of sorted slot 0 of the tile
  }
  __syncthreads();
  const uint32_t total = sm.total;
  for (uint32_t i = tid; i < total; i += kWsThreads) {
    const uint32_t k = lds_u32(srt_a + 4 * i);
    a.hits[lds_u32(gofs_a + 4 * (k >> shift)) + i] = k & smask;
  }
}

static_assert(kWkWarps * WkSmem::R <= (int)kScTrash && kWsChunk <= (int)kScTrash, "trash area too small");
static_assert(kWsThreads >= kScBins, "one thread per bin in k_wave_sort");

// invariant check of a wave's far records (ERATO_GPU_CHECK_INVARIANTS): each
// lies inside the wave's tiles
__global__ void __launch_bounds__(256) k_check_wrecs(const uint32_t* __restrict__ in, const uint32_t* __restrict__ in_count,
                                                     uint32_t wcap, uint32_t lim, int* bad,
                                                     unsigned long long* nrec) {
  const uint32_t n = min(*in_count, wcap);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(nrec, (unsigned long long)n);
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    if (in[j] >= lim) atomicExch(bad, 1);
}

// ---------------------------------------------------------------------------
// Base primes: odd primes < 2^16 in one CTA (sieve in smem + block compaction).
__global__ void __launch_bounds__(1024) k_small_primes(uint32_t* __restrict__ out, uint32_t* __restrict__ count) {
  __shared__ uint32_t bits[1024];  // 32768 odd numbers 1..65535
  __shared__ uint32_t s_scan[1024];
  const uint32_t tid = threadIdx.x;
  bits[tid] = tid == 0 ? 1u : 0u;  // number 1 is not prime
  __syncthreads();
  for (uint32_t i = 3; i * i < 65536; i += 2) {
    if (!((bits[i >> 6] >> ((i >> 1) & 31)) & 1)) {
      for (uint32_t j = i * i + 2 * i * tid; j < 65536; j += 2 * i * blockDim.x)
        atomicOr(&bits[j >> 6], 1u << ((j >> 1) & 31));
    }
    __syncthreads();
  }
  const uint32_t free_bits = ~bits[tid];
  const uint32_t c = __popc(free_bits);
  s_scan[tid] = c;
  __syncthreads();
  for (uint32_t o = 1; o < 1024; o <<= 1) {
    const uint32_t v = tid >= o ? s_scan[tid - o] : 0;
    __syncthreads();
    s_scan[tid] += v;
    __syncthreads();
  }
  uint32_t pos = s_scan[tid] - c;
  uint32_t fb = free_bits;
  while (fb) {
    const uint32_t b = __ffs(fb) - 1;
    fb &= fb - 1;
    out[pos++] = 2 * (tid * 32 + b) + 1;
  }
  if (tid == 1023) *count = s_scan[1023];
}


// ---- compaction of a bit table to the sorted list of its zero bits ---------
// Block = 1024 words (32768 bits).  Zero bit j (lo <= j < nbits) -> value
// base + 2*j (u64) or 2*j+1 (u32 base primes).
constexpr int kCompactWords = 1024;

__global__ void __launch_bounds__(1024) k_count_zeros_blocks(const uint32_t* __restrict__ bits, uint64_t nbits,
                                                            uint64_t lo, uint32_t* __restrict__ bcnt) {
  __shared__ uint32_t s_red[32];
  const uint64_t w = (uint64_t)blockIdx.x * kCompactWords + threadIdx.x;
  uint32_t c = 0;
  if (w * 32 < nbits) {
    uint32_t v = ~bits[w];
    const uint64_t b0 = w * 32;
    if (nbits - b0 < 32) v &= (1u << (nbits - b0)) - 1;
    if (b0 < lo) v &= lo - b0 >= 32 ? 0u : ~((1u << (lo - b0)) - 1);
    c = __popc(v);
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t t = s_red[threadIdx.x];
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
    if (threadIdx.x == 0) bcnt[blockIdx.x] = t;
  }
}

// exclusive scan of n u32 counts into u64 offsets (single CTA); total -> *total
__global__ void __launch_bounds__(1024) k_scan_counts(const uint32_t* __restrict__ c, uint32_t n,
                                                     uint64_t* __restrict__ off, uint64_t* __restrict__ total) {
  __shared__ uint64_t s[1024];
  const uint32_t tid = threadIdx.x;
  const uint32_t per = (n + 1023) / 1024;
  const uint32_t b = tid * per, e = min(n, b + per);
  uint64_t sum = 0;
  for (uint32_t i = b; i < e; ++i) sum += c[i];
  s[tid] = sum;
  __syncthreads();
  for (uint32_t o = 1; o < 1024; o <<= 1) {
    const uint64_t v = tid >= o ? s[tid - o] : 0;
    __syncthreads();
    s[tid] += v;
    __syncthreads();
  }
  uint64_t run = s[tid] - sum;
  for (uint32_t i = b; i < e; ++i) {
    off[i] = run;
    run += c[i];
  }
  if (tid == 1023) *total = s[1023];
}

template <typename T>
__global__ void __launch_bounds__(1024) k_write_zeros(const uint32_t* __restrict__ bits, uint64_t nbits, uint64_t lo,
                                                     const uint64_t* __restrict__ boff, uint64_t base,
                                                     T* __restrict__ out, uint64_t cap) {
  __shared__ uint32_t s_scan[1024];
  const uint32_t tid = threadIdx.x;
  const uint64_t w = (uint64_t)blockIdx.x * kCompactWords + tid;
  uint32_t v = 0;
  if (w * 32 < nbits) {
    v = ~bits[w];
    const uint64_t b0 = w * 32;
    if (nbits - b0 < 32) v &= (1u << (nbits - b0)) - 1;
    if (b0 < lo) v &= lo - b0 >= 32 ? 0u : ~((1u << (lo - b0)) - 1);
  }
  const uint32_t c = __popc(v);
  s_scan[tid] = c;
  __syncthreads();
  for (uint32_t o = 1; o < 1024; o <<= 1) {
    const uint32_t x = tid >= o ? s_scan[tid - o] : 0;
    __syncthreads();
    s_scan[tid] += x;
    __syncthreads();
  }
  uint64_t pos = boff[blockIdx.x] + s_scan[tid] - c;
  while (v) {
    const uint32_t b = __ffs(v) - 1;
    v &= v - 1;
    if (pos < cap) out[pos] = (T)(base + 2 * (w * 32 + b));
    ++pos;
  }
}

// number of entries of a sorted array <= x, for several thresholds;
// out[nthr] = the largest entry (0 if none)
__global__ void k_bounds(const uint32_t* __restrict__ p, const uint64_t* __restrict__ n_ptr,
                         const uint64_t* __restrict__ thr, int nthr, uint64_t* __restrict__ out) {
  const int i = threadIdx.x;
  const uint64_t n = *n_ptr;
  if (i == nthr) out[i] = n ? p[n - 1] : 0;
  if (i >= nthr) return;
  const uint64_t x = thr[i];
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((uint64_t)p[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  out[i] = lo;
}

// ---- large-prime setup: first hits -> ML state, initial far buckets ------
struct SetupArgs {
  const uint32_t* primes;
  uint64_t i0, i_ml_end, i_end;  // ML = [i0, i_ml_end), far = [i_ml_end, i_end)
  uint64_t x0;                   // 2*g0 + 1
  uint2* ml;
  uint64_t* far_buckets;
  uint32_t* far_bcount;
  uint32_t ring, bcap;
  uint64_t nwaves;
  uint32_t WS;
  double inv_ws;
  int* overflow;
  int inject;  // test-only fault injection on the first far prime: 1 drop its entry, 2 corrupt its q
  int far7;    // far entries in the mod-210 format (far7_pack)
  int ml7;     // ML states in the mod-210 format (ml7_pack)
  // wheel mode (default path): ML states pos | idx << 32, far states farw_pack(pos, idx); idx = rank of the
  // first hit's cofactor among the residues coprime to wM
  uint64_t* fst;
  uint64_t* mlst;
  const uint32_t* wnext;  // [wM], for c mod wM coprime to 30: index of the first wheel residue >= c | half the gap to it << 16
  uint32_t wM, wR32, wmask;  // wR32 = 2^32 mod wM; wmask: bit 0/1/2 = the wheel also excludes cofactors divisible by 7/11/13
};

constexpr int kSetupThreads = 1024;

__global__ void __launch_bounds__(kSetupThreads) k_setup_large(const SetupArgs a) {
  __shared__ uint32_t s_cnt[kScBins], s_base[kScBins];
  if (!a.wnext) {  // (legacy bucket appends only; uniform over the grid)
    for (uint32_t b = threadIdx.x; b < kScBins; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
  }
  const uint64_t i = a.i0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool app = false;
  uint32_t slotb = 0;
  uint64_t ne = 0;
  if (i < a.i_end) {
    const uint32_t p = a.primes[i];
    uint32_t s;
    // cofactor >= 2 (-> >= 7 after the wheel): never marks p itself and
    // keeps the first hit within 3.5p of the interval start in overlap runs
    uint64_t cof = 0;
    uint64_t pos = first_hit(p, a.x0, 2, s, &cof);
    if (a.wnext) {
      // from the first cofactor coprime to 30 to the first one on the whole wheel: one table entry per
      // cofactor residue (its index on the wheel, and how far ahead it is); the cofactor mod the wheel
      // modulus without a 64-bit division: 2^32 = wR32 (mod wM)
      const uint32_t cm = (((uint32_t)(cof >> 32) % a.wM) * a.wR32 + (uint32_t)cof % a.wM) % a.wM;
      const uint32_t nx = a.wnext[cm];
      EG_CHECK(nx != 0xffffffffu, "cofactor not coprime to 30 p=%u", p);
      pos += (uint64_t)(nx >> 16) * p;
      const uint32_t wi = nx & 0xffffu;
      if (i < a.i_ml_end) {
        EG_CHECK(pos < (1ull << 32), "first ML hit beyond 32 bits p=%u", p);
        a.mlst[i - a.i0] = pos | ((uint64_t)wi << 32);
      } else {
        if (a.inject == 1 && i == a.i_ml_end) pos = kFarPosMask;  // test-only: the prime never hits
        a.fst[i - a.i_ml_end] = farw_pack(pos, wi);
      }
    } else if (i < a.i_ml_end) {
      if (a.ml7) {  // skip a first hit whose cofactor 7 divides (the next one cannot)
        uint32_t c7 = (uint32_t)(cof % 7);
        if (c7 == 0) {
          const uint32_t D = wheel_D(s);
          pos += (uint64_t)D * p;
          c7 = 2 * D;
          s = (s + 1) & 7;
        }
        a.ml[i - a.i0] = ml7_pack(p, (uint32_t)pos, s, c7);
      } else {
        a.ml[i - a.i0] = make_uint2(p | (s << 29), (uint32_t)pos);
      }
    } else {
      uint32_t c7 = 0;
      if (a.far7) {  // cofactor mod 7 of the first hit; skip it if 7 divides it (the next one cannot)
        c7 = (uint32_t)(cof % 7);
        if (c7 == 0) {
          const uint32_t D = wheel_D(s);
          pos += (uint64_t)D * p;
          c7 = 2 * D;
          s = (s + 1) & 7;
        }
      }
      // d = pos / WS: fp64 estimate (pos < 2^40, off by at most one), exact fix
      uint64_t d = __double2ull_rz(__dmul_rz(__ull2double_rz(pos), a.inv_ws));
      if (d * a.WS > pos) --d;
      if ((d + 1) * a.WS <= pos) ++d;
      if (d < a.nwaves) {
        app = true;
        slotb = (uint32_t)d % a.ring;
        const uint32_t q = (uint32_t)(pos - d * a.WS);
        ne = a.far7 ? far7_pack(p, q, s, c7) : (uint64_t)p | ((uint64_t)(q | (s << 29)) << 32);
        if (a.inject && i == a.i_ml_end) {
          if (a.inject == 1) app = false;
          else ne |= a.far7 ? (uint64_t)0xfffffffu << 30 : (uint64_t)0x1fffffffu << 32;  // q beyond the wave
        }
      }
    }
  }
  if (a.wnext) return;  // (wheel mode: no bucket appends; uniform over the grid)
  // CTA-level aggregation of the bucket appends: the first hits of all far
  // primes fall into the first few waves, so per-warp atomics on those few
  // counters would serialise
  uint32_t rank = 0;
  if (app) rank = atomicAdd(&s_cnt[slotb], 1u);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < a.ring; b += blockDim.x) {
    const uint32_t c = s_cnt[b];
    if (c) s_base[b] = atomicAdd(&a.far_bcount[b], c);
  }
  __syncthreads();
  if (app) {
    const uint32_t pos = s_base[slotb] + rank;
    if (pos < a.bcap) a.far_buckets[(uint64_t)slotb * a.bcap + pos] = ne;
    else atomicExch(a.overflow, 1);
  }
}

// ---- invariant checks (ERATO_GPU_CHECK_INVARIANTS), separate launches so
// the wave kernels are untouched.  Per wave, between the scatter and the
// tiles: sum the hit records the tiles are about to consume, and check that
// every far entry of the wave's bucket hits inside the wave.
__global__ void __launch_bounds__(256) k_check_wave(const uint32_t* __restrict__ hitcnt, uint32_t ntiles_w,
                                                    uint32_t hcap, const uint64_t* __restrict__ far_in,
                                                    const uint32_t* __restrict__ far_in_count, uint32_t bcap,
                                                    uint32_t WS, unsigned long long* rec_count, int* bad, int far7) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ntiles_w) atomicAdd(rec_count, (unsigned long long)min(hitcnt[i], hcap));
  if (far_in) {
    const uint32_t nfar = min(*far_in_count, bcap);
    for (uint32_t j = i; j < nfar; j += gridDim.x * blockDim.x)
      if (far_q(far_in[j], far7 != 0) >= WS) atomicExch(bad, 1);
  }
}

// ---- invariant check: admissible multiples of the large primes in the tiles
// (ERATO_GPU_CHECK_INVARIANTS).  For prime p the hit records are the
// multiples c*p, c coprime to 30 and c >= 2, of odd numbers in [x_lo, x_hi]
// (the run's tiles; the first hit uses cofactor >= 2, k_setup_large).
__device__ __forceinline__ uint64_t coprime30_upto(uint64_t n) {  // #{1 <= c <= n : gcd(c, 30) = 1}
  constexpr uint8_t cnt[30] = {0, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 4, 4, 4, 4, 5, 5, 6, 6, 6, 6, 7, 7, 7, 7, 7, 7, 8};
  return 8 * (n / 30) + cnt[n % 30];
}
__device__ __forceinline__ uint64_t coprime210_upto(uint64_t n) {  // #{1 <= c <= n : gcd(c, 210) = 1}
  return coprime30_upto(n) - coprime30_upto(n / 7);  // c coprime to 30 and divisible by 7: c = 7c', c' coprime to 30
}
// #{1 <= c <= n : gcd(c, 30) = 1 and none of the primes selected by mask (bit 0/1/2 = 7/11/13) divides c}
__device__ __forceinline__ uint64_t coprime_wheel_upto(uint64_t n, uint32_t mask) {
  const uint32_t q[3] = {7, 11, 13};
  uint64_t tot = 0;
  for (uint32_t sub = 0; sub < 8; ++sub) {  // inclusion-exclusion over the subsets of the selected primes
    if (sub & ~mask) continue;
    uint64_t d = 1;
    for (int k = 0; k < 3; ++k)
      if (sub >> k & 1) d *= q[k];
    const uint64_t t = coprime30_upto(n / d);
    tot = (__popc(sub) & 1) ? tot - t : tot + t;
  }
  return tot;
}
__device__ __forceinline__ uint64_t div_floor(uint64_t x, uint32_t p) {
  // fp64 estimate (off by at most one), exact fix on the remainder in
  // wrap-around u64 arithmetic (q*p may pass 2^64 when x is near it)
  uint64_t q = __double2ull_rz(__dmul_rz(__ull2double_rz(x), __drcp_rn((double)p)));
  int64_t r = (int64_t)(x - q * p);
  if (r < 0) --q;
  else if (r >= (int64_t)p) ++q;
  return q;
}
__global__ void __launch_bounds__(256) k_expected_records(const uint32_t* __restrict__ primes, uint64_t i0,
                                                          uint64_t i1, uint64_t x_lo, uint64_t x_hi,
                                                          unsigned long long* __restrict__ out, uint64_t i7_lo,
                                                          uint64_t i7_hi, uint32_t wmask) {
  const uint64_t i = i0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long cnt = 0;
  if (i < i1) {
    const uint32_t p = primes[i];
    uint64_t c_lo = div_floor(x_lo - 1, p) + 1;  // ceil(x_lo / p)
    if (c_lo < 2) c_lo = 2;
    const uint64_t c_hi = div_floor(x_hi, p);
    if (c_hi >= c_lo)
      cnt = i >= i7_lo && i < i7_hi ? coprime_wheel_upto(c_hi, wmask) - coprime_wheel_upto(c_lo - 1, wmask)
                                    : coprime30_upto(c_hi) - coprime30_upto(c_lo - 1);
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, cnt);
}

}  // namespace eg
