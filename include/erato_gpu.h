/* erato_gpu.h — C ABI of the B200-native segmented odd-only sieve.
 *
 * Drop-in for the reference sieve path `run_sieve` of erato
 * (/root/reference/proj/include/erato/driver.hpp:91, src/driver.cpp:83-120).
 * The reference exposes a C++ API, not an FFI; each entry point below names
 * the reference interface it replaces.  INTEGRATION.md shows the binding a
 * maintainer would add on the reference side.
 *
 * Conventions
 *  - Plain C types only; no torch, no CUDA types in the signatures.
 *  - Return value: 0 on success, else 1 + the ordinal of erato::errc
 *    (/root/reference/proj/include/erato/params.hpp:18-29), so the same
 *    codes/names (L_OUT_OF_RANGE, F_ZERO_OR_OVERLAP, ...) come back.
 *    Parameter errors are codes 1..5 (CLI exit 1), runtime errors 6..
 *    (CLI exit 2), as in /root/reference/proj/tools/erato.cpp:21-33.
 *  - Table layout (driver.hpp:6-8): bit j of the table is bit (j mod 8) of
 *    byte floor(j/8); 1 = 2(f*2^l+j)+1 is composite, 0 = prime.
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    point fails with ERATO_GPU_E_NO_DEVICE.
 */
#ifndef ERATO_GPU_H
#define ERATO_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errc ordinals + 1 (params.hpp:18-29) */
enum {
  ERATO_GPU_OK = 0,
  ERATO_GPU_L_OUT_OF_RANGE = 1,
  ERATO_GPU_F_ZERO_OR_OVERLAP = 2,
  ERATO_GPU_N_OUT_OF_RANGE = 3,
  ERATO_GPU_OVERFLOW = 4,
  ERATO_GPU_INDEX_OUT_OF_RANGE = 5,
  ERATO_GPU_NOT_ADMISSIBLE = 6,
  ERATO_GPU_ALLOC_LIMIT = 7,
  ERATO_GPU_LIMIT_TOO_LARGE = 8,
  ERATO_GPU_RANGE_TOO_LARGE = 9,
  ERATO_GPU_IO_ERROR = 10,
  /* GPU-side runtime errors (no reference counterpart; CLI exit 2) */
  ERATO_GPU_E_CUDA = 64,
  ERATO_GPU_E_NO_DEVICE = 65,
  ERATO_GPU_E_INVALID_ARG = 66,
  ERATO_GPU_E_INVARIANT = 67, /* ERATO_GPU_CHECK_INVARIANTS found a large-prime bookkeeping error */
};

/* flags */
#define ERATO_GPU_TEST_MODE 0x1u     /* l >= 4 instead of 10 (params.hpp:58-60) */
#define ERATO_GPU_ALLOW_OVERLAP 0x2u /* accept u^2 <= v incl. f = 0 (SURVEY §8c convention:
                                        multiples from max(u, p^2); 1 and primes stay 0) */
#define ERATO_GPU_CHECK_INVARIANTS 0x200u /* device checks of the large-prime path (the analog of
                                             validate_circle_invariants, src/kernels.cpp:103-179,
                                             and acceptance.cpp:122-161 "each multiple exactly
                                             once"): every far entry read from a wave's bucket hits
                                             inside that wave, and the hit records consumed by the
                                             tiles equal the admissible multiples of the large
                                             primes in the tiles (counted per prime in closed
                                             form); a violation fails with ERATO_GPU_E_INVARIANT */
#define ERATO_GPU_PHASE_TIMING 0x100u /* CUDA events around every launch: fills small_s (tile
                                         kernel) and large_s (bucket scatter) in the stats */

/* RunStats (driver.hpp:24-32).  Times are seconds of device time (CUDA
 * events); small_s covers masks+medium (tile kernel), large_s the bucket
 * scatter, output_s the D2H / file part of the call. */
typedef struct {
  uint64_t prime_count; /* zero bits over the run */
  uint64_t segments;    /* n */
  double init_s;
  double small_s;
  double large_s;
  double output_s;
  double total_s;
  uint64_t base_primes; /* odd primes <= isqrt(v) */
  uint64_t tiles;       /* GPU tiles (2^log_tile bits each) */
  uint32_t log_tile;
  uint32_t waves;
  uint32_t kernel_launches;
  uint32_t retries; /* capacity re-runs after a bucket overflow */
  double gen_s;     /* with ERATO_GPU_PHASE_TIMING: ML walk per wave (k_ml_walk; k_scatter_ml / k_gen on the legacy paths) */
  double bin_s;     /* with ERATO_GPU_PHASE_TIMING: far primes (k_far_walk per window + k_wave_sort per wave;
                       k_scatter_far / k_bin on the legacy paths) */
  uint64_t large_records; /* with ERATO_GPU_CHECK_INVARIANTS: hit records consumed by the tiles */
  double masks_s; /* with ERATO_GPU_PHASE_TIMING: the small-prime pattern phase of the tile kernel
                     (apply_small_masks, driver.cpp:97-99), %globaltimer in CTA 0 of each launch */
  uint64_t medium_primes; /* base primes sieved inside the tiles (61 < p <= tile) */
  uint64_t ml_primes;     /* large primes walked every wave (tile < p <= wave span) */
  uint64_t far_primes;    /* large primes walked once per window of waves (p > wave span / far_div) */
  uint32_t skip7;         /* bit 0: far primes, bit 1: ML primes skip cofactors divisible by 7 */
  uint32_t wheel;         /* wheel modulus of the large primes (30, 210, 2310, 30030); 0 on the legacy paths */
  uint64_t far_records;   /* with ERATO_GPU_CHECK_INVARIANTS: hit records of the far primes (of large_records) */
  double walk_s;          /* with ERATO_GPU_PHASE_TIMING: the k_far_walk part of bin_s */
  uint32_t far_windows;   /* k_far_walk launches (windows of waves) of the run */
  uint32_t reserved1;
} erato_gpu_stats;

/* Count written to a caller's dev_count when a bucket / hit-list capacity
 * overflowed (only possible with sync = 0; sync = 1 re-runs with doubled
 * capacities until the run is exact). */
#define ERATO_GPU_COUNT_OVERFLOW UINT64_MAX

/* ---- host-side parameter logic (no device needed) ---------------------- */

/* validate_params (src/params.cpp:23-44); u/v may be NULL. */
int erato_gpu_validate(unsigned l, uint64_t f, uint64_t n, unsigned flags, uint64_t* u,
                       uint64_t* v);
/* params_from_midpoint (src/params.cpp:64-77), decimal 10^e. */
int erato_gpu_f_from_midpoint(unsigned e, unsigned l, uint64_t n, unsigned flags, uint64_t* f);
/* isqrt (src/params.cpp:79-85). */
uint64_t erato_gpu_isqrt(uint64_t x);
/* first_offset, Lemma 1 (src/wheel.cpp:43-47). */
uint32_t erato_gpu_first_offset(uint32_t p, unsigned l, uint64_t f);
/* Host twin of the device start-offset logic (sieve_kernels.cuh first_hit):
 * index offset (c*p - x)/2 of the first multiple c*p >= x (x odd) whose
 * cofactor c >= cmin is coprime to 30, and c's wheel class (0..7 for
 * c mod 30 = 1,7,11,13,17,19,23,29).  With x = u this is Lemma 1 +
 * wheel_align (src/wheel.cpp:43-69) in one step. */
int erato_gpu_first_hit(uint32_t p, uint64_t x, uint64_t cmin, uint64_t* offset, unsigned* wheel_class);
/* The large primes' wheel (the reference's mod-30 wheel, src/wheel.cpp:10-34,
 * taken to modulus M = 30, 210, 2310 or 30030): writes delta[i] = half the gap
 * from the i-th odd residue coprime to M to the next one (wrapping) for
 * i < min(count, cap) and returns the residue count (8, 48, 480, 5760), 0 for
 * another M.  A large prime p marks c*p only for cofactors c on this wheel;
 * the index offset from one hit to the next is delta[i] * p. */
size_t erato_gpu_wheel_deltas(uint32_t M, uint8_t* delta, size_t cap);
/* table_filename (src/driver.cpp:17-20); returns bytes needed incl. NUL. */
size_t erato_gpu_table_filename(unsigned l, uint64_t f, uint64_t n, char* out, size_t cap);
/* errc_name (src/params.cpp:7-21) for codes 1..10, plus the GPU codes. */
const char* erato_gpu_errc_name(int code);
/* Message of the last failure on this thread. */
const char* erato_gpu_last_error(void);

/* ---- device context ----------------------------------------------------- */
/* Owns the device buffers, stream and cached tables for one CUDA device, so
 * repeated runs (bench) reuse allocations.  Not thread-safe; one context per
 * host thread / device.  device < 0 = current device. */
typedef struct erato_gpu_ctx erato_gpu_ctx;
int erato_gpu_create(int device, erato_gpu_ctx** out);
void erato_gpu_destroy(erato_gpu_ctx* ctx);
/* Cap on the number of base primes, RunOptions::max_base_pairs / the CLI's
 * --max-base-pairs (driver.hpp:84, base.cpp:24-27); default 2^27 as in the
 * reference (base.hpp:87).  Runs above it fail with ALLOC_LIMIT. */
int erato_gpu_set_max_base_pairs(erato_gpu_ctx* ctx, uint64_t max_pairs);
/* Number of CUDA devices visible (0 when none). */
int erato_gpu_device_count(void);

/* ---- the hot path: run_sieve (src/driver.cpp:83-120) --------------------- */

/* Sieve (l, f, n) on the context's device.
 *   dev_table  device pointer receiving n*2^(l-3) bytes (NULL = count only,
 *              the NullSink path of bench.cpp:11-16);
 *   dev_count  optional device pointer (uint64) receiving the zero-bit count
 *              (lets a caller all-reduce it without a host round trip);
 *   stream     cudaStream_t as void* (NULL = the context's stream);
 *   sync       1: wait, check the capacities (re-running with doubled ones
 *              after an overflow) and fill stats.
 *              0: return once every wave is enqueued (one host sync happens
 *              during init, for the prime-class boundaries); results are
 *              valid after the stream drains, stats->prime_count is NOT
 *              filled, and a capacity overflow — which would drop marks —
 *              is reported on the device: *dev_count = ERATO_GPU_COUNT_OVERFLOW
 *              (re-run with sync = 1).  ERATO_GPU_CHECK_INVARIANTS needs sync = 1.
 * The interval may be a shard of a larger run; see erato_gpu_shard. */
int erato_gpu_run(erato_gpu_ctx* ctx, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                  void* dev_table, uint64_t* dev_count, void* stream, int sync,
                  erato_gpu_stats* stats);

/* SegmentSink equivalent (driver.hpp:34-39): the table is streamed to fn in
 * order, as contiguous byte slices covering [0, n*2^(l-3)) exactly once
 * (one slice per wave of tiles, <= ~20 MB), from a library thread while the
 * next waves sieve.  `bytes` is valid only during the call (it is a pinned
 * staging slot); a nonzero return aborts the run with ERATO_GPU_IO_ERROR.
 * Only kOutSlots wave slices are in flight, so neither HBM nor host memory
 * holds the whole table (the reference's one-segment-at-a-time FileSink,
 * driver.cpp:29-51). */
typedef int (*erato_gpu_sink_fn)(void* user, const uint8_t* bytes, uint64_t offset, uint64_t nbytes);
int erato_gpu_run_to_sink(erato_gpu_ctx* ctx, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                          erato_gpu_sink_fn fn, void* user, erato_gpu_stats* stats);

/* TableSink equivalent (driver.hpp:72-80): the whole table into host memory
 * dst (dst_cap >= n*2^(l-3) bytes).  Pinned dst: each wave's slice is copied
 * straight into it while the next waves sieve; pageable dst: through the
 * pinned staging slots of erato_gpu_run_to_sink. */
int erato_gpu_sieve_to_host(erato_gpu_ctx* ctx, unsigned l, uint64_t f, uint64_t n,
                            unsigned flags, uint8_t* dst, size_t dst_cap, erato_gpu_stats* stats);

/* NullSink run (count only): bench_run's timed_run (src/bench.cpp:11-16). */
int erato_gpu_count(erato_gpu_ctx* ctx, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                    uint64_t* count, erato_gpu_stats* stats);

/* FileSink / write_table (driver.hpp:45-58, :98-99): writes
 * out_dir/erato_l{l}_f{f}_n{n}.bits (exactly n*2^(l-3) bytes) and returns
 * the path.  The table is streamed (erato_gpu_run_to_sink + pwrite).
 *  - (part_f, part_n) == (f, n): the whole table, written to a temporary file
 *    that is renamed to the reference name only on success.
 *  - otherwise (part_f, part_n) is one shard of (f, n) (erato_gpu_shard): only
 *    its bytes are pwrite()n at their offset into the shared file, which is
 *    created / sized to the full length if needed; part_n = 0 is an empty
 *    shard (nothing is sieved). */
int erato_gpu_write_table(erato_gpu_ctx* ctx, const char* out_dir, unsigned l, uint64_t f,
                          uint64_t n, uint64_t part_f, uint64_t part_n, unsigned flags,
                          char* path_out, size_t path_cap, erato_gpu_stats* stats);

/* Contiguous range shard of (f, n) for rank `rank` of `world`:
 * rank g gets segments [f + floor(g*n/world), f + floor((g+1)*n/world)). */
void erato_gpu_shard(uint64_t f, uint64_t n, int rank, int world, uint64_t* f_out,
                     uint64_t* n_out);

/* Ascending primes represented by the clear bits of an interval
 * (extract_primes, src/driver.cpp:65-81), computed on the device.
 * Writes up to cap primes to host dst; returns the count in *count. */
int erato_gpu_extract_primes(erato_gpu_ctx* ctx, unsigned l, uint64_t f, uint64_t n,
                             unsigned flags, uint64_t* dst, uint64_t cap, uint64_t* count);

/* The device base-prime list: the odd primes <= limit (limit <= 2^32 - 1),
 * ascending, computed exactly as a run computes its base primes
 * (build_base / simple_sieve(isqrt v), src/base.cpp:19-53, src/oracle.cpp:8-23):
 * writes up to cap of them to host dst, *count = their number. */
int erato_gpu_base_primes(erato_gpu_ctx* ctx, uint64_t limit, uint32_t* dst, uint64_t cap, uint64_t* count);

/* ---- multi-GPU run_sieve -------------------------------- */
/* num_gpus contiguous range shards (erato_gpu_shard), one host thread and one
 * context per shard.  Each shard recomputes its own base primes and offsets
 * (no data-path collective); the only collective is one
 * ncclAllReduce(uint64, sum) of the shards' device count words over NVLink /
 * NVSwitch.  devices: num_gpus CUDA ordinals (NULL = 0..num_gpus-1).  NCCL
 * (libnccl.so.2, loaded at run time) needs distinct devices; a list that
 * repeats a device (a test topology on a 1-GPU box) sums the counts on the
 * host instead — see erato_gpu_multi_uses_nccl. */
typedef struct erato_gpu_multi erato_gpu_multi;
int erato_gpu_multi_create(int num_gpus, const int* devices, erato_gpu_multi** out);
void erato_gpu_multi_destroy(erato_gpu_multi* m);
int erato_gpu_multi_uses_nccl(const erato_gpu_multi* m);
/* NullSink run over all shards; *count = the all-reduced count.  stats: device
 * times are the max over shards, tiles / launches the sum. */
int erato_gpu_multi_count(erato_gpu_multi* m, unsigned l, uint64_t f, uint64_t n, unsigned flags,
                          uint64_t* count, erato_gpu_stats* stats);
/* write_table over all shards: each shard streams its bytes into the one
 * out_dir/erato_l{l}_f{f}_n{n}.bits at its offset (temporary file, renamed
 * on success). */
int erato_gpu_multi_write_table(erato_gpu_multi* m, const char* out_dir, unsigned l, uint64_t f,
                                uint64_t n, unsigned flags, char* path_out, size_t path_cap,
                                uint64_t* count, erato_gpu_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* ERATO_GPU_H */
