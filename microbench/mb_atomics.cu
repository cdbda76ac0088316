// Microbenchmark: shared-memory atomicOr / byte-store / global RED.OR rates on B200.
// Used to pick the marking primitive for the tile kernel.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t lcg(uint32_t& s) { s = s * 1664525u + 1013904223u; return s; }

// random smem atomicOr over a WORDS-word tile
template <int WORDS>
__global__ void k_smem_atom(int iters, uint32_t* out) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u + 1;
  for (int i = 0; i < iters; ++i) {
    uint32_t r = lcg(st);
    atomicOr(&s[(r >> 8) & (WORDS - 1)], 1u << (r & 31));
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[st & (WORDS - 1)];
}

// sieve-like: each thread has its own stride p (odd) and walks q += p over the bit tile
template <int WORDS>
__global__ void k_smem_atom_stride(int iters, uint32_t* out) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const uint32_t nbits = WORDS * 32u;
  uint32_t p = 2049u + 2u * (blockIdx.x * blockDim.x + threadIdx.x) % 60000u;
  uint32_t q = (threadIdx.x * 7919u) % p % nbits;
  for (int i = 0; i < iters; ++i) {
    atomicOr(&s[q >> 5], 1u << (q & 31));
    q += p; while (q >= nbits) q -= nbits;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[q >> 5 & (WORDS-1)];
}

// same but plain byte stores (byte-per-number tile, race-free since all write 1)
template <int BYTES>
__global__ void k_smem_u8_stride(int iters, uint32_t* out) {
  extern __shared__ uint8_t sb[];
  for (int i = threadIdx.x; i < BYTES; i += blockDim.x) sb[i] = 0;
  __syncthreads();
  uint32_t p = 2049u + 2u * (blockIdx.x * blockDim.x + threadIdx.x) % 60000u;
  uint32_t q = (threadIdx.x * 7919u) % p % BYTES;
  for (int i = 0; i < iters; ++i) {
    asm volatile("st.shared.u8 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(sb + q)), "r"(1u) : "memory");
    q += p; while (q >= BYTES) q -= BYTES;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sb[q & (BYTES-1)];
}

// plain (racy) RMW on 32-bit words: ld.shared + or + st.shared — measures non-atomic ceiling
template <int WORDS>
__global__ void k_smem_rmw_stride(int iters, uint32_t* out) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const uint32_t nbits = WORDS * 32u;
  uint32_t p = 2049u + 2u * (blockIdx.x * blockDim.x + threadIdx.x) % 60000u;
  uint32_t q = (threadIdx.x * 7919u) % p;
  volatile uint32_t* vs = s;
  for (int i = 0; i < iters; ++i) {
    vs[q >> 5] |= 1u << (q & 31);
    q += p; while (q >= nbits) q -= nbits;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[q >> 5 & (WORDS-1)];
}

// Pure ATOMS issue rate: 16 addresses per thread precomputed in registers,
// the timed loop is 16 unrolled atomicOr per iteration plus one loop counter
// (no address arithmetic).  CONFLICT_FREE: lane j always hits bank j (the
// shared pipe's ceiling); else random words (the sieve's ~3.1-way conflicts).
template <int WORDS, bool CONFLICT_FREE>
__global__ void k_smem_atom_pure(int iters, uint32_t* out) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u + 1;
  uint32_t a[16], m[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t r = lcg(st);
    const uint32_t w = CONFLICT_FREE ? (((r >> 8) & (WORDS - 1)) & ~31u) | (threadIdx.x & 31) : (r >> 8) & (WORDS - 1);
    a[k] = (uint32_t)__cvta_generic_to_shared(s + w);
    m[k] = 1u << (r & 31);
  }
  for (int i = 0; i < iters; i += 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a[k]), "r"(m[k]) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[st & (WORDS - 1)];
}

// global RED.OR random over a region of `words` words
__global__ void k_gred(uint32_t* tab, uint64_t words_mask, int iters) {
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u + 1;
  uint32_t st2 = st ^ 0x9e3779b9u;
  for (int i = 0; i < iters; ++i) {
    uint64_t r = ((uint64_t)lcg(st) << 32) | lcg(st2);
    atomicOr(&tab[(r >> 5) & words_mask], 1u << (r & 31));
  }
}

// streaming copy of 8-byte entries (bucket traffic proxy)
__global__ void k_copy8(const uint2* __restrict__ a, uint2* __restrict__ b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint2 x = a[i]; x.y += x.x; b[i] = x;
  }
}

template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int nsm = pr.multiProcessorCount;
  printf("device %s SMs %d smemOptin %zu L2 %d\n", pr.name, nsm, pr.sharedMemPerBlockOptin, pr.l2CacheSize);
  uint32_t* out; CK(cudaMalloc(&out, 1 << 20));
  const int iters = 4096;
  struct Cfg { int threads, ctas_per_sm; };
  Cfg cfgs[] = {{1024, 1}, {512, 2}, {256, 4}};
  for (auto c : cfgs) {
    int grid = nsm * c.ctas_per_sm * 4;
    {  // 128 KiB tile (32768 words) — only 1 CTA/SM fits
      const int W = 32768; size_t sm = W * 4;
      if (c.ctas_per_sm == 1) {
        CK(cudaFuncSetAttribute(k_smem_atom<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        CK(cudaFuncSetAttribute(k_smem_atom_stride<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        CK(cudaFuncSetAttribute(k_smem_rmw_stride<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        CK(cudaFuncSetAttribute(k_smem_u8_stride<W*4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        double ops = (double)grid * c.threads * iters;
        float t1 = timeit([&] { k_smem_atom<W><<<grid, c.threads, sm>>>(iters, out); });
        float t2 = timeit([&] { k_smem_atom_stride<W><<<grid, c.threads, sm>>>(iters, out); });
        float t3 = timeit([&] { k_smem_rmw_stride<W><<<grid, c.threads, sm>>>(iters, out); });
        float t4 = timeit([&] { k_smem_u8_stride<W*4><<<grid, c.threads, sm>>>(iters, out); });
        printf("tile128K thr%d: atom_rand %.3g/s  atom_stride %.3g/s  rmw_stride %.3g/s  u8_stride %.3g/s\n",
               c.threads, ops / t1 * 1e3, ops / t2 * 1e3, ops / t3 * 1e3, ops / t4 * 1e3);
        CK(cudaFuncSetAttribute(k_smem_atom_pure<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        CK(cudaFuncSetAttribute(k_smem_atom_pure<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        float t5 = timeit([&] { k_smem_atom_pure<W, false><<<grid, c.threads, sm>>>(iters, out); });
        float t6 = timeit([&] { k_smem_atom_pure<W, true><<<grid, c.threads, sm>>>(iters, out); });
        printf("tile128K thr%d: pure unrolled ATOMS random words %.3g/s  conflict-free %.3g/s\n", c.threads,
               ops / t5 * 1e3, ops / t6 * 1e3);
      }
    }
    {  // 32 KiB tile (8192 words) — many CTAs/SM
      const int W = 8192; size_t sm = W * 4;
      CK(cudaFuncSetAttribute(k_smem_atom_stride<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      CK(cudaFuncSetAttribute(k_smem_u8_stride<W*4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      double ops = (double)grid * c.threads * iters;
      float t2 = timeit([&] { k_smem_atom_stride<W><<<grid, c.threads, sm>>>(iters, out); });
      float t4 = timeit([&] { k_smem_u8_stride<W*4><<<grid, c.threads, sm>>>(iters, out); });
      printf("tile32K thr%d x%d/SM: atom_stride %.3g/s  u8_stride %.3g/s\n", c.threads, c.ctas_per_sm, ops / t2 * 1e3, ops / t4 * 1e3);
    }
  }
  // global RED.OR
  uint32_t* tab; size_t big = (size_t)4 << 30; CK(cudaMalloc(&tab, big)); CK(cudaMemset(tab, 0, big));
  for (size_t region : {(size_t)16 << 20, (size_t)64 << 20, (size_t)big}) {
    uint64_t wm = region / 4 - 1; int grid = nsm * 8, thr = 256, it = 1024;
    double ops = (double)grid * thr * it;
    float t = timeit([&] { k_gred<<<grid, thr>>>(tab, wm, it); });
    printf("global RED.OR random region %zu MB: %.3g ops/s\n", region >> 20, ops / t * 1e3);
  }
  {
    uint64_t n = (uint64_t)1 << 28;  // 2 GiB of entries
    uint2* a = (uint2*)tab; uint2* b = (uint2*)((char*)tab + (n * 8));
    float t = timeit([&] { k_copy8<<<nsm * 8, 256>>>(a, b, n); });
    printf("copy8 (r+w) %.1f GB/s\n", 16.0 * n / t / 1e6);
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
