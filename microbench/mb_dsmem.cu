// Microbenchmark: DSMEM (cluster shared memory) atomicOr throughput on B200,
// vs local smem atomics.  Decides whether tiles of a cluster can exchange
// hit records through distributed shared memory instead of HBM lists.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint32_t lcg(uint32_t& s) { s = s * 1664525u + 1013904223u; return s; }

template <int CL, bool REMOTE>
__global__ void k(int iters, uint32_t* out) {
  extern __shared__ uint32_t s[];
  constexpr int W = 32768;
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < W; i += blockDim.x) s[i] = 0;
  cl.sync();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u + 1;
  uint32_t* peers[CL];
  for (int r = 0; r < CL; ++r) peers[r] = cl.map_shared_rank(s, r);
  for (int i = 0; i < iters; ++i) {
    uint32_t r = lcg(st);
    uint32_t* base = REMOTE ? peers[(r >> 28) % CL] : s;
    atomicOr(&base[(r >> 8) & (W - 1)], 1u << (r & 31));
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = s[st & (W - 1)];
}

template <int CL, bool REMOTE>
void run(int nsm, uint32_t* out) {
  const int smem = 32768 * 4, thr = 1024, iters = 2048;
  CK(cudaFuncSetAttribute(k<CL, REMOTE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (CL > 8) CK(cudaFuncSetAttribute(k<CL, REMOTE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int grid = (nsm / CL) * CL * 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid; cfg.blockDim = thr; cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  CK(cudaLaunchKernelEx(&cfg, k<CL, REMOTE>, iters, out)); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < 3; ++r) CK(cudaLaunchKernelEx(&cfg, k<CL, REMOTE>, iters, out));
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  double ops = 3.0 * grid * thr * iters;
  printf("cluster %2d %s: %.3g atomicOr/s\n", CL, REMOTE ? "spread over cluster" : "local only        ", ops / ms * 1e3);
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  uint32_t* out; CK(cudaMalloc(&out, 1 << 20));
  run<2, false>(pr.multiProcessorCount, out);
  run<2, true>(pr.multiProcessorCount, out);
  run<4, true>(pr.multiProcessorCount, out);
  run<8, true>(pr.multiProcessorCount, out);
  run<16, true>(pr.multiProcessorCount, out);
  printf("done\n");
}
