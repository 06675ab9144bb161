// Throughput of shared-memory atomics to the own CTA vs to other CTAs of a
// thread-block cluster (DSMEM, atom/red.shared::cluster).
// usage: probe_dsmem <cluster size C> <remote fraction 0|1>
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
namespace cg = cooperative_groups;

__global__ void k(unsigned *out, int words, int iters, int remote, unsigned seed) {
  extern __shared__ unsigned acc[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < words; i += blockDim.x) acc[i] = 0;
  cl.sync();
  const unsigned C = cl.num_blocks();
  const unsigned me = cl.block_rank();
  unsigned x = seed ^ (blockIdx.x * 7919u + threadIdx.x * 104729u);
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    const unsigned w = (x >> 8) % words;
    const unsigned dst = remote ? (me + 1 + (x & 7) % (C > 1 ? C - 1 : 1)) % C : me;
    unsigned *p = cl.map_shared_rank(acc, dst);
    if (remote) atomicAdd(p + w, 1u);
    else atomicAdd(acc + w, 1u);
  }
  cl.sync();
  unsigned s = 0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) s += acc[i];
  atomicAdd(out, s);
}

int main(int argc, char **argv) {
  const int C = argc > 1 ? atoi(argv[1]) : 2;
  const int remote = argc > 2 ? atoi(argv[2]) : 1;
  const int words = 24 * 1024, threads = 1024, iters = 2048;
  unsigned *out;
  cudaMalloc(&out, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4);
  if (C > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148 / C * C);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = words * 4;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, k, out, words, iters, remote, 12345u + rep);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); return 1; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double n = double(cfg.gridDim.x) * threads * iters;
    printf("C=%d remote=%d  %.3f ms  %.3f T atomics/s\n", C, remote, ms, n / ms / 1e9);
  }
  return 0;
}
