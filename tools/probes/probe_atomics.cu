// Probe: scatter-add throughput on B200 (throwaway measurement).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void k(float* outf, unsigned* outu, uint32_t n_out, int iters) {
  __shared__ float sf[6144];
  __shared__ unsigned su[6144];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (MODE >= 2) { for (int i = threadIdx.x; i < 6144; i += blockDim.x) { sf[i] = 0; su[i] = 0; } __syncthreads(); }
  uint32_t h = hash(t);
  for (int i = 0; i < iters; ++i) {
    h = hash(h + i);
    if (MODE == 0) atomicAdd(outf + (h % n_out), 1.0f);
    if (MODE == 1) atomicAdd(outu + (h % n_out), 1u);
    if (MODE == 2) atomicAdd(su + (h % 6144), 1u);
    if (MODE == 3) atomicAdd(sf + (h % 6144), 1.0f);
  }
  if (MODE >= 2) { __syncthreads(); if (threadIdx.x < 32) outu[blockIdx.x * 32 + threadIdx.x] += su[threadIdx.x] + (unsigned)sf[threadIdx.x]; }
}

int main() {
  float* f; unsigned* u; cudaMalloc(&f, 64 << 20); cudaMalloc(&u, 64 << 20);
  cudaMemset(f, 0, 64 << 20); cudaMemset(u, 0, 64 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern, uint32_t n_out, int grid, int block, int iters) {
    kern<<<grid, block>>>(f, u, n_out, iters);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kern<<<grid, block>>>(f, u, n_out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = 5.0 * grid * block * iters;
    printf("%-32s n_out %9u grid %5d: %8.1f G ops/s\n", name, n_out, grid, ops / (ms / 1e3) / 1e9);
  };
  for (uint32_t n_out : {100000u, 1000000u, 12500000u}) {
    run("REDG.F32 global", k<0>, n_out, 148 * 8, 256, 256);
    run("REDG.U32 global", k<1>, n_out, 148 * 8, 256, 256);
  }
  run("ATOMS.ADD.U32 smem (12k)", k<2>, 1, 148 * 4, 256, 256);
  run("ATOMS f32 CAS smem (12k)", k<3>, 1, 148 * 4, 256, 256);
  run("ATOMS.ADD.U32 smem 1024thr", k<2>, 1, 148 * 2, 1024, 256);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
