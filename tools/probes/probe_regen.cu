// Probe: cost of JIT row regeneration alone vs with binning, 27.5k rows,
// fan-out 80 (12.5M-neuron network), warp-per-row.  Throwaway measurement.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2311_05106_b200/csrc/rng.cuh"
using namespace bp;

template <int MODE>
__global__ void __launch_bounds__(256) k_regen(const int32_t* active, int n_active, uint64_t seed,
    uint32_t K, uint32_t n, int* counts, unsigned long long* out_sum) {
  const uint32_t lane = threadIdx.x & 31;
  const int warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int k = warp0; k < n_active; k += nw) {
    const uint32_t row = MODE >= 10 ? (uint32_t)k : (uint32_t)active[k];
    u32x4 g = philox_block(seed, 0, row, 0, lane);
    uint32_t start = first_offset(seed, K, row, 0);
    uint32_t chunk = 0;
    while (start < n) {
      const uint32_t g0 = bounded(1u, K, g.x), g1 = bounded(1u, K, g.y);
      const uint32_t g2 = bounded(1u, K, g.z), g3 = bounded(1u, K, g.w);
      const uint32_t p1 = g0, p2 = g0 + g1, p3 = p2 + g2, t = p3 + g3;
      uint32_t incl = t;
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= (uint32_t)off) incl += v;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t pos0 = start + (incl - t);
      const uint32_t pos[4] = {pos0, pos0 + p1, pos0 + p2, pos0 + p3};
      for (int q = 0; q < 4; ++q) if (pos[q] < n) {
        if (MODE % 10 == 0) acc += pos[q];
        else if (MODE % 10 == 1) atomicAdd(counts + (pos[q] >> 12) * 64, 1);
        else if (MODE % 10 == 2) atomicAdd(counts + pos[q], 1);   // RED into dense
      }
      start += total; ++chunk;
      if (start < n) g = philox_block(seed, 0, row, 0, chunk * 32 + lane);
    }
  }
  if (MODE % 10 == 0 && acc == 0x12345678) out_sum[0] = acc;
}

int main() {
  const uint32_t n = 12500000; const uint32_t K = 312499; const int n_active = 27500;
  int32_t* active; int* counts; unsigned long long* o;
  cudaMalloc(&active, n_active * 4); cudaMalloc(&counts, (size_t)n * 4); cudaMalloc(&o, 8);
  int32_t* h = new int32_t[n_active];
  for (int i = 0; i < n_active; ++i) h[i] = (int32_t)(((uint64_t)i * 2654435761u) % n);
  cudaMemcpy(active, h, n_active * 4, cudaMemcpyHostToDevice);
  cudaMemset(counts, 0, (size_t)n * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern, int grid, int block) {
    for (int w = 0; w < 3; ++w) kern<<<grid, block>>>(active, n_active, 7, K, n, counts, o);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) kern<<<grid, block>>>(active, n_active, 7, K, n, counts, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-40s grid %5d x %4d : %8.2f us\n", name, grid, block, ms * 1000 / 20);
  };
  for (int grid : {148 * 4, 148 * 8, 148 * 16, 3438}) {
    run("regen only (active list)", k_regen<0>, grid, 256);
    run("regen only (rows = index)", k_regen<10>, grid, 256);
    run("regen + tile-counter ATOMG", k_regen<1>, grid, 256);
    run("regen + dense RED", k_regen<2>, grid, 256);
  }
  // same kernels right after a 300 MB streaming copy (L2 full of dirty lines)
  char *sa, *sb; cudaMalloc(&sa, 300 << 20); cudaMalloc(&sb, 300 << 20);
  auto run_after_copy = [&](const char* name, auto kern, int grid, int block) {
    float tot = 0;
    for (int r = 0; r < 23; ++r) {
      cudaMemcpyAsync(sb, sa, 300 << 20, cudaMemcpyDeviceToDevice);
      cudaEventRecord(a);
      kern<<<grid, block>>>(active, n_active, 7, K, n, counts, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 3) tot += ms;
    }
    printf("%-40s after copy grid %5d: %8.2f us\n", name, grid, tot * 1000 / 20);
  };
  run_after_copy("regen only", k_regen<0>, 1184, 256);
  run_after_copy("regen + tile-counter ATOMG", k_regen<1>, 1184, 256);
  run_after_copy("regen + dense RED", k_regen<2>, 1184, 256);
  auto run_single = [&](const char* name, auto kern, int grid, int block) {
    float tot = 0;
    for (int r = 0; r < 23; ++r) {
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      kern<<<grid, block>>>(active, n_active, 7, K, n, counts, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 3) tot += ms;
    }
    printf("%-40s single grid %5d: %8.2f us\n", name, grid, tot * 1000 / 20);
  };
  run_single("regen only", k_regen<0>, 1184, 256);
  run_single("regen + tile-counter ATOMG", k_regen<1>, 1184, 256);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
