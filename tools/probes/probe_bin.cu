// Probe: phase timing of k_bin_sorted on the 12.5M-neuron config (27.5k rows).
#define BP_BIN_TIMING 1
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2311_05106_b200/csrc/step.cuh"
using namespace bp;

int main(int argc, char** argv) {
  // args: n_total, seg_len (= local partition), n_active, lane_rows
  const uint32_t n = argc > 1 ? (uint32_t)atoll(argv[1]) : 12500000u;
  const uint32_t L = argc > 2 ? (uint32_t)atoll(argv[2]) : n;
  const int n_active = argc > 3 ? atoi(argv[3]) : 27500;
  const int lane_rows = argc > 4 ? atoi(argv[4]) : 0;
  const uint32_t n_exc = n / 5 * 4, K = n / 40 - 1;
  const uint32_t n_tiles = (L + kTile - 1) / kTile, cap = 17408;
  int32_t *active, *count; cudaMalloc(&active, n_active * 4); cudaMalloc(&count, 4);
  std::vector<int32_t> h(n_active);
  for (int i = 0; i < n_active; ++i) h[i] = (int32_t)(((uint64_t)i * 2654435761u) % n);
  cudaMemcpy(active, h.data(), n_active * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(count, &n_active, 4, cudaMemcpyHostToDevice);
  Buckets bk{}; cudaMalloc(&bk.cnt, (size_t)n_tiles * kCntStride * 4); cudaMalloc(&bk.flag, n_tiles * 4);
  cudaMalloc(&bk.buf, (size_t)n_tiles * cap * 4); cudaMalloc(&bk.spill, (size_t)2 * L * 4);
  cudaMemset(bk.flag, 0, n_tiles * 4); cudaMemset(bk.spill, 0, (size_t)2 * L * 4);
  BinTarget bt{bk, cap, L, 0};
  ConnArgs c{}; c.conn = 0; c.split = n_exc; c.n_cols = n; c.lane_rows = lane_rows;
  c.je = JitSide{0x5EED0001, K, L, 0, 1, 0.6f, 0.f, 0, nullptr};
  c.ji = JitSide{0x5EED0002, K, L, 0, 1, 6.7f, 0.f, 0, nullptr};
  printf("n %u L %u K %u rows %d lane_rows %d tiles %u\n", n, L, K, n_active, lane_rows, n_tiles);
  unsigned long long* ev; cudaMalloc(&ev, 8);
  const size_t smem = (2 * (size_t)kBinStage + 2 * n_tiles) * 4;
  cudaFuncSetAttribute(k_bin_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) {
    cudaMemset(bk.cnt, 0, (size_t)n_tiles * kCntStride * 4);
    cudaEventRecord(a);
    k_bin_sorted<<<148, kBinThreads, smem>>>(c, bt, active, count, ev, n_tiles);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long t[1024][6]; cudaMemcpyFromSymbol(t, g_bin_t, sizeof(t));
    unsigned long long t0 = ~0ull; for (int i = 0; i < 148; ++i) t0 = std::min(t0, t[i][0]);
    double ph[5] = {0}; double mx[5] = {0};
    for (int i = 0; i < 148; ++i) for (int k = 0; k < 5; ++k) {
      double v = (k == 0 ? (double)(t[i][0] - t0) : (double)(t[i][k] - t[i][k - 1])) / 1e3;
      ph[k] += v / 148; mx[k] = std::max(mx[k], v);
    }
    double end = 0; for (int i = 0; i < 148; ++i) end = std::max(end, (double)(t[i][4] - t0) / 1e3);
    double scan = 0; for (int i = 0; i < 148; ++i) scan += (double)(t[i][5] - t[i][1]) / 1e3 / 148;
    printf("scan %.1f us | ", scan);
    printf("event %.1f us | last block end %.1f us | start-skew avg %.1f max %.1f | A %.1f/%.1f B %.1f/%.1f C %.1f/%.1f D %.1f/%.1f (avg/max us)\n",
           ms * 1e3, end, ph[0], mx[0], ph[1], mx[1], ph[2], mx[2], ph[3], mx[3], ph[4], mx[4]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
