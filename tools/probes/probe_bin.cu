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
  // args: n_total, seg_len (= local partition), n_active, group lanes S
  const uint32_t n = argc > 1 ? (uint32_t)atoll(argv[1]) : 12500000u;
  const uint32_t L = argc > 2 ? (uint32_t)atoll(argv[2]) : n;
  const int n_active = argc > 3 ? atoi(argv[3]) : 27500;
  const int group = argc > 4 ? atoi(argv[4]) : 32;
  const uint32_t n_exc = n / 5 * 4, K = argc > 5 ? (uint32_t)atoll(argv[5]) : n / 40 - 1;
  // LOCAL=1: a rank's partition = the first segment [0, L) only (weak
  // scaling: the remote rows' events restricted to the local segment)
  const bool local = getenv("LOCAL") && atoi(getenv("LOCAL"));
  const uint32_t n_loc = local ? L : n;
  const uint32_t n_tiles = (n_loc + kTile - 1) / kTile, cap = 17408;
  int32_t *active, *count; cudaMalloc(&active, n_active * 4); cudaMalloc(&count, 4);
  std::vector<int32_t> h(n_active);
  for (int i = 0; i < n_active; ++i) h[i] = (int32_t)(((uint64_t)i * 2654435761u) % n);
  // the library's lists are (nearly) ascending: compaction of the spike
  // words in order, k_step's appends tile by tile -- E and I rows do not mix
  // within a warp's items except at the boundary
  if (!getenv("UNSORTED")) std::sort(h.begin(), h.end());
  cudaMemcpy(active, h.data(), n_active * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(count, &n_active, 4, cudaMemcpyHostToDevice);
  Buckets bk{}; cudaMalloc(&bk.cnt, (size_t)n_tiles * kCntStride * 4); cudaMalloc(&bk.flag, n_tiles * 4);
  cudaMalloc(&bk.buf, (size_t)n_tiles * cap * 4); cudaMalloc(&bk.spill, (size_t)2 * n * 4);
  const uint32_t n_seg = local ? 1u : (n + L - 1) / L;
  cudaMemset(bk.flag, 0, n_tiles * 4); cudaMemset(bk.spill, 0, (size_t)2 * n * 4);
  BinTarget bt{bk, cap, n_loc, 0};
  NetProj tab[2] = {};
  tab[0].pre_begin = 0; tab[0].pre_end = n_exc; tab[0].conn = 0; tab[0].cls = 0;
  tab[0].j = JitSide{0x5EED0001, K, L, 0, n_seg, 0.6f, 0.f, 0, nullptr};
  tab[1].pre_begin = n_exc; tab[1].pre_end = n; tab[1].conn = 0; tab[1].cls = 1;
  tab[1].j = JitSide{0x5EED0002, K, L, 0, n_seg, 6.7f, 0.f, 0, nullptr};
  NetProj *dtab; cudaMalloc(&dtab, sizeof tab);
  cudaMemcpy(dtab, tab, sizeof tab, cudaMemcpyHostToDevice);
  ConnArgs c{}; c.proj = dtab; c.n_proj = 2; c.all_jit = 1; c.n_cols = n;
  c.group_lanes = group; c.n_seg_max = n_seg;
  printf("n %u L %u K %u rows %d S %d tiles %u\n", n, L, K, n_active, group, n_tiles);
  unsigned long long* ev; cudaMalloc(&ev, 8);
  const size_t smem = (2 * (size_t)kBinStage + 2 * n_tiles) * 4;
  cudaFuncSetAttribute(k_bin_sorted<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) {
    cudaMemset(bk.cnt, 0, (size_t)n_tiles * kCntStride * 4);
    cudaEventRecord(a);
    k_bin_sorted<false><<<148, kBinThreads, smem>>>(c, bt, active, count, WordRange{}, ev, n_tiles);
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
    printf("event %.1f us | last block end %.1f us | start-skew avg %.1f max %.1f | A %.1f/%.1f B %.1f/%.1f C %.1f/%.1f D %.1f/%.1f (avg/max us)\n",
           ms * 1e3, end, ph[0], mx[0], ph[1], mx[1], ph[2], mx[2], ph[3], mx[3], ph[4], mx[4]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
