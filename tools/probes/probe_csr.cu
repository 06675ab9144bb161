// Phase timing of the streamed CSR scatter (k_csr_split + k_csr_stream) on a
// synthetic 100k x 100k matrix with rows of exactly p*n sorted columns.
// usage: probe_csr <p> <density> <homo 0|1> <fused 0|1>  (fused: cooperative, in-kernel
// compaction and reduction; else separate compaction, partials only)
#define BP_CSR_TIMING 1
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_2311_05106_b200/csrc/csr_stream.cuh"

__global__ void k_fill(int32_t *idx, float *dat, int64_t n, int L) {
  const int64_t r = blockIdx.x;
  const int step = static_cast<int>(n / L);
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    uint32_t h = static_cast<uint32_t>(r * 2654435761u) ^ (j * 40503u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    idx[r * L + j] = j * step + static_cast<int32_t>(h % step);
    if (dat) dat[r * L + j] = (h & 1023) * 1e-4f - 0.05f;
  }
}
__global__ void k_pat(uint32_t *w, int64_t words, double d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= words) return;
  uint32_t v = 0;
  for (int b = 0; b < 32; ++b) {
    uint32_t h = static_cast<uint32_t>(i * 32 + b) * 2246822519u; h ^= h >> 15; h *= 3266489917u; h ^= h >> 16;
    if (h < d * 4294967296.0) v |= 1u << b;
  }
  w[i] = v;
}
__global__ void k_compact(const uint32_t *s, int64_t n, int32_t *act, int32_t *cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i * 32 >= n) return;
  uint32_t v = s[i];
  while (v) { int b = __ffs(v) - 1; v &= v - 1; act[atomicAdd(cnt, 1)] = (int32_t)(i * 32 + b); }
}

int main(int argc, char **argv) {
  const double p = atof(argv[1]), d = atof(argv[2]);
  const bool homo = atoi(argv[3]) != 0, fused = atoi(argv[4]) != 0;
  const int64_t n = 100000;
  const int L = static_cast<int>(p * n);
  int32_t *idx, *act, *cnt; float *dat = nullptr; int64_t *indptr, *bounds; uint32_t *sp;
  cudaMalloc(&idx, n * L * 4);
  if (!homo) cudaMalloc(&dat, n * L * 4);
  std::vector<int64_t> ip(n + 1);
  for (int64_t r = 0; r <= n; ++r) ip[r] = r * L;
  cudaMalloc(&indptr, (n + 1) * 8);
  cudaMemcpy(indptr, ip.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
  k_fill<<<n, 256>>>(idx, dat, n, L);
  cudaMalloc(&sp, n / 8 + 64);
  k_pat<<<(n / 32 + 255) / 256, 256>>>(sp, n / 32 + 1, d);
  cudaMalloc(&act, n * 4); cudaMalloc(&cnt, 4);
  cudaMemset(cnt, 0, 4);
  k_compact<<<(n / 32 + 255) / 256, 256>>>(sp, n, act, cnt);
  int na; cudaMemcpy(&na, cnt, 4, cudaMemcpyDeviceToHost);
  const int acc = 4;
  const size_t fixed = bp::stream_smem(0, acc, homo).total + bp::kStreamStaticSmem + 256;
  const int64_t max_cols = ((232448 - fixed) / acc) & ~3LL;
  const int nt = (int)((n + max_cols - 1) / max_cols);
  const int tile_cols = (int)(((n + nt - 1) / nt + 3) & ~3LL);
  const int G = 148 / nt;
  int32_t *split;
  cudaMalloc(&split, (size_t)n * (nt + 1) * 4);
  void *partials, *out;
  cudaMalloc(&partials, (size_t)nt * G * tile_cols * 4);
  cudaMalloc(&out, n * 4);
  bp::CsrSplitArgs sa{indptr, idx, nullptr, nullptr, n, split, nt, tile_cols, n};   // plan
  bp::k_csr_split<<<148 * 16, 256>>>(sa);
  bp::CsrStreamArgs ca{idx, dat, indptr, split, act, cnt, indptr + n, partials, tile_cols, G, nt,
                       0, n, fused ? out : nullptr, 0.6f, 0};
  const size_t smem = bp::stream_smem(tile_cols, acc, homo).total;
  auto kern = homo ? bp::k_csr_stream<0, true> : bp::k_csr_stream<0, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(232448 - bp::kStreamStaticSmem));
  cudaEvent_t e0, e1, e2; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  if (getenv("CARVEOUT")) {   // keep the SM's shared-memory carveout at max across kernels
    cudaFuncSetAttribute(k_compact, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  printf("p=%g d=%g homo=%d fused=%d active=%d tiles=%d groups=%d tile_cols=%d smem=%zu\n",
         p, d, homo, fused, na, nt, G, tile_cols, smem);
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    cudaMemsetAsync(cnt, 0, 4);
    k_compact<<<(n / 32 + 255) / 256, 256>>>(sp, n, act, cnt);
    cudaEventRecord(e1);
    void *args[] = {&ca};
    if (fused) cudaLaunchCooperativeKernel((const void *)kern, dim3(nt * G), dim3(1024), args, smem, 0);
    else kern<<<nt * G, 1024, smem>>>(ca);
    cudaEventRecord(e2);
    cudaEventSynchronize(e2);
    if (cudaGetLastError() != cudaSuccess) { printf("error\n"); return 1; }
    float t1, t2; cudaEventElapsedTime(&t1, e0, e1); cudaEventElapsedTime(&t2, e1, e2);
    unsigned long long T[1024][8];
    cudaMemcpyFromSymbol(T, bp::g_csr_t, sizeof(T));
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < nt * G; ++b) t0 = std::min(t0, T[b][0]);
    double ph[8] = {0}, mx[8] = {0};
    for (int b = 0; b < nt * G; ++b)
      for (int k = 0; k < 8; ++k) { double v = (T[b][k] - t0) / 1e3; ph[k] += v / (nt * G); mx[k] = std::max(mx[k], v); }
    printf("compact %.1f us  stream %.1f us | mean/max since first CTA start (us):", t1 * 1e3, t2 * 1e3);
    const char *nm[7] = {"start", "init", "w0loop", "allloop", "flush", "gsync", "end"};
    for (int k = 0; k < (fused ? 7 : 5); ++k) printf(" %s %.1f/%.1f", nm[k], ph[k], mx[k]);
    printf("\n");
  }
  return 0;
}
