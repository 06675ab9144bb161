// Probe: achievable DRAM bandwidth for the k_step access pattern (V r/w f32,
// ref r u8, gE/gI r/w f32) with no compute, vs a plain copy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NPT>
__global__ void __launch_bounds__(256) k_pattern(float* v, const uint8_t* ref, float* ge, float* gi, int64_t n) {
  int64_t i0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 4;
  int64_t stride = (int64_t)gridDim.x * 256 * 4;
  for (int64_t i = i0; i + 3 < n; i += stride) {
    float4 a = *reinterpret_cast<float4*>(v + i);
    uint32_t r = *reinterpret_cast<const uint32_t*>(ref + i);
    float4 e = *reinterpret_cast<float4*>(ge + i);
    float4 f = *reinterpret_cast<float4*>(gi + i);
    a.x += 1.f + (r & 1); e.x *= 0.9f; f.x *= 0.9f;
    *reinterpret_cast<float4*>(v + i) = a;
    *reinterpret_cast<float4*>(ge + i) = e;
    *reinterpret_cast<float4*>(gi + i) = f;
  }
}
__global__ void k_copy(const float4* a, float4* b, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  const int64_t n = 12500000;
  float *v, *ge, *gi; uint8_t* ref;
  cudaMalloc(&v, n * 4); cudaMalloc(&ge, n * 4); cudaMalloc(&gi, n * 4); cudaMalloc(&ref, n);
  cudaMemset(v, 0, n * 4); cudaMemset(ge, 0, n * 4); cudaMemset(gi, 0, n * 4); cudaMemset(ref, 0, n);
  float *ca, *cb; int64_t cn = 1ll << 28; cudaMalloc(&ca, cn * 4); cudaMalloc(&cb, cn * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {592, 1184, 2368, 12207}) {
    for (int w = 0; w < 3; ++w) k_pattern<4><<<grid, 256>>>(v, ref, ge, gi, n);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) k_pattern<4><<<grid, 256>>>(v, ref, ge, gi, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = n * (4 + 4 + 1 + 16 + 0.0);  // V r+w, ref r, g r+w = 25 B
    printf("pattern grid %5d: %.1f us  %.0f GB/s (25 B/neuron)\n", grid, ms * 1000 / 20, bytes / (ms / 20 / 1e3) / 1e9);
  }
  for (int w = 0; w < 3; ++w) k_copy<<<148 * 8, 256>>>((float4*)ca, (float4*)cb, cn / 4);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) k_copy<<<148 * 8, 256>>>((float4*)ca, (float4*)cb, cn / 4);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("copy 1 GiB: %.0f GB/s\n", 2.0 * cn * 4 / (ms / 10 / 1e3) / 1e9);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
