// Probe: how fast can the network state (V f32, g_E f32, g_I f32, ref u8 --
// 25 B per neuron read + written) be streamed with k_step's block shape,
// with no counting and no neuron arithmetic?  Variants: passes in flight
// per thread (2 = k_step's, 4 = the whole tile's), and a grid-stride
// persistent layout.  Prints GB/s of algorithmic bytes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kTile = 4096;
struct S { float *v, *ge, *gi; uint8_t *ref; int64_t n; };

template <int INFLIGHT, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_stream(S s, int flip) {
  constexpr int passes = kTile / (4 * NT);
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  float4 V[INFLIGHT], E[INFLIGHT], I[INFLIGHT];
  uint32_t R[INFLIGHT];
  auto load = [&](int slot, int p) {
    const int64_t i = base + p * 4 * NT + 4 * threadIdx.x;
    V[slot] = *reinterpret_cast<const float4 *>(s.v + i);
    E[slot] = *reinterpret_cast<const float4 *>(s.ge + i);
    I[slot] = *reinterpret_cast<const float4 *>(s.gi + i);
    R[slot] = *reinterpret_cast<const uint32_t *>(s.ref + i);
  };
  auto store = [&](int slot, int p) {
    const int64_t i = base + p * 4 * NT + 4 * threadIdx.x;
    float4 v = V[slot]; v.x += 1.f;
    float4 e = E[slot]; e.y *= 0.98f;
    float4 g = I[slot]; g.z *= 0.99f;
    *reinterpret_cast<float4 *>(s.v + i) = v;
    *reinterpret_cast<float4 *>(s.ge + i) = e;
    *reinterpret_cast<float4 *>(s.gi + i) = g;
    if (flip) *reinterpret_cast<uint32_t *>(s.ref + i) = R[slot] + 1u;
  };
#pragma unroll
  for (int p = 0; p < INFLIGHT && p < passes; ++p) load(p, p);
#pragma unroll
  for (int p = 0; p < passes; ++p) {
    store(p % INFLIGHT, p);
    if (p + INFLIGHT < passes) load(p % INFLIGHT, p + INFLIGHT);
  }
}

int main() {
  const int64_t n = 12500000 / kTile * kTile;
  S s{};
  s.n = n;
  cudaMalloc(&s.v, n * 4); cudaMalloc(&s.ge, n * 4); cudaMalloc(&s.gi, n * 4); cudaMalloc(&s.ref, n);
  cudaMemset(s.v, 0, n * 4); cudaMemset(s.ge, 0, n * 4); cudaMemset(s.gi, 0, n * 4); cudaMemset(s.ref, 0, n);
  const int grid = static_cast<int>(n / kTile);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char *name, auto kern, int nt) {
    for (int w = 0; w < 3; ++w) kern<<<grid, nt>>>(s, w & 1);
    cudaEventRecord(a);
    const int reps = 50;
    for (int r = 0; r < reps; ++r) kern<<<grid, nt>>>(s, r & 1);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / reps;
    printf("%-28s %7.2f us  %7.0f GB/s (25 B/neuron alg.)\n", name, us, 25.0 * n / us / 1e3);
  };
  run("256 thr, 2 passes in flight", k_stream<2, 256>, 256);
  run("256 thr, 4 passes in flight", k_stream<4, 256>, 256);
  run("512 thr, 2 passes in flight", k_stream<2, 512>, 512);
  run("128 thr, 2 passes in flight", k_stream<2, 128>, 128);
  run("128 thr, 4 passes in flight", k_stream<4, 128>, 128);
  run("1024 thr, 1 pass", k_stream<1, 1024>, 1024);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
