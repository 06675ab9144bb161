// csr_grad.cuh -- gather-orientation event csrmv and the reverse mode of
// the event scatter (reading G1; BrainPy's
// csrmv(..., transpose=False) and the gradient behind the paper's
// differentiability claim).  Both walk CSR rows (one warp per row,
// lanes stride the row) and need no atomics on their outputs: each output
// is owned by one warp, so fixed-point results are exact and fp32 results
// are deterministic (a fixed warp-tree reduction order).
#pragma once
#include <cstdint>

#include "rng.cuh"

namespace bp {

constexpr int kGatherThreads = 256;

__device__ __forceinline__ bool spike_bit(const uint32_t *words, int64_t i) {
  return (__ldg(words + (i >> 5)) >> (i & 31)) & 1u;
}

struct CsrGatherArgs {
  const int64_t *indptr;
  const int32_t *indices;
  const float *data;        // nullptr -> homogeneous w
  float w;
  long long q;              // quantize(w)
  int64_t n_rows;           // outputs
  const uint32_t *spikes;   // n_cols bits (the event vector)
  void *out;                // n_rows, f32 or int64 fixed point
  int accumulate;
};

// out[r] (+)= sum_{k in row r} w_k [s[indices[k]]]
template <int KIND>
__global__ void __launch_bounds__(kGatherThreads) k_csr_gather(CsrGatherArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * kGatherThreads) >> 5;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * kGatherThreads + threadIdx.x) >> 5;
       r < a.n_rows; r += nw) {
    const int64_t lo = __ldg(a.indptr + r), hi = __ldg(a.indptr + r + 1);
    unsigned n = 0;
    float f = 0.f;
    long long fx = 0;
    for (int64_t k = lo + lane; k < hi; k += 32) {
      if (!spike_bit(a.spikes, __ldg(a.indices + k))) continue;
      if (a.data == nullptr) ++n;
      else if (KIND == 0) f = __fadd_rn(f, __ldg(a.data + k));
      else fx += quantize(__ldg(a.data + k));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      n += __shfl_xor_sync(0xffffffffu, n, o);
      f = __fadd_rn(f, __shfl_xor_sync(0xffffffffu, f, o));
      fx += __shfl_xor_sync(0xffffffffu, fx, o);
    }
    if (lane != 0) continue;
    if (KIND == 0) {
      const float v = a.data == nullptr ? __fmul_rn(static_cast<float>(n), a.w) : f;
      float *o = static_cast<float *>(a.out) + r;
      *o = a.accumulate ? __fadd_rn(*o, v) : v;
    } else {
      const long long v = a.data == nullptr ? static_cast<long long>(n) * a.q : fx;
      long long *o = static_cast<long long *>(a.out) + r;
      *o = a.accumulate ? *o + v : v;
    }
  }
}

struct CsrGradArgs {
  const int64_t *indptr;
  const int32_t *indices;
  const float *data;        // nullptr -> homogeneous w
  float w;
  int64_t n_rows;
  const uint32_t *spikes;   // n_rows bits
  const float *gy;          // n_cols upstream gradient
  float *grad_data;         // nullable [nnz]
  float *grad_events;       // nullable [n_rows]
  double *grad_w;           // nullable, homogeneous weight (pre-zeroed)
};

// Reverse mode of y = M^T s: grad_data[k] = s[r] gy[c_k];
// grad_events[r] = sum_k w_k gy[c_k]; grad_w = sum_{r: s[r]} sum_k gy[c_k].
__global__ void __launch_bounds__(kGatherThreads) k_csr_grad(CsrGradArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * kGatherThreads) >> 5;
  double gw = 0.0;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * kGatherThreads + threadIdx.x) >> 5;
       r < a.n_rows; r += nw) {
    const int64_t lo = __ldg(a.indptr + r), hi = __ldg(a.indptr + r + 1);
    const bool s = spike_bit(a.spikes, r);
    float ge = 0.f;
    double gsum = 0.0;
    for (int64_t k = lo + lane; k < hi; k += 32) {
      const float g = __ldg(a.gy + __ldg(a.indices + k));
      if (a.grad_data) a.grad_data[k] = s ? g : 0.f;
      if (a.grad_events) ge = __fmaf_rn(a.data ? __ldg(a.data + k) : a.w, g, ge);
      if (s) gsum += static_cast<double>(g);
    }
    if (a.grad_events) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) ge = __fadd_rn(ge, __shfl_xor_sync(0xffffffffu, ge, o));
      if (lane == 0) a.grad_events[r] = ge;
    }
    gw += gsum;
  }
  if (a.grad_w) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) gw += __shfl_xor_sync(0xffffffffu, gw, o);
    if (lane == 0 && gw != 0.0) atomicAdd(a.grad_w, gw);
  }
}

}  // namespace bp
