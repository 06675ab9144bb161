// cache.cuh -- L2 eviction-priority hints (PTX createpolicy + .L2::cache_hint).
//
// The network keeps its conductance arrays g_E/g_I resident in the 126 MB L2
// across steps: the neuron update and the scatter REDs touch them with an
// evict_last policy covering a fraction of the lines (the fraction the L2
// budget allows, deterministic per address), while the streamed state
// (V, refractory counters) uses evict_first so it does not displace them.
#pragma once
#include <cstdint>

namespace bp {

__device__ __forceinline__ uint64_t policy_keep(float fraction) {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, %1;"
               : "=l"(p) : "f"(fraction));
  return p;
}
__device__ __forceinline__ uint64_t policy_stream() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_neutral() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// keep_frac > 0: (evict_last on that fraction of g lines, evict_first on the
// streamed state); keep_frac == 0: leave the L2 policy unchanged.
struct Policies {
  uint64_t keep, stream;
};
__device__ __forceinline__ Policies make_policies(float keep_frac) {
  Policies p;
  if (keep_frac > 0.0f) {
    p.keep = policy_keep(keep_frac);
    p.stream = policy_stream();
  } else {
    p.keep = p.stream = policy_neutral();
  }
  return p;
}

__device__ __forceinline__ float ld_f32(const float *p, uint64_t pol) {
  float x;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(x) : "l"(p), "l"(pol));
  return x;
}
__device__ __forceinline__ long long ld_s64(const long long *p, uint64_t pol) {
  long long x;
  asm volatile("ld.global.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(x) : "l"(p), "l"(pol));
  return x;
}
__device__ __forceinline__ uint32_t ld_u8(const uint8_t *p, uint64_t pol) {
  uint32_t x;
  asm volatile("ld.global.L2::cache_hint.u8 %0, [%1], %2;" : "=r"(x) : "l"(p), "l"(pol));
  return x;
}
__device__ __forceinline__ void st_f32(float *p, float x, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(x), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_s64(long long *p, long long x, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.s64 [%0], %1, %2;" ::"l"(p), "l"(x), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_u8(uint8_t *p, uint32_t x, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(p), "r"(x), "l"(pol) : "memory");
}
// Fire-and-forget reductions (REDG) with a cache policy.
__device__ __forceinline__ void red_add_f32(float *p, float x, uint64_t pol) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f32 [%0], %1, %2;"
               ::"l"(p), "f"(x), "l"(pol) : "memory");
}
__device__ __forceinline__ void red_add_u64(unsigned long long *p, unsigned long long x,
                                            uint64_t pol) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;"
               ::"l"(p), "l"(x), "l"(pol) : "memory");
}

}  // namespace bp
