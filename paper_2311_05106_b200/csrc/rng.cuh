// rng.cuh -- counter-based randomness of the JIT connectivity (DESIGN.md
// rules J2, J3, J5, J7), written for sm_100a.
//
// Philox4x32-10: 10 rounds of two 32x32->64 multiplies (IMAD.WIDE.U32 /
// IMAD.HI) and xors with a Weyl-sequence key schedule.  A JIT row is a pure
// function of (seed, row, segment, draw index), so any lane can regenerate
// any edge with no connectivity memory (App. C).
#pragma once
#include <cstdint>

namespace bp {

struct u32x4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ u32x4 philox4x32_10(uint32_t c0, uint32_t c1,
                                               uint32_t c2, uint32_t c3,
                                               uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const uint32_t lo0 = 0xD2511F53u * c0;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

// Block of 4 words j = 4*blk .. 4*blk+3 of stream (tag, row, seg):
// counter = (blk, row, seg, tag), key = (lo32(seed), hi32(seed)).
__device__ __forceinline__ u32x4 philox_block(uint64_t seed, uint32_t tag,
                                              uint32_t row, uint32_t seg,
                                              uint32_t blk) {
  return philox4x32_10(blk, row, seg, tag, static_cast<uint32_t>(seed),
                       static_cast<uint32_t>(seed >> 32));
}

__device__ __forceinline__ uint32_t word_of(const u32x4 &b, uint32_t k) {
  return k == 0 ? b.x : (k == 1 ? b.y : (k == 2 ? b.z : b.w));
}

// Rule J3: lo + floor(x * (hi - lo + 1) / 2^32).
__device__ __forceinline__ uint32_t bounded(uint32_t lo, uint32_t span,
                                            uint32_t x) {
  return lo + __umulhi(x, span);
}
// span == 2^32 cannot occur: K < 2^31.

enum : uint32_t { kTagGap = 0, kTagWeight = 1, kTagFirst = 2 };

// Rule J5: stationary first offset a in [0, K) of (row, seg):
// a = U[0,K-1](w0), b = U[0,K](w1), b <= a -> a = K-1-a.
__device__ __forceinline__ uint32_t first_offset(uint64_t seed, uint32_t K,
                                                 uint32_t row, uint32_t seg) {
  const u32x4 b = philox_block(seed, kTagFirst, row, seg, 0);
  uint32_t a = bounded(0u, K, b.x);
  const uint32_t c = bounded(0u, K + 1u, b.y);
  if (c <= a) a = K - 1u - a;
  return a;
}

// Rule J7 weights.  uniform: u = (x >> 8) 2^-24, w = fmaf(u, hi - lo, lo).
__device__ __forceinline__ float uniform_weight(uint32_t x, float lo,
                                                float span) {
  const float u = __uint2float_rn(x >> 8) * 0x1p-24f;
  return __fmaf_rn(u, span, lo);
}

// Rule J10 (geometric-gap sampler; NEXT 4): op-for-op specified fp32
// natural log on (0, 1] -- the oracle runs the same operations, so both
// sides draw identical gaps.  u = m 2^e; m in [sqrt(1/2), sqrt 2];
// log m = 2 atanh(s), s = (m-1)/(m+1), as 2s + 2s z r(z), z = s^2.
__device__ __forceinline__ float logf_j10(float u) {
  const uint32_t b = __float_as_uint(u);
  int e = static_cast<int>(b >> 23) - 127;
  float m = __uint_as_float((b & 0x7FFFFFu) | 0x3F800000u);
  if (m > 1.41421353816986083984375f) {
    m = __fmul_rn(m, 0.5f);
    e += 1;
  }
  const float f = __fsub_rn(m, 1.0f);
  const float s = __fdiv_rn(f, __fadd_rn(2.0f, f));
  const float z = __fmul_rn(s, s);
  float r = __fmaf_rn(z, 1.0f / 11.0f, 1.0f / 9.0f);
  r = __fmaf_rn(z, r, 1.0f / 7.0f);
  r = __fmaf_rn(z, r, 1.0f / 5.0f);
  r = __fmaf_rn(z, r, 1.0f / 3.0f);
  const float zr = __fmul_rn(z, r);
  const float s2 = __fadd_rn(s, s);
  const float lm = __fmaf_rn(s2, zr, s2);
  const float ef = static_cast<float>(e);
  return __fmaf_rn(ef, 0.693145751953125f, __fmaf_rn(ef, 1.428606765330187e-6f, lm));
}

// Rule J10 gap G ~ Geo(p) from one word: u = ((x >> 8) + 1) 2^-24 in (0, 1],
// t = log(u) / c with c = fl32(log1p(-p)) (IEEE division), G = ceil(t)
// clamped to [1, cap], cap = L + 1 (a gap that long leaves the segment).
__device__ __forceinline__ uint32_t geo_gap(uint32_t x, float c, uint32_t cap) {
  const float u = __fmul_rn(__uint2float_rn((x >> 8) + 1u), 0x1p-24f);
  const float t = __fdiv_rn(logf_j10(u), c);
  if (!(t < __uint2float_rn(cap))) return cap;
  const float ct = ceilf(t);
  if (ct < 1.0f) return 1u;
  const uint32_t g = __float2uint_rz(ct);
  return g > cap ? cap : g;
}

// Reading J7n: cos(2 pi u) for u in [0, 1), op-for-op specified in fp32 (the
// oracle runs the same operations): reduce by symmetry to b in [0, 1/4],
// Taylor cos (to theta^10) for b <= 1/8, else sin of 2 pi (1/4 - b) (to
// theta^9), Horner with fmaf.
__device__ __forceinline__ float cos2pi_j7(float u) {
  const float v = __fsub_rn(u, rintf(u));
  float a = fabsf(v);
  float sgn = 1.0f;
  if (a > 0.25f) {
    a = __fsub_rn(0.5f, a);
    sgn = -1.0f;
  }
  float r;
  if (a <= 0.125f) {
    const float t = __fmul_rn(6.28318548202514648438f, a);
    const float t2 = __fmul_rn(t, t);
    float p = __fmaf_rn(t2, -2.7557319e-7f, 2.4801587e-5f);
    p = __fmaf_rn(t2, p, -1.3888889e-3f);
    p = __fmaf_rn(t2, p, 4.1666668e-2f);
    p = __fmaf_rn(t2, p, -0.5f);
    r = __fmaf_rn(t2, p, 1.0f);
  } else {
    const float t = __fmul_rn(6.28318548202514648438f, __fsub_rn(0.25f, a));
    const float t2 = __fmul_rn(t, t);
    float p = __fmaf_rn(t2, 2.7557319e-6f, -1.9841270e-4f);
    p = __fmaf_rn(t2, p, 8.3333338e-3f);
    p = __fmaf_rn(t2, p, -0.16666667f);
    r = __fmaf_rn(__fmul_rn(t, t2), p, t);
  }
  return __fmul_rn(sgn, r);
}

// Rule J7 / reading J7n, normal weights: Box-Muller in fp32, u1 = ((x1 >> 8)
// + 1) 2^-24 in (0,1], u2 = (x2 >> 8) 2^-24, z = sqrt(-2 logf_j10(u1)) *
// cos2pi_j7(u2) (IEEE sqrt), w = fmaf(sigma, z, mu).
__device__ __forceinline__ float normal_weight(uint32_t x1, uint32_t x2, float mu,
                                               float sigma) {
  const float u1 = __fmul_rn(__uint2float_rn((x1 >> 8) + 1u), 0x1p-24f);
  const float u2 = __fmul_rn(__uint2float_rn(x2 >> 8), 0x1p-24f);
  const float radius = __fsqrt_rn(__fmul_rn(-2.0f, logf_j10(u1)));
  return __fmaf_rn(sigma, __fmul_rn(radius, cos2pi_j7(u2)), mu);
}

// Rule F1: q(w) = round-half-even(w * 2^32) as int64.
__device__ __forceinline__ long long quantize(float w) {
  return __double2ll_rn(__dmul_rn(static_cast<double>(w), 4294967296.0));
}

}  // namespace bp
