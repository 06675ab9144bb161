// neuron.cuh -- fused exponential synapse (AlignPost) + COBA + LIF / HH step
// for sm_100a.
//
// One thread per neuron; a warp covers 32 consecutive neurons = one spike
// word, so the new spike bits leave the kernel as one __ballot_sync per warp
// (no separate compaction pass for local spikes) and the active-row list of
// the next step is appended with one atomicAdd per spiking warp.
//
// Numerics (DESIGN.md rules N1, F1, H1): the library is compiled with
// -fmad=false, so the only fused multiply-adds are the explicit __fmaf_rn
// calls the rules write; division is IEEE; no flush-to-zero.
#pragma once
#include <cstdint>

#include "cache.cuh"

namespace bp {

struct NeuronArgs {
  // LIF (rule N1)
  float v_rest, v_reset, v_th, r, i_ext, e_exc, e_inh, alpha_v;
  double alpha_e, alpha_i;      // fixed-point decay factors (fp64)
  float alpha_e32, alpha_i32;   // fp32 decay factors = fl32(alpha)
  int32_t ref_steps;
  // HH (rule H1)
  float c_m, g_l, e_l, g_na, e_na, g_k, e_k, v_t, dt, v_spike;
  // state
  float *v;
  void *g_e, *g_i;
  uint8_t *ref;
  float *m, *h, *nk;
  int64_t n;
  uint32_t *spikes;      // word 0 <-> neurons 0..31 of this range
  uint32_t *raster;      // nullable, same layout
  int32_t *active;       // nullable
  int32_t *count;
  int32_t active_base;
  float keep_frac;       // L2 evict_last fraction for g (0: no hints)
  int32_t frac_bits;     // BP_OUT_FIX32: fractional bits F
  double inv_scale;      // 2^-F
  float inv_scale32;     // 2^-F (exact in fp32)
  long long a_e_q, a_i_q;  // rule F2 decay: llrint(alpha * 2^32)
};

// Rule F2 decay: g' = (g * A + 2^31) >> 32 (round half up).  With
// A = 2^32 + A' (A' = A - 2^32 < 0 fits int32) this is exactly
// g + hi32(g * A' + 2^31): one IMAD.WIDE (s32 x s32) and a 64-bit add.
__device__ __forceinline__ int32_t fix32_decay(int32_t g, long long A) {
  const int32_t a_m = static_cast<int32_t>(A - (1ll << 32));
  const long long p = static_cast<long long>(g) * a_m + (1ll << 31);
  return g + static_cast<int32_t>(p >> 32);
}

// Rule F2 read: fl32(g * 2^-F) = fl32(g) * 2^-F (power-of-two scaling is
// exact for F <= 30), so one I2F + one FMUL instead of fp64.
__device__ __forceinline__ float fix32_read(int32_t g, float inv_scale32) {
  return __fmul_rn(__int2float_rn(g), inv_scale32);
}

template <int KIND>
__device__ __forceinline__ float g_load(const void *g, int64_t i, uint64_t pol,
                                        float inv_scale = 0.f) {
  if (KIND == 1) {
    const long long q = ld_s64(static_cast<const long long *>(g) + i, pol);
    return __double2float_rn(__dmul_rn(__ll2double_rn(q), 0x1p-32));
  }
  if (KIND == 2) return fix32_read(static_cast<const int32_t *>(g)[i], inv_scale);
  return ld_f32(static_cast<const float *>(g) + i, pol);
}

// g' = decay(g): fixed point llrint(g * alpha) in fp64 (rule F1), fp32 g * fl32(alpha).
template <int KIND>
__device__ __forceinline__ void g_decay(void *g, int64_t i, double a64, float a32,
                                        long long a_q, uint64_t pol) {
  if (KIND == 1) {
    long long *q = static_cast<long long *>(g) + i;
    st_s64(q, __double2ll_rn(__dmul_rn(__ll2double_rn(ld_s64(q, pol)), a64)), pol);
  } else if (KIND == 2) {
    int32_t *q = static_cast<int32_t *>(g) + i;
    *q = fix32_decay(*q, a_q);
  } else {
    float *f = static_cast<float *>(g) + i;
    st_f32(f, __fmul_rn(ld_f32(f, pol), a32), pol);
  }
}

// Spike word, raster word and active-list append for the calling warp.
__device__ __forceinline__ void emit_spikes(const NeuronArgs &a, int64_t i,
                                            bool spike) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned ballot = __ballot_sync(0xffffffffu, spike);
  const int64_t word = i >> 5;
  if (lane == 0 && (word << 5) < a.n) {
    a.spikes[word] = ballot;
    if (a.raster) a.raster[word] = ballot;
  }
  if (a.active != nullptr && ballot != 0u) {
    int slot = 0;
    if (lane == 0) slot = atomicAdd(a.count, __popc(ballot));
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (spike)
      a.active[slot + __popc(ballot & ((1u << lane) - 1u))] =
          a.active_base + static_cast<int32_t>(i);
  }
}

template <int KIND>
__global__ void __launch_bounds__(256) k_lif(NeuronArgs a) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const Policies pol = make_policies(a.keep_frac);
  bool spike = false;
  if (i < a.n) {
    const float V = ld_f32(a.v + i, pol.stream);
    const uint32_t ref = ld_u8(a.ref + i, pol.stream);
    // g is read once and written once: load both, then store the decayed values
    float gE, gI;
    long long qE = 0, qI = 0;
    float fE = 0.f, fI = 0.f;
    if (KIND == 1) {
      qE = ld_s64(static_cast<const long long *>(a.g_e) + i, pol.keep);
      qI = ld_s64(static_cast<const long long *>(a.g_i) + i, pol.keep);
      gE = __double2float_rn(__dmul_rn(__ll2double_rn(qE), 0x1p-32));
      gI = __double2float_rn(__dmul_rn(__ll2double_rn(qI), 0x1p-32));
    } else if (KIND == 2) {
      qE = static_cast<const int32_t *>(a.g_e)[i];
      qI = static_cast<const int32_t *>(a.g_i)[i];
      gE = fix32_read(static_cast<int32_t>(qE), a.inv_scale32);
      gI = fix32_read(static_cast<int32_t>(qI), a.inv_scale32);
    } else {
      fE = ld_f32(static_cast<const float *>(a.g_e) + i, pol.keep);
      fI = ld_f32(static_cast<const float *>(a.g_i) + i, pol.keep);
      gE = fE;
      gI = fI;
    }
    const float I = __fmaf_rn(gI, a.e_inh - V, __fmaf_rn(gE, a.e_exc - V, a.i_ext));
    const float Vinf = __fmaf_rn(a.r, I, a.v_rest);
    const float Vc = __fmaf_rn(V - Vinf, a.alpha_v, Vinf);
    if (ref > 0) {
      st_u8(a.ref + i, ref - 1u, pol.stream);      // hold V while refractory
    } else if (Vc > a.v_th) {                      // strict '>'
      st_f32(a.v + i, a.v_reset, pol.stream);
      st_u8(a.ref + i, static_cast<uint32_t>(a.ref_steps), pol.stream);
      spike = true;
    } else {
      st_f32(a.v + i, Vc, pol.stream);
    }
    if (KIND == 1) {
      st_s64(static_cast<long long *>(a.g_e) + i,
             __double2ll_rn(__dmul_rn(__ll2double_rn(qE), a.alpha_e)), pol.keep);
      st_s64(static_cast<long long *>(a.g_i) + i,
             __double2ll_rn(__dmul_rn(__ll2double_rn(qI), a.alpha_i)), pol.keep);
    } else if (KIND == 2) {
      static_cast<int32_t *>(a.g_e)[i] = fix32_decay(static_cast<int32_t>(qE), a.a_e_q);
      static_cast<int32_t *>(a.g_i)[i] = fix32_decay(static_cast<int32_t>(qI), a.a_i_q);
    } else {
      st_f32(static_cast<float *>(a.g_e) + i, __fmul_rn(fE, a.alpha_e32), pol.keep);
      st_f32(static_cast<float *>(a.g_i) + i, __fmul_rn(fI, a.alpha_i32), pol.keep);
    }
  }
  emit_spikes(a, i, spike);
}

// Rule H1-exp: clamp to [-87, 88], k = rint(x log2 e), two-step Cody-Waite
// reduction by ln 2, degree-7 Taylor polynomial (coefficients fl32(1/n!)),
// scale by 2^k through the exponent bits.
__device__ __forceinline__ float hh_exp(float x) {
  if (x > 88.0f) x = 88.0f;
  if (x < -87.0f) x = -87.0f;
  const float k = rintf(__fmul_rn(x, 1.44269502162933349609375f));
  float r = __fmaf_rn(k, -0.693145751953125f, x);
  r = __fmaf_rn(k, -1.428606765330187045e-06f, r);
  float q = 1.0f / 5040.0f;
  q = __fmaf_rn(q, r, 1.0f / 720.0f);
  q = __fmaf_rn(q, r, 1.0f / 120.0f);
  q = __fmaf_rn(q, r, 1.0f / 24.0f);
  q = __fmaf_rn(q, r, 1.0f / 6.0f);
  q = __fmaf_rn(q, r, 0.5f);
  q = __fmaf_rn(q, r, 1.0f);
  q = __fmaf_rn(q, r, 1.0f);
  return __fmul_rn(q, __int_as_float((static_cast<int>(k) + 127) << 23));
}

// u / (e^{u/k} - 1), removable singularity: k - u/2 for |u| < 1e-4.
__device__ __forceinline__ float hh_efrac(float u, float k) {
  if (fabsf(u) < 1e-4f) return __fmaf_rn(-0.5f, u, k);
  return u / (hh_exp(u / k) - 1.0f);
}

template <int KIND>
__global__ void __launch_bounds__(256) k_hh(NeuronArgs a) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const Policies pol = make_policies(a.keep_frac);
  bool spike = false;
  if (i < a.n) {
    const float V = a.v[i], M = a.m[i], H = a.h[i], Nk = a.nk[i];
    const float gE = g_load<KIND>(a.g_e, i, pol.keep, a.inv_scale32);
    const float gI = g_load<KIND>(a.g_i, i, pol.keep, a.inv_scale32);
    const float x = V - a.v_t;
    const float am = 0.32f * hh_efrac(13.0f - x, 4.0f);
    const float bm = 0.28f * hh_efrac(x - 40.0f, 5.0f);
    const float ah = 0.128f * hh_exp((17.0f - x) / 18.0f);
    const float bh = 4.0f / (1.0f + hh_exp((40.0f - x) / 5.0f));
    const float an = 0.032f * hh_efrac(15.0f - x, 5.0f);
    const float bn = 0.5f * hh_exp((10.0f - x) / 40.0f);
    const float sm = am + bm, sh = ah + bh, sn = an + bn;
    const float m_inf = am / sm, h_inf = ah / sh, n_inf = an / sn;
    const float m_new = __fmaf_rn(M - m_inf, hh_exp(-(a.dt * sm)), m_inf);
    const float h_new = __fmaf_rn(H - h_inf, hh_exp(-(a.dt * sh)), h_inf);
    const float n_new = __fmaf_rn(Nk - n_inf, hh_exp(-(a.dt * sn)), n_inf);
    const float gna = a.g_na * (M * M * M) * H;
    const float n2 = Nk * Nk;
    const float gk = a.g_k * (n2 * n2);
    const float G = a.g_l + gna + gk + gE + gI;
    const float num = a.g_l * a.e_l + gna * a.e_na + gk * a.e_k + gE * a.e_exc +
                      gI * a.e_inh + a.i_ext;
    const float Vinf = num / G;
    const float V_new = __fmaf_rn(V - Vinf, hh_exp(-(a.dt * G / a.c_m)), Vinf);
    spike = V_new >= a.v_spike && V < a.v_spike;   // upward crossing
    a.v[i] = V_new;
    a.m[i] = m_new;
    a.h[i] = h_new;
    a.nk[i] = n_new;
    g_decay<KIND>(a.g_e, i, a.alpha_e, a.alpha_e32, a.a_e_q, pol.keep);
    g_decay<KIND>(a.g_i, i, a.alpha_i, a.alpha_i32, a.a_i_q, pol.keep);
  }
  emit_spikes(a, i, spike);
}

}  // namespace bp
