// step.cuh -- the network step on one device, two launches per timestep:
//   k_step     : fold the binned events of spikes_{n-1} into g, update
//                Expon + COBA + LIF/HH, emit spikes_n as bits and as an
//                active-row list;
//   k_bin_rows : regenerate (JIT) or read (CSR) the rows of spikes_n and
//                bin their synaptic events for step n+1 (a2-a4).
//
// Why binning: the events of a step land on random postsynaptic neurons
// (fan-out 80 over millions of columns).  Adding them straight into g costs
// one random 32-byte DRAM read-modify-write per event (the g arrays do not
// fit in L2 next to the streamed state).  Instead every event is appended,
// as a 4-byte (projection, offset) record, to the bucket of its
// 4096-neuron postsynaptic tile (bucket appends stay L2-resident: ~8 MB per
// step at the 12.5M-neuron config).  The next step's block for that tile
// counts its bucket into shared memory (native int32 ATOMS) and folds the
// counts into g while streaming the tile's state exactly once:
//   fixed point: g += count * q(w)  -- equal to summing q(w) count times;
//   fp32       : g += (float)count * w  (one rounding; rule T3 parity).
// Homogeneous projection weights (Listing S3's EventJitFPHomoLinear) are
// what make a count sufficient.
//
// Bucket overflow (a tile receiving more than `cap` events in one step) is
// handled exactly: the surplus goes to a dense per-neuron spill counter and
// the tile is flagged; the consumer adds and clears it.
//
// Tiles are visited in alternating (snake) order on even/odd steps so the
// state the previous step touched last -- still in L2 -- is touched first.
#pragma once
#include <cstdint>

#include "cache.cuh"
#include "neuron.cuh"
#include "rng.cuh"
#include "scatter.cuh"

namespace bp {

constexpr int kTileShift = 12;
constexpr int kTile = 1 << kTileShift;   // postsynaptic neurons per tile/block
constexpr int kStepThreads = 256;        // 16 neurons per thread
constexpr uint32_t kProjBit = 0x80000000u;

// Per-tile bucket counters sit on their own 256-byte line: the 2M
// slot-claiming atomics of a step then spread over all L2 slices instead of
// the handful a dense 12 KB counter array maps to.
constexpr int kCntStride = 64;

struct Buckets {
  int32_t *cnt;      // [n_tiles * kCntStride], counter of tile t at t*kCntStride
  uint32_t *buf;     // [n_tiles][cap]
  int32_t *spill;    // [2][n_local] dense event counts (E, I) on overflow
  int32_t *flag;     // [n_tiles] spill present
};

struct BinTarget {
  Buckets out;
  uint32_t cap;
  uint32_t n_local;
  uint32_t col_begin;
};

__device__ __forceinline__ uint32_t bin_record(uint32_t proj, uint32_t loc) {
  return (proj ? kProjBit : 0u) | (loc & (kTile - 1));
}

__device__ __forceinline__ void bin_store(const BinTarget &b, uint32_t proj,
                                          uint32_t loc, int slot) {
  const uint32_t tile = loc >> kTileShift;
  if (static_cast<uint32_t>(slot) < b.cap) {
    b.out.buf[static_cast<size_t>(tile) * b.cap + slot] = bin_record(proj, loc);
  } else {
    atomicAdd(b.out.spill + static_cast<size_t>(proj) * b.n_local + loc, 1);
    b.out.flag[tile] = 1;
  }
}

// Append one event (projection proj, local postsynaptic index loc).
__device__ __forceinline__ void bin_event(const BinTarget &b, uint32_t proj,
                                          uint32_t loc) {
  const int slot = atomicAdd(b.out.cnt + (loc >> kTileShift) * kCntStride, 1);
  bin_store(b, proj, loc, slot);
}

struct ConnArgs {
  int conn;                 // BP_CONN_JIT / BP_CONN_CSR (uniform per launch)
  JitSide je, ji;           // JIT: seed, K, L, local segments
  CsrSide ce, ci;           // CSR: column-sliced rows, indices local
  int64_t split;            // n_exc: rows >= split belong to projection I
  uint32_t n_cols;          // all neurons (columns of both projections)
};

// Regenerate (JIT) or read (CSR) the local targets of presynaptic neuron r
// (global id) and bin them.  Called by a whole warp (warp-uniform r).
// Returns the number of events this lane binned.
__device__ __forceinline__ uint32_t deliver_row(const ConnArgs &c, const BinTarget &b,
                                                int64_t r) {
  const uint32_t lane = threadIdx.x & 31u;
  const bool inh = r >= c.split;
  const uint32_t proj = inh ? 1u : 0u;
  const int64_t row64 = inh ? r - c.split : r;
  uint32_t ev = 0;
  if (c.conn == 1) {
    const CsrSide s = pick(inh, c.ce, c.ci);
    const int64_t begin = __ldg(s.indptr + row64), end = __ldg(s.indptr + row64 + 1);
    for (int64_t j = begin + lane; j < end; j += 32) {
      bin_event(b, proj, static_cast<uint32_t>(__ldg(s.indices + j)));
      ++ev;
    }
    return ev;
  }
  const JitSide s = pick(inh, c.je, c.ji);
  const uint32_t row = static_cast<uint32_t>(row64);
  for (uint32_t sidx = 0; sidx < s.n_seg; ++sidx) {
    const uint32_t seg = s.seg_first + sidx;
    const uint32_t seg_begin = seg * s.L;
    const uint32_t seg_end = min(seg_begin + s.L, c.n_cols);
    u32x4 g = philox_block(s.seed, kTagGap, row, seg, lane);
    uint32_t start = seg_begin + first_offset(s.seed, s.K, row, seg);
    uint32_t chunk = 0;
    while (start < seg_end) {                      // warp-uniform
      const uint32_t g0 = bounded(1u, s.K, g.x), g1 = bounded(1u, s.K, g.y);
      const uint32_t g2 = bounded(1u, s.K, g.z), g3 = bounded(1u, s.K, g.w);
      const uint32_t p1 = g0, p2 = g0 + g1, p3 = p2 + g2, t = p3 + g3;
      uint32_t incl = t;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= static_cast<uint32_t>(off)) incl += v;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t pos0 = start + (incl - t);
      const uint32_t pos[4] = {pos0, pos0 + p1, pos0 + p2, pos0 + p3};
      // claim all slots first so the four atomics are in flight together
      int slot[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        slot[k] = pos[k] < seg_end
                      ? atomicAdd(b.out.cnt + ((pos[k] - b.col_begin) >> kTileShift) * kCntStride, 1)
                      : 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (pos[k] < seg_end) {
          bin_store(b, proj, pos[k] - b.col_begin, slot[k]);
          ++ev;
        }
      }
      start += total;
      ++chunk;
      if (start < seg_end) g = philox_block(s.seed, kTagGap, row, seg, chunk * 32u + lane);
    }
  }
  return ev;
}

struct StepArgs {
  NeuronArgs nrn;           // params, local state, n = n_local, spikes/raster words
  int model;                // BP_MODEL_LIF / BP_MODEL_HH
  ConnArgs conn;
  float w_e, w_i;           // homogeneous weights (fp32 mode)
  long long q_e, q_i;       // quantised weights (fixed point)
  Buckets in;               // events for this step (consumed, then cleared)
  BinTarget out;            // events for the next step
  uint32_t n_tiles;
  int reverse;              // snake order
  unsigned long long *events;
  unsigned long long *spikes;
  int32_t *step_spikes;     // nullable: += spikes of this step
  int32_t *active;          // spikes_n as global ids, appended at *active_count
  int32_t *active_count;
  int32_t *zero_count;      // set to 0 (the other ping-pong list counter)
};

// ---------------------------------------------------------------- helpers
template <int KIND>
struct GVec;  // 4 consecutive conductances of one kind
template <>
struct GVec<0> {
  float v[4];
  __device__ __forceinline__ void load(const void *g, int64_t i, uint64_t pol) {
    const float *p = static_cast<const float *>(g) + i;
    float4 x;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "l"(p), "l"(pol));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
  __device__ __forceinline__ void store(void *g, int64_t i, uint64_t pol) const {
    float *p = static_cast<float *>(g) + i;
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "l"(pol) : "memory");
  }
};
template <>
struct GVec<1> {
  long long v[4];
  __device__ __forceinline__ void load(const void *g, int64_t i, uint64_t pol) {
    const long long *p = static_cast<const long long *>(g) + i;
    asm volatile("ld.global.L2::cache_hint.v2.s64 {%0,%1}, [%2], %3;"
                 : "=l"(v[0]), "=l"(v[1]) : "l"(p), "l"(pol));
    asm volatile("ld.global.L2::cache_hint.v2.s64 {%0,%1}, [%2], %3;"
                 : "=l"(v[2]), "=l"(v[3]) : "l"(p + 2), "l"(pol));
  }
  __device__ __forceinline__ void store(void *g, int64_t i, uint64_t pol) const {
    long long *p = static_cast<long long *>(g) + i;
    asm volatile("st.global.L2::cache_hint.v2.s64 [%0], {%1,%2}, %3;"
                 ::"l"(p), "l"(v[0]), "l"(v[1]), "l"(pol) : "memory");
    asm volatile("st.global.L2::cache_hint.v2.s64 [%0], {%1,%2}, %3;"
                 ::"l"(p + 2), "l"(v[2]), "l"(v[3]), "l"(pol) : "memory");
  }
};

// g_n = (pre-decayed g) + increments of this step; returns the fp32 value
// the neuron update reads, leaves the state value in `g` (rule F1 / fp32).
__device__ __forceinline__ float g_fold(long long &g, int32_t cnt, long long q) {
  g += static_cast<long long>(cnt) * q;
  return __double2float_rn(__dmul_rn(__ll2double_rn(g), 0x1p-32));
}
__device__ __forceinline__ float g_fold(float &g, int32_t cnt, float w) {
  if (cnt) g = __fadd_rn(g, __fmul_rn(__int2float_rn(cnt), w));
  return g;
}
__device__ __forceinline__ void g_after(long long &g, double a64, float) {
  g = __double2ll_rn(__dmul_rn(__ll2double_rn(g), a64));
}
__device__ __forceinline__ void g_after(float &g, double, float a32) {
  g = __fmul_rn(g, a32);
}

// One LIF neuron (rule N1); returns spike.
__device__ __forceinline__ bool lif_one(const NeuronArgs &a, float &V, uint32_t &ref,
                                        float gE, float gI) {
  const float I = __fmaf_rn(gI, a.e_inh - V, __fmaf_rn(gE, a.e_exc - V, a.i_ext));
  const float Vinf = __fmaf_rn(a.r, I, a.v_rest);
  const float Vc = __fmaf_rn(V - Vinf, a.alpha_v, Vinf);
  if (ref > 0) {
    ref -= 1u;
    return false;
  }
  if (Vc > a.v_th) {
    V = a.v_reset;
    ref = static_cast<uint32_t>(a.ref_steps);
    return true;
  }
  V = Vc;
  return false;
}

// One HH neuron (rule H1, same op order as k_hh); returns spike.
__device__ __forceinline__ bool hh_one(const NeuronArgs &a, float &V, float &M, float &H,
                                       float &Nk, float gE, float gI) {
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
  const bool spike = V_new >= a.v_spike && V < a.v_spike;
  V = V_new; M = m_new; H = h_new; Nk = n_new;
  return spike;
}

__device__ __forceinline__ float4 ld4(const float *p, uint64_t pol) {
  float4 x;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "l"(p), "l"(pol));
  return x;
}
__device__ __forceinline__ void st4(float *p, const float *v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
               ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "l"(pol) : "memory");
}

// ---------------------------------------------------------------- kernel
template <int MODEL, int KIND>
__global__ void __launch_bounds__(kStepThreads)
k_step(StepArgs a) {
  __shared__ int32_t cnt_e[kTile];
  __shared__ int32_t cnt_i[kTile];
  __shared__ unsigned long long block_sp;
  const int tid = threadIdx.x;
  const uint32_t lane = tid & 31u, warp = tid >> 5;
  const uint32_t tile = a.reverse ? a.n_tiles - 1u - blockIdx.x : blockIdx.x;
  const int64_t base = static_cast<int64_t>(tile) << kTileShift;
  const NeuronArgs &nr = a.nrn;
  const Policies pol = make_policies(nr.keep_frac);

  // 1. count this tile's incoming events (bucket + rare spill)
  for (int j = tid; j < kTile; j += kStepThreads) { cnt_e[j] = 0; cnt_i[j] = 0; }
  if (tid == 0) block_sp = 0;
  __syncthreads();
  const int32_t n_in = min(static_cast<uint32_t>(a.in.cnt[tile * kCntStride]), a.out.cap);
  const uint32_t *buf = a.in.buf + static_cast<size_t>(tile) * a.out.cap;
  for (int k = tid; k < n_in; k += kStepThreads) {
    const uint32_t e = __ldcs(buf + k);
    atomicAdd((e & kProjBit) ? &cnt_i[e & (kTile - 1)] : &cnt_e[e & (kTile - 1)], 1);
  }
  if (a.in.flag[tile]) {                       // overflow spill (exact, rare)
    for (int j = tid; j < kTile && base + j < nr.n; j += kStepThreads) {
      int32_t *se = a.in.spill + base + j;
      int32_t *si = a.in.spill + a.out.n_local + base + j;
      atomicAdd(&cnt_e[j], *se);
      atomicAdd(&cnt_i[j], *si);
      *se = 0;
      *si = 0;
    }
  }
  __syncthreads();
  if (tid == 0) {
    a.in.cnt[tile * kCntStride] = 0;
    a.in.flag[tile] = 0;
    if (blockIdx.x == 0) *a.zero_count = 0;
  }

  // 2. update the tile: 4 passes of 1024 neurons, 4 consecutive per thread
  uint32_t my_sp = 0;
  for (int pass = 0; pass < kTile / 1024; ++pass) {
    const int j0 = pass * 1024 + 4 * tid;               // offset in tile
    const int64_t i0 = base + j0;                        // local neuron
    uint32_t nib = 0;
    if (i0 < nr.n) {
      if (i0 + 4 <= nr.n) {
        GVec<KIND> ge, gi;
        ge.load(nr.g_e, i0, pol.keep);
        gi.load(nr.g_i, i0, pol.keep);
        float gEf[4], gIf[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if constexpr (KIND == 1) {
            gEf[q] = g_fold(reinterpret_cast<long long &>(ge.v[q]), cnt_e[j0 + q], a.q_e);
            gIf[q] = g_fold(reinterpret_cast<long long &>(gi.v[q]), cnt_i[j0 + q], a.q_i);
          } else {
            gEf[q] = g_fold(reinterpret_cast<float &>(ge.v[q]), cnt_e[j0 + q], a.w_e);
            gIf[q] = g_fold(reinterpret_cast<float &>(gi.v[q]), cnt_i[j0 + q], a.w_i);
          }
          g_after(ge.v[q], nr.alpha_e, nr.alpha_e32);
          g_after(gi.v[q], nr.alpha_i, nr.alpha_i32);
        }
        const float4 V4 = ld4(nr.v + i0, pol.stream);
        float V[4] = {V4.x, V4.y, V4.z, V4.w};
        if constexpr (MODEL == 0) {
          uint32_t R4;
          asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;"
                       : "=r"(R4) : "l"(nr.ref + i0), "l"(pol.stream));
          uint32_t Rn = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t r = (R4 >> (8 * q)) & 0xFFu;
            if (lif_one(nr, V[q], r, gEf[q], gIf[q])) nib |= 1u << q;
            Rn |= r << (8 * q);
          }
          if (Rn != R4)
            asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;"
                         ::"l"(nr.ref + i0), "r"(Rn), "l"(pol.stream) : "memory");
        } else {
          const float4 M4 = ld4(nr.m + i0, pol.stream), H4 = ld4(nr.h + i0, pol.stream);
          const float4 N4 = ld4(nr.nk + i0, pol.stream);
          float M[4] = {M4.x, M4.y, M4.z, M4.w}, H[4] = {H4.x, H4.y, H4.z, H4.w};
          float Nn[4] = {N4.x, N4.y, N4.z, N4.w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (hh_one(nr, V[q], M[q], H[q], Nn[q], gEf[q], gIf[q])) nib |= 1u << q;
          st4(nr.m + i0, M, pol.stream);
          st4(nr.h + i0, H, pol.stream);
          st4(nr.nk + i0, Nn, pol.stream);
        }
        st4(nr.v + i0, V, pol.stream);
        ge.store(nr.g_e, i0, pol.keep);
        gi.store(nr.g_i, i0, pol.keep);
      } else {
        // ragged tail of the last tile: scalar path
        for (int q = 0; q < 4 && i0 + q < nr.n; ++q) {
          const int64_t i = i0 + q;
          float gEf, gIf;
          if constexpr (KIND == 1) {
            long long *pe = static_cast<long long *>(nr.g_e) + i;
            long long *pi = static_cast<long long *>(nr.g_i) + i;
            long long ge = *pe, gi = *pi;
            gEf = g_fold(ge, cnt_e[j0 + q], a.q_e);
            gIf = g_fold(gi, cnt_i[j0 + q], a.q_i);
            g_after(ge, nr.alpha_e, 0.f); g_after(gi, nr.alpha_i, 0.f);
            *pe = ge; *pi = gi;
          } else {
            float *pe = static_cast<float *>(nr.g_e) + i;
            float *pi = static_cast<float *>(nr.g_i) + i;
            float ge = *pe, gi = *pi;
            gEf = g_fold(ge, cnt_e[j0 + q], a.w_e);
            gIf = g_fold(gi, cnt_i[j0 + q], a.w_i);
            g_after(ge, 0.0, nr.alpha_e32); g_after(gi, 0.0, nr.alpha_i32);
            *pe = ge; *pi = gi;
          }
          float V = nr.v[i];
          if constexpr (MODEL == 0) {
            uint32_t r = nr.ref[i];
            if (lif_one(nr, V, r, gEf, gIf)) nib |= 1u << q;
            nr.ref[i] = static_cast<uint8_t>(r);
          } else {
            float M = nr.m[i], H = nr.h[i], Nk = nr.nk[i];
            if (hh_one(nr, V, M, H, Nk, gEf, gIf)) nib |= 1u << q;
            nr.m[i] = M; nr.h[i] = H; nr.nk[i] = Nk;
          }
          nr.v[i] = V;
        }
      }
    }
    // 3. spike words: lanes 8w..8w+7 of this warp hold the 32 neurons of word w
    uint32_t word = nib << (4u * (lane & 7u));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    word |= __shfl_xor_sync(0xffffffffu, word, 4);
    const int64_t wi = (base + pass * 1024 + warp * 128) / 32 + (lane >> 3);
    if ((lane & 7u) == 0 && wi * 32 < nr.n) {
      nr.spikes[wi] = word;
      if (nr.raster) nr.raster[wi] = word;
    }
    my_sp += __popc(nib);
    // 4. append the new spikes to the active list (one atomic per warp);
    //    k_bin_rows regenerates their rows and bins the events
    const uint32_t warp_sp = __reduce_add_sync(0xffffffffu, __popc(nib));
    if (warp_sp) {
      uint32_t incl = __popc(nib);
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= static_cast<uint32_t>(off)) incl += v;
      }
      int slot = 0;
      if (lane == 0) slot = atomicAdd(a.active_count, static_cast<int>(warp_sp));
      slot = __shfl_sync(0xffffffffu, slot, 0) + static_cast<int>(incl - __popc(nib));
      uint32_t bits = nib;
      while (bits) {
        const int q = __ffs(bits) - 1;
        bits &= bits - 1u;
        a.active[slot++] = nr.active_base + static_cast<int32_t>(i0 + q);
      }
    }
  }
  // 5. counters
  my_sp = __reduce_add_sync(0xffffffffu, my_sp);
  if (lane == 0 && my_sp) atomicAdd(&block_sp, static_cast<unsigned long long>(my_sp));
  __syncthreads();
  if (tid == 0) {
    if (block_sp) {
      atomicAdd(a.spikes, block_sp);
      if (a.step_spikes) atomicAdd(a.step_spikes, static_cast<int32_t>(block_sp));
    }
  }
}

// Remote (or initial) spikes: bin the events of every active row in
// `active[0..*count)` whose targets fall in this partition.
__global__ void __launch_bounds__(kScatterThreads)
k_bin_rows(ConnArgs conn, BinTarget out, const int32_t *active, const int32_t *count,
           unsigned long long *events) {
  const int n_active = *count;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  unsigned long long ev = 0;
  for (int64_t k = warp0; k < n_active; k += n_warps) ev += deliver_row(conn, out, active[k]);
  count_events(events, ev);
}

}  // namespace bp
