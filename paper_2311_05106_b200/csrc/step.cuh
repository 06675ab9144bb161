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
#include <type_traits>

#include "cache.cuh"
#include "neuron.cuh"
#include "rng.cuh"
#include "scatter.cuh"

namespace bp {

// Programmatic dependent launch (sm_90+): let the next kernel in the stream
// be scheduled while this one drains, and wait for the previous kernel's
// completion + memory flush before touching its outputs.  No-ops when the
// kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#ifndef BP_TILE_SHIFT
#define BP_TILE_SHIFT 12
#endif
constexpr int kTileShift = BP_TILE_SHIFT;
constexpr int kTile = 1 << kTileShift;   // postsynaptic neurons per tile/block
#ifndef BP_STEP_THREADS
#define BP_STEP_THREADS 256
#endif
constexpr int kStepThreads = BP_STEP_THREADS;   // LIF block size (4 neurons per thread per pass)
// Event records carry the WEIGHT CLASS of their projection in the top two
// bits: projections that add the same homogeneous weight into the same
// conductance share a class (one count array in k_step), projections with
// other weights or receptors get their own.  At most kMaxCls classes.
constexpr int kMaxProj = 8;        // projections per network (BP_MAX_PROJ)
constexpr int kMaxCls = 4;         // weight classes
constexpr int kClsShift = 30;
constexpr uint32_t kClsMask = 3u << kClsShift;
constexpr uint32_t kLocMask = (1u << kClsShift) - 1u;   // staged local index < 2^30

// Per-tile bucket counters sit on their own 256-byte line: the 2M
// slot-claiming atomics of a step then spread over all L2 slices instead of
// the handful a dense 12 KB counter array maps to.
constexpr int kCntStride = 64;

struct Buckets {
  int32_t *cnt;      // [n_tiles * kCntStride], counter of tile t at t*kCntStride
  uint32_t *buf;     // [n_tiles][cap]
  int32_t *spill;    // [n_cls][n_local] dense event counts per class on overflow
  int32_t *flag;     // [n_tiles] spill present
};

struct BinTarget {
  Buckets out;
  uint32_t cap;
  uint32_t n_local;
  uint32_t col_begin;
};

__device__ __forceinline__ uint32_t bin_record(uint32_t cls, uint32_t loc) {
  return (cls << kClsShift) | (loc & (kTile - 1));
}

__device__ __forceinline__ void bin_store(const BinTarget &b, uint32_t cls,
                                          uint32_t loc, int slot) {
  const uint32_t tile = loc >> kTileShift;
  if (static_cast<uint32_t>(slot) < b.cap) {
    b.out.buf[static_cast<size_t>(tile) * b.cap + slot] = bin_record(cls, loc);
  } else {
    atomicAdd(b.out.spill + static_cast<size_t>(cls) * b.n_local + loc, 1);
    b.out.flag[tile] = 1;
  }
}

// Append one event (weight class cls, local postsynaptic index loc).
// Dense delivery (b.cap == 0): one atomic on the neuron's count.
__device__ __forceinline__ void bin_event(const BinTarget &b, uint32_t cls,
                                          uint32_t loc) {
  if (b.cap == 0) {
    atomicAdd(b.out.spill + static_cast<size_t>(cls) * b.n_local + loc, 1);
    return;
  }
  const int slot = atomicAdd(b.out.cnt + (loc >> kTileShift) * kCntStride, 1);
  bin_store(b, cls, loc, slot);
}

// One projection of a network (include/bp.h bp_projection), device view.
// The table lives in device memory (a runtime index into the kernel
// parameters would copy them to local memory); a row's projection is
// loaded once per row.
struct NetProj {
  uint32_t pre_begin, pre_end;  // presynaptic rows = global neurons [pre_begin, pre_end)
  int32_t conn;                 // BP_CONN_JIT / BP_CONN_CSR
  uint32_t cls;                 // weight class of its events
  JitSide j;                    // JIT: seed, K, L, local segments
  CsrSide c;                    // CSR: column-sliced rows, indices local
};

// ConnArgs::group_lanes value: one warp per (row, segment) item
constexpr int kWarpPerItem = 64;

struct ConnArgs {
  const NetProj *proj;      // device table [n_proj]
  int n_proj;
  int all_jit;              // every projection is JIT (the warp-batched path)
  uint32_t n_cols;          // all neurons (columns of every projection)
  int group_lanes;          // JIT binning split: 2 or 4 lanes per (row, segment)
                            // item, 32 = a warp per row (its segments in turn),
                            // or kWarpPerItem = a warp per (row, segment) item
  uint32_t n_seg_max;       // JIT: most local segments of any projection
};

__device__ __forceinline__ bool proj_has(const NetProj *P, int64_t r, uint32_t &row) {
  const uint32_t lo = P->pre_begin, hi = P->pre_end;
  row = static_cast<uint32_t>(r) - lo;
  return static_cast<uint32_t>(r) >= lo && static_cast<uint32_t>(r) < hi;
}

__device__ __forceinline__ JitSide load_jit(const NetProj *P) {
  JitSide s;
  s.seed = P->j.seed;
  s.K = P->j.K;
  s.L = P->j.L;
  s.seg_first = P->j.seg_first;
  s.n_seg = P->j.n_seg;
  return s;
}

// Regenerate (JIT) or read (CSR) the local targets of presynaptic neuron r
// (global id) in every projection it belongs to and bin them.  Called by a
// whole warp (warp-uniform r).  Returns the number of events this lane binned.
__device__ __forceinline__ uint32_t deliver_row(const ConnArgs &c, const BinTarget &b,
                                                int64_t r) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t ev = 0;
  for (int p = 0; p < c.n_proj; ++p) {
    const NetProj *P = c.proj + p;
    uint32_t row;
    if (!proj_has(P, r, row)) continue;
    const uint32_t cls = P->cls;
    if (P->conn == 1) {
      const int64_t *indptr = P->c.indptr;
      const int32_t *indices = P->c.indices;
      const int64_t begin = __ldg(indptr + row), end = __ldg(indptr + row + 1);
      for (int64_t j = begin + lane; j < end; j += 32) {
        bin_event(b, cls, static_cast<uint32_t>(__ldg(indices + j)));
        ++ev;
      }
      continue;
    }
    const JitSide s = load_jit(P);
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
          slot[k] = (pos[k] < seg_end && b.cap)
                        ? atomicAdd(b.out.cnt + ((pos[k] - b.col_begin) >> kTileShift) * kCntStride, 1)
                        : 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (pos[k] < seg_end) {
            if (b.cap) bin_store(b, cls, pos[k] - b.col_begin, slot[k]);
            else bin_event(b, cls, pos[k] - b.col_begin);
            ++ev;
          }
        }
        start += total;
        ++chunk;
        if (start < seg_end) g = philox_block(s.seed, kTagGap, row, seg, chunk * 32u + lane);
      }
    }
  }
  return ev;
}

struct StepArgs {
  NeuronArgs nrn;           // params, local state, n = n_local, spikes/raster words
  int model;                // BP_MODEL_LIF / BP_MODEL_HH
  int n_cls;                // weight classes in use (<= NCLS of the kernel)
  float w[kMaxCls];         // class weight (fp32 mode, one class per receptor)
  long long q[kMaxCls];     // class weight quantised: 2^32 (fix64, multi-class fp32) or
                            // 2^F (fix32); 0 for unused classes
  int rec[kMaxCls];         // class receptor: 0 -> g_e, 1 -> g_i
  unsigned long long *saturated;   // rule F2 saturations
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
  int32_t *tile_counter;    // k_step_persist: next tile index of this step
  int32_t *zero_tile_counter;   // the next step's, set to 0
  ConnArgs conn;            // FUSED kernels: deliver this step's spikes into `out`
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

template <>
struct GVec<2> {
  int32_t v[4];
  __device__ __forceinline__ void load(const void *g, int64_t i, uint64_t pol) {
    const int32_t *p = static_cast<const int32_t *>(g) + i;
    asm volatile("ld.global.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "l"(p), "l"(pol));
  }
  __device__ __forceinline__ void store(void *g, int64_t i, uint64_t pol) const {
    int32_t *p = static_cast<int32_t *>(g) + i;
    asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;"
                 ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "l"(pol) : "memory");
  }
};

// Rule F2: g32 += cnt * q with saturation at the int32 range (counted).
__device__ __forceinline__ float g_fold32(int32_t &g, int32_t cnt, long long q,
                                          float inv_scale, uint32_t &sat) {
  // branch-free: cnt * q fits int64; clamp to the int32 range, count clamps
  const long long v = static_cast<long long>(g) + static_cast<long long>(cnt) * q;
  const long long c = v > 2147483647ll ? 2147483647ll : (v < -2147483648ll ? -2147483648ll : v);
  sat += c != v;
  g = static_cast<int32_t>(c);
  return fix32_read(g, inv_scale);
}
__device__ __forceinline__ void g_after32(int32_t &g, long long a_q) { g = fix32_decay(g, a_q); }

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

// Several weight classes into one conductance (AlignPost merging):
// the step's increment is the exact sum S = sum_c cnt_c q_c (int64).
//   fixed point (F1): g += S;  F2: g += S with saturation;
//   fp32 (rule N1-f32): g = fl32(g + fl32(S 2^-32)) -- the exactly rounded
//   sum of the increments (the host requires every w = q 2^-32 exactly).
__device__ __forceinline__ float g_add(long long &g, long long S) {
  g += S;
  return __double2float_rn(__dmul_rn(__ll2double_rn(g), 0x1p-32));
}
__device__ __forceinline__ float g_add32(int32_t &g, long long S, float inv_scale,
                                         uint32_t &sat) {
  const long long v = static_cast<long long>(g) + S;
  const long long c = v > 2147483647ll ? 2147483647ll : (v < -2147483648ll ? -2147483648ll : v);
  sat += c != v;
  g = static_cast<int32_t>(c);
  return fix32_read(g, inv_scale);
}
__device__ __forceinline__ float g_add(float &g, long long S) {
  if (S) g = __fadd_rn(g, __fmul_rn(__ll2float_rn(S), 0x1p-32f));
  return g;
}

// Fold the counts of neuron j (class c at cnt[c * stride + j]) into its two
// conductances, return the values the neuron reads (gEf, gIf) and leave the
// pre-decayed state in ge / gi.  NCLS == 2: class 0 -> g_e, class 1 -> g_i,
// one class per receptor (Listing S3's network); else the general merge.
template <int KIND, int NCLS, typename G>
__device__ __forceinline__ void fold_pair(const StepArgs &a, G &ge, G &gi, const int32_t *cnt,
                                          int stride, int j, uint32_t &sat, float &gEf,
                                          float &gIf) {
  const NeuronArgs &nr = a.nrn;
  if constexpr (NCLS == 2) {
    const int32_t ce = cnt[j], ci = cnt[stride + j];
    if constexpr (KIND == 2) {
      gEf = g_fold32(ge, ce, a.q[0], nr.inv_scale32, sat);
      gIf = g_fold32(gi, ci, a.q[1], nr.inv_scale32, sat);
    } else if constexpr (KIND == 1) {
      gEf = g_fold(ge, ce, a.q[0]);
      gIf = g_fold(gi, ci, a.q[1]);
    } else {
      gEf = g_fold(ge, ce, a.w[0]);
      gIf = g_fold(gi, ci, a.w[1]);
    }
  } else {
    long long se = 0, si = 0;
#pragma unroll
    for (int c = 0; c < NCLS; ++c) {
      const long long t = static_cast<long long>(cnt[c * stride + j]) * a.q[c];
      if (a.rec[c]) si += t;
      else se += t;
    }
    if constexpr (KIND == 2) {
      gEf = g_add32(ge, se, nr.inv_scale32, sat);
      gIf = g_add32(gi, si, nr.inv_scale32, sat);
    } else {
      gEf = g_add(ge, se);
      gIf = g_add(gi, si);
    }
  }
  if constexpr (KIND == 2) {
    g_after32(ge, nr.a_e_q);
    g_after32(gi, nr.a_i_q);
  } else {
    g_after(ge, nr.alpha_e, nr.alpha_e32);
    g_after(gi, nr.alpha_i, nr.alpha_i32);
  }
}

// One LIF neuron (rule N1); returns spike.  SELECT: the three cases as
// selects, no divergence (measured, same box: fp32 k_step 61.8 -> 59.8 us,
// fix32 71.8 -> 69.8 us, fix64 unchanged; tools/lib_ab.sh).
template <bool SELECT = true>
__device__ __forceinline__ bool lif_one(const NeuronArgs &a, float &V, uint32_t &ref,
                                        float gE, float gI) {
  const float I = __fmaf_rn(gI, a.e_inh - V, __fmaf_rn(gE, a.e_exc - V, a.i_ext));
  const float Vinf = __fmaf_rn(a.r, I, a.v_rest);
  const float Vc = __fmaf_rn(V - Vinf, a.alpha_v, Vinf);
  if constexpr (SELECT) {
    // refractory -> hold V, count down; else Vc > V_th -> reset, spike; else V = Vc
    const bool free = ref == 0u;
    const bool spike = free && Vc > a.v_th;
    V = free ? (spike ? a.v_reset : Vc) : V;
    ref = free ? (spike ? static_cast<uint32_t>(a.ref_steps) : 0u) : ref - 1u;
    return spike;
  }
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
// The state of 4 consecutive neurons (one thread, one pass of 1024).
template <int MODEL, int KIND>
struct Pass {
  bool full;            // all 4 neurons exist (else the scalar tail path)
  float4 V;
  uint32_t R;           // LIF refractory counters, 4 x u8
  float4 M, H, N;       // HH gates
  GVec<KIND> ge, gi;
};

template <int MODEL, int KIND>
__device__ __forceinline__ void pass_load(Pass<MODEL, KIND> &p, const NeuronArgs &nr,
                                          int64_t i0, const Policies &pol) {
  p.full = i0 + 4 <= nr.n;
  if (!p.full) return;
  p.ge.load(nr.g_e, i0, pol.keep);
  p.gi.load(nr.g_i, i0, pol.keep);
  p.V = ld4(nr.v + i0, pol.stream);
  if constexpr (MODEL == 0) {
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(p.R) : "l"(nr.ref + i0), "l"(pol.stream));
  } else {
    p.M = ld4(nr.m + i0, pol.stream);
    p.H = ld4(nr.h + i0, pol.stream);
    p.N = ld4(nr.nk + i0, pol.stream);
  }
}

// Update the 4 neurons of pass p (offset j0 in the tile, local index i0);
// returns their spike nibble.
// ZERO: the counts this pass consumed are reset to 0 right after the fold
// (the persistent kernel then needs no zeroing pass and barrier per tile).
template <int MODEL, int KIND, int NCLS, bool ZERO = false>
__device__ __forceinline__ uint32_t pass_update(Pass<MODEL, KIND> &p, const StepArgs &a,
                                                int32_t *cnt, int stride,
                                                int j0, int64_t i0, const Policies &pol,
                                                uint32_t &sat) {
  const NeuronArgs &nr = a.nrn;
  uint32_t nib = 0;
  if (i0 >= nr.n) return 0;
  if (p.full) {
    float gEf[4], gIf[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      fold_pair<KIND, NCLS>(a, p.ge.v[q], p.gi.v[q], cnt, stride, j0 + q, sat, gEf[q], gIf[q]);
    if constexpr (ZERO) {
#pragma unroll
      for (int c = 0; c < NCLS; ++c)
        *reinterpret_cast<int4 *>(cnt + c * stride + j0) = make_int4(0, 0, 0, 0);
    }
    float V[4] = {p.V.x, p.V.y, p.V.z, p.V.w};
    if constexpr (MODEL == 0) {
      uint32_t Rn = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t r = (p.R >> (8 * q)) & 0xFFu;
        if (lif_one(nr, V[q], r, gEf[q], gIf[q])) nib |= 1u << q;
        Rn |= r << (8 * q);
      }
      if (Rn != p.R)
        asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;"
                     ::"l"(nr.ref + i0), "r"(Rn), "l"(pol.stream) : "memory");
    } else {
      float M[4] = {p.M.x, p.M.y, p.M.z, p.M.w}, H[4] = {p.H.x, p.H.y, p.H.z, p.H.w};
      float Nn[4] = {p.N.x, p.N.y, p.N.z, p.N.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (hh_one(nr, V[q], M[q], H[q], Nn[q], gEf[q], gIf[q])) nib |= 1u << q;
      st4(nr.m + i0, M, pol.stream);
      st4(nr.h + i0, H, pol.stream);
      st4(nr.nk + i0, Nn, pol.stream);
    }
    st4(nr.v + i0, V, pol.stream);
    p.ge.store(nr.g_e, i0, pol.keep);
    p.gi.store(nr.g_i, i0, pol.keep);
    return nib;
  }
  // ragged tail of the last tile: scalar path
  for (int q = 0; q < 4 && i0 + q < nr.n; ++q) {
    const int64_t i = i0 + q;
    float gEf, gIf;
    using G = typename std::conditional<KIND == 1, long long,
                                        typename std::conditional<KIND == 2, int32_t, float>::type>::type;
    G *pe = static_cast<G *>(nr.g_e) + i;
    G *pi = static_cast<G *>(nr.g_i) + i;
    G ge = *pe, gi = *pi;
    fold_pair<KIND, NCLS>(a, ge, gi, cnt, stride, j0 + q, sat, gEf, gIf);
    if constexpr (ZERO) {
#pragma unroll
      for (int c = 0; c < NCLS; ++c) cnt[c * stride + j0 + q] = 0;
    }
    *pe = ge;
    *pi = gi;
    float V = nr.v[i];
    if constexpr (MODEL == 0) {
      uint32_t r = nr.ref[i];
      if (lif_one(nr, V, r, gEf, gIf)) nib |= 1u << q;
      nr.ref[i] = static_cast<uint8_t>(r);
    } else {
      float M = nr.m[i], H = nr.h[i], Nk = nr.nk[i];
      if (hh_one(nr, V, M, H, Nk, gEf, gIf)) nib |= 1u << q;
      nr.m[i] = M;
      nr.h[i] = H;
      nr.nk[i] = Nk;
    }
    nr.v[i] = V;
  }
  return nib;
}

// Spike words of one pass (lanes 8w..8w+7 hold the 32 neurons of word w)
// and the active-list append (one atomic per warp with spikes).
__device__ __forceinline__ void pass_emit(const StepArgs &a, uint32_t nib, int64_t base,
                                          int pass_off, uint32_t &my_sp) {
  const NeuronArgs &nr = a.nrn;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t word = nib << (4u * (lane & 7u));
  word |= __shfl_xor_sync(0xffffffffu, word, 1);
  word |= __shfl_xor_sync(0xffffffffu, word, 2);
  word |= __shfl_xor_sync(0xffffffffu, word, 4);
  const int64_t wi = (base + pass_off + warp * 128) / 32 + (lane >> 3);
  if ((lane & 7u) == 0 && wi * 32 < nr.n) {
    nr.spikes[wi] = word;
    if (nr.raster) nr.raster[wi] = word;
  }
  const uint32_t c = __popc(nib);
  my_sp += c;
  const uint32_t warp_sp = __reduce_add_sync(0xffffffffu, c);
  if (warp_sp) {
    uint32_t incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= static_cast<uint32_t>(off)) incl += v;
    }
    int slot = 0;
    if (lane == 0) slot = atomicAdd(a.active_count, static_cast<int>(warp_sp));
    slot = __shfl_sync(0xffffffffu, slot, 0) + static_cast<int>(incl - c);
    const int64_t i0 = base + pass_off + 4 * static_cast<int64_t>(threadIdx.x);
    uint32_t bits = nib;
    while (bits) {
      const int q = __ffs(bits) - 1;
      bits &= bits - 1u;
      a.active[slot++] = nr.active_base + static_cast<int32_t>(i0 + q);
    }
  }
}

// ---------------------------------------------------------------- kernel
// The first two passes' state loads are issued before the bucket-counting
// phase so their DRAM latency overlaps it; passes 2 and 3 are loaded while
// 0 and 1 compute (register double buffering).
// LIF (memory-bound): 256 threads, 4 passes, register double buffering.
// HH (FP32-latency-bound): 512 threads, 2 passes (more warps, 128 registers).
// NCLS count arrays of kTile int32 in dynamic shared memory (2: 32 KB,
// Listing S3's E + I; 4: 64 KB, merged projections with several weights).
template <int MODEL, int KIND, int NCLS>
#ifndef BP_STEP_MINB
#define BP_STEP_MINB (1024 / BP_STEP_THREADS)
#endif
__global__ void __launch_bounds__(MODEL == 0 ? kStepThreads : 512, MODEL == 0 ? BP_STEP_MINB : 1)
k_step(StepArgs a) {
  extern __shared__ __align__(16) int32_t cnt[];   // [NCLS][kTile]
  __shared__ unsigned long long block_sp;
  const int tid = threadIdx.x;
  constexpr int nthreads = MODEL == 0 ? kStepThreads : 512;
  constexpr int passes = kTile / (4 * nthreads);
  constexpr int pstride = 4 * nthreads;   // neurons per pass
  const uint32_t lane = tid & 31u;
  const uint32_t tile = a.reverse ? a.n_tiles - 1u - blockIdx.x : blockIdx.x;
  const int64_t base = static_cast<int64_t>(tile) << kTileShift;
  const NeuronArgs &nr = a.nrn;
  const Policies pol = make_policies(nr.keep_frac);

  pdl_trigger();
  pdl_wait();               // state and buckets of the previous kernels are final
  Pass<MODEL, KIND> pa, pb;
  pass_load(pa, nr, base + 4 * tid, pol);
  pass_load(pb, nr, base + pstride + 4 * tid, pol);

  // 1. count this tile's incoming events per weight class (bucket + rare spill)
  for (int j = tid; j < NCLS * kTile; j += nthreads) cnt[j] = 0;
  if (tid == 0) block_sp = 0;
  __syncthreads();
  const int32_t n_in = min(static_cast<uint32_t>(a.in.cnt[tile * kCntStride]), a.out.cap);
  const uint32_t *buf = a.in.buf + static_cast<size_t>(tile) * a.out.cap;
  for (int k = tid; k < n_in; k += nthreads) {
    const uint32_t e = __ldcs(buf + k);
    atomicAdd(&cnt[(e >> kClsShift) * kTile + (e & (kTile - 1))], 1);
  }
  if (a.in.flag[tile]) {                       // overflow spill (exact, rare)
    for (int j = tid; j < kTile && base + j < nr.n; j += nthreads) {
#pragma unroll
      for (int c = 0; c < NCLS; ++c) {
        int32_t *sp = a.in.spill + static_cast<size_t>(c) * a.out.n_local + base + j;
        atomicAdd(&cnt[c * kTile + j], *sp);
        *sp = 0;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    a.in.cnt[tile * kCntStride] = 0;
    a.in.flag[tile] = 0;
    if (blockIdx.x == 0) *a.zero_count = 0;
  }

  // 2. update the tile: 4 passes of 1024 neurons, 4 consecutive per thread
  uint32_t my_sp = 0, sat = 0;
#pragma unroll
  for (int p = 0; p < passes; ++p) {
    Pass<MODEL, KIND> &cur = (p & 1) ? pb : pa;
    const int off = p * pstride;
    const uint32_t nib = pass_update<MODEL, KIND, NCLS>(cur, a, cnt, kTile, off + 4 * tid,
                                                        base + off + 4 * tid, pol, sat);
    if (p + 2 < passes) pass_load(cur, nr, base + off + 2 * pstride + 4 * tid, pol);
    pass_emit(a, nib, base, off, my_sp);
  }

  // 3. counters
  if (KIND == 2 && sat) atomicAdd(a.saturated, static_cast<unsigned long long>(sat));
  my_sp = __reduce_add_sync(0xffffffffu, my_sp);
  if (lane == 0 && my_sp) atomicAdd(&block_sp, static_cast<unsigned long long>(my_sp));
  __syncthreads();
  if (tid == 0 && block_sp) {
    atomicAdd(a.spikes, block_sp);
    if (a.step_spikes) atomicAdd(a.step_spikes, static_cast<int32_t>(block_sp));
  }
}

constexpr int kPfRecs = 4 * kStepThreads;   // bucket records prefetched per tile

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Persistent variant of k_step (LIF): the grid is the resident capacity
// (4 blocks of 256 threads per SM) and every block takes tiles from a
// per-step counter, so there is no partial last wave, and while it updates
// passes 2 and 3 of its tile it already loads passes 0 and 1 of its NEXT
// tile -- two passes of state in flight at every moment, also across tiles.
// Same per-tile code (count -> fold + update -> emit) as k_step, hence
// bit-identical results.
template <int MODEL, int KIND, int NCLS>
__global__ void __launch_bounds__(kStepThreads, BP_STEP_MINB)
k_step_persist(StepArgs a) {
  extern __shared__ __align__(16) int32_t cnt[];   // [NCLS][kTile]
  __shared__ unsigned long long block_sp;
  __shared__ int32_t next_s;
  __shared__ __align__(16) uint32_t pf_rec[kPfRecs];   // next tile's first records
  __shared__ int32_t pf_n;                             // next tile's bucket count
  const int tid = threadIdx.x;
  constexpr int nthreads = kStepThreads;
  constexpr int passes = kTile / (4 * nthreads);
  static_assert(passes >= 2, "two passes in flight");
  constexpr int pstride = 4 * nthreads;
  const uint32_t lane = tid & 31u;
  const NeuronArgs &nr = a.nrn;
  const Policies pol = make_policies(nr.keep_frac);
  const int n_tiles = static_cast<int>(a.n_tiles);
  auto tile_of = [&](int idx) -> uint32_t {
    return a.reverse ? static_cast<uint32_t>(n_tiles - 1 - idx) : static_cast<uint32_t>(idx);
  };

  pdl_trigger();
  pdl_wait();               // state and buckets of the previous kernels are final
  if (tid == 0) {
    block_sp = 0;
    next_s = atomicAdd(a.tile_counter, 1);
    if (blockIdx.x == 0) {
      *a.zero_count = 0;
      *a.zero_tile_counter = 0;
    }
  }
  // the count arrays are zeroed once; every fold then resets what it read
  for (int j = tid; j < NCLS * kTile; j += nthreads) cnt[j] = 0;
  __syncthreads();
  int idx = next_s;
  uint32_t my_sp = 0, sat = 0;
  Pass<MODEL, KIND> pa, pb;
  // The next tile's bucket count and first kPfRecs records are copied into
  // shared memory (cp.async, no registers) while this tile updates, so the
  // counting phase waits for no L2 round trip (records beyond kPfRecs, rare,
  // are read as before).  Needs 16-byte rows of records: cap % 4 == 0.
  const bool pf_ok = (a.out.cap & 3u) == 0u;
  auto prefetch = [&](uint32_t t) {
    if (pf_ok && 4u * tid + 4u <= a.out.cap)
      cp_async16(&pf_rec[4 * tid], a.in.buf + static_cast<size_t>(t) * a.out.cap + 4 * tid);
    if (tid == 0) cp_async4(&pf_n, a.in.cnt + t * kCntStride);
    cp_async_commit();
  };
  if (idx < n_tiles) {
    const int64_t base0 = static_cast<int64_t>(tile_of(idx)) << kTileShift;
    prefetch(tile_of(idx));
    pass_load(pa, nr, base0 + 4 * tid, pol);
    pass_load(pb, nr, base0 + pstride + 4 * tid, pol);
  }
  while (idx < n_tiles) {
    const uint32_t tile = tile_of(idx);
    const int64_t base = static_cast<int64_t>(tile) << kTileShift;
    cp_async_wait_all();
    __syncthreads();        // the previous tile's counts consumed (and reset); prefetch landed
    const int32_t n_in = min(static_cast<uint32_t>(pf_n), a.out.cap);
    const int32_t n_pf = pf_ok ? min(n_in, kPfRecs) : 0;
    for (int k = tid; k < n_pf; k += nthreads) {
      const uint32_t e = pf_rec[k];
      atomicAdd(&cnt[(e >> kClsShift) * kTile + (e & (kTile - 1))], 1);
    }
    const uint32_t *buf = a.in.buf + static_cast<size_t>(tile) * a.out.cap;
    for (int k = n_pf + tid; k < n_in; k += nthreads) {
      const uint32_t e = __ldcs(buf + k);
      atomicAdd(&cnt[(e >> kClsShift) * kTile + (e & (kTile - 1))], 1);
    }
    if (a.in.flag[tile]) {                     // overflow spill (exact, rare)
      for (int j = tid; j < kTile && base + j < nr.n; j += nthreads) {
#pragma unroll
        for (int c = 0; c < NCLS; ++c) {
          int32_t *sp = a.in.spill + static_cast<size_t>(c) * a.out.n_local + base + j;
          atomicAdd(&cnt[c * kTile + j], *sp);
          *sp = 0;
        }
      }
    }
    if (tid == 0) next_s = atomicAdd(a.tile_counter, 1);
    __syncthreads();        // counts complete; every thread is done with pf_rec / pf_n
    const int nxt = next_s;
    if (tid == 0) {
      a.in.cnt[tile * kCntStride] = 0;
      a.in.flag[tile] = 0;
    }
    if (nxt < n_tiles) prefetch(tile_of(nxt));
    const int64_t nbase = nxt < n_tiles ? static_cast<int64_t>(tile_of(nxt)) << kTileShift : 0;
#pragma unroll
    for (int p = 0; p < passes; ++p) {
      Pass<MODEL, KIND> &cur = (p & 1) ? pb : pa;
      const int off = p * pstride;
      const uint32_t nib = pass_update<MODEL, KIND, NCLS, true>(cur, a, cnt, kTile, off + 4 * tid,
                                                                base + off + 4 * tid, pol, sat);
      if (p + 2 < passes) pass_load(cur, nr, base + off + 2 * pstride + 4 * tid, pol);
      else if (nxt < n_tiles) pass_load(cur, nr, nbase + (p + 2 - passes) * pstride + 4 * tid, pol);
      pass_emit(a, nib, base, off, my_sp);
    }
    idx = nxt;
  }
  if (KIND == 2 && sat) atomicAdd(a.saturated, static_cast<unsigned long long>(sat));
  my_sp = __reduce_add_sync(0xffffffffu, my_sp);
  if (lane == 0 && my_sp) atomicAdd(&block_sp, static_cast<unsigned long long>(my_sp));
  __syncthreads();
  if (tid == 0 && block_sp) {
    atomicAdd(a.spikes, block_sp);
    if (a.step_spikes) atomicAdd(a.step_spikes, static_cast<int32_t>(block_sp));
  }
}

// Dense delivery (small, compute-bound networks -- config 4's 400 k HH
// neurons fill only 98 tiles of 4096): events arrive as per-neuron counts
// (one global atomic each, bin_event with cap 0) and every block updates
// DENSE_NT * 4 neurons in one pass, so the grid covers every SM.  The block
// moves its neurons' counts into shared memory (and clears them) and then
// runs the same pass code as k_step.
constexpr int kDenseThreads = 128;

template <int MODEL, int KIND>
__global__ void __launch_bounds__(kDenseThreads, MODEL == 0 ? 8 : 4)
k_step_dense(StepArgs a) {
  __shared__ __align__(16) int32_t cnt[2 * 4 * kDenseThreads];   // class 0 (E), class 1 (I)
  __shared__ unsigned long long block_sp;
  const int tid = threadIdx.x;
  const uint32_t lane = tid & 31u;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * (4 * kDenseThreads);
  const NeuronArgs &nr = a.nrn;
  const Policies pol = make_policies(nr.keep_frac);
  pdl_trigger();
  pdl_wait();               // counts of the previous binning are final
  Pass<MODEL, KIND> pa;
  pass_load(pa, nr, base + 4 * tid, pol);
  if (tid == 0) {
    block_sp = 0;
    if (blockIdx.x == 0 && a.zero_count) *a.zero_count = 0;
  }
  for (int j = tid; j < 4 * kDenseThreads; j += kDenseThreads) {
    const int64_t i = base + j;
    int32_t ce = 0, ci = 0;
    if (i < nr.n) {
      int32_t *se = a.in.spill + i;
      int32_t *si = a.in.spill + a.out.n_local + i;
      ce = *se;
      ci = *si;
      if (ce) *se = 0;
      if (ci) *si = 0;
    }
    cnt[j] = ce;
    cnt[4 * kDenseThreads + j] = ci;
  }
  __syncthreads();
  uint32_t my_sp = 0, sat = 0;
  const uint32_t nib = pass_update<MODEL, KIND, 2>(pa, a, cnt, 4 * kDenseThreads, 4 * tid,
                                                   base + 4 * tid, pol, sat);
  pass_emit(a, nib, base, 0, my_sp);
  if (KIND == 2 && sat) atomicAdd(a.saturated, static_cast<unsigned long long>(sat));
  my_sp = __reduce_add_sync(0xffffffffu, my_sp);
  if (lane == 0 && my_sp) atomicAdd(&block_sp, static_cast<unsigned long long>(my_sp));
  __syncthreads();
  if (tid == 0 && block_sp) {
    atomicAdd(a.spikes, block_sp);
    if (a.step_spikes) atomicAdd(a.step_spikes, static_cast<int32_t>(block_sp));
  }
}

// HH with dense delivery: few neurons per thread.  The HH update is a long
// dependent fp32 chain (~490 instructions per neuron); at 400 k neurons four
// neurons per thread leave ~21 warps per SM and the per-warp chain sets the
// time, so here a thread takes kHHPerThread neurons (the same rule H1 code and
// count folding as the 4-wide pass, hence bit-identical results).
constexpr int kHHThreads = 256;

template <int KIND>
__device__ __forceinline__ bool hh_dense_one(const StepArgs &a, int64_t i, uint32_t &sat) {
  const NeuronArgs &nr = a.nrn;
  int32_t *se = a.in.spill + i;
  int32_t *si = a.in.spill + a.out.n_local + i;
  const int32_t ce = *se, ci = *si;
  if (ce) *se = 0;
  if (ci) *si = 0;
  float gEf, gIf;
  using G = typename std::conditional<KIND == 1, long long,
                                      typename std::conditional<KIND == 2, int32_t, float>::type>::type;
  G *pe = static_cast<G *>(nr.g_e) + i;
  G *pi = static_cast<G *>(nr.g_i) + i;
  G ge = *pe, gi = *pi;
  const int32_t cnt2[2] = {ce, ci};
  fold_pair<KIND, 2>(a, ge, gi, cnt2, 1, 0, sat, gEf, gIf);
  *pe = ge;
  *pi = gi;
  float V = nr.v[i], M = nr.m[i], H = nr.h[i], Nk = nr.nk[i];
  const bool spike = hh_one(nr, V, M, H, Nk, gEf, gIf);
  nr.v[i] = V;
  nr.m[i] = M;
  nr.h[i] = H;
  nr.nk[i] = Nk;
  return spike;
}

// kHHPerThread neurons per thread, kHHThreads apart (measured at 400 k
// neurons: 1 -> 14.7 us per step, 2 -> 16.4 us).
constexpr int kHHPerThread = 1;

// FUSED: the kernel also delivers its own spikes (dense delivery: every
// event is a fire-and-forget RED on the next step's per-neuron count, so the
// delivering warp never waits on an atomic) -- the separate binning launch of
// the ~60 spikes per step of config 4 goes away.  The row delivery is an
// out-of-line call so its registers do not burden the HH update.
__device__ __noinline__ uint32_t deliver_row_call(ConnArgs c, BinTarget b, int64_t r) {
  return deliver_row(c, b, r);
}

template <int KIND, bool FUSED = false>
__global__ void __launch_bounds__(kHHThreads, 8) k_hh_dense1(StepArgs a) {
  const NeuronArgs &nr = a.nrn;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kHHThreads * kHHPerThread;
  const uint32_t lane = threadIdx.x & 31u;
  pdl_trigger();
  pdl_wait();               // counts of the previous binning are final
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.zero_count) *a.zero_count = 0;
  bool spike[kHHPerThread];
  uint32_t sat = 0;
#pragma unroll
  for (int k = 0; k < kHHPerThread; ++k) {
    const int64_t i = base + k * kHHThreads + threadIdx.x;
    spike[k] = i < nr.n ? hh_dense_one<KIND>(a, i, sat) : false;
  }
#pragma unroll
  for (int k = 0; k < kHHPerThread; ++k) {
    // spike word of the warp's 32 neurons, active-list append, counters
    const int64_t i = base + k * kHHThreads + threadIdx.x;
    const uint32_t ballot = __ballot_sync(0xffffffffu, spike[k]);
    const int64_t w0 = i - lane;
    if (lane == 0 && w0 < nr.n) {
      nr.spikes[w0 >> 5] = ballot;
      if (nr.raster) nr.raster[w0 >> 5] = ballot;
    }
    if (ballot) {
      const int c = __popc(ballot);
      int slot = 0;
      if (lane == 0) {
        if (!FUSED && a.active) slot = atomicAdd(a.active_count, c);
        atomicAdd(a.spikes, static_cast<unsigned long long>(c));
        if (a.step_spikes) atomicAdd(a.step_spikes, c);
      }
      if constexpr (FUSED) {
        uint32_t m = ballot, ev = 0;
        while (m) {
          const int src = __ffs(m) - 1;
          m &= m - 1u;
          ev += deliver_row_call(a.conn, a.out, nr.active_base + w0 + src);
        }
        ev = __reduce_add_sync(0xffffffffu, ev);
        if (lane == 0 && ev && a.events) atomicAdd(a.events, static_cast<unsigned long long>(ev));
      } else {
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (spike[k] && a.active)
          a.active[slot + __popc(ballot & ((1u << lane) - 1u))] =
              nr.active_base + static_cast<int32_t>(i);
      }
    }
  }
  if (KIND == 2) {
    sat = __reduce_add_sync(0xffffffffu, sat);
    if (lane == 0 && sat) atomicAdd(a.saturated, static_cast<unsigned long long>(sat));
  }
}

// Debug check (BP_DEBUG_NAN=1, the SPEC's NaN abort turned into a counter):
// counts the non-finite membrane potentials after a step.
__global__ void __launch_bounds__(256) k_count_nonfinite(const float *v, int64_t n,
                                                         unsigned long long *counter) {
  uint32_t bad = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad += isfinite(v[i]) ? 0u : 1u;
  bad = __reduce_add_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31u) == 0 && bad) atomicAdd(counter, static_cast<unsigned long long>(bad));
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

// ---------------------------------------------------------------------------
// Block-aggregated binning (one 1024-thread block per SM).  A block's share
// of the active rows is regenerated into shared memory, counting-sorted by
// tile there, and then each non-empty tile costs ONE global slot-claiming
// atomic per block and its records leave as a contiguous run -- ~5x fewer L2
// atomics and sectors than one atomic + one 4-byte store per event.
// Events that do not fit the shared staging area take the per-event path.
constexpr int kBinThreads = 1024;
#ifndef BP_BIN_STAGE
#define BP_BIN_STAGE 16384
#endif
constexpr int kBinStage = BP_BIN_STAGE;   // staged records per block

#ifdef BP_BIN_TIMING
__device__ unsigned long long g_bin_t[1024][6];
#define BP_BIN_MARK(k)                                                       \
  do {                                                                       \
    if (threadIdx.x == 0) {                                                  \
      unsigned long long t_;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                \
      g_bin_t[blockIdx.x][k] = t_;                                           \
    }                                                                        \
  } while (0)
#else
#define BP_BIN_MARK(k) do {} while (0)
#endif

__device__ __forceinline__ uint32_t stage_record(uint32_t cls, uint32_t loc) {
  return (cls << kClsShift) | loc;    // loc < 2^30
}

// Stage up to 4 locs per lane (valid[k]) through one warp-wide slot claim;
// events past the staging area take the per-event path.  Whole warp.
__device__ __forceinline__ uint32_t stage_emit4(const BinTarget &b, uint32_t cls,
                                                const uint32_t *loc, const bool *valid,
                                                uint32_t *staged, int32_t *n_staged,
                                                int32_t *hist) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t mine = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) mine += valid[k];
  uint32_t incl = mine;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= static_cast<uint32_t>(off)) incl += v;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0) return 0;
  int base = 0;
  if (lane == 31) base = atomicAdd(n_staged, static_cast<int>(total));
  base = __shfl_sync(0xffffffffu, base, 31);
  int slot = base + static_cast<int>(incl - mine);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (!valid[k]) continue;
    if (slot < kBinStage) {
      staged[slot] = stage_record(cls, loc[k]);
      atomicAdd(hist + (loc[k] >> kTileShift), 1);
    } else {
      bin_event(b, cls, loc[k]);
    }
    ++slot;
  }
  return mine;
}

// Generate the local targets of row r (global id) in every projection it
// belongs to into the block's staging area (or the global per-event path
// when it is full).  Whole warp, warp-uniform r.  Any mix of CSR and JIT.
__device__ __forceinline__ uint32_t stage_row(const ConnArgs &c, const BinTarget &b, int64_t r,
                                              uint32_t *staged, int32_t *n_staged,
                                              int32_t *hist) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t ev = 0;
  for (int p = 0; p < c.n_proj; ++p) {
    const NetProj *P = c.proj + p;
    uint32_t row;
    if (!proj_has(P, r, row)) continue;
    const uint32_t cls = P->cls;
    if (P->conn == 1) {
      const int64_t *indptr = P->c.indptr;
      const int32_t *indices = P->c.indices;
      const int64_t begin = __ldg(indptr + row), end = __ldg(indptr + row + 1);
      for (int64_t j0 = begin; j0 < end; j0 += 128) {
        uint32_t loc[4];
        bool valid[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t j = j0 + k * 32 + lane;
          valid[k] = j < end;
          loc[k] = valid[k] ? static_cast<uint32_t>(__ldg(indices + j)) : 0u;
        }
        ev += stage_emit4(b, cls, loc, valid, staged, n_staged, hist);
      }
      continue;
    }
    const JitSide s = load_jit(P);
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
        uint32_t loc[4];
        bool valid[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          valid[k] = pos[k] < seg_end;
          loc[k] = pos[k] - b.col_begin;
        }
        ev += stage_emit4(b, cls, loc, valid, staged, n_staged, hist);
        start += total;
        ++chunk;
        if (start < seg_end) g = philox_block(s.seed, kTagGap, row, seg, chunk * 32u + lane);
      }
    }
  }
  return ev;
}

// JIT rows active[k0 + 32 i] (i < 32, k0 + 32 i < k_end) for one warp, every
// projection JIT.  Per projection, the lanes whose row belongs to it first
// compute the stationary first offset of that row (one Philox per lane
// instead of one per row); then the warp walks those rows one by one: one
// Philox block of 4 gaps per lane per chunk of 128 gaps.  Positions grow
// with (lane, k), so the valid events are a prefix of that order and their
// staging slots follow from four ballots -- no second scan.
__device__ __forceinline__ uint32_t stage_rows_jit(const ConnArgs &c, const BinTarget &b,
                                                   const int32_t *active, int k0, int k_end,
                                                   uint32_t *staged, int32_t *n_staged,
                                                   int32_t *hist) {
  const uint32_t lane = threadIdx.x & 31u;
  // rows k0, k0 + 32, k0 + 64, ... (stride = warps per block)
  const int nrows = min(32, (k_end - k0 + 31) / 32);
  const int64_t r_l = lane < static_cast<uint32_t>(nrows) ? active[k0 + 32 * lane] : -1;
  uint32_t ev = 0;
  for (int p = 0; p < c.n_proj; ++p) {
    const NetProj *P = c.proj + p;
    uint32_t row_l;
    const bool mem = r_l >= 0 && proj_has(P, r_l, row_l);
    const uint32_t members = __ballot_sync(0xffffffffu, mem);
    if (!members) continue;
    const JitSide s = load_jit(P);
    const uint32_t pbit = P->cls << kClsShift;
    for (uint32_t sidx = 0; sidx < s.n_seg; ++sidx) {
      const uint32_t seg = s.seg_first + sidx;
      const uint32_t seg_end = min(seg * s.L + s.L, c.n_cols);
      // lane-parallel first offsets of the member rows in this segment
      uint32_t first_l = 0;
      if (mem) first_l = seg * s.L + first_offset(s.seed, s.K, row_l, seg);
      uint32_t todo = members;
      while (todo) {
        const int jl = __ffs(todo) - 1;
        todo &= todo - 1u;
        const uint32_t row = __shfl_sync(0xffffffffu, row_l, jl);
        uint32_t start = __shfl_sync(0xffffffffu, first_l, jl);
        uint32_t chunk = 0;
        while (start < seg_end) {                            // warp-uniform
          const u32x4 g = philox_block(s.seed, kTagGap, row, seg, chunk * 32u + lane);
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
          bool v[4];
          uint32_t n_valid = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            v[k] = pos[k] < seg_end;
            n_valid += __popc(__ballot_sync(0xffffffffu, v[k]));
          }
          int base = 0;
          if (lane == 0) base = atomicAdd(n_staged, static_cast<int>(n_valid));
          base = __shfl_sync(0xffffffffu, base, 0) + static_cast<int>(4 * lane);
          if (base - static_cast<int>(4 * lane) + static_cast<int>(n_valid) <= kBinStage) {
            // common case, warp-uniform: predicated stores + histogram atomics
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (v[k]) {
                const uint32_t loc = pos[k] - b.col_begin;
                staged[base + k] = pbit | loc;
                atomicAdd(hist + (loc >> kTileShift), 1);
              }
            }
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (!v[k]) continue;
              const uint32_t loc = pos[k] - b.col_begin;
              if (base + k < kBinStage) {
                staged[base + k] = pbit | loc;
                atomicAdd(hist + (loc >> kTileShift), 1);
              } else {
                bin_event(b, pbit >> kClsShift, loc);
              }
            }
          }
          ev += static_cast<uint32_t>(v[0]) + v[1] + v[2] + v[3];
          start += total;
          ++chunk;
        }
      }
    }
  }
  return ev;
}

// JIT items (active row k, segment sidx) of every projection the row
// belongs to, S lanes per item (32 / S items per warp at a time) -- for
// networks whose rows have few events per segment (the ~10 of a multi-GPU
// partition or of a strong-scaling segment), where a whole warp per row
// would regenerate 128 gaps for 10 events.  The first 32 / S lanes compute
// the stationary first offsets of the warp's items (one Philox each); lane
// q of an item then draws Philox block `chunk * S + q` (4 gaps) and a scan
// over the S lanes turns the gaps into positions (4 S gaps per step).
// Positions grow with (lane, k) within an item, so an item's valid events
// are a prefix; the staging slots come from one warp-wide scan of the
// per-lane counts and one shared atomic per warp and step.
template <int S>
__device__ __forceinline__ uint32_t stage_items(const ConnArgs &c, const BinTarget &b,
                                                const int32_t *active, int r_lo, int r_hi,
                                                uint32_t n_seg_max, uint32_t *staged,
                                                int32_t *n_staged, int32_t *hist) {
  constexpr int IPW = 32 / S;                 // items per warp
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t sub = lane & (S - 1);
  const uint32_t gi = lane / S;               // item slot of this lane's group
  const int64_t n_items = static_cast<int64_t>(r_hi - r_lo) * n_seg_max;
  const int64_t stride = (kBinThreads / 32) * IPW;
  uint32_t ev = 0;
  for (int64_t base = (threadIdx.x >> 5) * IPW; base < n_items; base += stride) {
    // lane j < IPW decodes item base + j (first offsets); every lane its group's
    const int64_t it_l = base + (lane < IPW ? lane : 0);
    const bool have_l = lane < IPW && it_l < n_items;
    const int64_t r_l = have_l ? active[r_lo + it_l / n_seg_max] : -1;
    const uint32_t sidx_l = have_l ? static_cast<uint32_t>(it_l % n_seg_max) : 0u;
    for (int p = 0; p < c.n_proj; ++p) {
      const NetProj *P = c.proj + p;
      uint32_t row_l = 0;
      const JitSide s = load_jit(P);
      const bool mem_l = have_l && proj_has(P, r_l, row_l) && sidx_l < s.n_seg;
      if (!__ballot_sync(0xffffffffu, mem_l)) continue;
      const uint32_t cbits = P->cls << kClsShift;
      uint32_t first_l = 0;
      if (mem_l) {
        const uint32_t seg = s.seg_first + sidx_l;
        first_l = seg * s.L + first_offset(s.seed, s.K, row_l, seg);
      }
      // this lane's item (group gi)
      const bool mine = __shfl_sync(0xffffffffu, static_cast<int>(mem_l), gi) != 0;
      const uint32_t row = __shfl_sync(0xffffffffu, row_l, gi);
      const uint32_t seg = s.seg_first + __shfl_sync(0xffffffffu, sidx_l, gi);
      const uint32_t first = __shfl_sync(0xffffffffu, first_l, gi);
      const uint32_t seg_end = min(seg * s.L + s.L, c.n_cols);
      uint32_t start = mine ? first : seg_end;
      uint32_t chunk = 0;
      while (__any_sync(0xffffffffu, start < seg_end)) {
        // finished groups compute along (their results are masked off)
        const bool go = start < seg_end;              // uniform within the group
        const u32x4 g = philox_block(s.seed, kTagGap, row, seg, chunk * S + sub);
        const uint32_t g0 = bounded(1u, s.K, g.x), g1 = bounded(1u, s.K, g.y);
        const uint32_t g2 = bounded(1u, s.K, g.z), g3 = bounded(1u, s.K, g.w);
        const uint32_t p1 = g0, p2 = g0 + g1, p3 = p2 + g2, t = p3 + g3;
        uint32_t incl_g = t;
#pragma unroll
        for (int off = 1; off < S; off <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, incl_g, off, S);
          if (sub >= static_cast<uint32_t>(off)) incl_g += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl_g, S - 1, S);
        const uint32_t pos0 = start + (incl_g - t);
        uint32_t pos[4] = {pos0, pos0 + p1, pos0 + p2, pos0 + p3};
        if (!go) pos[0] = pos[1] = pos[2] = pos[3] = seg_end;
        uint32_t nv = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) nv += pos[k] < seg_end;
        // warp-wide exclusive scan of the per-lane counts -> staging slots
        uint32_t incl = nv;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= static_cast<uint32_t>(off)) incl += v;
        }
        const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
        int slot0 = 0;
        if (lane == 31 && wtot) slot0 = atomicAdd(n_staged, static_cast<int>(wtot));
        slot0 = __shfl_sync(0xffffffffu, slot0, 31);
        int slot = slot0 + static_cast<int>(incl - nv);
        if (slot0 + static_cast<int>(wtot) <= kBinStage) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (pos[k] < seg_end) {
              const uint32_t loc = pos[k] - b.col_begin;
              staged[slot++] = cbits | loc;
              atomicAdd(hist + (loc >> kTileShift), 1);
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (pos[k] < seg_end) {
              const uint32_t loc = pos[k] - b.col_begin;
              if (slot < kBinStage) {
                staged[slot] = cbits | loc;
                atomicAdd(hist + (loc >> kTileShift), 1);
              } else {
                bin_event(b, cbits >> kClsShift, loc);
              }
              ++slot;
            }
          }
        }
        ev += nv;
        start += total;
        ++chunk;
      }
    }
  }
  return ev;
}

// Exclusive scan of v[0..n) in place (block-wide, kBinThreads threads);
// returns the total.
__device__ __forceinline__ int32_t block_exclusive_scan(int32_t *v, int n, int32_t *warp_sums) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + kBinThreads - 1) / kBinThreads;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int32_t sum = 0;
  for (int i = lo; i < hi; ++i) sum += v[i];
  int32_t incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int32_t t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int32_t w = warp_sums[lane];
    int32_t wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t t = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += t;
    }
    warp_sums[lane] = wi - w;          // exclusive warp offsets
    if (lane == 31) warp_sums[32] = wi;
  }
  __syncthreads();
  int32_t run = warp_sums[warp] + incl - sum;
  for (int i = lo; i < hi; ++i) {
    const int32_t x = v[i];
    v[i] = run;
    run += x;
  }
  const int32_t total = warp_sums[32];
  __syncthreads();
  return total;
}

// Phase A of the binning for the rows list[r_lo, r_hi): regenerate (JIT) or
// read (CSR) them into the shared staging area + tile histogram.
__device__ __forceinline__ uint32_t stage_list(const ConnArgs &conn, const BinTarget &out,
                                               const int32_t *list, int r_lo, int r_hi,
                                               uint32_t *staged, int32_t *n_staged,
                                               int32_t *hist) {
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t ev = 0;
  if (!conn.all_jit) {
    for (int k = r_lo + static_cast<int>(warp); k < r_hi; k += kBinThreads / 32)
      ev += stage_row(conn, out, list[k], staged, n_staged, hist);
  } else if (conn.group_lanes == 2) {
    // ~10 events per item, one segment per row: 2 lanes per item
    ev = stage_items<2>(conn, out, list, r_lo, r_hi, conn.n_seg_max, staged, n_staged, hist);
  } else if (conn.group_lanes < 32) {
    // few events per (row, segment): 4 lanes per item
    ev = stage_items<4>(conn, out, list, r_lo, r_hi, conn.n_seg_max, staged, n_staged, hist);
  } else if (conn.group_lanes == kWarpPerItem) {
    // long (row, segment) items, few rows: a whole warp per item, so a
    // row's segments run on different warps
    ev = stage_items<32>(conn, out, list, r_lo, r_hi, conn.n_seg_max, staged, n_staged, hist);
  } else {
    // warp w takes rows r_lo + w + 32 i (i = 0, 1, ...), 32 rows per batch
    for (int k0 = r_lo + static_cast<int>(warp); k0 < r_hi; k0 += kBinThreads)
      ev += stage_rows_jit(conn, out, list, k0, r_hi, staged, n_staged, hist);
  }
  return ev;
}

// k_bin_sorted<true>: the rows are the set bits of spike words [w_begin,
// w_end) without [skip_b, skip_e) (a partition's remote words on both sides
// of its own range), bits >= n ignored -- each block lists the rows of its
// contiguous share of those words itself (no compaction launch, no global
// list, no count memset).
struct WordRange {
  const uint32_t *vec;      // spike vector, word w = neurons 32 w .. 32 w + 31
  int64_t w_begin, w_end;
  int64_t skip_b, skip_e;
  int64_t n;
};

// Per-event binning of the set bits of a WordRange (dense delivery, or tile
// tables too large for the block-aggregated kernel): each warp takes `wpw`
// (<= 32) consecutive words of the range per iteration and delivers the rows
// of their set bits one by one -- no compaction launch, no list, no memset.
// (The host picks wpw so that every resident warp gets words: a warp's rows
// are delivered serially.)
__global__ void __launch_bounds__(kScatterThreads)
k_bin_rows_words(ConnArgs conn, BinTarget out, WordRange wr, int wpw,
                 unsigned long long *events) {
  const uint32_t lane = threadIdx.x & 31u;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t sb = min(max(wr.skip_b, wr.w_begin), wr.w_end);
  const int64_t se = min(max(wr.skip_e, sb), wr.w_end);
  const int64_t W1 = sb - wr.w_begin, Wt = W1 + (wr.w_end - se);
  auto word_of = [&](int64_t v) { return v < W1 ? wr.w_begin + v : se + (v - W1); };
  unsigned long long ev = 0;
  for (int64_t v0 = warp0 * wpw; v0 < Wt; v0 += n_warps * wpw) {
    const int64_t v = v0 + lane;
    uint32_t w = 0;
    if (lane < static_cast<uint32_t>(wpw) && v < Wt) {
      const int64_t wi = word_of(v);
      w = wr.vec[wi];
      const int64_t rem = wr.n - wi * 32;
      if (rem < 32) w &= rem > 0 ? (1u << rem) - 1u : 0u;
    }
    uint32_t m = __ballot_sync(0xffffffffu, w != 0u);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1u;
      uint32_t bits = __shfl_sync(0xffffffffu, w, src);
      const int64_t wi = word_of(v0 + src);
      while (bits) {
        const int q = __ffs(bits) - 1;
        bits &= bits - 1u;
        ev += deliver_row(conn, out, wi * 32 + q);
      }
    }
  }
  count_events(events, ev);
}

// Block-wide exclusive scan of one value per thread; *total = the sum.
__device__ __forceinline__ int32_t block_scan1(int32_t c, int32_t *warp_sums, int32_t *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t incl = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int32_t t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int32_t w = warp_sums[lane];
    int32_t wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t t = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += t;
    }
    warp_sums[lane] = wi - w;
    if (lane == 31) warp_sums[32] = wi;
  }
  __syncthreads();
  *total = warp_sums[32];
  return warp_sums[warp] + incl - c;
}

#ifndef BP_WORDS_PT
#define BP_WORDS_PT 4
#endif
constexpr int kWordsPT = BP_WORDS_PT;   // spike words per thread and listing round

template <bool WORDS>
__global__ void __launch_bounds__(kBinThreads, 1)
k_bin_sorted(ConnArgs conn_g, BinTarget out, const int32_t *active, const int32_t *count,
             WordRange wr, unsigned long long *events, uint32_t n_tiles) {
  extern __shared__ uint32_t smem[];
  uint32_t *staged = smem;                                  // [kBinStage]
  uint32_t *sorted = staged + kBinStage;                    // [kBinStage]
  int32_t *hist = reinterpret_cast<int32_t *>(sorted + kBinStage);   // [n_tiles]
  int32_t *gbase = hist + n_tiles;                          // [n_tiles]
  __shared__ int32_t n_staged;
  __shared__ int32_t warp_sums[33];
  __shared__ unsigned long long block_ev;
  __shared__ NetProj proj_s[kMaxProj];
  const int tid = threadIdx.x;
  const uint32_t lane = tid & 31u;
  // the projection table in shared memory: every row's membership test and
  // JIT parameters are then one shared load, not an L1/L2 round trip on the
  // regeneration's dependency chain
  ConnArgs conn = conn_g;
  {
    const uint32_t *src = reinterpret_cast<const uint32_t *>(conn_g.proj);
    uint32_t *dst = reinterpret_cast<uint32_t *>(proj_s);
    constexpr int words = static_cast<int>(sizeof(NetProj) / 4);
    for (int i = tid; i < conn_g.n_proj * words; i += kBinThreads) dst[i] = src[i];
    conn.proj = proj_s;
  }
  pdl_trigger();
  pdl_wait();               // the active list / spike words of the producers are final
  uint32_t ev = 0;
  if constexpr (!WORDS) {
    const int n_active = *count;
    // this block's contiguous share of the active rows
    const int per = (n_active + gridDim.x - 1) / gridDim.x;
    const int r_lo = min(n_active, static_cast<int>(blockIdx.x) * per);
    const int r_hi = min(n_active, r_lo + per);
    BP_BIN_MARK(0);
    if (r_lo >= r_hi) return;
    for (uint32_t t = tid; t < n_tiles; t += kBinThreads) hist[t] = 0;
    if (tid == 0) { n_staged = 0; block_ev = 0; }
    __syncthreads();
    // A. regenerate this block's rows into shared memory + tile histogram
    ev = stage_list(conn, out, active, r_lo, r_hi, staged, &n_staged, hist);
  } else {
    // the remote words as one virtual range [0, W1 + W2)
    const int64_t sb = min(max(wr.skip_b, wr.w_begin), wr.w_end);
    const int64_t se = min(max(wr.skip_e, sb), wr.w_end);
    const int64_t W1 = sb - wr.w_begin, Wt = W1 + (wr.w_end - se);
    const int64_t per = (Wt + gridDim.x - 1) / gridDim.x;
    const int64_t v_lo = min(Wt, static_cast<int64_t>(blockIdx.x) * per);
    const int64_t v_hi = min(Wt, v_lo + per);
    BP_BIN_MARK(0);
    if (v_lo >= v_hi) return;
    for (uint32_t t = tid; t < n_tiles; t += kBinThreads) hist[t] = 0;
    if (tid == 0) { n_staged = 0; block_ev = 0; }
    // A0 + A. list the rows of kWordsPT * 1024 words at a time (all loads in
    //    flight together) into sorted[] (unused until the sort) and stage
    //    them whenever the list is full
    int32_t *list = reinterpret_cast<int32_t *>(sorted);
    int list_n = 0, rows = 0;                     // block-uniform
    auto word_of = [&](int64_t v) { return v < W1 ? wr.w_begin + v : se + (v - W1); };
    for (int64_t v0 = v_lo; v0 < v_hi; v0 += kWordsPT * kBinThreads) {
      uint32_t w[kWordsPT];
      int32_t c = 0;
#pragma unroll
      for (int j = 0; j < kWordsPT; ++j) {
        const int64_t v = v0 + tid + j * kBinThreads;
        w[j] = v < v_hi ? wr.vec[word_of(v)] : 0u;
      }
#pragma unroll
      for (int j = 0; j < kWordsPT; ++j) {
        const int64_t rem = wr.n - word_of(v0 + tid + j * kBinThreads) * 32;
        if (rem < 32) w[j] &= rem > 0 ? (1u << rem) - 1u : 0u;
        c += __popc(w[j]);
      }
      int32_t total;
      const int32_t excl = block_scan1(c, warp_sums, &total);
      rows += total;
      for (int done = 0; done < total;) {         // (several rounds only for bursts)
        const int take = min(kBinStage - list_n, total - done);
        int o = excl;
#pragma unroll
        for (int j = 0; j < kWordsPT; ++j) {
          uint32_t bits = w[j];
          if (!bits) continue;
          const int64_t wi = word_of(v0 + tid + j * kBinThreads);
          while (bits) {
            const int q = __ffs(bits) - 1;
            bits &= bits - 1u;
            if (o >= done && o < done + take)
              list[list_n + o - done] = static_cast<int32_t>(wi * 32 + q);
            ++o;
          }
        }
        list_n += take;
        done += take;
        __syncthreads();
        if (list_n == kBinStage) {
          ev += stage_list(conn, out, list, 0, list_n, staged, &n_staged, hist);
          list_n = 0;
          __syncthreads();
        }
      }
      __syncthreads();                            // warp_sums reused by the next scan
    }
    if (rows == 0) return;
    if (list_n) ev += stage_list(conn, out, list, 0, list_n, staged, &n_staged, hist);
  }
  __syncthreads();
  BP_BIN_MARK(1);
  const int ns = min(n_staged, kBinStage);

  // B. tile offsets; one global slot claim per non-empty tile.  The claims'
  //    results are first needed in D, so (up to kClaimRegs tiles per thread)
  //    they stay in flight across the sort (measured, B200, config 5: binning
  //    B + C 7.1 -> 6.8 us; the ~150 same-address atomics per tile counter
  //    are L2-throughput-bound, so most of their time remains).
  block_exclusive_scan(hist, static_cast<int>(n_tiles), warp_sums);
  BP_BIN_MARK(5);
  constexpr int kClaimRegs = 4;
  if (n_tiles <= kClaimRegs * kBinThreads) {
    int32_t base[kClaimRegs];
#pragma unroll
    for (int u = 0; u < kClaimRegs; ++u) {
      const uint32_t t = tid + u * kBinThreads;
      base[u] = 0;
      if (t < n_tiles) {
        const int32_t begin = hist[t];
        const int32_t end = (t + 1 < n_tiles) ? hist[t + 1] : ns;
        if (end > begin) base[u] = atomicAdd(out.out.cnt + t * kCntStride, end - begin);
      }
    }
    __syncthreads();          // every offset read before the sort moves them
    BP_BIN_MARK(2);
    // C. counting sort by tile (hist[] becomes the running cursor)
    for (int i = tid; i < ns; i += kBinThreads) {
      const uint32_t rec = staged[i];
      const uint32_t t = (rec & kLocMask) >> kTileShift;
      sorted[atomicAdd(hist + t, 1)] = rec;
    }
#pragma unroll
    for (int u = 0; u < kClaimRegs; ++u)
      if (tid + u * kBinThreads < n_tiles) gbase[tid + u * kBinThreads] = base[u];
  } else {
    // a thread's slot claims are independent: issue 4 before using any result
    for (uint32_t t0 = tid; t0 < n_tiles; t0 += 4 * kBinThreads) {
      int32_t base[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t t = t0 + u * kBinThreads;
        base[u] = 0;
        if (t < n_tiles) {
          const int32_t begin = hist[t];
          const int32_t end = (t + 1 < n_tiles) ? hist[t + 1] : ns;
          if (end > begin) base[u] = atomicAdd(out.out.cnt + t * kCntStride, end - begin);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (t0 + u * kBinThreads < n_tiles) gbase[t0 + u * kBinThreads] = base[u];
    }
    __syncthreads();
    BP_BIN_MARK(2);
    // C. counting sort by tile (hist[] becomes the running cursor)
    for (int i = tid; i < ns; i += kBinThreads) {
      const uint32_t rec = staged[i];
      const uint32_t t = (rec & kLocMask) >> kTileShift;
      sorted[atomicAdd(hist + t, 1)] = rec;
    }
  }
  __syncthreads();

  BP_BIN_MARK(3);
  // D. write the runs.  After the sort hist[t] is the END of tile t's run in
  //    sorted[], so the run begins at hist[t-1] (tiles are in order).
  for (int i = tid; i < ns; i += kBinThreads) {
    const uint32_t rec = sorted[i];
    const uint32_t loc = rec & kLocMask;
    const uint32_t t = loc >> kTileShift;
    const int32_t run_begin = (t == 0) ? 0 : hist[t - 1];
    const int32_t slot = gbase[t] + (i - run_begin);
    bin_store(out, rec >> kClsShift, loc, slot);
  }
  // events counter
  ev = __reduce_add_sync(0xffffffffu, ev);
  if (lane == 0 && ev) atomicAdd(&block_ev, static_cast<unsigned long long>(ev));
  __syncthreads();
  BP_BIN_MARK(4);
  if (tid == 0 && block_ev && events) atomicAdd(events, block_ev);
}

}  // namespace bp

namespace bp {

// ---------------------------------------------------------------------------
// Small networks (config 1: 4000 neurons): ONE CTA runs the whole time loop
// with the network state in shared memory.  Per step ~9 neurons spike, i.e.
// ~700 events -- microseconds of work that two kernel launches per step
// would dominate.  Per step: (1) the warps deliver last step's spikes (one
// warp per spiking row, CSR row loads or JIT regeneration) as int32 event
// counts in shared memory; (2) barrier; (3) every thread updates 4 neurons
// (rule N1/H1 with the same helpers as k_step) and appends spikes; (4)
// barrier.  State is loaded once and written back once.
constexpr int kSmallMax = 4096;
constexpr int kSmallThreads = 1024;

struct SmallArgs {
  NeuronArgs nrn;          // global state (n = N <= kSmallMax), spikes, raster
  ConnArgs conn;
  float w_e, w_i;
  long long q_e, q_i;
  int64_t n_steps;
  int32_t *step_counts;    // nullable, device [n_steps]
  int32_t *active_io;      // in: initial active list, out: last step's list
  int32_t *count_io;       // in/out: its length
  unsigned long long *events;
  unsigned long long *spikes;
  unsigned long long *saturated;
};

template <int MODEL, int KIND>
__global__ void __launch_bounds__(kSmallThreads, 1)
k_small_net(SmallArgs a) {
  extern __shared__ unsigned char sm[];
  const NeuronArgs &nr = a.nrn;
  const int n = static_cast<int>(nr.n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  using G = typename std::conditional<KIND == 1, long long,
                                      typename std::conditional<KIND == 2, int32_t, float>::type>::type;
  G *gE = reinterpret_cast<G *>(sm);
  G *gI = gE + kSmallMax;
  float *V = reinterpret_cast<float *>(gI + kSmallMax);
  float *M = V + kSmallMax;                  // HH only
  float *H = M + kSmallMax;
  float *Nk = H + kSmallMax;
  int32_t *cE = reinterpret_cast<int32_t *>(MODEL == 0 ? (V + kSmallMax) : (Nk + kSmallMax));
  int32_t *cI = cE + kSmallMax;
  int32_t *act = cI + kSmallMax;             // active list (spikes of the last step)
  uint8_t *R = reinterpret_cast<uint8_t *>(act + kSmallMax);
  __shared__ int32_t n_act, n_next;
  __shared__ unsigned long long ev_total, sp_total;

  for (int i = tid; i < kSmallMax; i += kSmallThreads) {
    const bool in = i < n;
    gE[i] = in ? static_cast<G *>(nr.g_e)[i] : G(0);
    gI[i] = in ? static_cast<G *>(nr.g_i)[i] : G(0);
    V[i] = in ? nr.v[i] : 0.f;
    if (MODEL == 0) R[i] = in ? nr.ref[i] : 0;
    else { M[i] = in ? nr.m[i] : 0.f; H[i] = in ? nr.h[i] : 0.f; Nk[i] = in ? nr.nk[i] : 0.f; }
    cE[i] = 0;
    cI[i] = 0;
  }
  if (tid == 0) { n_act = *a.count_io; ev_total = 0; sp_total = 0; }
  __syncthreads();
  for (int i = tid; i < n_act; i += kSmallThreads) act[i] = a.active_io[i];
  __syncthreads();

  uint32_t my_ev = 0, my_sp = 0, sat = 0;
  for (int64_t step = 0; step < a.n_steps; ++step) {
    // (1) deliver spikes_{n-1}: count events per postsynaptic neuron
    for (int k = warp; k < n_act; k += kSmallThreads / 32) {
      const int64_t r = act[k];
      for (int pj = 0; pj < a.conn.n_proj; ++pj) {
        const NetProj *P = a.conn.proj + pj;
        uint32_t row;
        if (!proj_has(P, r, row)) continue;
        int32_t *cnt = P->cls ? cI : cE;       // standard layout: class = receptor
        if (P->conn == 1) {
          const int64_t *indptr = P->c.indptr;
          const int32_t *indices = P->c.indices;
          const int64_t b = __ldg(indptr + row), e = __ldg(indptr + row + 1);
          for (int64_t j = b + lane; j < e; j += 32) {
            atomicAdd(cnt + __ldg(indices + j), 1);
            ++my_ev;
          }
          continue;
        }
        const JitSide s = load_jit(P);
        for (uint32_t sidx = 0; sidx < s.n_seg; ++sidx) {
          const uint32_t seg = s.seg_first + sidx;
          const uint32_t seg_end = min(seg * s.L + s.L, a.conn.n_cols);
          u32x4 g = philox_block(s.seed, kTagGap, row, seg, lane);
          uint32_t start = seg * s.L + first_offset(s.seed, s.K, row, seg);
          uint32_t chunk = 0;
          while (start < seg_end) {
            const uint32_t g0 = bounded(1u, s.K, g.x), g1 = bounded(1u, s.K, g.y);
            const uint32_t g2 = bounded(1u, s.K, g.z), g3 = bounded(1u, s.K, g.w);
            const uint32_t p1 = g0, p2 = g0 + g1, p3 = p2 + g2, t = p3 + g3;
            uint32_t incl = t;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
              if (lane >= off) incl += v;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            const uint32_t pos0 = start + (incl - t);
            const uint32_t pos[4] = {pos0, pos0 + p1, pos0 + p2, pos0 + p3};
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (pos[q] < seg_end) { atomicAdd(cnt + pos[q], 1); ++my_ev; }
            start += total;
            ++chunk;
            if (start < seg_end) g = philox_block(s.seed, kTagGap, row, seg, chunk * 32u + lane);
          }
        }
      }
    }
    if (tid == 0) n_next = 0;
    __syncthreads();
    // (3) update, 4 consecutive neurons per thread
    const int j0 = 4 * tid;
    uint32_t nib = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = j0 + q;
      if (i >= n) break;
      float gEf, gIf;
      if constexpr (KIND == 2) {
        gEf = g_fold32(gE[i], cE[i], a.q_e, nr.inv_scale32, sat);
        gIf = g_fold32(gI[i], cI[i], a.q_i, nr.inv_scale32, sat);
      } else if constexpr (KIND == 1) {
        gEf = g_fold(gE[i], cE[i], a.q_e);
        gIf = g_fold(gI[i], cI[i], a.q_i);
      } else {
        gEf = g_fold(gE[i], cE[i], a.w_e);
        gIf = g_fold(gI[i], cI[i], a.w_i);
      }
      cE[i] = 0;
      cI[i] = 0;
      if constexpr (KIND == 2) {
        g_after32(gE[i], nr.a_e_q);
        g_after32(gI[i], nr.a_i_q);
      } else {
        g_after(gE[i], nr.alpha_e, nr.alpha_e32);
        g_after(gI[i], nr.alpha_i, nr.alpha_i32);
      }
      bool sp;
      if constexpr (MODEL == 0) {
        uint32_t r = R[i];
        sp = lif_one(nr, V[i], r, gEf, gIf);
        R[i] = static_cast<uint8_t>(r);
      } else {
        sp = hh_one(nr, V[i], M[i], H[i], Nk[i], gEf, gIf);
      }
      if (sp) nib |= 1u << q;
    }
    uint32_t word = nib << (4u * (lane & 7u));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    word |= __shfl_xor_sync(0xffffffffu, word, 4);
    const int wi = (warp * 128) / 32 + (lane >> 3);
    if ((lane & 7u) == 0 && wi * 32 < n) {
      nr.spikes[wi] = word;
      if (nr.raster) nr.raster[step * ((n + 31) / 32) + wi] = word;
    }
    if (nib) {
      const int c = __popc(nib);
      int slot = atomicAdd(&n_next, c);
      my_sp += c;
      uint32_t bits = nib;
      while (bits) {
        const int q = __ffs(bits) - 1;
        bits &= bits - 1u;
        act[slot++] = j0 + q;
      }
    }
    __syncthreads();
    if (tid == 0) {
      n_act = n_next;
      if (a.step_counts) a.step_counts[step] = n_next;
    }
    __syncthreads();
  }
  // write back state and the final active list
  for (int i = tid; i < n; i += kSmallThreads) {
    static_cast<G *>(nr.g_e)[i] = gE[i];
    static_cast<G *>(nr.g_i)[i] = gI[i];
    nr.v[i] = V[i];
    if (MODEL == 0) nr.ref[i] = R[i];
    else { nr.m[i] = M[i]; nr.h[i] = H[i]; nr.nk[i] = Nk[i]; }
  }
  for (int i = tid; i < n_act; i += kSmallThreads) a.active_io[i] = act[i];
  if (tid == 0) *a.count_io = n_act;
  my_ev = __reduce_add_sync(0xffffffffu, my_ev);
  my_sp = __reduce_add_sync(0xffffffffu, my_sp);
  if (lane == 0) {
    atomicAdd(&ev_total, static_cast<unsigned long long>(my_ev));
    atomicAdd(&sp_total, static_cast<unsigned long long>(my_sp));
  }
  __syncthreads();
  if (tid == 0) {
    atomicAdd(a.events, ev_total);
    atomicAdd(a.spikes, sp_total);
  }
  if (KIND == 2 && sat) atomicAdd(a.saturated, static_cast<unsigned long long>(sat));
}

inline size_t small_net_smem(int model, int kind) {
  const size_t g = kind == 1 ? 8 : 4;   // f32 and FIX32: 4 bytes
  const size_t per = 2 * g + 4 + (model == 1 ? 12 : 0) + 4 + 4 + 4 + (model == 0 ? 1 : 0);
  return per * kSmallMax;
}

}  // namespace bp
