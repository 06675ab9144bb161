// jit_tiled.cuh -- JIT-connectivity event scatter (a3 + a4, Listing S2) with
// shared-memory column tiles instead of one global RED per event.
//
// The stateless bp_jitconn_event_mv_* spends its time in random global REDs
// (~0.11-0.19 T/s on B200, k_jit_scatter).  Regeneration reads no memory, so
// the whole shared memory of an SM can hold accumulators: columns are cut
// into tiles of up to ~57 k f32 / int32 counts (28 k int64), CTA (tile t,
// group g) regenerates its share of the active (row, segment) items, keeps
// the events inside its tile in shared memory (native int32 counts for
// homogeneous weights, two int32 words for fixed point, f32 CAS otherwise),
// and stops each gap chain at the tile's end.  A row segment that spans
// several tiles is regenerated from its start by every tile it reaches, so
// later tiles do more work: they get proportionally more CTAs.  The partial
// tiles are reduced in the same cooperative kernel (tile_reduce).  (Adding
// the non-zero columns of sparse CTAs with atomics instead, to spare small
// calls the 148 dense partials, measured slower at every size.)
#pragma once
#include <cstdint>

#include "csr_stream.cuh"

namespace bp {

constexpr int kJitTiledThreads = 1024;
constexpr int kJitMaxTiles = 16;

struct JitTiledArgs {
  JitSide s;                   // the projection (one per call)
  uint32_t n_cols, col_begin, col_end;
  const int32_t *active;       // event mode: the spiking rows
  const int32_t *count;
  const float *v;              // vector mode (mv_prob_*, reading MV1): every row r, v[r] * w
  int64_t n_rows;
  void *partials;              // [CTA][tile_cols]
  void *out;                   // indexed c - col_begin
  int accumulate;
  int32_t tile_cols, n_tiles;
  int32_t cta0[kJitMaxTiles + 1];   // first CTA of each tile (CTA-major partials)
  unsigned long long *events;       // nullable
  int cta_ok;                       // n_cols + 4096 max_gap < 2^32: CTA-parallel chains allowed
  int row_chunks;                   // expected 128-gap chunks of a row in the partition
};

// VEC: non-event product with a float vector (every row, contribution v[r] w:
// fl32 product in f32 mode, the exact fp64 product rounded once in fixed point)
// C16 (homogeneous only): 16-bit counts, two per 32-bit word, added with a
// native 32-bit ATOMS of 1 << 16 (c & 1) -- exact while a CTA's count of a
// column stays below 2^16 (the host checks: a (row, segment) adds at most
// one event per column).  Twice the columns per tile: 100 k columns fit one
// tile, so no gap chain is regenerated twice.
template <int LAW, int KIND, bool VEC, bool GEO, bool C16 = false>
__global__ void __launch_bounds__(kJitTiledThreads, 1) k_jit_tiled(JitTiledArgs a) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr bool HOMO = LAW == 0 && !VEC;     // count events, scale once
  static_assert(!C16 || HOMO, "16-bit counts for homogeneous weights only");
  constexpr int acc_bytes = C16 ? 2 : ((HOMO || KIND == 0) ? 4 : 8);
  int tile = 0;
  while (tile + 1 < a.n_tiles && static_cast<int>(blockIdx.x) >= a.cta0[tile + 1]) ++tile;
  const int group = blockIdx.x - a.cta0[tile];
  const int groups = a.cta0[tile + 1] - a.cta0[tile];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t W = a.col_end - a.col_begin;
  const uint32_t t0 = static_cast<uint32_t>(tile) * a.tile_cols;
  const uint32_t g0 = a.col_begin + t0;                        // global tile range
  const uint32_t g1 = a.col_begin + min(W, t0 + a.tile_cols);
  const int width = static_cast<int>(g1 - g0);
  const int n_zero32 = ((width + 1) * acc_bytes + 3) / 4;        // tile + sink slot
  for (int c = tid; c < n_zero32; c += kJitTiledThreads) reinterpret_cast<uint32_t *>(sm)[c] = 0u;
  __syncthreads();
  const JitSide &s = a.s;
  auto add = [&](uint32_t pos, float w, float vr) {
    const uint32_t lc = min(pos - g0, static_cast<uint32_t>(width));
    if (C16) atomicAdd(reinterpret_cast<uint32_t *>(sm) + (lc >> 1), 1u << ((lc & 1u) * 16u));
    else if (HOMO) atomicAdd(reinterpret_cast<uint32_t *>(sm) + lc, 1u);
    else if (KIND == 0) atomicAdd(reinterpret_cast<float *>(sm) + lc, VEC ? __fmul_rn(vr, w) : w);
    else {
      unsigned *p = reinterpret_cast<unsigned *>(sm) + 2 * lc;   // int64 as 2 x int32 + carry
      const unsigned long long qq = static_cast<unsigned long long>(
          VEC ? __double2ll_rn(__dmul_rn(static_cast<double>(vr), static_cast<double>(w)) *
                               4294967296.0)
              : quantize(w));
      const unsigned lo = static_cast<unsigned>(qq);
      const unsigned old = atomicAdd(p, lo);
      atomicAdd(p + 1, static_cast<unsigned>(qq >> 32) + (old + lo < old ? 1u : 0u));
    }
  };

  const int64_t n_items = (VEC ? a.n_rows : static_cast<int64_t>(*a.count)) * s.n_seg;
  const int64_t NW = static_cast<int64_t>(groups) * (kJitTiledThreads / 32);
  uint32_t ev = 0;
  // one chunk of 128 gaps of (row, seg): lane holds gaps g (one Philox
  // block), its inclusive warp prefix incl and the chunk start; emits the
  // lane's events inside [g0, stop)
  auto emit = [&](uint32_t row, uint32_t seg, uint32_t blk, uint32_t q0, uint32_t q1,
                  uint32_t q2, uint32_t t, uint32_t incl, uint32_t start, uint32_t stop,
                  float vr) {
    const uint32_t pos0 = start + (incl - t);
    const uint32_t pos[4] = {pos0, pos0 + q0, pos0 + q0 + q1, pos0 + q0 + q1 + q2};
    // this lane's events inside the tile (positions ascend along the chain)
    if (!(pos0 < stop && pos[3] >= g0)) return;
    if constexpr (HOMO) {
      // counts only: branch-free, an event outside [g0, stop) (at most the
      // boundary lane's) is counted into the sink slot `width`, never flushed
      uint32_t nv = 0;
      uint32_t *acc = reinterpret_cast<uint32_t *>(sm);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool ok = pos[k] >= g0 && pos[k] < stop;
        nv += ok;
        const uint32_t lc = ok ? pos[k] - g0 : static_cast<uint32_t>(width);
        if (C16) atomicAdd(acc + (lc >> 1), 1u << ((lc & 1u) * 16u));
        else atomicAdd(acc + lc, 1u);
      }
      ev += nv;
      return;
    }
    float w[4] = {s.w0, s.w0, s.w0, s.w0};
    if (LAW == 1) {
      const u32x4 x = philox_block(s.seed, kTagWeight, row, seg, blk);
      w[0] = uniform_weight(x.x, s.w0, s.w1); w[1] = uniform_weight(x.y, s.w0, s.w1);
      w[2] = uniform_weight(x.z, s.w0, s.w1); w[3] = uniform_weight(x.w, s.w0, s.w1);
    } else if (LAW == 2) {
      const u32x4 x = philox_block(s.seed, kTagWeight, row, seg, 2u * blk);
      if (pos[0] >= g0) w[0] = normal_weight(x.x, x.y, s.w0, s.w1);
      if (pos[1] >= g0 && pos[1] < stop) w[1] = normal_weight(x.z, x.w, s.w0, s.w1);
      if (pos[2] < stop && pos[3] >= g0) {
        const u32x4 y = philox_block(s.seed, kTagWeight, row, seg, 2u * blk + 1u);
        if (pos[2] >= g0) w[2] = normal_weight(y.x, y.y, s.w0, s.w1);
        if (pos[3] < stop) w[3] = normal_weight(y.z, y.w, s.w0, s.w1);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (pos[k] >= g0 && pos[k] < stop) {
        add(pos[k], w[k], vr);
        ++ev;
      }
    }
  };
  auto warp_scan = [&](uint32_t t) {
    uint32_t incl = t;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    return incl;
  };

  // CTA-parallel chains for long rows (>= 32 chunks of 128 gaps) when a
  // CTA's share of items, each ~4 chunk-times per round of 32 chunks
  // (barriers, and every used CTA flushes and reduces a partial tile), beats
  // a warp taking a whole row (measured on the config-2 cells: 100 rows of
  // 5,000 events 53 -> 31 us; 1,000 such rows are faster per warp)
  const int64_t ipc = (n_items + groups - 1) / groups;
  const int rounds = (a.row_chunks + 31) / 32;
  const bool cta_mode = a.cta_ok && a.row_chunks >= 32 &&
                        4 * ipc * rounds <= static_cast<int64_t>(a.row_chunks);
  if (cta_mode) {
    // few items (long rows, low density): the chain of one item is
    // regenerated by the whole CTA, 32 chunks per round -- warp w takes
    // chunk 32 r + w, the chunk starts follow from a block prefix of the 32
    // chunk totals (Philox blocks do not depend on the running position)
    __shared__ uint32_t chunk_tot[32];
    for (int64_t item = group; item < n_items; item += groups) {   // block-uniform
      const uint32_t row = static_cast<uint32_t>(VEC ? item / s.n_seg : a.active[item / s.n_seg]);
      float vr = 1.f;
      if (VEC) {
        vr = __ldg(a.v + row);
        if (vr == 0.f) continue;
      }
      const uint32_t seg = s.seg_first + static_cast<uint32_t>(item % s.n_seg);
      const uint32_t seg_begin = seg * s.L;
      const uint32_t seg_end = min(seg_begin + s.L, a.n_cols);
      const uint32_t stop = min(seg_end, g1);
      if (seg_begin >= g1 || seg_end <= g0) continue;
      uint32_t round_start = seg_begin + jit_first<GEO>(s, row, seg);
      for (uint32_t r = 0; round_start < stop; ++r) {              // block-uniform
        const uint32_t chunk = 32u * r + static_cast<uint32_t>(warp);
        const u32x4 g = philox_block(s.seed, kTagGap, row, seg, chunk * 32u + lane);
        const uint32_t q0 = jit_gap<GEO>(s, g.x), q1 = jit_gap<GEO>(s, g.y);
        const uint32_t q2 = jit_gap<GEO>(s, g.z), q3 = jit_gap<GEO>(s, g.w);
        const uint32_t t = q0 + q1 + q2 + q3;
        const uint32_t incl = warp_scan(t);
        if (lane == 31) chunk_tot[warp] = incl;
        __syncthreads();
        uint32_t before = 0, round_total = 0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const uint32_t v = chunk_tot[k];
          before += k < warp ? v : 0u;
          round_total += v;
        }
        emit(row, seg, chunk * 32u + lane, q0, q1, q2, t, incl, round_start + before, stop, vr);
        round_start += round_total;
        __syncthreads();                                           // chunk_tot reused
      }
    }
  } else {
    for (int64_t item = static_cast<int64_t>(group) * (kJitTiledThreads / 32) + warp;
         item < n_items; item += NW) {
      const uint32_t row = static_cast<uint32_t>(VEC ? item / s.n_seg : a.active[item / s.n_seg]);
      float vr = 1.f;
      if (VEC) {
        vr = __ldg(a.v + row);
        if (vr == 0.f) continue;                                  // contributes nothing
      }
      const uint32_t seg = s.seg_first + static_cast<uint32_t>(item % s.n_seg);
      const uint32_t seg_begin = seg * s.L;
      const uint32_t seg_end = min(seg_begin + s.L, a.n_cols);
      const uint32_t stop = min(seg_end, g1);
      if (seg_begin >= g1 || seg_end <= g0) continue;             // warp-uniform
      u32x4 g = philox_block(s.seed, kTagGap, row, seg, lane);
      uint32_t start = seg_begin + jit_first<GEO>(s, row, seg);
      uint32_t chunk = 0;
      while (start < stop) {                                      // warp-uniform
        const uint32_t q0 = jit_gap<GEO>(s, g.x), q1 = jit_gap<GEO>(s, g.y);
        const uint32_t q2 = jit_gap<GEO>(s, g.z), q3 = jit_gap<GEO>(s, g.w);
        const uint32_t t = q0 + q1 + q2 + q3;
        const uint32_t incl = warp_scan(t);
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        emit(row, seg, chunk * 32u + lane, q0, q1, q2, t, incl, start, stop, vr);
        start += total;
        ++chunk;
        if (start < stop) g = philox_block(s.seed, kTagGap, row, seg, chunk * 32u + lane);
      }
    }
  }
  __syncthreads();
  // items are dealt 32 per CTA in order: only the first `used` CTAs of the
  // tile got any, and only their partials are written and reduced
  const int64_t cta_items = cta_mode ? n_items : (n_items + 31) / 32;
  const int used = cta_items < groups ? static_cast<int>(cta_items) : groups;
  if (group < used) {
    char *dst = static_cast<char *>(a.partials) +
                static_cast<size_t>(blockIdx.x) * a.tile_cols * acc_bytes;
    const int n16 = width * acc_bytes / 16;
    for (int k = tid; k < n16; k += kJitTiledThreads)
      reinterpret_cast<uint4 *>(dst)[k] = reinterpret_cast<const uint4 *>(sm)[k];
    for (int b = n16 * 16 + tid; b < width * acc_bytes; b += kJitTiledThreads) dst[b] = sm[b];
  }
  if (a.events) {
    ev = __reduce_add_sync(0xffffffffu, ev);
    if (lane == 0 && ev) atomicAdd(a.events, static_cast<unsigned long long>(ev));
  }
  __threadfence();
  cg::this_grid().sync();
  tile_reduce<KIND, HOMO, kJitTiledThreads, C16>(a.partials, static_cast<size_t>(a.cta0[tile]),
                                                 group, groups, used, a.tile_cols, width, t0,
                                                 a.out, a.accumulate, s.w0, s.q);
}

}  // namespace bp
