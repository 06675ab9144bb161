// csr_stream.cuh -- CSR event scatter (a2, Listing S1) with the row data
// streamed into shared memory by the bulk-copy (TMA) engine.
//
// Why: the register-staged tiled kernel (scatter.cuh, k_csr_tiled) reaches
// only ~2.9 TB/s on the config-2 cells (ncu: long-scoreboard stalls, 64
// registers per thread leave ~2 KB per warp in flight, and every warp pays a
// dependent 32-way search per row).  Here
//  * k_csr_split finds, once per active row, where the row crosses each
//    column-tile boundary (warp-wide 128-entry window at the interpolated
//    position: one dependent load for uniformly spread columns, a 32-way
//    search otherwise) -> split[row][t-1] (per call for the active rows, or
//    once for all rows by bp_csrmv_plan when the matrix is reused);
//  * k_csr_stream: CTA (tile t, group g) owns column tile t in shared memory;
//    each of its 32 warps streams its own active rows' in-tile index (and
//    weight) ranges through a private ring of buffers filled by
//    cp.async.bulk (mbarrier complete_tx), so ~96 KB per SM are in flight
//    without registers, and turns them into shared-memory atomics.  Only 32-bit integer shared atomics are native on
//    sm_100a (f32 and 64-bit adds compile to CAS loops): homogeneous weights
//    count events (POPC.INC), fixed-point weights add int64 as two 32-bit
//    words with a carry, fp32 weights use the CAS add.  The tile is stored
//    as a partial and k_csr_reduce (scatter.cuh) sums the groups in order --
//    no global atomics.
// Indices must ascend within each row (canonical CSR, include/bp.h); entries
// outside the tile are skipped, so unsorted input cannot corrupt memory.
#pragma once
#include <cstdint>

#include <cooperative_groups.h>

#include "scatter.cuh"

namespace bp {
namespace cg = cooperative_groups;

// ----------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in hardware instead
// of spinning, so it does not take issue slots from the producer warp
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT;\n}" ::"r"(smem_u32(b)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, size % 16 == 0), completion
// counted on the mbarrier's transaction count
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

// --------------------------------------------------------------- split
struct CsrSplitArgs {
  const int64_t *indptr;
  const int32_t *indices;
  const int32_t *active;   // nullptr: every row (the plan of bp_csrmv_plan)
  const int32_t *count;    // nullptr: n_rows rows
  int64_t n_rows;
  int32_t *split;          // [row][n_tiles - 1]: first entry with column >= t*tile_cols, - indptr[row]
  int32_t n_tiles, tile_cols;
  int64_t n_cols;
};

// One warp per row r (active[k], or k itself): split[r][t-1] = (first entry
// of row r with column >= t * tile_cols) - indptr[r], t = 1 .. n_tiles-1.
// The boundaries are searched 4 at a time, 8 lanes each: a 128-entry window
// (4 int4 loads per lane, all in flight) at the interpolated position --
// columns of a random row are spread evenly -- so a row costs 3 dependent
// loads (active, indptr, windows); a boundary outside its window falls back
// to the warp-wide search.
__global__ void __launch_bounds__(256) k_csr_split(CsrSplitArgs a) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
  const int nt = a.n_tiles;
  const int64_t n_items = a.count ? *a.count : a.n_rows;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
       k < n_items; k += nw) {
    const int64_t r = a.active ? a.active[k] : k;
    const int64_t lo = __ldg(a.indptr + r), hi = __ldg(a.indptr + r + 1);
    int32_t *b = a.split + r * (nt - 1) - 1;      // b[t], t = 1 .. nt-1
    for (int t0 = 1; t0 < nt; t0 += 4) {
      const int t = t0 + grp;
      const bool mine = t < nt;
      const int32_t x = mine ? t * a.tile_cols : 0;
      int64_t r0 = lo, r1 = lo;          // counted region of the window
      int n_lt = 0;
      if (mine && hi > lo) {
        const int64_t g = lo + static_cast<int64_t>(static_cast<double>(hi - lo) * x /
                                                    static_cast<double>(a.n_cols));
        int64_t w0 = g - 64;
        w0 = w0 > hi - 128 ? hi - 128 : w0;
        w0 = (w0 < lo ? lo : w0) & ~int64_t{3};        // 16-byte aligned window start
        r0 = w0 > lo ? w0 : lo;
        r1 = w0 + 128 < hi ? w0 + 128 : hi;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int64_t j = w0 + 16 * gl + 4 * v;
          int32_t e4[4];
          if (j >= r0 && j + 4 <= r1) {
            const int4 q = __ldg(reinterpret_cast<const int4 *>(a.indices + j));
            e4[0] = q.x; e4[1] = q.y; e4[2] = q.z; e4[3] = q.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              e4[e] = (j + e >= r0 && j + e < r1) ? __ldg(a.indices + j + e) : INT32_MAX;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) n_lt += e4[e] < x ? 1 : 0;
        }
      }
#pragma unroll
      for (int o = 4; o >= 1; o >>= 1) n_lt += __shfl_xor_sync(0xffffffffu, n_lt, o);
      // the window decides unless every counted entry is < x with more row
      // beyond it, or none is < x with row before it
      const bool below = mine && hi > lo && n_lt == 0 && r0 > lo;
      const bool above = mine && hi > lo && r0 + n_lt == r1 && r1 < hi;
      if (mine && gl == 0 && !below && !above)
        b[t] = static_cast<int32_t>((hi > lo ? r0 + n_lt : lo) - lo);
      const int64_t w0 = r0, w1 = r1;
      unsigned fb = __ballot_sync(0xffffffffu, (below || above) && gl == 0);
      while (fb) {                                  // rare: warp-wide search
        const int src = __ffs(fb) - 1;
        fb &= fb - 1;
        const int ts = t0 + (src >> 3);
        const bool bl = __shfl_sync(0xffffffffu, below, src);
        const int64_t sw0 = __shfl_sync(0xffffffffu, w0, src);
        const int64_t sw1 = __shfl_sync(0xffffffffu, w1, src);
        const int32_t xs = ts * a.tile_cols;
        const int64_t j = bl ? warp_lower_bound(a.indices, lo, sw0, xs)
                             : warp_lower_bound(a.indices, sw1, hi, xs);
        if (lane == 0) b[ts] = static_cast<int32_t>(j - lo);
      }
    }
  }
}

// --------------------------------------------------------------- stream
// Every warp streams its own rows: a private ring of NB buffers of BE
// entries, filled by cp.async.bulk issued from lane 0 (one mbarrier per
// buffer, transaction-counted), so up to NB-1 chunks per warp are in flight
// while the warp turns the current one into shared-memory atomics.  There is
// no cross-warp synchronisation inside the loop (a single producer warp per
// CTA could not keep up: one row costs ~100 issue slots).
#ifndef BP_STREAM_BUFS
#define BP_STREAM_BUFS 2
#endif
#ifndef BP_STREAM_BUF_BYTES
#define BP_STREAM_BUF_BYTES 2048
#endif
#ifndef BP_STREAM_THREADS
#define BP_STREAM_THREADS 1024
#endif
constexpr int kStreamThreads = BP_STREAM_THREADS;
// static shared memory of k_csr_stream
constexpr size_t kStreamStaticSmem = 0;
constexpr int kStreamWarps = kStreamThreads / 32;
constexpr int kStreamBufs = BP_STREAM_BUFS;
// entries per buffer: BP_STREAM_BUF_BYTES of indices (+ as many of weights)
__host__ __device__ constexpr int stream_buf_ent(bool homo) {
  return homo ? BP_STREAM_BUF_BYTES / 4 : BP_STREAM_BUF_BYTES / 8;
}

#ifndef BP_STREAM_SEGS
#define BP_STREAM_SEGS 8
#endif
constexpr int kStreamSegs = BP_STREAM_SEGS;   // row pieces per buffer

struct StreamChunk {   // one row piece in a buffer
  int32_t dst;     // first buffer slot of the piece (multiple of 4)
  int32_t len;     // slots of the piece (multiple of 4)
  int32_t v0, v1;  // valid entries [v0, v1) relative to a0
  int32_t gl;      // entries >= gl were not copied (end of the array): read from global
  int32_t pad;
  int64_t a0;      // global index of slot dst (16-byte aligned)
};
struct StreamBuf {
  int32_t nseg, fill, pad[2];
  StreamChunk seg[kStreamSegs];
};

struct CsrStreamArgs {
  const int32_t *indices;
  const float *data;         // nullptr -> homogeneous: count events per column
  const int64_t *indptr;
  const int32_t *split;      // [row][n_tiles - 1] (k_csr_split / bp_csrmv_plan)
  const int32_t *active;
  const int32_t *count;
  const int64_t *nnz;        // &indptr[n_rows]
  void *partials;            // [tile][group][tile_cols]
  int32_t tile_cols, groups, n_tiles, accumulate;
  int64_t n_cols;
  void *out;                 // fused reduction (cooperative launch)
  float w;                   // homogeneous weight
  long long q;               // quantize(w)
  int32_t fix_bits;          // KIND 2 (rule T4): weights accumulated at 2^-fix_bits
  int32_t absw;              // accumulate |w| (bp_csrmv_plan's column bound)
  int64_t n_rows_all;        // active == nullptr: every row 0 .. n_rows_all - 1
};

// Shared-memory layout (host and device agree through this function).
struct StreamSmem {
  size_t idx, dat, meta, bar, total;
};
__host__ __device__ inline StreamSmem stream_smem(int tile_cols, int acc_bytes, bool homo) {
  auto up = [](size_t x) { return (x + 127) & ~size_t{127}; };
  const size_t ring = static_cast<size_t>(kStreamWarps) * kStreamBufs * stream_buf_ent(homo) * 4;
  StreamSmem s{};
  s.idx = up(static_cast<size_t>(tile_cols + 4) * acc_bytes);   // + sink slot
  s.dat = s.idx + ring;
  s.meta = s.dat + (homo ? 0 : ring);
  s.bar = up(s.meta + static_cast<size_t>(kStreamWarps) * kStreamBufs * sizeof(StreamBuf));
  s.total = s.bar + static_cast<size_t>(kStreamWarps) * kStreamBufs * 8;
  return s;
}

#ifdef BP_CSR_TIMING
__device__ unsigned long long g_csr_t[1024][8];
#define CSR_MARK(k)                                                            \
  do {                                                                         \
    if (threadIdx.x == 0) {                                                    \
      unsigned long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
      g_csr_t[blockIdx.x][k] = t_;                                             \
    }                                                                          \
  } while (0)
#else
#define CSR_MARK(k) do {} while (0)
#endif

// Sum a tile's partials (CTA-major: partial of CTA b of the tile at
// (first + b) * tile_cols) over its `groups` CTAs in ascending order; CTA
// `group` handles column slice `group` and writes out[c0 + column]
// (accumulate: +=).  Homogeneous partials are event counts: fl32(n * w) or
// n * q.  Deterministic for counts and fixed point.
// C16: homogeneous partials are 16-bit counts (k_jit_tiled's packed tiles).
// Only the first `used` CTAs of a tile received work (rows / items are
// dealt kStreamWarps per CTA in order), so only their partials are summed -- a call
// with few active rows does not read 148 empty partial tiles.
template <int KIND, bool HOMO, int NT, bool C16 = false>
__device__ __forceinline__ void tile_reduce(const void *partials, size_t first, int group,
                                            int groups, int used, int tile_cols, int width,
                                            int64_t c0, void *out, int accumulate, float w,
                                            long long q, int fix_bits = 0) {
  const int per = (width + groups - 1) / groups;
  const int s0 = group * per, s1 = min(width, s0 + per);
  const size_t stride = static_cast<size_t>(tile_cols);
  const size_t base = first * stride;
  for (int cc = s0 + static_cast<int>(threadIdx.x); cc < s1; cc += NT) {
    const int64_t c = c0 + cc;
    if (HOMO) {
      unsigned long long n = 0;
      if (C16) {
        const unsigned short *p = static_cast<const unsigned short *>(partials) + base + cc;
        for (int g = 0; g < used; ++g) n += __ldcg(p + g * stride);
      } else {
        const unsigned *p = static_cast<const unsigned *>(partials) + base + cc;
        for (int g = 0; g < used; ++g) n += __ldcg(p + g * stride);
      }
      if (KIND == 0) {
        const float v = __fmul_rn(__ull2float_rn(n), w);
        float *o = static_cast<float *>(out) + c;
        *o = accumulate ? __fadd_rn(*o, v) : v;
      } else {
        const long long v = static_cast<long long>(n) * q;
        long long *o = static_cast<long long *>(out) + c;
        *o = accumulate ? *o + v : v;
      }
    } else if (KIND == 0) {
      const float *p = static_cast<const float *>(partials) + base + cc;
      float v = 0.f;
      for (int g = 0; g < used; ++g) v = __fadd_rn(v, __ldcg(p + g * stride));
      float *o = static_cast<float *>(out) + c;
      *o = accumulate ? __fadd_rn(*o, v) : v;
    } else if (KIND == 2) {
      const int2 *p = static_cast<const int2 *>(partials) + base + cc;
      long long hi = 0;
      unsigned long long lo = 0;
      for (int g = 0; g < used; ++g) {
        const int2 x = __ldcg(p + g * stride);
        hi += x.x;
        lo += static_cast<unsigned>(x.y);
      }
      const float v = fix2_value(hi, lo, fix_bits);
      float *o = static_cast<float *>(out) + c;
      *o = accumulate ? __fadd_rn(*o, v) : v;
    } else {
      const long long *p = static_cast<const long long *>(partials) + base + cc;
      long long v = 0;
      for (int g = 0; g < used; ++g) v += __ldcg(p + g * stride);
      long long *o = static_cast<long long *>(out) + c;
      *o = accumulate ? *o + v : v;
    }
  }
}

// KIND: 0 f32 partials, 1 int64 fixed-point partials; HOMO: uint32 counts,
// or (C16) 16-bit counts packed two per word -- exact while a CTA streams
// fewer than 2^16 rows (the host's check; canonical rows hold a column at
// most once), and half the shared memory per column, so fewer column tiles.
template <int KIND, bool HOMO, bool C16 = false>
__global__ void __launch_bounds__(kStreamThreads, 1) k_csr_stream(CsrStreamArgs a) {
  extern __shared__ __align__(128) unsigned char sm[];
  static_assert(!C16 || HOMO, "16-bit counts for homogeneous weights only");
  constexpr int acc_bytes = C16 ? 2 : ((HOMO || KIND == 0) ? 4 : 8);
  constexpr int BE = stream_buf_ent(HOMO);
  constexpr int NB = kStreamBufs;
  const StreamSmem L = stream_smem(a.tile_cols, acc_bytes, HOMO);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int32_t *bidx = reinterpret_cast<int32_t *>(sm + L.idx) + warp * NB * BE;
  float *bdat = reinterpret_cast<float *>(sm + L.dat) + warp * NB * BE;
  StreamBuf *meta = reinterpret_cast<StreamBuf *>(sm + L.meta) + warp * NB;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + L.bar) + warp * NB;

  const int tile = blockIdx.x / a.groups, group = blockIdx.x % a.groups;
  const int64_t c0 = static_cast<int64_t>(tile) * a.tile_cols;
  const int64_t c1 = min(c0 + a.tile_cols, a.n_cols);
  const int width = static_cast<int>(c1 - c0);
  const int32_t c0i = static_cast<int32_t>(c0);
  const float fix_scale = __int_as_float((127 + (KIND == 2 ? a.fix_bits : 0)) << 23);  // 2^fix_bits
  CSR_MARK(0);

  const int n_zero32 = ((width + 1) * acc_bytes + 3) / 4;      // tile + sink slot
  for (int c = tid; c < n_zero32; c += kStreamThreads) reinterpret_cast<uint32_t *>(sm)[c] = 0u;
  if (lane < NB) mbar_init(bar + lane, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::
                   : "memory");
  __syncthreads();

  CSR_MARK(1);
  const int nt = a.n_tiles;
  const int64_t nnz4 = __ldg(a.nnz) & ~int64_t{3};
  int64_t issued_total = 0, used_total = 0;
  // Stream the rows list[w], list[w + NW], ... (n_active entries) of this
  // warp through its ring into the tile.
  auto stream_rows = [&](const int32_t *list, bool list_smem, int64_t n_active, int64_t w,
                         int64_t NW) {
    // lane j holds the tile range of the warp's row 32 b + j; next batch prefetched
    auto load_range = [&](int64_t kb, int64_t &lo_r, int64_t &hi_r) {
      const int64_t k = w + (kb + lane) * NW;
      lo_r = 0;
      hi_r = 0;
      if (k < n_active) {
        const int64_t r = list == nullptr ? k : (list_smem ? list[k] : __ldg(list + k));
        const int64_t p0 = __ldg(a.indptr + r), p1 = __ldg(a.indptr + r + 1);
        const int32_t *sp = a.split + r * (nt - 1) - 1;      // sp[t], t = 1 .. nt-1
        lo_r = tile > 0 ? p0 + __ldg(sp + tile) : p0;
        hi_r = tile < nt - 1 ? p0 + __ldg(sp + tile + 1) : p1;
        lo_r = min(max(lo_r, p0), p1);          // a stale plan cannot leave the row
        hi_r = min(max(hi_r, lo_r), p1);
      }
    };
    const int64_t my_rows = n_active > w ? (n_active - w + NW - 1) / NW : 0;
    int64_t blo, bhi, nlo, nhi;             // current / next batch (per lane)
    load_range(0, blo, bhi);
    load_range(32, nlo, nhi);
    // issue cursor (warp-uniform): row index ir, position pos in [pos, hi)
    int64_t ir = 0, pos = 0, hi = 0;
    auto row_at = [&](int64_t r) {          // broadcast row r's range (r in current batch)
      const int j = static_cast<int>(r & 31);
      pos = __shfl_sync(0xffffffffu, blo, j);
      hi = __shfl_sync(0xffffffffu, bhi, j);
    };
    if (my_rows > 0) row_at(0);
    // fill buffer b with the next row pieces (up to kStreamSegs, BE slots);
    // false when the rows are exhausted
    auto issue = [&](int b) -> bool {
      int fill = 0, nseg = 0;
      // the buffer's sentinel slots were written through the generic proxy:
      // order them before the bulk copies (async proxy) overwrite the buffer
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      while (nseg < kStreamSegs && fill <= BE - 4) {
        while (ir < my_rows && pos >= hi) { // advance to the next non-empty row
          ++ir;
          if (ir >= my_rows) break;
          if ((ir & 31) == 0) {
            blo = nlo;
            bhi = nhi;
            load_range(ir + 32, nlo, nhi);
          }
          row_at(ir);
        }
        if (ir >= my_rows) break;
        const int64_t a0 = pos & ~int64_t{3};
        const int64_t a1 = min((hi + 3) & ~int64_t{3}, a0 + (BE - fill));
        const int64_t piece_hi = min(hi, a1);
        const int64_t ac = min(a1, max(nnz4, a0));         // copyable end
        const uint32_t bytes = static_cast<uint32_t>(ac - a0) * 4u;
        if (lane == 0) {
          StreamChunk &m = meta[b].seg[nseg];
          m.dst = fill;
          m.len = static_cast<int32_t>(a1 - a0);
          m.v0 = static_cast<int32_t>(pos - a0);
          m.v1 = static_cast<int32_t>(piece_hi - a0);
          m.gl = static_cast<int32_t>(ac - a0);
          m.a0 = a0;
          if (bytes) {
            mbar_expect_tx(bar + b, HOMO ? bytes : 2u * bytes);
            bulk_g2s(bidx + b * BE + fill, a.indices + a0, bytes, bar + b);
            if (!HOMO) bulk_g2s(bdat + b * BE + fill, a.data + a0, bytes, bar + b);
          }
        }
        fill += static_cast<int>(a1 - a0);
        ++nseg;
        pos = piece_hi;
      }
      if (nseg == 0) return false;
      if (lane == 0) {
        meta[b].nseg = nseg;
        meta[b].fill = fill;
        mbar_arrive(bar + b);
      }
      return true;
    };

    // lc = col - c0 clamped to the sink slot `width` (entries of an unsorted
    // row that fall outside the tile land there and are never flushed):
    // branch-free, one clamp per entry
    auto add = [&](int32_t col, float wgt) {
      const uint32_t lc = min(static_cast<uint32_t>(col - c0i), static_cast<uint32_t>(width));
      if (C16) atomicAdd(reinterpret_cast<uint32_t *>(sm) + (lc >> 1), 1u << ((lc & 1u) * 16u));
      else if (HOMO) atomicAdd(reinterpret_cast<uint32_t *>(sm) + lc, 1u);
      else if (KIND == 0) atomicAdd(reinterpret_cast<float *>(sm) + lc, a.absw ? fabsf(wgt) : wgt);
      else if (KIND == 2) {
        // rule T4: q = rint(w 2^fix_bits) as hi = q >> 8 and lo = q & 255,
        // two independent native 32-bit ATOMS (no carry, no return value)
        const long long qq = __float2ll_rn(__fmul_rn(wgt, fix_scale));
        unsigned *p = reinterpret_cast<unsigned *>(sm) + 2 * lc;
        atomicAdd(p, static_cast<unsigned>(static_cast<int>(qq >> 8)));
        atomicAdd(p + 1, static_cast<unsigned>(qq & 255));
      } else {
        // int64 add as two native 32-bit ATOMS (a 64-bit shared add is a CAS
        // loop on sm_100a): low word with return, carry into the high word --
        // exact modulo 2^64, like an int64 add
        unsigned *p = reinterpret_cast<unsigned *>(sm) + 2 * lc;
        const unsigned long long qq = static_cast<unsigned long long>(quantize(wgt));
        const unsigned lo = static_cast<unsigned>(qq);
        const unsigned old = atomicAdd(p, lo);
        atomicAdd(p + 1, static_cast<unsigned>(qq >> 32) + (old + lo < old ? 1u : 0u));
      }
    };
    auto add4 = [&](const int4 &ci, const float4 &wi) {
      add(ci.x, wi.x);
      add(ci.y, wi.y);
      add(ci.z, wi.z);
      add(ci.w, wi.w);
    };

    // buffer of the i-th chunk: i % NB, its mbarrier phase (i / NB) & 1;
    // the counts run on across calls of this lambda
    const int64_t used0 = used_total;
    for (int j = 0; j < NB; ++j)
      if (issue(static_cast<int>(issued_total % NB))) ++issued_total;
    for (int64_t used = used0; used < issued_total; ++used) {
      const int b = static_cast<int>(used % NB);
      mbar_wait(bar + b, static_cast<uint32_t>((used / NB) & 1));
      // lane i sanitises piece i: slots outside [v0, v1) (16-byte alignment
      // padding, <= 3 each side) get a column that clamps into the sink slot,
      // entries past the last copied 16 bytes of the array (<= 3) are loaded
      int32_t *si = bidx + b * BE;
      float *sd = bdat + b * BE;
      if (lane < meta[b].nseg) {
        const StreamChunk m = meta[b].seg[lane];
        int32_t *pi = si + m.dst;
        for (int o = 0; o < m.v0; ++o) pi[o] = INT32_MIN;
        for (int o = m.v1; o < m.len; ++o) pi[o] = INT32_MIN;
        for (int o = m.gl; o < m.v1; ++o) {
          pi[o] = __ldg(a.indices + m.a0 + o);
          if (!HOMO) sd[m.dst + o] = __ldg(a.data + m.a0 + o);
        }
      }
      __syncwarp();
      // every slot of the buffer: two quads per lane per iteration, no checks
      const int fill = meta[b].fill;
      for (int q = 4 * lane; q < fill; q += 256) {
        const bool two = q + 128 < fill;
        const int4 c1 = *reinterpret_cast<const int4 *>(si + q);
        const int4 c2 = two ? *reinterpret_cast<const int4 *>(si + q + 128) : c1;
        float4 w1 = make_float4(0.f, 0.f, 0.f, 0.f), w2 = w1;
        if (!HOMO) {
          w1 = *reinterpret_cast<const float4 *>(sd + q);
          if (two) w2 = *reinterpret_cast<const float4 *>(sd + q + 128);
        }
        add4(c1, w1);
        if (two) add4(c2, w2);
      }
      __syncwarp();                                 // buffer b consumed by every lane
      if (issue(b)) ++issued_total;
    }
    used_total = issued_total;
  };

  // rows from the active list: warp w of the tile takes k = w, w + NW, ... --
  // dealt evenly over the tile's CTAs (a per-CTA compaction of its slice of
  // the spike words avoids the compaction launch but leaves ~12 % imbalance)
  const int64_t n_active_rows = a.active ? static_cast<int64_t>(*a.count) : a.n_rows_all;
  stream_rows(a.active, false, n_active_rows, static_cast<int64_t>(group) * kStreamWarps + warp,
              static_cast<int64_t>(a.groups) * kStreamWarps);
  CSR_MARK(2);
  __syncthreads();
  CSR_MARK(3);
  // partial tile -> [tile][group][tile_cols], 16-byte stores.  Rows are
  // dealt kStreamWarps per CTA in order, so only the first `used` CTAs of a tile got
  // any; with the fused reduction the others skip the flush (it reads only
  // the first `used` partials), k_csr_reduce reads them all.
  const int64_t cta_rows = (n_active_rows + kStreamWarps - 1) / kStreamWarps;
  const int used = cta_rows < a.groups ? static_cast<int>(cta_rows) : a.groups;
  if (a.out == nullptr || group < used) {
    char *dst = static_cast<char *>(a.partials) +
                (static_cast<size_t>(tile) * a.groups + group) * a.tile_cols * acc_bytes;
    const int n16 = width * acc_bytes / 16;
    for (int k = tid; k < n16; k += kStreamThreads)
      reinterpret_cast<uint4 *>(dst)[k] = reinterpret_cast<const uint4 *>(sm)[k];
    for (int b = n16 * 16 + tid; b < width * acc_bytes; b += kStreamThreads) dst[b] = sm[b];
  }
  CSR_MARK(4);
  if (a.out == nullptr) return;
  // fused reduction (cooperative launch: every CTA is resident): after a
  // grid-wide barrier, CTA g of tile t sums column slice g of the tile over
  // the groups in ascending order (L2-resident partials, deterministic)
  __threadfence();
  cg::this_grid().sync();
  CSR_MARK(5);
  tile_reduce<KIND, HOMO, kStreamThreads, C16>(a.partials, static_cast<size_t>(tile) * a.groups,
                                               group, a.groups, used, a.tile_cols, width, c0,
                                               a.out, a.accumulate, a.w, a.q, a.fix_bits);
  CSR_MARK(6);
}

}  // namespace bp
