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
//    search otherwise) -> bounds[k][0..n_tiles];
//  * k_csr_stream: CTA (tile t, group g) owns column tile t in shared memory
//    and active rows k = g, g+G, ...  One producer warp issues
//    cp.async.bulk copies of the rows' in-tile index (and weight) ranges into
//    a ring of S stages of E entries (several rows per stage, mbarrier
//    complete_tx), so S*E*4 bytes per SM are in flight without registers;
//    15 consumer warps turn staged entries into shared-memory atomics and
//    release the stage.  Only 32-bit integer shared atomics are native on
//    sm_100a (f32 and 64-bit adds compile to CAS loops): homogeneous weights
//    count events (POPC.INC), fixed-point weights add int64 as two 32-bit
//    words with a carry, fp32 weights use the CAS add.  The tile is stored
//    as a partial and k_csr_reduce (scatter.cuh) sums the groups in order --
//    no global atomics.
// Indices must ascend within each row (canonical CSR, include/bp.h); entries
// outside the tile are skipped, so unsorted input cannot corrupt memory.
#pragma once
#include <cstdint>

#include "scatter.cuh"

namespace bp {

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
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
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
// First j in [lo, hi) with idx[j] >= x, starting from a guess g: one 128-entry
// window (4 per lane) around g, a 32-way search only if the answer is outside.
__device__ __forceinline__ int64_t window_lower_bound(const int32_t *__restrict__ idx,
                                                      int64_t lo, int64_t hi, int32_t x,
                                                      int64_t g) {
  if (hi - lo <= 128) {
    const int lane = threadIdx.x & 31;
    int n_lt = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t j = lo + 4 * lane + e;
      n_lt += (j < hi && __ldg(idx + j) < x) ? 1 : 0;
    }
    return lo + __reduce_add_sync(0xffffffffu, static_cast<unsigned>(n_lt));
  }
  const int lane = threadIdx.x & 31;
  int64_t w0 = g - 64;
  w0 = w0 < lo ? lo : (w0 > hi - 128 ? hi - 128 : w0);
  int n_lt = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) n_lt += __ldg(idx + w0 + 4 * lane + e) < x ? 1 : 0;
  n_lt = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(n_lt)));
  if (n_lt == 0 && w0 > lo) return warp_lower_bound(idx, lo, w0, x);
  if (n_lt == 128 && w0 + 128 < hi) return warp_lower_bound(idx, w0 + 128, hi, x);
  return w0 + n_lt;
}

struct CsrSplitArgs {
  const int64_t *indptr;
  const int32_t *indices;
  const int32_t *active;
  const int32_t *count;
  int64_t *bounds;       // [k][n_tiles + 1]
  int32_t n_tiles, tile_cols;
  int64_t n_cols;
};

// One warp per active row: bounds[k][t] = first entry of row active[k] with
// column >= t * tile_cols (t = 0 and n_tiles: the row's ends).
__global__ void __launch_bounds__(256) k_csr_split(CsrSplitArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t n_active = *a.count;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int nt = a.n_tiles;
  for (int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
       k < n_active; k += nw) {
    const int64_t r = a.active[k];
    const int64_t lo = __ldg(a.indptr + r), hi = __ldg(a.indptr + r + 1);
    int64_t *b = a.bounds + k * (nt + 1);
    int64_t cur = lo;
    for (int t = 1; t < nt; ++t) {
      const int32_t x = t * a.tile_cols;
      // columns of a random row are spread evenly: interpolate the position
      int64_t g = lo + static_cast<int64_t>(static_cast<double>(hi - lo) * x /
                                            static_cast<double>(a.n_cols));
      g = g < cur ? cur : (g > hi ? hi : g);
      const int64_t j = cur < hi ? window_lower_bound(a.indices, cur, hi, x, g) : hi;
      if (lane == 0) b[t] = j;
      cur = j;
    }
    if (lane == 0) {
      b[0] = lo;
      b[nt] = hi;
    }
  }
}

// --------------------------------------------------------------- stream
constexpr int kStreamThreads = 512;       // warp 0 produces, 15 warps consume
constexpr int kStreamConsumers = kStreamThreads / 32 - 1;
constexpr int kStreamSegs = 16;           // row pieces per stage
constexpr int kStreamEnt = 4096;          // entries per stage

struct StreamSeg {
  int32_t dst;     // first stage slot of the copy (multiple of 4)
  int32_t len;     // slots of the copy (multiple of 4)
  int32_t v0, v1;  // valid entries [v0, v1) relative to a0
  int32_t gl;      // entries >= gl were not copied (end of the array): read from global
  int32_t pad;
  int64_t a0;      // global index of slot dst (16-byte aligned)
};
struct StreamMeta {
  int32_t nseg;    // < 0: no more stages
  int32_t fill;
  int32_t pad[2];
  StreamSeg seg[kStreamSegs];
};

struct CsrStreamArgs {
  const int32_t *indices;
  const float *data;         // nullptr -> homogeneous: count events per column
  const int64_t *bounds;
  const int32_t *count;
  const int64_t *nnz;        // &indptr[n_rows]
  void *partials;            // [tile][group][tile_cols]
  int32_t tile_cols, groups, n_tiles, stages;
  int64_t n_cols;
};

// Shared-memory layout (host and device agree through this function).
struct StreamSmem {
  size_t acc, idx, dat, meta, bar, total;
};
__host__ __device__ inline StreamSmem stream_smem(int tile_cols, int acc_bytes, int stages,
                                                  bool homo) {
  auto up = [](size_t x) { return (x + 127) & ~size_t{127}; };
  StreamSmem s{};
  s.acc = 0;
  s.idx = up(static_cast<size_t>(tile_cols) * acc_bytes);
  s.dat = s.idx + static_cast<size_t>(stages) * kStreamEnt * 4;
  s.meta = s.dat + (homo ? 0 : static_cast<size_t>(stages) * kStreamEnt * 4);
  s.bar = up(s.meta + static_cast<size_t>(stages) * sizeof(StreamMeta));
  s.total = s.bar + static_cast<size_t>(2 * stages) * 8;
  return s;
}

// KIND: 0 f32 partials, 1 int64 fixed-point partials; HOMO: uint32 counts.
template <int KIND, bool HOMO>
__global__ void __launch_bounds__(kStreamThreads, 1) k_csr_stream(CsrStreamArgs a) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int acc_bytes = (HOMO || KIND == 0) ? 4 : 8;
  const int S = a.stages;
  const StreamSmem L = stream_smem(a.tile_cols, acc_bytes, S, HOMO);
  int32_t *sidx = reinterpret_cast<int32_t *>(sm + L.idx);
  float *sdat = reinterpret_cast<float *>(sm + L.dat);
  StreamMeta *meta = reinterpret_cast<StreamMeta *>(sm + L.meta);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + L.bar);
  uint64_t *empty = full + S;

  const int tile = blockIdx.x / a.groups, group = blockIdx.x % a.groups;
  const int64_t c0 = static_cast<int64_t>(tile) * a.tile_cols;
  const int64_t c1 = min(c0 + a.tile_cols, a.n_cols);
  const int width = static_cast<int>(c1 - c0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int c = tid; c < width; c += kStreamThreads) {
    if (acc_bytes == 4) reinterpret_cast<uint32_t *>(sm)[c] = 0u;
    else reinterpret_cast<unsigned long long *>(sm)[c] = 0ull;
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kStreamConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::
                     : "memory");
  }
  __syncthreads();
  const int64_t n_active = *a.count;
  const int nt = a.n_tiles, G = a.groups;

  if (warp == 0) {
    // ---- producer: pack the rows' in-tile ranges into stages
    const int64_t nnz4 = __ldg(a.nnz) & ~int64_t{3};
    int s = 0, nseg = 0, fill = 0;
    uint32_t ph = 0;
    mbar_wait(empty + s, ph ^ 1u);
    auto commit = [&]() {
      if (lane == 0) {
        meta[s].nseg = nseg;
        meta[s].fill = fill;
        mbar_arrive(full + s);
      }
      if (++s == S) { s = 0; ph ^= 1u; }
      nseg = 0;
      fill = 0;
      mbar_wait(empty + s, ph ^ 1u);
    };
    for (int64_t kb = group; kb < n_active; kb += 32LL * G) {
      const int64_t k = kb + static_cast<int64_t>(lane) * G;
      int64_t lo_l = 0, hi_l = 0;
      if (k < n_active) {
        lo_l = __ldg(a.bounds + k * (nt + 1) + tile);
        hi_l = __ldg(a.bounds + k * (nt + 1) + tile + 1);
      }
      for (int j = 0; j < 32; ++j) {
        int64_t lo = __shfl_sync(0xffffffffu, lo_l, j);
        const int64_t hi = __shfl_sync(0xffffffffu, hi_l, j);
        while (lo < hi) {
          const int room = kStreamEnt - fill;
          if (room < 4 || nseg == kStreamSegs) {
            commit();
            continue;
          }
          const int64_t a0 = lo & ~int64_t{3};
          const int64_t a1 = min((hi + 3) & ~int64_t{3}, a0 + room);
          const int64_t piece_hi = min(hi, a1);
          const int64_t ac = min(a1, max(nnz4, a0));     // copyable end
          const uint32_t bytes = static_cast<uint32_t>(ac - a0) * 4u;
          if (lane == 0) {
            StreamSeg &sg = meta[s].seg[nseg];
            sg.dst = fill;
            sg.len = static_cast<int32_t>(a1 - a0);
            sg.v0 = static_cast<int32_t>(lo - a0);
            sg.v1 = static_cast<int32_t>(piece_hi - a0);
            sg.gl = static_cast<int32_t>(ac - a0);
            sg.a0 = a0;
            if (bytes) {
              mbar_expect_tx(full + s, HOMO ? bytes : 2u * bytes);
              bulk_g2s(sidx + static_cast<size_t>(s) * kStreamEnt + fill, a.indices + a0,
                       bytes, full + s);
              if (!HOMO)
                bulk_g2s(sdat + static_cast<size_t>(s) * kStreamEnt + fill, a.data + a0,
                         bytes, full + s);
            }
          }
          fill += static_cast<int>(a1 - a0);
          ++nseg;
          lo = piece_hi;
        }
      }
    }
    if (nseg) commit();
    if (lane == 0) {
      meta[s].nseg = -1;
      mbar_arrive(full + s);
    }
  } else {
    // ---- consumers: staged entries -> shared-memory atomics
    const int c = tid - 32;
    constexpr int NC = kStreamThreads - 32;
    const int32_t c0i = static_cast<int32_t>(c0);
    int s = 0;
    uint32_t ph = 0;
    for (;;) {
      mbar_wait(full + s, ph);
      const StreamMeta &m = meta[s];
      const int nseg = m.nseg;
      if (nseg < 0) break;
      const int fill = m.fill;
      const int32_t *si = sidx + static_cast<size_t>(s) * kStreamEnt;
      const float *sd = sdat + static_cast<size_t>(s) * kStreamEnt;
      int i = 0;
      int seg_end = m.seg[0].len;      // seg[0].dst == 0
      for (int q = 4 * c; q < fill; q += 4 * NC) {
        while (q >= seg_end) {
          ++i;
          seg_end = m.seg[i].dst + m.seg[i].len;
        }
        const StreamSeg &sg = m.seg[i];
        const int off = q - sg.dst;
        const int4 ci = *reinterpret_cast<const int4 *>(si + q);
        float4 wi = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!HOMO) wi = *reinterpret_cast<const float4 *>(sd + q);
        const int32_t cv[4] = {ci.x, ci.y, ci.z, ci.w};
        const float wv[4] = {wi.x, wi.y, wi.z, wi.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int o = off + e;
          if (o < sg.v0 || o >= sg.v1) continue;
          int32_t col = cv[e];
          float w = wv[e];
          if (o >= sg.gl) {                    // tail past the last 16-byte boundary
            col = __ldg(a.indices + sg.a0 + o);
            if (!HOMO) w = __ldg(a.data + sg.a0 + o);
          }
          const uint32_t lc = static_cast<uint32_t>(col - c0i);
          if (lc >= static_cast<uint32_t>(width)) continue;   // unsorted row: skip
          if (HOMO) atomicAdd(reinterpret_cast<uint32_t *>(sm) + lc, 1u);
          else if (KIND == 0) atomicAdd(reinterpret_cast<float *>(sm) + lc, w);
          else {
            // int64 add as two native 32-bit ATOMS (a 64-bit shared add is
            // a CAS loop on sm_100a): low word with return, carry into the
            // high word -- exact modulo 2^64, like an int64 add
            unsigned *p = reinterpret_cast<unsigned *>(sm) + 2 * lc;
            const unsigned long long qq = static_cast<unsigned long long>(quantize(w));
            const unsigned lo = static_cast<unsigned>(qq);
            const unsigned old = atomicAdd(p, lo);
            atomicAdd(p + 1, static_cast<unsigned>(qq >> 32) + (old + lo < old ? 1u : 0u));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (++s == S) { s = 0; ph ^= 1u; }
    }
  }
  __syncthreads();
  // partial tile -> [tile][group][tile_cols], 16-byte stores
  char *dst = static_cast<char *>(a.partials) +
              (static_cast<size_t>(tile) * a.groups + group) * a.tile_cols * acc_bytes;
  const int n16 = width * acc_bytes / 16;
  for (int k = tid; k < n16; k += kStreamThreads)
    reinterpret_cast<uint4 *>(dst)[k] = reinterpret_cast<const uint4 *>(sm)[k];
  for (int b = n16 * 16 + tid; b < width * acc_bytes; b += kStreamThreads) dst[b] = sm[b];
}

}  // namespace bp
