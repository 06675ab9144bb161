// scatter.cuh -- spike compaction (a1), CSR event scatter (a2) and JIT
// connectivity regeneration + scatter (a3, a4) for sm_100a.
//
// Design:
//  * compaction: one thread per 32-bit spike word; warp inclusive scan of
//    popcounts, one atomicAdd per warp claims a slice of the active list.
//  * CSR: one warp per active row (grid-stride).  A row's indices/data are
//    read as 128-byte coalesced warp loads, 4 loads in flight per lane, and
//    every synaptic event is one fire-and-forget RED (no return value).
//  * JIT: one warp per (active row, segment).  Lane l of chunk c owns gap
//    draws 128c+4l..128c+4l+3 (one Philox block), a warp scan turns gaps into
//    positions, and each lane scatters its (up to) 4 edges.  No connectivity
//    bytes are read at all.
#pragma once
#include <cstdint>

#include "cache.cuh"
#include "rng.cuh"

namespace bp {

constexpr int kScatterThreads = 256;

__device__ __forceinline__ void add_f32(void *out, int64_t c, float w, uint64_t pol) {
  red_add_f32(static_cast<float *>(out) + c, w, pol);
}
__device__ __forceinline__ void add_fix(void *out, int64_t c, long long q, uint64_t pol) {
  red_add_u64(reinterpret_cast<unsigned long long *>(out) + c,
              static_cast<unsigned long long>(q), pol);
}

// Block-wide sum of per-thread event counts, one atomic per block.
__device__ __forceinline__ void count_events(unsigned long long *counter,
                                             unsigned long long mine) {
  if (counter == nullptr) return;
  __shared__ unsigned long long block_sum;
  if (threadIdx.x == 0) block_sum = 0;
  __syncthreads();
  mine = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(mine));
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&block_sum, mine);
  __syncthreads();
  if (threadIdx.x == 0 && block_sum) atomicAdd(counter, block_sum);
}

// ---------------------------------------------------------------- a1
// Words [skip_b, skip_e) count as empty (a partition's own words in
// bp_network_scatter).  Short vectors (config-2 calls): warps warp0, warp0 + n_warps, ... each
// take 32 spike words: warp scan of the popcounts, one atomicAdd per warp
// claims a slice of the active list (no block barriers).
__device__ __forceinline__ void compact_words(const uint32_t *__restrict__ spikes, int64_t n,
                                              int32_t *__restrict__ active,
                                              int32_t *__restrict__ count, int32_t id_base,
                                              int64_t warp0, int64_t n_warps,
                                              int64_t skip_b, int64_t skip_e) {
  const int lane = threadIdx.x & 31;
  const int64_t n_words = (n + 31) >> 5;
  for (int64_t base = warp0 * 32; base < n_words; base += n_warps * 32) {
    const int64_t wi = base + lane;
    uint32_t word = 0;
    if (wi < n_words && (wi < skip_b || wi >= skip_e)) {
      word = __ldg(spikes + wi);
      const int64_t valid = n - (wi << 5);
      if (valid < 32) word &= (1u << valid) - 1u;
    }
    const int c = __popc(word);
    int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    int slot = 0;
    if (lane == 31) slot = atomicAdd(count, total);
    slot = __shfl_sync(0xffffffffu, slot, 31) + incl - c;
    while (word) {
      const int b = __ffs(word) - 1;
      active[slot++] = id_base + static_cast<int32_t>((wi << 5) + b);
      word &= word - 1u;
    }
  }
}

__global__ void __launch_bounds__(256)
k_compact_warp(const uint32_t *__restrict__ spikes, int64_t n,
          int32_t *__restrict__ active, int32_t *__restrict__ count,
          int32_t id_base, int64_t skip_b, int64_t skip_e) {
  compact_words(spikes, n, active, count, id_base,
                (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5,
                (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5, skip_b, skip_e);
}

// Long vectors (the remote words of a partitioned network): block-aggregated
// compaction.  Each block takes 1024 consecutive spike
// words per iteration (4 per thread), ranks their set bits with a block
// scan of the popcounts and claims its slice of the active list with ONE
// atomic per non-empty iteration.  (A claim per warp of 32 words put ~10^5
// returning atomics on the single counter for a 10^8-neuron vector --
// 55 us at 0.22 % density, serialised on one L2 address.)
// WPT words per thread: 4 for long vectors (fewer claims), 1 for short ones
// (more blocks in flight).
constexpr int kCompactThreads = 256;

template <int WPT>
__global__ void __launch_bounds__(kCompactThreads)
k_compact(const uint32_t *__restrict__ spikes, int64_t n,
          int32_t *__restrict__ active, int32_t *__restrict__ count,
          int32_t id_base, int64_t skip_b, int64_t skip_e) {
  __shared__ int32_t warp_tot[kCompactThreads / 32];
  __shared__ int32_t block_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n_words = (n + 31) >> 5;
  constexpr int BW = WPT * kCompactThreads;     // words per block iteration
  for (int64_t w0 = static_cast<int64_t>(blockIdx.x) * BW; w0 < n_words;
       w0 += static_cast<int64_t>(gridDim.x) * BW) {
    uint32_t wd[WPT];
    int c = 0;
    const int64_t wt = w0 + WPT * tid;             // this thread's first word
    if (WPT % 4 == 0 && wt + WPT <= n_words && (wt + WPT <= skip_b || wt >= skip_e) &&
        (n & 31) == 0 && (reinterpret_cast<uintptr_t>(spikes) & 15) == 0) {
      // whole 16-byte groups inside the vector and outside the skip range
#pragma unroll
      for (int k = 0; k < WPT; k += 4) {
        const uint4 q = __ldg(reinterpret_cast<const uint4 *>(spikes + wt + k));
        wd[k] = q.x; wd[k + 1] = q.y; wd[k + 2] = q.z; wd[k + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < WPT; ++k) {
        const int64_t wi = wt + k;
        uint32_t word = 0;
        if (wi < n_words && (wi < skip_b || wi >= skip_e)) {
          word = __ldg(spikes + wi);
          const int64_t valid = n - (wi << 5);
          if (valid < 32) word &= (1u << valid) - 1u;
        }
        wd[k] = word;
      }
    }
#pragma unroll
    for (int k = 0; k < WPT; ++k) c += __popc(wd[k]);
    int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kCompactThreads / 32; ++k) {
      const int v = warp_tot[k];
      before += k < warp ? v : 0;
      total += v;
    }
    if (tid == 0 && total) block_base = atomicAdd(count, total);
    __syncthreads();                 // block_base ready; warp_tot reusable
    if (total == 0) continue;        // block-uniform
    int slot = block_base + before + incl - c;
#pragma unroll
    for (int k = 0; k < WPT; ++k) {
      uint32_t word = wd[k];
      while (word) {
        const int b = __ffs(word) - 1;
        word &= word - 1u;
        active[slot++] = id_base + static_cast<int32_t>(((w0 + WPT * tid + k) << 5) + b);
      }
    }
  }
}

// ---------------------------------------------------------------- a2
struct CsrSide {
  const int64_t *indptr;
  const int32_t *indices;
  const float *data;  // nullptr -> homogeneous w
  float w;
  long long q;        // quantize(w)
  void *out;
};

struct CsrScatterArgs {
  CsrSide e, i;          // rows < split -> e (row), else i (row - split)
  int64_t split;
  const int32_t *active;
  const int32_t *count;
  int32_t *zero_count;   // nullable; set to 0 by thread 0 (ping-pong list)
  unsigned long long *events;   // nullable
  unsigned long long *spikes;   // nullable; += *count once
  float keep_frac;              // L2 evict_last fraction of the outputs (0: none)
};

// Field-wise select keeps the chosen projection in registers (a runtime
// reference into the kernel-parameter struct would spill it to local memory).
__device__ __forceinline__ CsrSide pick(bool second, const CsrSide &x,
                                        const CsrSide &y) {
  CsrSide s;
  s.indptr = second ? y.indptr : x.indptr;
  s.indices = second ? y.indices : x.indices;
  s.data = second ? y.data : x.data;
  s.w = second ? y.w : x.w;
  s.q = second ? y.q : x.q;
  s.out = second ? y.out : x.out;
  return s;
}

template <int KIND>
__device__ __forceinline__ void csr_emit(const CsrSide &s, int32_t c, float w,
                                         uint64_t pol) {
  if (KIND == 0) add_f32(s.out, c, w, pol);
  else add_fix(s.out, c, s.data ? quantize(w) : s.q, pol);
}

template <int KIND>
__global__ void __launch_bounds__(kScatterThreads)
k_csr_scatter(CsrScatterArgs a) {
  const int n_active = *a.count;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (a.zero_count) *a.zero_count = 0;
    if (a.spikes) atomicAdd(a.spikes, static_cast<unsigned long long>(n_active));
  }
  const int lane = threadIdx.x & 31;
  const int warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int n_warps = (gridDim.x * blockDim.x) >> 5;
  const uint64_t pol = make_policies(a.keep_frac).keep;
  unsigned long long ev = 0;
  for (int k = warp0; k < n_active; k += n_warps) {
    const int64_t r = a.active[k];
    const bool inh = r >= a.split;
    const CsrSide s = pick(inh, a.e, a.i);
    const int64_t row = inh ? r - a.split : r;
    const int64_t begin = __ldg(s.indptr + row);
    const int64_t end = __ldg(s.indptr + row + 1);
    if (lane == 0) ev += static_cast<unsigned long long>(end - begin);
    int64_t j = begin + lane;
    // 4 independent 128-byte warp loads in flight before the REDs.
    for (; j + 96 < end; j += 128) {
      const int32_t c0 = __ldg(s.indices + j), c1 = __ldg(s.indices + j + 32);
      const int32_t c2 = __ldg(s.indices + j + 64), c3 = __ldg(s.indices + j + 96);
      float w0 = s.w, w1 = s.w, w2 = s.w, w3 = s.w;
      if (s.data) {
        w0 = __ldg(s.data + j); w1 = __ldg(s.data + j + 32);
        w2 = __ldg(s.data + j + 64); w3 = __ldg(s.data + j + 96);
      }
      csr_emit<KIND>(s, c0, w0, pol); csr_emit<KIND>(s, c1, w1, pol);
      csr_emit<KIND>(s, c2, w2, pol); csr_emit<KIND>(s, c3, w3, pol);
    }
    for (; j < end; j += 32) {
      const int32_t c = __ldg(s.indices + j);
      csr_emit<KIND>(s, c, s.data ? __ldg(s.data + j) : s.w, pol);
    }
  }
  count_events(a.events, ev);
}


// ---------------------------------------------------------------- a2, tiled
// Column-tiled CSR scatter for outputs that fit a few shared-memory tiles
// (config 2: 100k columns = two 50k-float tiles).  Random global REDs run at
// ~0.19 T/s on B200 while shared-memory atomics run at 0.7 (f32 CAS) to 1.5
// (int32) T/s (tools/probes/probe_atomics.cu), so each CTA owns one column
// tile in shared memory, walks its share of the active rows, and adds only
// the entries inside its tile -- the row's sub-range is found with a
// 32-way warp search (<= 3 dependent loads for rows of 5000) -- then flushes
// the tile with coalesced REDs (skipping untouched zeros).
constexpr int kTiledThreads = 1024;

// First j in [lo, hi) with idx[j] >= x (idx ascending); warp-cooperative.
__device__ __forceinline__ int64_t warp_lower_bound(const int32_t *__restrict__ idx, int64_t lo,
                                                    int64_t hi, int32_t x) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t j = lo + lane * step;
    const bool ge = j < hi ? (__ldg(idx + j) >= x) : true;
    const unsigned m = __ballot_sync(0xffffffffu, ge);
    if (m == 0u) {                       // every probe < x: answer after the last probe
      lo = lo + 31 * step + 1;
      continue;
    }
    const int f = __ffs(m) - 1;
    if (f == 0) return lo;               // idx[lo] >= x
    const int64_t nlo = lo + (f - 1) * step + 1;
    const int64_t nhi = lo + f * step;   // idx[nhi] >= x (or nhi >= hi)
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
  }
  const int64_t j = lo + lane;
  const bool ge = j < hi ? (__ldg(idx + j) >= x) : true;
  const unsigned m = __ballot_sync(0xffffffffu, ge);
  return m ? lo + (__ffs(m) - 1) : hi;
}

struct CsrTiledArgs {
  const int64_t *indptr;
  const int32_t *indices;
  const float *data;          // nullptr -> homogeneous w
  float w;
  long long q;
  void *out;
  int64_t n_cols;
  int32_t tile_cols;
  int32_t groups;             // CTAs per tile
  const int32_t *active;
  const int32_t *count;
  void *partials;             // nullable: [tile][group][tile_cols] partial sums
  int accumulate;             // reduce: out += sum (else out = sum)
  int vec;                    // indices (and data) 16-byte aligned: 128-bit loads
  int32_t fix_bits;           // KIND 2 partials (k_csr_stream): fixed point 2^-fix_bits
};

// Rule T4 (heterogeneous fp32 output through scaled fixed point): a column's
// partial is a (hi int32, lo uint32) pair with value hi 2^8 + lo in units
// of 2^-fix_bits (each weight w adds q = rint(w 2^fix_bits) as hi = q >> 8,
// lo = q & 255: two independent native 32-bit shared atomics, exact, and
// order-free).  The sum of a column is rounded to fp32 once.
__device__ __forceinline__ float fix2_value(long long hi, unsigned long long lo, int fix_bits) {
  const long long t = hi * 256 + static_cast<long long>(lo);
  return __fmul_rn(__ll2float_rn(t), __int_as_float((127 - fix_bits) << 23));
}

template <int KIND>
__global__ void __launch_bounds__(kTiledThreads, 1)
k_csr_tiled(CsrTiledArgs a) {
  extern __shared__ __align__(16) unsigned char tile_raw[];
  const int tile = blockIdx.x / a.groups, group = blockIdx.x % a.groups;
  const int64_t c0 = static_cast<int64_t>(tile) * a.tile_cols;
  const int64_t c1 = min(c0 + a.tile_cols, a.n_cols);
  const int width = static_cast<int>(c1 - c0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float *accf = reinterpret_cast<float *>(tile_raw);
  unsigned long long *accq = reinterpret_cast<unsigned long long *>(tile_raw);
  // homogeneous weight: count the events per column (native int32 ATOMS)
  // and scale once at the flush -- count * q(w) equals the fixed-point sum;
  // fl32(count * w) is within rule T2 of the fp32 sum
  unsigned *accc = reinterpret_cast<unsigned *>(tile_raw);
  const bool homo = a.data == nullptr;
  for (int c = tid; c < width; c += kTiledThreads) {
    if (homo) accc[c] = 0u;
    else if (KIND == 0) accf[c] = 0.f;
    else accq[c] = 0ull;
  }
  __syncthreads();
  const int n_active = *a.count;
  // Work unit = (active row, quarter of its in-tile range); units are dealt
  // to the CTAs of the tile first, so a few long rows still spread over
  // many SMs instead of queueing on one warp.
  const int nwarp = a.groups * (kTiledThreads / 32);
  const int kChunks = n_active >= nwarp ? 1 : 4;     // split rows only when rows are few
  const int64_t n_units = static_cast<int64_t>(n_active) * kChunks;
  for (int64_t u = static_cast<int64_t>(warp) * a.groups + group; u < n_units; u += nwarp) {
    const int64_t r = a.active[u / kChunks];
    const int chunk = static_cast<int>(u % kChunks);
    int64_t lo = __ldg(a.indptr + r), hi = __ldg(a.indptr + r + 1);
    if (c0 > 0) lo = warp_lower_bound(a.indices, lo, hi, static_cast<int32_t>(c0));
    if (c1 < a.n_cols) hi = warp_lower_bound(a.indices, lo, hi, static_cast<int32_t>(c1));
    const int64_t span = hi - lo;
    hi = lo + span * (chunk + 1) / kChunks;
    lo = lo + span * chunk / kChunks;
    // entry j's contribution to the shared tile
    auto add = [&](int32_t col, float w) {
      if (static_cast<uint32_t>(col) >= static_cast<uint32_t>(width)) return;  // unsorted row
      if (homo) atomicAdd(accc + col, 1u);               // native ATOMS (POPC.INC)
      else if (KIND == 0) atomicAdd(accf + col, w);
      else atomicAdd(accq + col, static_cast<unsigned long long>(quantize(w)));
    };
    const int32_t c0i = static_cast<int32_t>(c0);
    if (!a.vec) {                                       // arrays not 16-byte aligned
      for (int64_t jj = lo + lane; jj < hi; jj += 32)
        add(__ldg(a.indices + jj) - c0i, a.data ? __ldg(a.data + jj) : a.w);
      continue;
    }
    // head up to a 16-byte boundary, 128-bit body (4 int4 loads = 16
    // entries in flight per lane), tail
    const int64_t a0 = min(hi, (lo + 3) & ~int64_t{3});
    const int64_t a1 = a0 + ((hi - a0) & ~int64_t{3});
    if (lo + lane < a0) {
      const int64_t jj = lo + lane;
      add(__ldg(a.indices + jj) - c0i, a.data ? __ldg(a.data + jj) : a.w);
    }
    if (a1 + lane < hi) {
      const int64_t jj = a1 + lane;
      add(__ldg(a.indices + jj) - c0i, a.data ? __ldg(a.data + jj) : a.w);
    }
    const int4 *iv = reinterpret_cast<const int4 *>(a.indices + a0);
    const float4 *dv = a.data ? reinterpret_cast<const float4 *>(a.data + a0) : nullptr;
    const int64_t nv = (a1 - a0) >> 2;                  // int4 vectors in the body
    for (int64_t v = lane; v < nv; v += 128) {
      int4 ci[4];
      float4 wi[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t vv = v + 32 * u;
        ci[u] = vv < nv ? __ldg(iv + vv) : make_int4(-1, -1, -1, -1);
        wi[u] = (dv && vv < nv) ? __ldg(dv + vv) : make_float4(a.w, a.w, a.w, a.w);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (ci[u].x < 0) continue;
        add(ci[u].x - c0i, wi[u].x);
        add(ci[u].y - c0i, wi[u].y);
        add(ci[u].z - c0i, wi[u].z);
        add(ci[u].w - c0i, wi[u].w);
      }
    }
  }
  __syncthreads();
  if (a.partials) {
    // coalesced 16-byte stores of the whole tile; k_csr_reduce sums the
    // groups in a fixed order (no global atomics, deterministic)
    const size_t elt = (homo || KIND == 0) ? 4 : 8;
    char *dst = static_cast<char *>(a.partials) +
                (static_cast<size_t>(tile) * a.groups + group) * a.tile_cols * elt;
    const int n16 = static_cast<int>(width * elt / 16);
    const uint4 *src = reinterpret_cast<const uint4 *>(tile_raw);
    for (int k = tid; k < n16; k += kTiledThreads) reinterpret_cast<uint4 *>(dst)[k] = src[k];
    for (int b = n16 * 16 + tid; b < static_cast<int>(width * elt); b += kTiledThreads)
      dst[b] = reinterpret_cast<const char *>(tile_raw)[b];
    return;
  }
  if (homo) {
    for (int c = tid; c < width; c += kTiledThreads) {
      const unsigned n = accc[c];
      if (n == 0u) continue;
      if (KIND == 0)
        atomicAdd(static_cast<float *>(a.out) + c0 + c, __fmul_rn(__uint2float_rn(n), a.w));
      else
        atomicAdd(static_cast<unsigned long long *>(a.out) + c0 + c,
                  static_cast<unsigned long long>(static_cast<long long>(n) * a.q));
    }
    return;
  }
  if (KIND == 0 && (c0 & 3) == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0) {
    // 16-byte vector REDs (red.global.add.v4.f32), all-zero quads skipped
    float *out = static_cast<float *>(a.out) + c0;
    const int quads = width / 4;
    for (int qd = tid; qd < quads; qd += kTiledThreads) {
      const float4 v = reinterpret_cast<const float4 *>(accf)[qd];
      if (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f)
        asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                     ::"l"(out + 4 * qd), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
    for (int c = 4 * quads + tid; c < width; c += kTiledThreads) {
      const float v = accf[c];
      if (v != 0.f) atomicAdd(out + c, v);
    }
    return;
  }
  for (int c = tid; c < width; c += kTiledThreads) {
    if (KIND == 0) {
      const float v = accf[c];
      if (v != 0.f) atomicAdd(static_cast<float *>(a.out) + c0 + c, v);
    } else {
      const unsigned long long v = accq[c];
      if (v != 0ull) atomicAdd(static_cast<unsigned long long *>(a.out) + c0 + c, v);
    }
  }
}

// Sum the per-CTA partial tiles of k_csr_tiled, groups in ascending order:
// homogeneous weights -> fl32(count * w) or count * q; else the f32 / int64
// partial sums.  One thread per output column.
template <int KIND>
__global__ void __launch_bounds__(256)
k_csr_reduce(CsrTiledArgs a, int homo, int c16 = 0) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= a.n_cols) return;
  const int64_t tile = c / a.tile_cols, cc = c - tile * a.tile_cols;
  const size_t stride = static_cast<size_t>(a.tile_cols);
  const size_t base = static_cast<size_t>(tile) * a.groups * stride + cc;
  if (homo) {
    unsigned long long n = 0;
    if (c16) {       // 16-bit counts (k_csr_stream C16)
      const unsigned short *p = static_cast<const unsigned short *>(a.partials) + base;
      for (int g = 0; g < a.groups; ++g) n += __ldcs(p + g * stride);
    } else {
      const unsigned *p = static_cast<const unsigned *>(a.partials) + base;
      for (int g = 0; g < a.groups; ++g) n += __ldcs(p + g * stride);
    }
    if (KIND == 0) {
      const float v = __fmul_rn(__ull2float_rn(n), a.w);
      float *o = static_cast<float *>(a.out) + c;
      *o = a.accumulate ? __fadd_rn(*o, v) : v;
    } else {
      const long long v = static_cast<long long>(n) * a.q;
      long long *o = static_cast<long long *>(a.out) + c;
      *o = a.accumulate ? *o + v : v;
    }
  } else if (KIND == 0) {
    const float *p = static_cast<const float *>(a.partials) + base;
    float v = 0.f;
    for (int g = 0; g < a.groups; ++g) v = __fadd_rn(v, __ldcs(p + g * stride));
    float *o = static_cast<float *>(a.out) + c;
    *o = a.accumulate ? __fadd_rn(*o, v) : v;
  } else if (KIND == 2) {
    const int2 *p = static_cast<const int2 *>(a.partials) + base;
    long long hi = 0;
    unsigned long long lo = 0;
    for (int g = 0; g < a.groups; ++g) {
      const int2 x = __ldcs(p + g * stride);
      hi += x.x;
      lo += static_cast<unsigned>(x.y);
    }
    const float v = fix2_value(hi, lo, a.fix_bits);
    float *o = static_cast<float *>(a.out) + c;
    *o = a.accumulate ? __fadd_rn(*o, v) : v;
  } else {
    const long long *p = static_cast<const long long *>(a.partials) + base;
    long long v = 0;
    for (int g = 0; g < a.groups; ++g) v += __ldcs(p + g * stride);
    long long *o = static_cast<long long *>(a.out) + c;
    *o = a.accumulate ? *o + v : v;
  }
}

// ---------------------------------------------------------------- a3 + a4
struct JitSide {
  uint64_t seed;
  uint32_t K, L;
  uint32_t seg_first, n_seg;   // local segments [seg_first, seg_first + n_seg)
  float w0, w1;                // homo: (w, -); uniform: (lo, hi-lo); normal: (mu, sigma)
  long long q;                 // quantize(w0) for homo
  void *out;                   // indexed c - col_begin
  float geo_c;                 // 0: uniform gaps (J3); else fl32(log1p(-p)) (rule J10)
  uint32_t geo_cap;            // L + 1
};

// Gap e of a JIT row from its word x: U[1, K] (rules J3, J6) or Geo(p)
// (rule J10).  A template parameter of the hot kernels, so the paper's
// uniform sampler pays nothing for the other one.  The network kernels
// (step.cuh) use the uniform rule only.
template <bool GEO>
__device__ __forceinline__ uint32_t jit_gap(const JitSide &s, uint32_t x) {
  if (GEO) return geo_gap(x, s.geo_c, s.geo_cap);
  return bounded(1u, s.K, x);
}
// Offset of the first target from the segment start: rule J5 or G_0 - 1 (J10).
template <bool GEO>
__device__ __forceinline__ uint32_t jit_first(const JitSide &s, uint32_t row, uint32_t seg) {
  if (GEO)
    return geo_gap(philox_block(s.seed, kTagFirst, row, seg, 0).x, s.geo_c, s.geo_cap) - 1u;
  return first_offset(s.seed, s.K, row, seg);
}

struct JitScatterArgs {
  JitSide e, i;
  const float *v;              // nullable: non-event product, every row, v[r] * w (MV1)
  int64_t n_rows;
  int64_t split;
  uint32_t n_seg_max;
  uint32_t n_cols, col_begin, col_end;
  const int32_t *active;
  const int32_t *count;
  int32_t *zero_count;
  unsigned long long *events;
  unsigned long long *spikes;
  float keep_frac;
};

__device__ __forceinline__ JitSide pick(bool second, const JitSide &x,
                                        const JitSide &y) {
  JitSide s;
  s.seed = second ? y.seed : x.seed;
  s.K = second ? y.K : x.K;
  s.L = second ? y.L : x.L;
  s.seg_first = second ? y.seg_first : x.seg_first;
  s.n_seg = second ? y.n_seg : x.n_seg;
  s.w0 = second ? y.w0 : x.w0;
  s.w1 = second ? y.w1 : x.w1;
  s.q = second ? y.q : x.q;
  s.out = second ? y.out : x.out;
  s.geo_c = second ? y.geo_c : x.geo_c;
  s.geo_cap = second ? y.geo_cap : x.geo_cap;
  return s;
}

template <int LAW, int KIND>
__device__ __forceinline__ void jit_emit(const JitSide &s, uint32_t pos,
                                         uint32_t col_begin, float w, uint64_t pol,
                                         const float *v, float vr) {
  const int64_t c = static_cast<int64_t>(pos) - col_begin;
  if (v) {                     // MV1: fl32(v w), or the exact product rounded once
    if (KIND == 0) add_f32(s.out, c, __fmul_rn(vr, w), pol);
    else
      add_fix(s.out, c,
              __double2ll_rn(__dmul_rn(static_cast<double>(vr), static_cast<double>(w)) *
                             4294967296.0),
              pol);
    return;
  }
  if (KIND == 0) add_f32(s.out, c, w, pol);
  else add_fix(s.out, c, LAW == 0 ? s.q : quantize(w), pol);
}

template <int LAW, int KIND, bool GEO>
__global__ void __launch_bounds__(kScatterThreads)
k_jit_scatter(JitScatterArgs a) {
  const int n_active = a.v ? 0 : *a.count;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (a.zero_count) *a.zero_count = 0;
    if (a.spikes) atomicAdd(a.spikes, static_cast<unsigned long long>(n_active));
  }
  const uint32_t lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t n_items = (a.v ? a.n_rows : static_cast<int64_t>(n_active)) * a.n_seg_max;
  const uint64_t pol = make_policies(a.keep_frac).keep;
  unsigned long long ev = 0;
  for (int64_t item = warp0; item < n_items; item += n_warps) {
    const int64_t r = a.v ? item / a.n_seg_max : a.active[item / a.n_seg_max];
    const float vr = a.v ? __ldg(a.v + r) : 1.f;
    if (a.v && vr == 0.f) continue;                // contributes nothing
    const uint32_t sidx = static_cast<uint32_t>(item % a.n_seg_max);
    const bool inh = r >= a.split;
    const JitSide s = pick(inh, a.e, a.i);
    if (sidx >= s.n_seg) continue;
    const uint32_t row = static_cast<uint32_t>(inh ? r - a.split : r);
    const uint32_t seg = s.seg_first + sidx;
    const uint32_t seg_begin = seg * s.L;
    const uint32_t seg_end = min(seg_begin + s.L, a.n_cols);
    // The first gap block does not depend on the first offset: issue both
    // Philox evaluations back to back so their 10-round chains overlap.
    u32x4 g = philox_block(s.seed, kTagGap, row, seg, lane);
    uint32_t start = seg_begin + jit_first<GEO>(s, row, seg);
    uint32_t chunk = 0;
    while (start < seg_end) {                      // warp-uniform
      const uint32_t blk = chunk * 32u + lane;
      const uint32_t g0 = jit_gap<GEO>(s, g.x), g1 = jit_gap<GEO>(s, g.y);
      const uint32_t g2 = jit_gap<GEO>(s, g.z), g3 = jit_gap<GEO>(s, g.w);
      const uint32_t p1 = g0, p2 = g0 + g1, p3 = p2 + g2, t = p3 + g3;
      uint32_t incl = t;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= static_cast<uint32_t>(off)) incl += v;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t pos0 = start + (incl - t);
      if (pos0 < seg_end) {
        const uint32_t pos[4] = {pos0, pos0 + p1, pos0 + p2, pos0 + p3};
        float w[4] = {s.w0, s.w0, s.w0, s.w0};
        if (LAW == 1) {
          const u32x4 x = philox_block(s.seed, kTagWeight, row, seg, blk);
          w[0] = uniform_weight(x.x, s.w0, s.w1); w[1] = uniform_weight(x.y, s.w0, s.w1);
          w[2] = uniform_weight(x.z, s.w0, s.w1); w[3] = uniform_weight(x.w, s.w0, s.w1);
        } else if (LAW == 2) {
          const u32x4 x = philox_block(s.seed, kTagWeight, row, seg, 2u * blk);
          w[0] = normal_weight(x.x, x.y, s.w0, s.w1);
          if (pos[1] < seg_end) w[1] = normal_weight(x.z, x.w, s.w0, s.w1);
          if (pos[2] < seg_end) {
            const u32x4 y = philox_block(s.seed, kTagWeight, row, seg, 2u * blk + 1u);
            w[2] = normal_weight(y.x, y.y, s.w0, s.w1);
            if (pos[3] < seg_end) w[3] = normal_weight(y.z, y.w, s.w0, s.w1);
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (pos[k] < seg_end && pos[k] >= a.col_begin && pos[k] < a.col_end) {
            jit_emit<LAW, KIND>(s, pos[k], a.col_begin, w[k], pol, a.v, vr);
            ++ev;
          }
        }
      }
      start += total;
      ++chunk;
      if (start < seg_end) g = philox_block(s.seed, kTagGap, row, seg, chunk * 32u + lane);
    }
  }
  count_events(a.events, ev);
}

// Row counts / materialisation with the kernel's own generator (debug;
// also the gap-sampler cost benchmark: row counts are gap chains only).
template <bool GEO>
__global__ void __launch_bounds__(kScatterThreads)
k_jit_rows(JitSide s, int64_t n_rows, uint32_t n_cols, int law,
           const int64_t *__restrict__ indptr, int64_t *__restrict__ counts,
           int32_t *__restrict__ indices, float *__restrict__ data) {
  const uint32_t lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp0; r < n_rows; r += n_warps) {
    const uint32_t row = static_cast<uint32_t>(r);
    int64_t out = indptr ? indptr[r] : 0;
    for (uint32_t seg = 0; seg < s.n_seg; ++seg) {
      const uint32_t seg_begin = seg * s.L;
      const uint32_t seg_end = min(seg_begin + s.L, n_cols);
      uint32_t start = seg_begin + jit_first<GEO>(s, row, seg);
      uint32_t chunk = 0;
      while (start < seg_end) {
        const uint32_t blk = chunk * 32u + lane;
        const u32x4 g = philox_block(s.seed, kTagGap, row, seg, blk);
        const uint32_t g0 = jit_gap<GEO>(s, g.x), g1 = jit_gap<GEO>(s, g.y);
        const uint32_t g2 = jit_gap<GEO>(s, g.z), g3 = jit_gap<GEO>(s, g.w);
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
        int nv = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) nv += pos[k] < seg_end;
        // edges before this lane in this chunk
        uint32_t nv_incl = nv;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, nv_incl, off);
          if (lane >= static_cast<uint32_t>(off)) nv_incl += v;
        }
        const uint32_t nv_total = __shfl_sync(0xffffffffu, nv_incl, 31);
        if (indices) {
          int64_t o = out + (nv_incl - nv);
          float w[4] = {s.w0, s.w0, s.w0, s.w0};
          if (nv > 0 && law == 1) {
            const u32x4 x = philox_block(s.seed, kTagWeight, row, seg, blk);
            w[0] = uniform_weight(x.x, s.w0, s.w1); w[1] = uniform_weight(x.y, s.w0, s.w1);
            w[2] = uniform_weight(x.z, s.w0, s.w1); w[3] = uniform_weight(x.w, s.w0, s.w1);
          } else if (nv > 0 && law == 2) {
            const u32x4 x = philox_block(s.seed, kTagWeight, row, seg, 2u * blk);
            const u32x4 y = philox_block(s.seed, kTagWeight, row, seg, 2u * blk + 1u);
            w[0] = normal_weight(x.x, x.y, s.w0, s.w1); w[1] = normal_weight(x.z, x.w, s.w0, s.w1);
            w[2] = normal_weight(y.x, y.y, s.w0, s.w1); w[3] = normal_weight(y.z, y.w, s.w0, s.w1);
          }
          for (int k = 0; k < nv; ++k) {
            indices[o + k] = static_cast<int32_t>(pos[k]);
            if (data) data[o + k] = w[k];
          }
        }
        out += nv_total;
        start += total;
        ++chunk;
      }
    }
    if (counts && lane == 0) counts[r] = out;
  }
}

}  // namespace bp
