// persist.cuh -- the whole single-device LIF network time loop in ONE
// cooperative kernel, with the neuron update (a5, a6) and the event binning
// (a2-a4 for the next step) overlapped inside every SM.
//
// Why: in the two-kernel step (step.cuh) the update k_step is HBM-bound
// (~50 % issue utilisation) and the binning k_bin_sorted is issue/latency
// bound; run back to back they cost 64 + 30 us per step.  Here each SM runs
// one 1024-thread CTA whose warps are specialised:
//  * warps 0-15: two update groups of 256 threads.  A group takes tiles from
//    a global counter (snake order), runs exactly the k_step tile body
//    (step_tile), then publishes the tile id in a ready queue (release);
//  * warps 16-31: the binning group.  It pops ready tiles (acquire), compacts
//    the tile's spike words into a shared row list, regenerates (JIT) or
//    reads (CSR) the rows' targets into shared staging with a per-tile
//    histogram, and flushes the staging as one global slot claim per
//    non-empty destination tile plus record stores.
// A grid barrier closes each step (the buckets written in step n are read in
// step n+1).  Tiles move between SMs from step to step, so every cross-step
// load bypasses L1 (ld.global.cg in step_tile).  Results are bit-identical to
// the two-kernel path: event counts are integers and the update is the same
// code.  Waits on the queue are bounded (globaltimer) -- a timeout sets an
// error word that bp_network_counters reports instead of hanging the GPU.
#pragma once
#include <cooperative_groups.h>

#include "step.cuh"

namespace bp {

constexpr int kPerThreads = 1024;
#ifndef BP_PER_UPD_GROUPS
#define BP_PER_UPD_GROUPS 2
#endif
constexpr int kPerUpdGroups = BP_PER_UPD_GROUPS;               // 256-thread tile groups
constexpr int kPerUpdThreads = kPerUpdGroups * kStepThreads;   // warps 0-15
constexpr int kPerBinThreads = kPerThreads - kPerUpdThreads;   // warps 16-31
constexpr int kPerBinWarps = kPerBinThreads / 32;
constexpr int kPerStage = 16384;        // staged event records (64 KB)
constexpr int kPerRows = kTile + 512;   // compacted rows (one fully spiking tile + slack)
constexpr int kPerRowBatch = 64;        // rows staged between staging-capacity checks
constexpr int kPerMaxTiles = 4096;
#ifdef BP_PER_NO_BIN
constexpr bool kPerNoBin = true;    // timing experiment only: update role alone, no delivery
#else
constexpr bool kPerNoBin = false;
#endif
// control words, each on its own 128-byte line: [parity] tile counter, queue
// tail, queue head, step spike count; error flag
enum { kCtlTile = 0, kCtlTail = 2, kCtlHead = 4, kCtlSpk = 6, kCtlErr = 8, kCtlWords = 10 };
constexpr int kCtlStride = 32;
constexpr unsigned long long kPerTimeoutNs = 500000000ull;   // 0.5 s

struct PersistArgs {
  // step arguments by bucket parity b (in = buckets b, out = b ^ 1, snake
  // order and step-spike counter of the steps that read b): indexed with a
  // compile-time constant so they stay in the parameter bank
  StepArgs st[2];
  int bpar0;                 // bucket parity read by the first step
  uint32_t step0;            // global index of the first step (snake order, queue tags)
  int64_t n_steps;
  uint32_t *raster;          // nullable [n_steps][n_words]
  uint32_t *spikes;          // spike words when raster == null
  int64_t n_words;
  int32_t *counts_out;       // nullable [n_steps]
  unsigned long long *queue; // [2][n_tiles] ready tiles: (step + 1) << 32 | tile
  uint32_t *ctl;             // [kCtlWords * kCtlStride]
};

__host__ __device__ inline size_t persist_smem(uint32_t n_tiles) {
  return static_cast<size_t>(kPerUpdGroups) * 2 * kTile * 4 + kPerStage * 4 + kPerRows * 4 +
         2 * static_cast<size_t>(n_tiles) * 4;
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifdef BP_PERSIST_TIMING
// per block, per step (first 64 steps): [0] step start, [1] update role done,
// [2] binning role done, [3] after the grid barrier
__device__ unsigned long long g_per_t[148][64][4];
#define PER_MARK(s, k)                                                         \
  do {                                                                         \
    if ((s) < 64 && blockIdx.x < 148) g_per_t[blockIdx.x][s][k] = globaltimer(); \
  } while (0)
#else
#define PER_MARK(s, k) do {} while (0)
#endif

// One step of the persistent loop (st = the step arguments of this step's
// bucket parity).
template <int KIND>
__device__ __forceinline__ void persist_step(const PersistArgs &a, const StepArgs &st,
                                             int64_t s, unsigned char *psm) {
  const uint32_t n_tiles = st.n_tiles;
  int32_t *cnt = reinterpret_cast<int32_t *>(psm);                   // [groups][2][kTile]
  uint32_t *staged = reinterpret_cast<uint32_t *>(cnt + kPerUpdGroups * 2 * kTile);
  int32_t *rows = reinterpret_cast<int32_t *>(staged + kPerStage);   // [kPerRows]
  int32_t *hist = rows + kPerRows;                                    // [n_tiles]
  int32_t *gbase = hist + n_tiles;                                    // [n_tiles]
  __shared__ unsigned long long s_sp[kPerUpdGroups];
  __shared__ uint32_t s_tile[kPerUpdGroups];
  __shared__ int32_t s_nstaged, s_nrows, s_wsum[8];
  __shared__ uint32_t s_h, s_btile;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t *ctl = a.ctl;
  auto C = [ctl](int w, int par) { return ctl + (w + par) * kCtlStride; };
  const uint32_t sd = a.step0 + static_cast<uint32_t>(s);
  const int par = static_cast<int>(sd & 1u);
  uint32_t *spk = a.raster ? a.raster + s * a.n_words : a.spikes;
  if (blockIdx.x == 0 && tid == 0) {
    // the other parity's words were last used in step s-1 (before the grid
    // barrier) and are next used in step s+1 (after the next one)
    *C(kCtlTile, par ^ 1) = 0;
    *C(kCtlTail, par ^ 1) = 0;
    *C(kCtlHead, par ^ 1) = 0;
    *C(kCtlSpk, par ^ 1) = 0;
  }
  unsigned long long *queue = a.queue + static_cast<size_t>(par) * n_tiles;
  const unsigned long long tag = static_cast<unsigned long long>(sd + 1u) << 32;
  if (tid == 0) PER_MARK(s, 0);

  if (tid < kPerUpdThreads) {
    // ---- update: tiles from the global counter, k_step's tile body
    const int g = warp >> 3, gt = tid & (kStepThreads - 1);
    int32_t *ce = cnt + g * 2 * kTile, *ci = ce + kTile;
    // the next tile index is claimed while the current tile streams
    uint32_t next = 0;
    if (gt == 0) next = atomicAdd(C(kCtlTile, par), 1u);
    for (;;) {
      if (gt == 0) s_tile[g] = next;
      named_sync(1 + g, kStepThreads);
      const uint32_t idx = s_tile[g];
      if (idx >= n_tiles) break;
      if (gt == 0) next = atomicAdd(C(kCtlTile, par), 1u);
      const uint32_t tile = st.reverse ? n_tiles - 1u - idx : idx;
      step_tile<0, KIND, kStepThreads>(st, tile, gt, ce, ci, &s_sp[g], false, spk, nullptr,
                                       [g] { named_sync(1 + g, kStepThreads); });
      // publish: the group barrier orders every thread's spike words before
      // the leader's fence + release store (cumulativity), so no thread
      // waits for its own state stores to drain
      named_sync(1 + g, kStepThreads);
      if (gt == 0) {
        __threadfence();
        const uint32_t pos = atomicAdd(C(kCtlTail, par), 1u);
        st_release_u64(queue + pos, tag | tile);
      }
    }
    if (tid == 0) PER_MARK(s, 1);
  } else if (!kPerNoBin) {
    // ---- binning of this step's spikes, tile by tile as they are ready
    const int bt = tid - kPerUpdThreads, bw = bt >> 5;
    auto bsync = [] { named_sync(1 + kPerUpdGroups, kPerBinThreads); };
    const BinTarget &out = st.out;
    const ConnArgs &conn = st.conn;
    for (uint32_t t = bt; t < n_tiles; t += kPerBinThreads) hist[t] = 0;
    if (bt == 0) {
      s_nstaged = 0;
      s_nrows = 0;
    }
    bsync();
    uint32_t ev = 0;
    auto flush = [&]() {                       // staging -> buckets
      bsync();
      const int ns = min(s_nstaged, kPerStage);
      for (uint32_t t = bt; t < n_tiles; t += kPerBinThreads) {
        const int32_t c = hist[t];
        if (c) {
          gbase[t] = atomicAdd(out.out.cnt + t * kCntStride, c);
          hist[t] = 0;
        }
      }
      bsync();
      for (int i = bt; i < ns; i += kPerBinThreads) {
        const uint32_t rec = staged[i];
        const uint32_t loc = rec & ~kProjBit;
        const int32_t slot = atomicAdd(gbase + (loc >> kTileShift), 1);
        bin_store(out, (rec & kProjBit) ? 1u : 0u, loc, slot);
      }
      bsync();
      if (bt == 0) s_nstaged = 0;
      bsync();
    };
    auto stage = [&](int k_lo, int k_hi) {     // rows[k_lo, k_hi) -> staging
      if (conn.conn == 1) {
        for (int k = k_lo + bw; k < k_hi; k += kPerBinWarps)
          ev += stage_row<kPerStage>(conn, out, rows[k], staged, &s_nstaged, hist);
      } else if (conn.lane_rows) {
        for (int k = k_lo + bt; k < k_hi; k += kPerBinThreads)
          ev += stage_row_lane<kPerStage>(conn, out, rows[k], staged, &s_nstaged, hist);
      } else {
        for (int k0 = k_lo + bw; k0 < k_hi; k0 += kPerBinWarps * 32)
          ev += stage_rows_jit<kPerBinWarps, kPerStage>(conn, out, rows, k0, k_hi, staged,
                                                        &s_nstaged, hist);
      }
    };
    bool more = true;
    for (;;) {
      if (more) {
        if (bt == 0) {
          const uint32_t h = atomicAdd(C(kCtlHead, par), 1u);
          uint32_t tile = ~0u;
          if (h < n_tiles) {
            const unsigned long long t0 = globaltimer();
            for (;;) {
              const unsigned long long v = ld_acquire_u64(queue + h);
              if ((v & ~0xFFFFFFFFull) == tag) {
                tile = static_cast<uint32_t>(v);
                break;
              }
              if (globaltimer() - t0 > kPerTimeoutNs) {
                atomicExch(ctl + kCtlErr * kCtlStride, 1u);
                break;
              }
              __nanosleep(64);
            }
          }
          s_h = h;
          s_btile = tile;
        }
        bsync();
        const uint32_t h = s_h, tile = s_btile;
        if (h >= n_tiles) {
          more = false;
        } else if (tile != ~0u) {
          // the tile's 128 spike words -> rows (4 warps, one word per lane)
          uint32_t word = 0;
          const int64_t wi = (static_cast<int64_t>(tile) << kTileShift) / 32 + bt;
          if (bt < kTile / 32 && wi < a.n_words) word = __ldcg(spk + wi);
          const int c = __popc(word);
          int incl = c;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
          }
          if (bt < kTile / 32 && lane == 31) s_wsum[bw] = incl;
          bsync();
          const int base = s_nrows;
          int woff = 0;
          for (int k = 0; k < bw && k < kTile / 1024; ++k) woff += s_wsum[k];
          if (bt < kTile / 32) {
            int slot = base + woff + incl - c;
            const int32_t r0 = static_cast<int32_t>(wi << 5) + st.nrn.active_base;
            while (word) {
              const int b = __ffs(word) - 1;
              rows[slot++] = r0 + b;
              word &= word - 1u;
            }
          }
          bsync();
          if (bt == 0) {
            int tot = 0;
            for (int k = 0; k < kTile / 1024; ++k) tot += s_wsum[k];
            s_nrows = base + tot;
          }
        }
        bsync();
      }
      const int nr = s_nrows;
      if (nr >= kPerRowBatch || (!more && nr > 0)) {
        for (int k_lo = 0; k_lo < nr; k_lo += kPerRowBatch) {
          // room for ~kPerRowBatch rows of a few hundred events each
          if (s_nstaged > kPerStage - kPerRowBatch * 160) flush();
          stage(k_lo, min(nr, k_lo + kPerRowBatch));
          bsync();
        }
        if (bt == 0) s_nrows = 0;
        bsync();
      }
      if (!more) break;
    }
    flush();
    ev = __reduce_add_sync(0xffffffffu, ev);
    if (lane == 0 && ev) atomicAdd(st.events, static_cast<unsigned long long>(ev));
    if (tid == kPerUpdThreads) PER_MARK(s, 2);
  }
}

template <int KIND>
__global__ void __launch_bounds__(kPerThreads, 1) k_net_persist(PersistArgs a) {
  extern __shared__ __align__(16) unsigned char psm[];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  int bpar = a.bpar0;
  for (int64_t s = 0; s < a.n_steps; ++s) {
    if (bpar == 0) persist_step<KIND>(a, a.st[0], s, psm);
    else persist_step<KIND>(a, a.st[1], s, psm);
    grid.sync();
    if (threadIdx.x == 0) PER_MARK(s, 3);
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.counts_out) {
      const int par = static_cast<int>((a.step0 + static_cast<uint32_t>(s)) & 1u);
      a.counts_out[s] = static_cast<int32_t>(a.ctl[(kCtlSpk + par) * kCtlStride]);
    }
    bpar ^= 1;
  }
}

}  // namespace bp
