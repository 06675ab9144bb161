// bp_api.cu -- host side of libbp.so: argument validation, launch geometry
// and the per-step orchestration of the network (include/bp.h).
#include <cuda_runtime.h>

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <mutex>
#include <vector>
#include <cstdarg>
#include <new>
#include <utility>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/bp.h"
#include "neuron.cuh"
#include "scatter.cuh"
#include "csr_stream.cuh"
#include "jit_tiled.cuh"
#include "csr_grad.cuh"
#include "step.cuh"

namespace {

thread_local std::string g_last_error;

bp_status fail(bp_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
bp_status fail(bp_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

#define BP_CHECK(cond, status, ...) \
  do {                              \
    if (!(cond)) return fail(status, __VA_ARGS__); \
  } while (0)

#define BP_CUDA(call)                                                       \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess)                                                  \
      return fail(BP_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_));    \
  } while (0)

struct DeviceInfo {
  int checked = 0;
  int ok = 0;
  int sms = 148;
};
DeviceInfo g_dev[64];

// Sticky-error check + sm_100 check, cached per device.
bp_status device_ready(int *sms) {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess)
    return fail(BP_ERR_CUDA, "pending CUDA error: %s", cudaGetErrorString(e));
  int dev = 0;
  BP_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(BP_ERR_UNSUPPORTED, "device id %d", dev);
  DeviceInfo &d = g_dev[dev];
  if (!d.checked) {
    int major = 0, minor = 0;
    BP_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    BP_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    BP_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    d.ok = (major == 10 && minor == 0);
    d.checked = 1;
  }
  if (!d.ok) return fail(BP_ERR_UNSUPPORTED, "libbp is built for sm_100a only");
  if (sms) *sms = d.sms;
  return BP_OK;
}

bp_status launched() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(BP_ERR_CUDA, "launch failed: %s", cudaGetErrorString(e));
  return BP_OK;
}

inline cudaStream_t as_stream(bp_stream s) { return static_cast<cudaStream_t>(s); }
inline bool aligned(const void *p, size_t a) {
  return (reinterpret_cast<uintptr_t>(p) % a) == 0;
}
constexpr int64_t kMaxDim = (int64_t{1} << 31) - 1;

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// cudaFuncSetAttribute applies to the CURRENT device only: a kernel's opt-in
// is remembered per device ordinal (bit d of `mask`), so a second GPU used
// from the same process gets its own call.  Returns true the first time on
// this device.
bool first_on_device(std::atomic<uint64_t> &mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = uint64_t{1} << (dev & 63);
  return (mask.fetch_or(bit) & bit) == 0;
}

// Dense event delivery (per-neuron atomic counts, one neuron per thread) for
// the compute-bound HH model up to 2 M local neurons: the counts stay
// L2-resident and 4096-neuron tiles would leave SMs idle.
bool dense_delivery(int model, int64_t n_local) {
  return model == BP_MODEL_HH && n_local <= (int64_t{2} << 20);
}

// Workspace of the stateless scatter calls: [count int32 | pad to 256]
// [active int32[n_rows]].
struct Ws {
  int32_t *count;
  int32_t *active;
};
bp_status carve_ws(void *ws, size_t ws_bytes, int64_t n_rows, Ws *out) {
  BP_CHECK(ws != nullptr, BP_ERR_WORKSPACE, "workspace is NULL");
  BP_CHECK(aligned(ws, 256), BP_ERR_WORKSPACE, "workspace must be 256-byte aligned");
  BP_CHECK(ws_bytes >= bp_workspace_bytes(n_rows), BP_ERR_WORKSPACE,
           "workspace %zu bytes < %zu required", ws_bytes, bp_workspace_bytes(n_rows));
  out->count = static_cast<int32_t *>(ws);
  out->active = reinterpret_cast<int32_t *>(static_cast<char *>(ws) + 256);
  return BP_OK;
}

bool n_tiles_ok(int64_t n_tiles) { return n_tiles >= 1 && n_tiles <= 4; }

int grid_for_items(int64_t items_upper, int sms) {
  // one warp per item; at most 8 resident 256-thread blocks per SM
  const int64_t warps_per_block = bp::kScatterThreads / 32;
  int64_t blocks = (items_upper + warps_per_block - 1) / warps_per_block;
  const int64_t cap = static_cast<int64_t>(sms) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

// a1: warp-level claims for short vectors (k_compact_warp, no barriers);
// block-aggregated claims (k_compact) from 64 k words on, 4 words per thread
// once the vector fills every SM with 8 blocks of 1024-word iterations
// a1 into a counter that need not be zeroed: memset + the compaction kernels.
void compact_fresh(const uint32_t *spikes, int64_t n, int32_t *active, int32_t *count,
                   int sms, cudaStream_t st);

void launch_compact(const uint32_t *spikes, int64_t n, int32_t *active, int32_t *count,
                    int sms, cudaStream_t st, int32_t id_base = 0, int64_t skip_b = 0,
                    int64_t skip_e = 0) {
  const int64_t words = (n + 31) / 32;
  const int64_t cap = static_cast<int64_t>(sms) * 8;
  if (words < (int64_t{1} << 16)) {
    int64_t blocks = (words + 255) / 256;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    bp::k_compact_warp<<<static_cast<int>(blocks), 256, 0, st>>>(spikes, n, active, count,
                                                                 id_base, skip_b, skip_e);
    return;
  }
  const bool wide = words >= cap * 4 * bp::kCompactThreads;
  const int64_t per = (wide ? 8 : 1) * bp::kCompactThreads;
  int64_t blocks = (words + per - 1) / per;
  // long vectors: one 2048-word iteration per block (all loads in flight at
  // once, 16-byte loads); the grid is not capped at the resident blocks
  if (!wide && blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (wide)
    bp::k_compact<8><<<static_cast<int>(blocks), bp::kCompactThreads, 0, st>>>(
        spikes, n, active, count, id_base, skip_b, skip_e);
  else
    bp::k_compact<1><<<static_cast<int>(blocks), bp::kCompactThreads, 0, st>>>(
        spikes, n, active, count, id_base, skip_b, skip_e);
}

void compact_fresh(const uint32_t *spikes, int64_t n, int32_t *active, int32_t *count,
                   int sms, cudaStream_t st) {
  // (a single-block compaction that writes the count itself, without the
  // memset, measured 4-6 us slower per call on the config-2 cells: one SM
  // ranks the whole vector in sequential rounds)
  cudaMemsetAsync(count, 0, sizeof(int32_t), st);
  launch_compact(spikes, n, active, count, sms, st);
}

// ------------------------------------------------------------- CSR plan
struct CsrPlan {
  bool tiled;
  int64_t n_tiles;
  int32_t tile_cols, groups;
  size_t acc;            // shared accumulator bytes per column
  size_t partials_off;   // workspace offset of the partial tiles
  size_t ws_bytes;       // workspace needed for the reduce path
};

CsrPlan csr_plan(int64_t n_rows, int64_t n_cols, int out_kind, int sms) {
  CsrPlan p{};
  p.acc = out_kind == BP_OUT_FIX64 ? 8 : 4;
  const int64_t tile_cols = static_cast<int64_t>(200 * 1000 / p.acc);
  p.n_tiles = (n_cols + tile_cols - 1) / tile_cols;
  p.tiled = n_tiles_ok(p.n_tiles) && !std::getenv("BP_CSR_DIRECT");
  // multiple of 4 columns: the partial tiles are stored with 16-byte stores
  p.tile_cols = static_cast<int32_t>(
      round_up(static_cast<size_t>(n_cols < tile_cols ? n_cols : tile_cols), 4));
  p.groups = static_cast<int32_t>(sms / p.n_tiles > 0 ? sms / p.n_tiles : 1);
  p.partials_off = bp_workspace_bytes(n_rows);
  p.ws_bytes = p.partials_off +
               round_up(static_cast<size_t>(p.n_tiles) * p.groups * p.tile_cols * p.acc, 256);
  return p;
}

// Streamed CSR plan (csr_stream.cuh): column tiles sized to the shared
// memory left after the bulk-copy stages; one CTA per SM.
constexpr size_t kSmemOptin = 232448;     // 227 KB dynamic shared memory per block
constexpr int kMaxDelay = 16;             // synaptic delay steps (reading D1)
constexpr int kMaxSlots = kMaxDelay + 1;
constexpr int kStreamMaxTiles = 16;

struct StreamPlan {
  bool ok;
  bool c16;            // homogeneous counts in 16 bits
  int32_t n_tiles, tile_cols, groups;
  size_t smem, split_off, partials_off, ws_bytes, plan_bytes;
};

StreamPlan stream_plan_acc(int64_t n_rows, int64_t n_cols, int acc, bool homo, int sms) {
  StreamPlan p{};
  const size_t fixed = bp::stream_smem(0, acc, homo).total + bp::kStreamStaticSmem + 256;
  if (n_rows < 1 || n_cols < 1 || fixed >= kSmemOptin) return p;
  const int64_t max_cols = static_cast<int64_t>((kSmemOptin - fixed) / acc) & ~int64_t{7};
  const int64_t nt = (n_cols + max_cols - 1) / max_cols;
  if (nt > kStreamMaxTiles || nt > sms) return p;
  p.n_tiles = static_cast<int32_t>(nt);
  // partial rows stay 16-byte aligned (uint4 flush): 8 columns for 2-byte counts
  p.tile_cols = static_cast<int32_t>(
      round_up(static_cast<size_t>((n_cols + nt - 1) / nt), acc == 2 ? 8 : 4));
  p.groups = sms / p.n_tiles;
  p.smem = bp::stream_smem(p.tile_cols, acc, homo).total;
  p.plan_bytes = round_up(static_cast<size_t>(n_rows) * (nt - 1) * sizeof(int32_t), 256);
  if (p.smem + bp::kStreamStaticSmem > kSmemOptin || p.plan_bytes > (size_t{1} << 30)) return p;
  p.split_off = bp_workspace_bytes(n_rows);
  p.partials_off = p.split_off + p.plan_bytes;
  p.ws_bytes = p.partials_off +
               round_up(static_cast<size_t>(nt) * p.groups * p.tile_cols * acc, 256);
  p.ok = true;
  return p;
}

// BP_CSR_C16=1: 16-bit homogeneous counts (fewer, wider column tiles).
// Measured (100 k x 100 k, 10 %): p = 0.001 30.6 -> 26.6 us, p = 0.01 equal,
// p = 0.05 61.8 -> 65.8 us (two columns per word: more same-word conflicts
// among the lanes' atomics) -- so opt-in, not the default.
StreamPlan stream_plan(int64_t n_rows, int64_t n_cols, int out_kind, bool homo, int sms,
                       bool fix2 = false) {
  if (fix2 && !homo) return stream_plan_acc(n_rows, n_cols, 8, false, sms);   // rule T4 pairs
  const char *c16_env = std::getenv("BP_CSR_C16");
  if (homo && c16_env != nullptr && std::atoi(c16_env) != 0) {
    // 16-bit counts while a CTA streams < 2^16 rows: CTA g of a tile takes the
    // active ranks k with (k / W) % groups == g (W = bp::kStreamWarps), at
    // most W ceil(n / (W G))
    constexpr int64_t W = bp::kStreamWarps;
    StreamPlan p = stream_plan_acc(n_rows, n_cols, 2, homo, sms);
    if (p.ok && W * ((n_rows + W * p.groups - 1) / (W * p.groups)) < 65535) {
      p.c16 = true;
      return p;
    }
  }
  return stream_plan_acc(n_rows, n_cols, homo ? 4 : (out_kind == BP_OUT_FIX64 ? 8 : 4), homo,
                         sms);
}

template <int KIND, bool HOMO, bool C16 = false>
void stream_attr() {
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(bp::k_csr_stream<KIND, HOMO, C16>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmemOptin - bp::kStreamStaticSmem));
}

// Cooperative launch (every CTA resident: grid barriers allowed); false if
// the launch is refused.
template <int KIND, bool HOMO, bool C16 = false>
bool stream_coop(bp::CsrStreamArgs a, const StreamPlan &p, cudaStream_t st) {
  stream_attr<KIND, HOMO, C16>();
  void *args[] = {&a};
  if (cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(bp::k_csr_stream<KIND, HOMO, C16>),
                                  dim3(p.n_tiles * p.groups), dim3(bp::kStreamThreads), args,
                                  p.smem, st) == cudaSuccess)
    return true;
  cudaGetLastError();
  return false;
}

// With a.out set, try the cooperative launch (the kernel reduces the
// partial tiles itself after a grid barrier); returns false when it ran
// without the reduction, so the caller runs k_csr_reduce.
template <int KIND, bool HOMO, bool C16 = false>
bool launch_stream(bp::CsrStreamArgs a, const StreamPlan &p, cudaStream_t st) {
  stream_attr<KIND, HOMO, C16>();
  if (a.out != nullptr && stream_coop<KIND, HOMO, C16>(a, p, st)) return true;
  a.out = nullptr;
  bp::k_csr_stream<KIND, HOMO, C16><<<p.n_tiles * p.groups, bp::kStreamThreads, p.smem, st>>>(a);
  return false;
}

// ------------------------------------------------------------- JIT helpers
struct JitResolved {
  uint32_t K, L;
  float geo_c;        // rule J10: fl32(log1p(-p)); 0 for uniform gaps
  uint32_t geo_cap;   // L + 1
  double density;     // expected connection probability: 2/(K+1) or p
};

bp_status resolve_jit(const bp_jitconn *spec, int64_t n_cols, JitResolved *r) {
  BP_CHECK(spec != nullptr, BP_ERR_INVALID_ARG, "jitconn spec is NULL");
  uint32_t K = spec->conn_len;
  if (K == 0) {
    BP_CHECK(spec->prob > 0.0 && spec->prob <= 1.0, BP_ERR_INVALID_ARG,
             "prob %g not in (0, 1]", spec->prob);
    K = bp_conn_len(spec->prob);
  }
  BP_CHECK(K >= 1 && K < (1u << 31), BP_ERR_INVALID_ARG, "conn_len %u invalid", K);
  const uint64_t reach = static_cast<uint64_t>(n_cols) + 128ull * K;
  BP_CHECK(reach < (1ull << 32), BP_ERR_UNSUPPORTED,
           "n_cols + 128*K = %llu exceeds 32-bit positions",
           static_cast<unsigned long long>(reach));
  uint32_t L = spec->seg_len ? spec->seg_len : static_cast<uint32_t>(n_cols);
  BP_CHECK(L >= 1, BP_ERR_INVALID_ARG, "seg_len 0 with n_cols 0");
  BP_CHECK(spec->reserved == 0, BP_ERR_INVALID_ARG, "bp_jitconn.reserved must be 0");
  r->K = K;
  r->L = L;
  r->geo_c = 0.f;
  r->geo_cap = 0;
  r->density = 2.0 / (K + 1.0);
  if (spec->gap_law == BP_GAP_GEOMETRIC) {
    // rule J10: gaps Geo(p) by inversion, c = fl32(log1p(-p)) (-inf at p = 1)
    BP_CHECK(spec->prob > 0.0 && spec->prob <= 1.0, BP_ERR_INVALID_ARG,
             "geometric gaps need prob in (0, 1], got %g", spec->prob);
    const uint64_t greach = static_cast<uint64_t>(n_cols) + 128ull * (L + 1ull);
    BP_CHECK(greach < (1ull << 32), BP_ERR_UNSUPPORTED,
             "n_cols + 128*(seg_len+1) = %llu exceeds 32-bit positions",
             static_cast<unsigned long long>(greach));
    r->geo_c = static_cast<float>(std::log1p(-spec->prob));
    BP_CHECK(r->geo_c != 0.f, BP_ERR_UNSUPPORTED, "prob %g too small for fp32 log1p",
             spec->prob);
    r->geo_cap = L + 1u;
    r->density = spec->prob;
  } else {
    BP_CHECK(spec->gap_law == BP_GAP_UNIFORM, BP_ERR_INVALID_ARG, "gap_law %d",
             spec->gap_law);
  }
  return BP_OK;
}

bp::JitSide jit_side(const bp_jitconn *spec, const JitResolved &jr, int law,
                     float w0, float w1, int64_t col_begin, int64_t col_end,
                     void *out) {
  bp::JitSide s{};
  s.seed = spec->seed;
  s.K = jr.K;
  s.L = jr.L;
  s.seg_first = static_cast<uint32_t>(col_begin / jr.L);
  const int64_t seg_last = col_end > col_begin ? (col_end - 1) / jr.L : -1;
  s.n_seg = col_end > col_begin ? static_cast<uint32_t>(seg_last - s.seg_first + 1) : 0u;
  s.w0 = w0;
  s.w1 = (law == BP_LAW_UNIFORM) ? (w1 - w0) : w1;   // uniform: fp32 span
  s.q = llrint(static_cast<double>(w0) * 4294967296.0);
  s.out = out;
  s.geo_c = jr.geo_c;
  s.geo_cap = jr.geo_cap;
  return s;
}

template <int LAW, bool GEO>
void launch_jit_law(const bp::JitScatterArgs &a, int kind, int grid,
                    cudaStream_t st) {
  if (kind == BP_OUT_FIX64)
    bp::k_jit_scatter<LAW, 1, GEO><<<grid, bp::kScatterThreads, 0, st>>>(a);
  else
    bp::k_jit_scatter<LAW, 0, GEO><<<grid, bp::kScatterThreads, 0, st>>>(a);
}

template <bool GEO>
void launch_jit_g(const bp::JitScatterArgs &a, int law, int kind, int grid,
                  cudaStream_t st) {
  if (law == BP_LAW_HOMO) launch_jit_law<0, GEO>(a, kind, grid, st);
  else if (law == BP_LAW_UNIFORM) launch_jit_law<1, GEO>(a, kind, grid, st);
  else launch_jit_law<2, GEO>(a, kind, grid, st);
}

// geometric gaps (rule J10) when the projection's geo_c is set
void launch_jit(const bp::JitScatterArgs &a, int law, int kind, int grid,
                cudaStream_t st) {
  if (a.e.geo_c != 0.f) launch_jit_g<true>(a, law, kind, grid, st);
  else launch_jit_g<false>(a, law, kind, grid, st);
}

void launch_csr(const bp::CsrScatterArgs &a, int kind, int grid, cudaStream_t st) {
  if (kind == BP_OUT_FIX64)
    bp::k_csr_scatter<1><<<grid, bp::kScatterThreads, 0, st>>>(a);
  else
    bp::k_csr_scatter<0><<<grid, bp::kScatterThreads, 0, st>>>(a);
}

bp_status check_out(void *out, int out_kind) {
  BP_CHECK(out != nullptr, BP_ERR_INVALID_ARG, "out is NULL");
  BP_CHECK(out_kind == BP_OUT_F32 || out_kind == BP_OUT_FIX64, BP_ERR_INVALID_ARG,
           "out_kind %d", out_kind);
  BP_CHECK(aligned(out, out_kind == BP_OUT_FIX64 ? 8 : 4), BP_ERR_INVALID_ARG,
           "out misaligned");
  return BP_OK;
}

// Column tiles for bp_jitconn_event_mv_*: as many columns per CTA as its
// shared memory holds; when a row segment spans tiles, tile t regenerates
// the chain from the segment start up to its own end (work ~ t + 1), so it
// gets proportionally more CTAs.
// room left for k_jit_tiled's static shared memory
constexpr size_t kJitStaticSmem = 1024;

struct JitTilePlan {
  bool ok;
  bool c16;            // homogeneous counts in 16 bits
  int32_t n_tiles, tile_cols, grid;
  int32_t cta0[bp::kJitMaxTiles + 1];
  size_t partials_off, ws_bytes, smem;
};

JitTilePlan jit_tile_plan_acc(int64_t n_rows, int64_t width, int acc, int law, uint32_t L,
                              int sms) {
  JitTilePlan p{};
  const int64_t max_cols =
      ((static_cast<int64_t>(kSmemOptin) - kJitStaticSmem) / acc - 4) & ~int64_t{7};
  const int64_t nt = (width + max_cols - 1) / max_cols;
  if (nt > bp::kJitMaxTiles || nt > sms) return p;
  p.n_tiles = static_cast<int32_t>(nt);
  // tile rows of the partials stay 16-byte aligned (uint4 flush): 8 columns for 2-byte counts
  p.tile_cols = static_cast<int32_t>(
      round_up(static_cast<size_t>((width + nt - 1) / nt), acc == 2 ? 8 : 4));
  // cost of tile t per row: gap chain up to the tile's end ((t + 1) / nt of
  // a row spanning all tiles) + weights of the tile's own events (1 / nt);
  // in units of one row's gap chain: uniform weights ~1 (one Philox word per
  // event), normal ~6 (two words + fp64 log/sqrt/cos per event)
  const double wcost = law == BP_LAW_HOMO ? 0.0 : (law == BP_LAW_UNIFORM ? 1.0 : 3.0);
  const bool spans = L >= static_cast<uint64_t>(p.tile_cols) * 2;
  double wsum = 0.0, wt[bp::kJitMaxTiles];
  for (int t = 0; t < nt; ++t) {
    wt[t] = (spans ? t + 1.0 : 1.0) + wcost;
    wsum += wt[t];
  }
  int given = 0;
  p.cta0[0] = 0;
  for (int t = 0; t < nt; ++t) {
    int c = static_cast<int>(sms * wt[t] / wsum);
    if (c < 1) c = 1;
    if (t == nt - 1) c = sms - given > 1 ? sms - given : 1;
    given += c;
    p.cta0[t + 1] = given;
  }
  p.grid = given;
  p.smem = static_cast<size_t>(p.tile_cols + 4) * acc;
  p.partials_off = bp_workspace_bytes(n_rows);
  p.ws_bytes = p.partials_off + round_up(static_cast<size_t>(p.grid) * p.tile_cols * acc, 256);
  p.ok = p.grid <= sms;
  return p;
}

// n_seg: segments of a row inside the partition
JitTilePlan jit_tile_plan(int64_t n_rows, int64_t width, int out_kind, int law, uint32_t L,
                          int sms, bool vec = false, int64_t n_seg = 1) {
  if (width < 1 || n_rows < 1) return JitTilePlan{};
  if (law == BP_LAW_HOMO && !vec && !std::getenv("BP_JIT_C32")) {
    // homogeneous counts in 16 bits (k_jit_tiled C16) while no CTA can count
    // 2^16 events in one column: a CTA of a tile with G CTAs takes at most
    // 32 ceil(items / (32 G)) (row, segment) items, each adding <= 1
    JitTilePlan p = jit_tile_plan_acc(n_rows, width, 2, law, L, sms);
    const int64_t items = n_rows * n_seg;
    bool fits = p.ok;
    for (int t = 0; fits && t < p.n_tiles; ++t) {
      const int64_t g = p.cta0[t + 1] - p.cta0[t];
      fits = 32 * ((items + 32 * g - 1) / (32 * g)) < 65535;
    }
    if (fits) {
      p.c16 = true;
      return p;
    }
  }
  const int acc = ((law == BP_LAW_HOMO && !vec) || out_kind == BP_OUT_F32) ? 4 : 8;
  return jit_tile_plan_acc(n_rows, width, acc, law, L, sms);
}

template <int LAW, int KIND, bool VEC, bool GEO, bool C16 = false>
bool jit_tiled_coop(bp::JitTiledArgs a, const JitTilePlan &p, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(bp::k_jit_tiled<LAW, KIND, VEC, GEO, C16>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmemOptin - kJitStaticSmem));
  void *args[] = {&a};
  if (cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(bp::k_jit_tiled<LAW, KIND, VEC, GEO, C16>),
                                  dim3(p.grid), dim3(bp::kJitTiledThreads), args, p.smem,
                                  st) == cudaSuccess)
    return true;
  cudaGetLastError();
  return false;
}

template <bool VEC, bool GEO>
bool launch_jit_tiled_v(const bp::JitTiledArgs &a, int law, bool fix, const JitTilePlan &p,
                        cudaStream_t st) {
  if (law == BP_LAW_HOMO) {
    if (!VEC && p.c16)
      return fix ? jit_tiled_coop<0, 1, false, GEO, true>(a, p, st)
                 : jit_tiled_coop<0, 0, false, GEO, true>(a, p, st);
    return fix ? jit_tiled_coop<0, 1, VEC, GEO>(a, p, st)
               : jit_tiled_coop<0, 0, VEC, GEO>(a, p, st);
  }
  if (law == BP_LAW_UNIFORM)
    return fix ? jit_tiled_coop<1, 1, VEC, GEO>(a, p, st)
               : jit_tiled_coop<1, 0, VEC, GEO>(a, p, st);
  return fix ? jit_tiled_coop<2, 1, VEC, GEO>(a, p, st)
             : jit_tiled_coop<2, 0, VEC, GEO>(a, p, st);
}

bool launch_jit_tiled(const bp::JitTiledArgs &a, int law, int out_kind, bool vec,
                      const JitTilePlan &p, cudaStream_t st) {
  const bool fix = out_kind == BP_OUT_FIX64;
  if (a.s.geo_c != 0.f)
    return vec ? launch_jit_tiled_v<true, true>(a, law, fix, p, st)
               : launch_jit_tiled_v<false, true>(a, law, fix, p, st);
  return vec ? launch_jit_tiled_v<true, false>(a, law, fix, p, st)
             : launch_jit_tiled_v<false, false>(a, law, fix, p, st);
}

// Event scatter (spikes) or non-event product (v, reading MV1); exactly one
// of spikes / v is used.
bp_status jit_event_mv(int law, const bp_jitconn *spec, float w0, float w1,
                       const uint32_t *spikes, int64_t n_rows, int64_t n_cols,
                       int64_t col_begin, int64_t col_end, void *out,
                       int out_kind, uint32_t flags, void *ws, size_t ws_bytes,
                       bp_stream stream, const float *v = nullptr) {
  const bool vec = v != nullptr;
  int sms = 0;
  bp_status s = device_ready(&sms);
  if (s != BP_OK) return s;
  BP_CHECK(n_rows >= 0 && n_rows <= kMaxDim && n_cols >= 1 && n_cols <= kMaxDim,
           BP_ERR_SHAPE, "n_rows=%lld n_cols=%lld", (long long)n_rows, (long long)n_cols);
  BP_CHECK(col_begin >= 0 && col_begin <= col_end && col_end <= n_cols, BP_ERR_SHAPE,
           "partition [%lld, %lld) outside [0, %lld)", (long long)col_begin,
           (long long)col_end, (long long)n_cols);
  BP_CHECK(n_rows == 0 || vec || spikes != nullptr, BP_ERR_INVALID_ARG, "spikes is NULL");
  if (col_end > col_begin) {
    s = check_out(out, out_kind);
    if (s != BP_OK) return s;
  }
  BP_CHECK(!std::isnan(w0) && !std::isnan(w1), BP_ERR_INVALID_ARG, "NaN weight parameter");
  if (law == BP_LAW_UNIFORM)
    BP_CHECK(w0 <= w1, BP_ERR_INVALID_ARG, "w_low %g > w_high %g", w0, w1);
  if (law == BP_LAW_NORMAL)
    BP_CHECK(w1 >= 0.0f, BP_ERR_INVALID_ARG, "w_sigma %g < 0", w1);
  JitResolved jr;
  s = resolve_jit(spec, n_cols, &jr);
  if (s != BP_OK) return s;
  BP_CHECK(col_begin % jr.L == 0 && (col_end % jr.L == 0 || col_end == n_cols),
           BP_ERR_SHAPE, "partition [%lld, %lld) not aligned to seg_len %u",
           (long long)col_begin, (long long)col_end, jr.L);
  Ws w;
  s = carve_ws(ws, ws_bytes, n_rows, &w);
  if (s != BP_OK) return s;
  cudaStream_t st = as_stream(stream);
  const size_t elt = out_kind == BP_OUT_FIX64 ? 8 : 4;
  const int64_t n_seg_part = col_end > col_begin
                                 ? (col_end - 1) / jr.L - col_begin / jr.L + 1 : 0;
  const JitTilePlan tp =
      jit_tile_plan(n_rows, col_end - col_begin, out_kind, law, jr.L, sms, vec, n_seg_part);
  // short rows (< ~1000 events per active row in the partition; < ~2500 for
  // normal weights, whose Box-Muller is the same on both paths): the partial
  // tiles cost more than the atomics they save (normal, 100 k x 100 k, 10 %:
  // tiled 366 vs 398 us at p = 0.05, 105 vs 92 us at p = 0.01)
  const double row_events = jr.density * static_cast<double>(col_end - col_begin);
  const bool tiled = tp.ok && n_rows > 0 && ws_bytes >= tp.ws_bytes &&
                     !std::getenv("BP_JIT_DIRECT") &&
                     ((row_events >= (law == BP_LAW_NORMAL ? 2500.0 : 1000.0)) ||
                      std::getenv("BP_JIT_TILED"));
  if (tiled) {
    // shared-memory column tiles + in-kernel reduction (every output
    // column of the partition is written: no memset)
    if (!vec) {
      compact_fresh(spikes, n_rows, w.active, w.count, sms, st);
    }
    bp::JitTiledArgs t{};
    t.v = v;
    t.n_rows = n_rows;
    t.s = jit_side(spec, jr, law, w0, w1, col_begin, col_end, out);
    t.n_cols = static_cast<uint32_t>(n_cols);
    t.col_begin = static_cast<uint32_t>(col_begin);
    t.col_end = static_cast<uint32_t>(col_end);
    t.active = w.active;
    t.count = w.count;
    t.partials = static_cast<char *>(ws) + tp.partials_off;
    t.out = out;
    t.accumulate = (flags & BP_ACCUMULATE) ? 1 : 0;
    t.tile_cols = tp.tile_cols;
    t.n_tiles = tp.n_tiles;
    for (int k = 0; k <= tp.n_tiles; ++k) t.cta0[k] = tp.cta0[k];
    // CTA-parallel chains advance 32 chunks (4096 gaps) per round
    const uint64_t max_gap = jr.geo_c != 0.f ? jr.geo_cap : jr.K;
    t.cta_ok = (static_cast<uint64_t>(n_cols) + 4096ull * max_gap < (1ull << 32)) &&
               !std::getenv("BP_JIT_NO_CTA_CHAINS");
    t.row_chunks = static_cast<int>(row_events / 128.0) + 1;
    if (launch_jit_tiled(t, law, out_kind, vec, tp, st)) return launched();
  }
  if (!(flags & BP_ACCUMULATE) && col_end > col_begin)
    BP_CUDA(cudaMemsetAsync(out, 0, elt * (col_end - col_begin), st));
  if (n_rows == 0 || col_end == col_begin) return launched();
  if (!vec) {
    compact_fresh(spikes, n_rows, w.active, w.count, sms, st);
  }
  bp::JitScatterArgs a{};
  a.v = v;
  a.n_rows = n_rows;
  a.e = jit_side(spec, jr, law, w0, w1, col_begin, col_end, out);
  a.i = a.e;
  a.split = n_rows;
  a.n_seg_max = a.e.n_seg;
  a.n_cols = static_cast<uint32_t>(n_cols);
  a.col_begin = static_cast<uint32_t>(col_begin);
  a.col_end = static_cast<uint32_t>(col_end);
  a.active = w.active;
  a.count = w.count;
  launch_jit(a, law, out_kind, grid_for_items(n_rows * a.n_seg_max, sms), st);
  return launched();
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int bp_abi_version(void) { return 2; }

const char *bp_status_string(int status) {
  switch (status) {
    case BP_OK: return "BP_OK";
    case BP_ERR_INVALID_ARG: return "BP_ERR_INVALID_ARG";
    case BP_ERR_SHAPE: return "BP_ERR_SHAPE";
    case BP_ERR_UNSUPPORTED: return "BP_ERR_UNSUPPORTED";
    case BP_ERR_WORKSPACE: return "BP_ERR_WORKSPACE";
    case BP_ERR_CUDA: return "BP_ERR_CUDA";
    case BP_ERR_NCCL: return "BP_ERR_NCCL";
    default: return "BP_ERR_UNKNOWN";
  }
}

const char *bp_last_error(void) { return g_last_error.c_str(); }

uint32_t bp_conn_len(double prob) {
  // Rule J1: floor(2/p - 1), snapped to the nearest integer within
  // 1e-9 relative, at least 1; 0 for p outside (0, 1].
  if (!(prob > 0.0) || !(prob <= 1.0)) return 0;
  const double x = 2.0 / prob - 1.0;
  const double nearest = std::nearbyint(x);
  const double tol = 1e-9 * (std::fabs(x) > 1.0 ? std::fabs(x) : 1.0);
  double k = std::fabs(x - nearest) <= tol ? nearest : std::floor(x);
  if (k < 1.0) k = 1.0;
  if (k > 2147483647.0) return 0;
  return static_cast<uint32_t>(k);
}

size_t bp_workspace_bytes(int64_t n_rows) {
  if (n_rows < 0) n_rows = 0;
  return 256 + round_up(static_cast<size_t>(n_rows) * sizeof(int32_t), 256);
}

size_t bp_csrmv_workspace_bytes(int64_t n_rows, int64_t n_cols, int out_kind) {
  int sms = 148;
  if (device_ready(&sms) != BP_OK) sms = 148;
  if (n_rows < 0 || n_cols < 1) return bp_workspace_bytes(n_rows);
  const CsrPlan p = csr_plan(n_rows, n_cols, out_kind, sms);
  size_t need = p.tiled ? p.ws_bytes : bp_workspace_bytes(n_rows);
  for (int homo = 0; homo < 2; ++homo) {
    for (int fix2 = 0; fix2 < 2; ++fix2) {
      const StreamPlan sp = stream_plan(n_rows, n_cols, out_kind, homo != 0, sms, fix2 != 0);
      if (sp.ok && sp.ws_bytes > need) need = sp.ws_bytes;
    }
  }
  return need;
}

size_t bp_jitconn_workspace_bytes(int64_t n_rows, int64_t col_begin, int64_t col_end,
                                  int out_kind) {
  int sms = 148;
  if (device_ready(&sms) != BP_OK) sms = 148;
  size_t need = bp_workspace_bytes(n_rows);
  // largest accumulator: int64 fixed point with per-edge weights
  const JitTilePlan p = jit_tile_plan(n_rows, col_end - col_begin, out_kind, BP_LAW_UNIFORM,
                                      0u, sms);
  if (p.ok && p.ws_bytes > need) need = p.ws_bytes;
  const JitTilePlan h = jit_tile_plan(n_rows, col_end - col_begin, out_kind, BP_LAW_HOMO, 0u, sms);
  if (h.ok && h.ws_bytes > need) need = h.ws_bytes;
  return need;
}

bp_status bp_compact_spikes(const uint32_t *spikes, int64_t n, int32_t *active,
                            int32_t *count, bp_stream stream) {
  int sms = 0;
  bp_status s = device_ready(&sms);
  if (s != BP_OK) return s;
  BP_CHECK(n >= 0 && n <= kMaxDim, BP_ERR_SHAPE, "n=%lld", (long long)n);
  BP_CHECK(count != nullptr && (n == 0 || (spikes && active)), BP_ERR_INVALID_ARG,
           "NULL pointer");
  cudaStream_t st = as_stream(stream);
  BP_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t), st));
  if (n > 0) launch_compact(spikes, n, active, count, sms, st);
  return launched();
}

namespace {
bp_status csrmv_impl(const void *plan, size_t plan_bytes, const int64_t *indptr,
                     const int32_t *indices, const float *data, float w_homo, int64_t n_rows,
                     int64_t n_cols, const uint32_t *spikes, void *out, int out_kind,
                     uint32_t flags, void *ws, size_t ws_bytes, bp_stream stream,
                     int32_t fix_bits = -1) {
  int sms = 0;
  bp_status s = device_ready(&sms);
  if (s != BP_OK) return s;
  BP_CHECK(n_rows >= 0 && n_rows <= kMaxDim && n_cols >= 1 && n_cols <= kMaxDim,
           BP_ERR_SHAPE, "n_rows=%lld n_cols=%lld", (long long)n_rows, (long long)n_cols);
  BP_CHECK(n_rows == 0 || (indptr && indices && spikes), BP_ERR_INVALID_ARG,
           "NULL indptr/indices/spikes");
  s = check_out(out, out_kind);
  if (s != BP_OK) return s;
  Ws w;
  s = carve_ws(ws, ws_bytes, n_rows, &w);
  if (s != BP_OK) return s;
  cudaStream_t st = as_stream(stream);
  const size_t elt = out_kind == BP_OUT_FIX64 ? 8 : 4;
  const bool homo = data == nullptr;
  // rule T4: heterogeneous fp32 output accumulated in scaled fixed point
  // (the plan's analysis chose fix_bits; -1 = fp32 atomics)
  const bool fix2 = !homo && out_kind == BP_OUT_F32 && fix_bits >= 0 &&
                    !std::getenv("BP_CSR_NO_T4");
  const StreamPlan sp = stream_plan(n_rows, n_cols, out_kind, homo, sms, fix2);
  if (sp.ok && ws_bytes >= sp.ws_bytes && aligned(indices, 16) && (homo || aligned(data, 16)) &&
      !std::getenv("BP_CSR_TILED") && !std::getenv("BP_CSR_ATOMIC_FLUSH") &&
      !std::getenv("BP_CSR_DIRECT")) {
    // a1 -> split points -> bulk-copy streamed tiles -> ordered reduction
    // (every output column written by the reduction: no memset)
    void *partials = static_cast<char *>(ws) + sp.partials_off;
    int32_t *split = static_cast<int32_t *>(const_cast<void *>(plan));
    const bool need_split = sp.n_tiles > 1 && (split == nullptr || plan_bytes < sp.plan_bytes);
    const bool coop = !std::getenv("BP_CSR_NO_FUSE");
    if (need_split) split = reinterpret_cast<int32_t *>(static_cast<char *>(ws) + sp.split_off);
    bp::CsrStreamArgs ca{indices, data, indptr, split, w.active, w.count, indptr + n_rows,
                         partials, sp.tile_cols, sp.groups, sp.n_tiles,
                         (flags & BP_ACCUMULATE) ? 1 : 0, n_cols, coop ? out : nullptr, w_homo,
                         llrint(static_cast<double>(w_homo) * 4294967296.0),
                         fix2 ? fix_bits : 0, 0, 0};
    auto stream_kernel = [&](const bp::CsrStreamArgs &c) {
      if (fix2) return launch_stream<2, false>(c, sp, st);
      if (homo)
        return sp.c16 ? (out_kind == BP_OUT_FIX64 ? launch_stream<1, true, true>(c, sp, st)
                                                  : launch_stream<0, true, true>(c, sp, st))
                      : (out_kind == BP_OUT_FIX64 ? launch_stream<1, true>(c, sp, st)
                                                  : launch_stream<0, true>(c, sp, st));
      return out_kind == BP_OUT_FIX64 ? launch_stream<1, false>(c, sp, st)
                                      : launch_stream<0, false>(c, sp, st);
    };
    compact_fresh(spikes, n_rows, w.active, w.count, sms, st);
    if (need_split) {
      bp::CsrSplitArgs sa{indptr, indices, w.active, w.count, n_rows, split, sp.n_tiles,
                          sp.tile_cols, n_cols};
      int64_t sblocks = (n_rows + 7) / 8;
      if (sblocks > static_cast<int64_t>(sms) * 8) sblocks = static_cast<int64_t>(sms) * 8;
      bp::k_csr_split<<<static_cast<int>(sblocks), 256, 0, st>>>(sa);
    }
    const bool fused = stream_kernel(ca);
    if (fused) return launched();
    bp::CsrTiledArgs t{};
    t.w = w_homo;
    t.q = ca.q;
    t.out = out;
    t.n_cols = n_cols;
    t.tile_cols = sp.tile_cols;
    t.groups = sp.groups;
    t.partials = partials;
    t.accumulate = ca.accumulate;
    t.fix_bits = ca.fix_bits;
    const int rgrid = static_cast<int>((n_cols + 255) / 256);
    if (fix2) bp::k_csr_reduce<2><<<rgrid, 256, 0, st>>>(t, 0, 0);
    else if (out_kind == BP_OUT_FIX64) bp::k_csr_reduce<1><<<rgrid, 256, 0, st>>>(t, homo, sp.c16);
    else bp::k_csr_reduce<0><<<rgrid, 256, 0, st>>>(t, homo, sp.c16);
    return launched();
  }
  CsrPlan tp = csr_plan(n_rows, n_cols, out_kind, sms);
  const bool reduce_path = tp.tiled && ws_bytes >= tp.ws_bytes && n_rows > 0 &&
                           !std::getenv("BP_CSR_ATOMIC_FLUSH");
  // the reduce kernel writes every output column: no memset needed there
  if (!(flags & BP_ACCUMULATE) && !reduce_path) BP_CUDA(cudaMemsetAsync(out, 0, elt * n_cols, st));
  if (n_rows == 0) return launched();
  compact_fresh(spikes, n_rows, w.active, w.count, sms, st);
  bp::CsrScatterArgs a{};
  a.e.indptr = indptr;
  a.e.indices = indices;
  a.e.data = data;
  a.e.w = w_homo;
  a.e.q = llrint(static_cast<double>(w_homo) * 4294967296.0);
  a.e.out = out;
  a.i = a.e;
  a.split = n_rows;
  a.active = w.active;
  a.count = w.count;
  // Column-tiled shared-memory aggregation when the output fits <= 4 tiles
  // of <= 200 KB (scatter.cuh, k_csr_tiled); partial tiles reduced by
  // k_csr_reduce when the workspace holds them, else flushed with REDs;
  // outputs wider than 4 tiles: one RED per event (k_csr_scatter).
  const size_t acc = tp.acc;
  const int64_t n_tiles = tp.n_tiles;
  if (tp.tiled) {
    bp::CsrTiledArgs t{};
    t.indptr = indptr; t.indices = indices; t.data = data; t.w = w_homo;
    t.q = a.e.q; t.out = out; t.n_cols = n_cols;
    t.tile_cols = tp.tile_cols;
    t.groups = tp.groups;
    t.active = w.active; t.count = w.count;
    t.partials = reduce_path ? static_cast<char *>(ws) + tp.partials_off : nullptr;
    t.accumulate = (flags & BP_ACCUMULATE) ? 1 : 0;
    t.vec = aligned(indices, 16) && (data == nullptr || aligned(data, 16)) ? 1 : 0;
    const size_t smem = static_cast<size_t>(t.tile_cols) * acc;
    static std::atomic<uint64_t> attr_set[2] = {{0}, {0}};
    if (first_on_device(attr_set[out_kind])) {
      if (out_kind == BP_OUT_FIX64)
        BP_CUDA(cudaFuncSetAttribute(bp::k_csr_tiled<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1000 + 1024));
      else
        BP_CUDA(cudaFuncSetAttribute(bp::k_csr_tiled<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1000 + 1024));
    }
    const int grid = static_cast<int>(n_tiles * t.groups);
    if (out_kind == BP_OUT_FIX64) bp::k_csr_tiled<1><<<grid, bp::kTiledThreads, smem, st>>>(t);
    else bp::k_csr_tiled<0><<<grid, bp::kTiledThreads, smem, st>>>(t);
    if (reduce_path) {
      const int rgrid = static_cast<int>((n_cols + 255) / 256);
      if (out_kind == BP_OUT_FIX64) bp::k_csr_reduce<1><<<rgrid, 256, 0, st>>>(t, data == nullptr);
      else bp::k_csr_reduce<0><<<rgrid, 256, 0, st>>>(t, data == nullptr);
    }
    return launched();
  }
  launch_csr(a, out_kind, grid_for_items(n_rows, sms), st);
  return launched();
}
}  // namespace

bp_status bp_event_csrmv(const int64_t *indptr, const int32_t *indices,
                         const float *data, float w_homo, int64_t n_rows,
                         int64_t n_cols, const uint32_t *spikes, void *out,
                         int out_kind, uint32_t flags, void *ws,
                         size_t ws_bytes, bp_stream stream) {
  return csrmv_impl(nullptr, 0, indptr, indices, data, w_homo, n_rows, n_cols, spikes, out,
                    out_kind, flags, ws, ws_bytes, stream);
}

bp_status bp_csrmv_gather(const int64_t *indptr, const int32_t *indices, const float *data,
                          float w_homo, int64_t n_rows, int64_t n_cols, const uint32_t *spikes,
                          void *out, int out_kind, uint32_t flags, bp_stream stream) {
  int sms = 0;
  bp_status s = device_ready(&sms);
  if (s != BP_OK) return s;
  BP_CHECK(n_rows >= 0 && n_rows <= kMaxDim && n_cols >= 1 && n_cols <= kMaxDim,
           BP_ERR_SHAPE, "n_rows=%lld n_cols=%lld", (long long)n_rows, (long long)n_cols);
  BP_CHECK(n_rows == 0 || (indptr && indices && spikes), BP_ERR_INVALID_ARG,
           "NULL indptr/indices/spikes");
  s = check_out(out, out_kind);
  if (s != BP_OK) return s;
  if (n_rows == 0) return BP_OK;
  bp::CsrGatherArgs a{indptr, indices, data, w_homo,
                      llrint(static_cast<double>(w_homo) * 4294967296.0), n_rows, spikes, out,
                      (flags & BP_ACCUMULATE) ? 1 : 0};
  int64_t blocks = (n_rows + 7) / 8;
  if (blocks > static_cast<int64_t>(sms) * 16) blocks = static_cast<int64_t>(sms) * 16;
  cudaStream_t st = as_stream(stream);
  if (out_kind == BP_OUT_FIX64)
    bp::k_csr_gather<1><<<static_cast<int>(blocks), bp::kGatherThreads, 0, st>>>(a);
  else
    bp::k_csr_gather<0><<<static_cast<int>(blocks), bp::kGatherThreads, 0, st>>>(a);
  return launched();
}

bp_status bp_event_csrmv_grad(const int64_t *indptr, const int32_t *indices, const float *data,
                              float w_homo, int64_t n_rows, int64_t n_cols,
                              const uint32_t *spikes, const float *gy, float *grad_data,
                              float *grad_events, double *grad_w, bp_stream stream) {
  int sms = 0;
  bp_status s = device_ready(&sms);
  if (s != BP_OK) return s;
  BP_CHECK(n_rows >= 0 && n_rows <= kMaxDim && n_cols >= 1 && n_cols <= kMaxDim,
           BP_ERR_SHAPE, "n_rows=%lld n_cols=%lld", (long long)n_rows, (long long)n_cols);
  BP_CHECK(n_rows == 0 || (indptr && indices && spikes && gy), BP_ERR_INVALID_ARG,
           "NULL indptr/indices/spikes/gy");
  BP_CHECK(grad_w == nullptr || data == nullptr, BP_ERR_INVALID_ARG,
           "grad_w is the gradient of the homogeneous weight (data must be NULL)");
  cudaStream_t st = as_stream(stream);
  if (grad_w) BP_CUDA(cudaMemsetAsync(grad_w, 0, sizeof(double), st));
  if (n_rows == 0) return launched();
  bp::CsrGradArgs a{indptr, indices, data, w_homo, n_rows, spikes, gy,
                    grad_data, grad_events, grad_w};
  int64_t blocks = (n_rows + 7) / 8;
  if (blocks > static_cast<int64_t>(sms) * 16) blocks = static_cast<int64_t>(sms) * 16;
  bp::k_csr_grad<<<static_cast<int>(blocks), bp::kGatherThreads, 0, st>>>(a);
  return launched();
}

size_t bp_csrmv_plan_bytes(int64_t n_rows, int64_t n_cols, int out_kind, int homo) {
  int sms = 148;
  if (device_ready(&sms) != BP_OK) sms = 148;
  const StreamPlan sp = stream_plan(n_rows, n_cols, out_kind, homo != 0, sms);
  size_t need = sp.ok && sp.n_tiles > 1 ? sp.plan_bytes : 0;
  if (!homo && out_kind == BP_OUT_F32) {
    // rule T4: the split points of the 8-byte-pair tiles, and the analysis's
    // column sums of |w| behind them
    const StreamPlan s2 = stream_plan(n_rows, n_cols, out_kind, false, sms, true);
    if (s2.ok)
      need = std::max(need, (s2.n_tiles > 1 ? s2.plan_bytes : 0) +
                                round_up(static_cast<size_t>(n_cols + 64) * 4, 256));
  }
  return need;
}

namespace {
// max of v[0..n) (non-negative floats) into *out: one block
__global__ void __launch_bounds__(1024) k_max_f32(const float *v, int64_t n, float *out) {
  __shared__ float red[32];
  float m = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, v[i]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = red[threadIdx.x];
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) *out = m;
  }
}

bp_status write_split(const int64_t *indptr, const int32_t *indices, int64_t n_rows,
                      int64_t n_cols, const StreamPlan &sp, int32_t *plan, int sms,
                      cudaStream_t st) {
  bp::CsrSplitArgs sa{indptr, indices, nullptr, nullptr, n_rows, plan, sp.n_tiles, sp.tile_cols,
                      n_cols};
  int64_t blocks = (n_rows + 7) / 8;
  if (blocks > static_cast<int64_t>(sms) * 16) blocks = static_cast<int64_t>(sms) * 16;
  bp::k_csr_split<<<static_cast<int>(blocks), 256, 0, st>>>(sa);
  return launched();
}
}  // namespace

bp_status bp_csrmv_plan(const int64_t *indptr, const int32_t *indices, const float *data,
                        int64_t n_rows, int64_t n_cols, int out_kind, int homo, void *plan,
                        size_t plan_bytes, bp_csrmv_plan_info *info, void *ws,
                        size_t ws_bytes, bp_stream stream) {
  int sms = 0;
  bp_status s = device_ready(&sms);
  if (s != BP_OK) return s;
  BP_CHECK(n_rows >= 0 && n_rows <= kMaxDim && n_cols >= 1 && n_cols <= kMaxDim,
           BP_ERR_SHAPE, "n_rows=%lld n_cols=%lld", (long long)n_rows, (long long)n_cols);
  BP_CHECK(out_kind == BP_OUT_F32 || out_kind == BP_OUT_FIX64, BP_ERR_INVALID_ARG,
           "out_kind %d", out_kind);
  BP_CHECK(homo || data != nullptr, BP_ERR_INVALID_ARG, "heterogeneous plan needs data");
  cudaStream_t st = as_stream(stream);
  bp_csrmv_plan_info inf{};
  inf.f32_fixed_bits = -1;
  const StreamPlan sp = stream_plan(n_rows, n_cols, out_kind, homo != 0, sms);
  inf.n_tiles = sp.ok ? sp.n_tiles : 0;
  if (info) *info = inf;
  if (!sp.ok || n_rows == 0) return BP_OK;                   // nothing to precompute
  BP_CHECK(indptr && indices && (plan || plan_bytes == 0), BP_ERR_INVALID_ARG,
           "NULL indptr/indices/plan");
  const size_t need = bp_csrmv_plan_bytes(n_rows, n_cols, out_kind, homo);
  BP_CHECK(plan_bytes >= need, BP_ERR_WORKSPACE, "plan %zu bytes < %zu required", plan_bytes,
           need);
  BP_CHECK(need == 0 || aligned(plan, 16), BP_ERR_WORKSPACE, "plan must be 16-byte aligned");
  int32_t *split = static_cast<int32_t *>(plan);
  if (sp.n_tiles > 1) {
    s = write_split(indptr, indices, n_rows, n_cols, sp, split, sms, st);
    if (s != BP_OK) return s;
  }
  const StreamPlan s2 = stream_plan(n_rows, n_cols, out_kind, false, sms, true);
  if (homo || out_kind != BP_OUT_F32 || !s2.ok || n_rows >= (int64_t{1} << 24) || !ws ||
      ws_bytes < std::max(sp.ws_bytes, s2.ws_bytes) || !aligned(indices, 16) ||
      !aligned(data, 16) || std::getenv("BP_CSR_NO_T4"))
    return BP_OK;
  // Rule T4 analysis: column sums of |w| over ALL rows (an fp32 atomic pass of
  // the stream kernel with every row active) bound every partial sum of any
  // call; from B = max column sum choose the largest F with
  // B 2^(F-8) + 2 n_rows < 2^31, so hi words never overflow, and lo words stay
  // below n_rows 2^8 < 2^32.
  Ws w;
  s = carve_ws(ws, ws_bytes, n_rows, &w);
  if (s != BP_OK) return s;
  const size_t colsum_off = s2.n_tiles > 1 ? s2.plan_bytes : 0;
  float *colsum = reinterpret_cast<float *>(static_cast<char *>(plan) + colsum_off);
  float *colmax = colsum + n_cols;
  bp::CsrStreamArgs ca{indices, data, indptr, split, nullptr, nullptr, indptr + n_rows,
                       static_cast<char *>(ws) + sp.partials_off, sp.tile_cols, sp.groups,
                       sp.n_tiles, 0, n_cols, colsum, 1.f, 0, 0, 1, n_rows};
  if (!launch_stream<0, false>(ca, sp, st)) {
    bp::CsrTiledArgs t{};
    t.out = colsum;
    t.n_cols = n_cols;
    t.tile_cols = sp.tile_cols;
    t.groups = sp.groups;
    t.partials = ca.partials;
    bp::k_csr_reduce<0><<<static_cast<int>((n_cols + 255) / 256), 256, 0, st>>>(t, 0, 0);
  }
  k_max_f32<<<1, 1024, 0, st>>>(colsum, n_cols, colmax);
  float bmax = 0.f;
  BP_CUDA(cudaMemcpyAsync(&bmax, colmax, sizeof(float), cudaMemcpyDeviceToHost, st));
  BP_CUDA(cudaStreamSynchronize(st));
  if (!std::isfinite(bmax)) return BP_OK;
  // the fp32 column sums carry <= n_rows 2^-24 relative rounding: 1 % margin
  const double B = std::max(static_cast<double>(bmax) * 1.01, 1e-30);
  const double room = 2147483648.0 - 2.0 * static_cast<double>(n_rows) - 16.0;
  int F = static_cast<int>(std::floor(std::log2(room / B))) + 8;
  if (F > 100) F = 100;
  if (F >= 8 && B * std::ldexp(1.0, F - 8) + 2.0 * n_rows < 2147483648.0) {
    inf.f32_fixed_bits = F;
    inf.n_tiles = s2.n_tiles;
    inf.max_col_abs_sum = bmax;
    if (s2.n_tiles > 1) {
      s = write_split(indptr, indices, n_rows, n_cols, s2, split, sms, st);
      if (s != BP_OK) return s;
    }
  }
  if (info) *info = inf;
  return BP_OK;
}

bp_status bp_event_csrmv_planned(const void *plan, size_t plan_bytes,
                                 const bp_csrmv_plan_info *info, const int64_t *indptr,
                                 const int32_t *indices, const float *data, float w_homo,
                                 int64_t n_rows, int64_t n_cols, const uint32_t *spikes,
                                 void *out, int out_kind, uint32_t flags, void *ws,
                                 size_t ws_bytes, bp_stream stream) {
  return csrmv_impl(plan, plan_bytes, indptr, indices, data, w_homo, n_rows, n_cols, spikes,
                    out, out_kind, flags, ws, ws_bytes, stream,
                    info ? info->f32_fixed_bits : -1);
}

bp_status bp_jitconn_event_mv_homo(const bp_jitconn *spec, float weight,
                                   const uint32_t *spikes, int64_t n_rows,
                                   int64_t n_cols, int64_t col_begin,
                                   int64_t col_end, void *out, int out_kind,
                                   uint32_t flags, void *ws, size_t ws_bytes,
                                   bp_stream stream) {
  return jit_event_mv(BP_LAW_HOMO, spec, weight, 0.0f, spikes, n_rows, n_cols,
                      col_begin, col_end, out, out_kind, flags, ws, ws_bytes,
                      stream);
}

bp_status bp_jitconn_event_mv_uniform(const bp_jitconn *spec, float w_low,
                                      float w_high, const uint32_t *spikes,
                                      int64_t n_rows, int64_t n_cols,
                                      int64_t col_begin, int64_t col_end,
                                      void *out, int out_kind, uint32_t flags,
                                      void *ws, size_t ws_bytes,
                                      bp_stream stream) {
  return jit_event_mv(BP_LAW_UNIFORM, spec, w_low, w_high, spikes, n_rows,
                      n_cols, col_begin, col_end, out, out_kind, flags, ws,
                      ws_bytes, stream);
}

bp_status bp_jitconn_event_mv_normal(const bp_jitconn *spec, float w_mu,
                                     float w_sigma, const uint32_t *spikes,
                                     int64_t n_rows, int64_t n_cols,
                                     int64_t col_begin, int64_t col_end,
                                     void *out, int out_kind, uint32_t flags,
                                     void *ws, size_t ws_bytes,
                                     bp_stream stream) {
  return jit_event_mv(BP_LAW_NORMAL, spec, w_mu, w_sigma, spikes, n_rows,
                      n_cols, col_begin, col_end, out, out_kind, flags, ws,
                      ws_bytes, stream);
}

bp_status bp_jitconn_mv_homo(const bp_jitconn *spec, float weight, const float *v,
                             int64_t n_rows, int64_t n_cols, int64_t col_begin,
                             int64_t col_end, void *out, int out_kind, uint32_t flags,
                             void *ws, size_t ws_bytes, bp_stream stream) {
  if (n_rows > 0 && v == nullptr) return fail(BP_ERR_INVALID_ARG, "v is NULL");
  return jit_event_mv(BP_LAW_HOMO, spec, weight, 0.0f, nullptr, n_rows, n_cols, col_begin,
                      col_end, out, out_kind, flags, ws, ws_bytes, stream,
                      v ? v : reinterpret_cast<const float *>(&weight));
}

bp_status bp_jitconn_mv_uniform(const bp_jitconn *spec, float w_low, float w_high,
                                const float *v, int64_t n_rows, int64_t n_cols,
                                int64_t col_begin, int64_t col_end, void *out, int out_kind,
                                uint32_t flags, void *ws, size_t ws_bytes, bp_stream stream) {
  if (n_rows > 0 && v == nullptr) return fail(BP_ERR_INVALID_ARG, "v is NULL");
  return jit_event_mv(BP_LAW_UNIFORM, spec, w_low, w_high, nullptr, n_rows, n_cols, col_begin,
                      col_end, out, out_kind, flags, ws, ws_bytes, stream,
                      v ? v : reinterpret_cast<const float *>(&w_low));
}

bp_status bp_jitconn_mv_normal(const bp_jitconn *spec, float w_mu, float w_sigma,
                               const float *v, int64_t n_rows, int64_t n_cols,
                               int64_t col_begin, int64_t col_end, void *out, int out_kind,
                               uint32_t flags, void *ws, size_t ws_bytes, bp_stream stream) {
  if (n_rows > 0 && v == nullptr) return fail(BP_ERR_INVALID_ARG, "v is NULL");
  return jit_event_mv(BP_LAW_NORMAL, spec, w_mu, w_sigma, nullptr, n_rows, n_cols, col_begin,
                      col_end, out, out_kind, flags, ws, ws_bytes, stream,
                      v ? v : reinterpret_cast<const float *>(&w_mu));
}

bp_status bp_jitconn_row_counts(const bp_jitconn *spec, int64_t n_rows,
                                int64_t n_cols, int64_t *counts,
                                bp_stream stream) {
  int sms = 0;
  bp_status s = device_ready(&sms);
  if (s != BP_OK) return s;
  BP_CHECK(n_rows >= 0 && n_rows <= kMaxDim && n_cols >= 1 && n_cols <= kMaxDim,
           BP_ERR_SHAPE, "bad shape");
  BP_CHECK(n_rows == 0 || counts, BP_ERR_INVALID_ARG, "counts is NULL");
  JitResolved jr;
  s = resolve_jit(spec, n_cols, &jr);
  if (s != BP_OK) return s;
  if (n_rows == 0) return BP_OK;
  bp::JitSide side = jit_side(spec, jr, BP_LAW_HOMO, 0.f, 0.f, 0, n_cols, nullptr);
  auto rows = side.geo_c != 0.f ? bp::k_jit_rows<true> : bp::k_jit_rows<false>;
  rows<<<grid_for_items(n_rows, sms), bp::kScatterThreads, 0, as_stream(stream)>>>(
      side, n_rows, static_cast<uint32_t>(n_cols), BP_LAW_HOMO, nullptr, counts, nullptr,
      nullptr);
  return launched();
}

}  // extern "C"

namespace {
// In-place inclusive scan of v[1..n] with v[0] = 0 (one block: the exclusive
// prefix of the row counts, i.e. a CSR indptr).
__global__ void __launch_bounds__(1024) k_indptr_scan(int64_t *v, int64_t n) {
  __shared__ long long part[1024];
  const int64_t per = (n + 1023) / 1024;
  const int64_t lo = 1 + threadIdx.x * per, hi = min(n + 1, lo + per);
  long long sum = 0;
  for (int64_t i = lo; i < hi; ++i) sum += v[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int t = 0; t < 1024; ++t) {
      const long long x = part[t];
      part[t] = run;
      run += x;
    }
    v[0] = 0;
  }
  __syncthreads();
  long long run = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) {
    run += v[i];
    v[i] = run;
  }
}
}  // namespace

extern "C" {

bp_status bp_jitconn_indptr(const bp_jitconn *spec, int64_t n_rows, int64_t n_cols,
                            int64_t *indptr, bp_stream stream) {
  BP_CHECK(indptr != nullptr, BP_ERR_INVALID_ARG, "indptr is NULL");
  bp_status s = bp_jitconn_row_counts(spec, n_rows, n_cols, indptr + 1, stream);
  if (s != BP_OK) return s;
  k_indptr_scan<<<1, 1024, 0, as_stream(stream)>>>(indptr, n_rows);
  return launched();
}

bp_status bp_jitconn_materialize(const bp_jitconn *spec, int law, float w0,
                                 float w1, int64_t n_rows, int64_t n_cols,
                                 const int64_t *indptr, int32_t *indices,
                                 float *data, bp_stream stream) {
  int sms = 0;
  bp_status s = device_ready(&sms);
  if (s != BP_OK) return s;
  BP_CHECK(n_rows >= 0 && n_rows <= kMaxDim && n_cols >= 1 && n_cols <= kMaxDim,
           BP_ERR_SHAPE, "bad shape");
  BP_CHECK(law >= 0 && law <= 2, BP_ERR_INVALID_ARG, "law %d", law);
  BP_CHECK(n_rows == 0 || (indptr && indices), BP_ERR_INVALID_ARG, "NULL indptr/indices");
  JitResolved jr;
  s = resolve_jit(spec, n_cols, &jr);
  if (s != BP_OK) return s;
  if (n_rows == 0) return BP_OK;
  bp::JitSide side = jit_side(spec, jr, law, w0, w1, 0, n_cols, nullptr);
  auto rows = side.geo_c != 0.f ? bp::k_jit_rows<true> : bp::k_jit_rows<false>;
  rows<<<grid_for_items(n_rows, sms), bp::kScatterThreads, 0, as_stream(stream)>>>(
      side, n_rows, static_cast<uint32_t>(n_cols), law, indptr, nullptr, indices, data);
  return launched();
}

}  // extern "C"

// ------------------------------------------------------------ neuron step
namespace {

bp_status fill_neuron_args(const bp_neuron_params *p, const bp_neuron_state *st,
                           int64_t n, bp::NeuronArgs *a) {
  BP_CHECK(p != nullptr && st != nullptr, BP_ERR_INVALID_ARG, "NULL params/state");
  BP_CHECK(p->model == BP_MODEL_LIF || p->model == BP_MODEL_HH, BP_ERR_INVALID_ARG,
           "model %d", p->model);
  BP_CHECK(st->g_kind == BP_OUT_F32 || st->g_kind == BP_OUT_FIX64 || st->g_kind == BP_OUT_FIX32,
           BP_ERR_INVALID_ARG, "g_kind %d", st->g_kind);
  BP_CHECK(st->g_kind != BP_OUT_FIX32 || (st->g_frac_bits >= 0 && st->g_frac_bits <= 30),
           BP_ERR_INVALID_ARG, "g_frac_bits %d not in [0, 30]", st->g_frac_bits);
  BP_CHECK(n >= 0 && n <= kMaxDim, BP_ERR_SHAPE, "n=%lld", (long long)n);
  if (n > 0) {
    BP_CHECK(st->v && st->g_exc && st->g_inh, BP_ERR_INVALID_ARG, "NULL v/g");
    if (p->model == BP_MODEL_LIF)
      BP_CHECK(st->ref != nullptr, BP_ERR_INVALID_ARG, "NULL ref");
    else
      BP_CHECK(st->m && st->h && st->n_gate, BP_ERR_INVALID_ARG, "NULL m/h/n");
    BP_CHECK(aligned(st->g_exc, st->g_kind == BP_OUT_FIX64 ? 8 : 4) &&
                 aligned(st->g_inh, st->g_kind == BP_OUT_FIX64 ? 8 : 4),
             BP_ERR_INVALID_ARG, "g misaligned");
  }
  BP_CHECK(p->ref_steps >= 0 && p->ref_steps <= 255, BP_ERR_INVALID_ARG,
           "ref_steps %d not in [0, 255]", p->ref_steps);
  *a = bp::NeuronArgs{};
  a->v_rest = p->v_rest; a->v_reset = p->v_reset; a->v_th = p->v_th; a->r = p->r;
  a->i_ext = p->i_ext; a->e_exc = p->e_exc; a->e_inh = p->e_inh; a->alpha_v = p->alpha_v;
  a->alpha_e = p->alpha_e; a->alpha_i = p->alpha_i;
  a->alpha_e32 = static_cast<float>(p->alpha_e);
  a->alpha_i32 = static_cast<float>(p->alpha_i);
  a->ref_steps = p->ref_steps;
  a->c_m = p->c_m; a->g_l = p->g_l; a->e_l = p->e_l; a->g_na = p->g_na; a->e_na = p->e_na;
  a->g_k = p->g_k; a->e_k = p->e_k; a->v_t = p->v_t; a->dt = p->dt; a->v_spike = p->v_spike;
  a->v = st->v; a->g_e = st->g_exc; a->g_i = st->g_inh; a->ref = st->ref;
  a->m = st->m; a->h = st->h; a->nk = st->n_gate;
  a->n = n;
  a->frac_bits = st->g_frac_bits ? st->g_frac_bits : 20;
  a->inv_scale = std::ldexp(1.0, -a->frac_bits);
  a->inv_scale32 = static_cast<float>(a->inv_scale);
  a->a_e_q = llrint(p->alpha_e * 4294967296.0);   // rule F2 decay factors
  a->a_i_q = llrint(p->alpha_i * 4294967296.0);
  return BP_OK;
}

void launch_neuron(const bp::NeuronArgs &a, int model, int g_kind, cudaStream_t st) {
  if (a.n == 0) return;
  const int blocks = static_cast<int>((a.n + 255) / 256);
  if (model == BP_MODEL_LIF) {
    if (g_kind == BP_OUT_FIX64) bp::k_lif<1><<<blocks, 256, 0, st>>>(a);
    else if (g_kind == BP_OUT_FIX32) bp::k_lif<2><<<blocks, 256, 0, st>>>(a);
    else bp::k_lif<0><<<blocks, 256, 0, st>>>(a);
  } else {
    if (g_kind == BP_OUT_FIX64) bp::k_hh<1><<<blocks, 256, 0, st>>>(a);
    else if (g_kind == BP_OUT_FIX32) bp::k_hh<2><<<blocks, 256, 0, st>>>(a);
    else bp::k_hh<0><<<blocks, 256, 0, st>>>(a);
  }
}

}  // namespace

extern "C" bp_status bp_neuron_step(const bp_neuron_params *params,
                                    const bp_neuron_state *state, int64_t n,
                                    uint32_t *spikes_out, int32_t *active_out,
                                    int32_t *count_out, int64_t active_base,
                                    bp_stream stream) {
  bp_status s = device_ready(nullptr);
  if (s != BP_OK) return s;
  bp::NeuronArgs a;
  s = fill_neuron_args(params, state, n, &a);
  if (s != BP_OK) return s;
  BP_CHECK(n == 0 || spikes_out != nullptr, BP_ERR_INVALID_ARG, "spikes_out is NULL");
  BP_CHECK(active_out == nullptr || count_out != nullptr, BP_ERR_INVALID_ARG,
           "active_out without count_out");
  BP_CHECK(active_base >= 0 && active_base + n <= kMaxDim, BP_ERR_SHAPE, "active_base");
  a.spikes = spikes_out;
  a.active = active_out;
  a.count = count_out;
  a.active_base = static_cast<int32_t>(active_base);
  launch_neuron(a, params->model, state->g_kind, as_stream(stream));
  return launched();
}

// ================================================================ NCCL
// NCCL is resolved at run time (dlopen), so libbp.so has no link-time NCCL
// dependency and shares the process's already loaded libnccl.so.2 (torch's)
// when there is one.
namespace {

struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int *) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bp_status nccl_load() {
  std::lock_guard<std::mutex> lock(g_nccl_mu);
  if (!g_nccl.tried) {
    g_nccl.tried = true;
    void *h = nullptr;
    if (const char *env = std::getenv("BP_NCCL_LIB")) h = dlopen(env, RTLD_NOW);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (h) {
      g_nccl.get_unique_id = reinterpret_cast<decltype(g_nccl.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
      g_nccl.comm_init_rank = reinterpret_cast<decltype(g_nccl.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
      g_nccl.all_gather = reinterpret_cast<decltype(g_nccl.all_gather)>(dlsym(h, "ncclAllGather"));
      g_nccl.comm_destroy = reinterpret_cast<decltype(g_nccl.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      g_nccl.error_string = reinterpret_cast<decltype(g_nccl.error_string)>(dlsym(h, "ncclGetErrorString"));
      g_nccl.get_version = reinterpret_cast<decltype(g_nccl.get_version)>(dlsym(h, "ncclGetVersion"));
      g_nccl.ok = g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.all_gather &&
                  g_nccl.comm_destroy && g_nccl.error_string;
    }
  }
  if (!g_nccl.ok) return fail(BP_ERR_NCCL, "NCCL not available (libnccl.so.2 not loadable)");
  return BP_OK;
}

#define BP_NCCL(call)                                                       \
  do {                                                                      \
    ncclResult_t r_ = (call);                                               \
    if (r_ != ncclSuccess)                                                  \
      return fail(BP_ERR_NCCL, "%s: %s", #call, g_nccl.error_string(r_));   \
  } while (0)

}  // namespace

extern "C" bp_status bp_nccl_version(int32_t *version) {
  BP_CHECK(version != nullptr, BP_ERR_INVALID_ARG, "version is NULL");
  bp_status s = nccl_load();
  if (s != BP_OK) return s;
  int v = 0;
  if (g_nccl.get_version) BP_NCCL(g_nccl.get_version(&v));
  *version = v;
  return BP_OK;
}

extern "C" bp_status bp_nccl_unique_id(uint8_t *out) {
  BP_CHECK(out != nullptr, BP_ERR_INVALID_ARG, "out is NULL");
  bp_status s = nccl_load();
  if (s != BP_OK) return s;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  BP_NCCL(g_nccl.get_unique_id(&id));
  std::memcpy(out, &id, sizeof id);
  return BP_OK;
}

// ================================================================ network
struct bp_network {
  bp_network_desc d;
  int sms;
  int64_t n_local, local_words, global_words;
  unsigned long long *counters;   // [0] spikes delivered, [1] events
  int32_t *count;                 // [2] ping-pong active counts
  int32_t *active[2];             // ping-pong active lists (n entries each)
  bp::NeuronArgs neuron;
  // weight classes (step.cuh): projections with the same (receptor, weight)
  // share one count array; ncls_kernel 2 = class 0 -> g_e, class 1 -> g_i
  int n_cls = 2, ncls_kernel = 2;
  float cls_w[bp::kMaxCls] = {};
  int cls_rec[bp::kMaxCls] = {};
  int proj_cls[BP_MAX_PROJ] = {};
  JitResolved jr[BP_MAX_PROJ] = {};
  bool all_jit = true;
  bp::NetProj *proj_dev = nullptr;  // device projection table (in bk_mem)
  // profiling: 3 events per step (before scatter, between, after update)
  cudaEvent_t *prof_ev = nullptr;
  cudaEvent_t xev = nullptr;      // bp_network_update_overlap: spike words final
  int64_t prof_cap = 0, prof_used = 0;
  float keep_frac = 0.f;          // L2 evict_last fraction of g (cache.cuh)
  // fused-step event buckets (step.cuh), owned by the network
  uint32_t n_tiles = 0, cap = 0;
  bp::Buckets bk[kMaxSlots] = {};  // ring of delay + 1 slots (reading D1)
  void *bk_mem = nullptr;
  size_t dev_bytes = 0;
  int delay = 1;                  // synaptic delay in steps (desc.delay_steps)
  int slots = 2;                  // bucket ring: step n reads slot n % slots and its
                                  // spikes are binned into slot (n + delay) % slots
  int64_t steps_done = 0;
  bp::ConnArgs conn{};
  // small networks (step.cuh k_small_net): whole time loop in one CTA
  bool small = false;
  int32_t *small_active = nullptr;   // pending spikes (global ids) + count
  int32_t *small_count = nullptr;
  int32_t *small_steps = nullptr;    // per-step spike counts scratch
  int64_t small_steps_cap = 0;
  int64_t prof_steps = 0;
  // dense delivery: events as per-neuron atomic counts (cap 0), small
  // blocks (k_step_dense) -- compute-bound networks that fill few tiles
  bool dense = false;
  bool debug_nan = false;         // BP_DEBUG_NAN=1: count non-finite V after every step
  bool hh_fused = true;           // dense HH kernel delivers its own spikes (BP_HH_FUSED)
  // BP_EXCHANGE_NCCL: the library's own spike all-gather
  bool nccl = false;
  ncclComm_t comm = nullptr;
  cudaStream_t comm_st = nullptr;
  cudaEvent_t ev_spk = nullptr;     // this step's local spike words are final
  cudaEvent_t ev_gath[2] = {};      // all-gather of step parity p done
  uint32_t *spk[2] = {};            // global spike vectors (D >= 2: alternate per step)
  int64_t part_words = 0;           // words per rank in the gathered vector
};

namespace {

struct NetWsLayout {
  size_t active0, active1, spk1, total;
};

NetWsLayout network_ws_layout(const bp_network_desc *d) {
  NetWsLayout l{};
  const size_t list = round_up(static_cast<size_t>(d->n) * sizeof(int32_t), 256);
  l.active0 = 256;
  l.active1 = 256 + list;
  l.spk1 = 256 + 2 * list;
  l.total = l.spk1;
  if (d->exchange == BP_EXCHANGE_NCCL && d->delay_steps > 1) {
    // second gathered spike vector (the exchange of step n overlaps step n + 1)
    const int64_t words = d->world > 0 && d->part_len > 0 ? d->world * (d->part_len / 32)
                                                          : (d->n + 31) / 32;
    l.total += round_up(static_cast<size_t>(words) * sizeof(uint32_t), 256);
  }
  return l;
}

bp_status validate_network(const bp_network_desc *d) {
  BP_CHECK(d != nullptr, BP_ERR_INVALID_ARG, "desc is NULL");
  BP_CHECK(d->n >= 1 && d->n <= kMaxDim, BP_ERR_SHAPE, "n=%lld", (long long)d->n);
  BP_CHECK(d->col_begin >= 0 && d->col_begin < d->col_end && d->col_end <= d->n,
           BP_ERR_SHAPE, "partition [%lld, %lld)", (long long)d->col_begin,
           (long long)d->col_end);
  BP_CHECK(d->col_end - d->col_begin < (int64_t{1} << 30), BP_ERR_SHAPE,
           "a process owns at most 2^30 - 1 neurons");
  BP_CHECK(d->col_begin % 32 == 0, BP_ERR_SHAPE, "col_begin not a multiple of 32");
  BP_CHECK(d->col_end % 32 == 0 || d->col_end == d->n, BP_ERR_SHAPE,
           "col_end must be a multiple of 32 or n");
  BP_CHECK(d->n_proj >= 1 && d->n_proj <= BP_MAX_PROJ, BP_ERR_INVALID_ARG,
           "n_proj %d not in [1, %d]", d->n_proj, BP_MAX_PROJ);
  for (int p = 0; p < d->n_proj; ++p) {
    const bp_projection &P = d->proj[p];
    BP_CHECK(P.conn == BP_CONN_JIT || P.conn == BP_CONN_CSR, BP_ERR_INVALID_ARG,
             "projection %d: conn %d", p, P.conn);
    BP_CHECK(P.receptor == BP_RECEPTOR_EXC || P.receptor == BP_RECEPTOR_INH,
             BP_ERR_INVALID_ARG, "projection %d: receptor %d", p, P.receptor);
    BP_CHECK(P.pre_begin >= 0 && P.pre_begin <= P.pre_end && P.pre_end <= d->n,
             BP_ERR_SHAPE, "projection %d: rows [%lld, %lld)", p, (long long)P.pre_begin,
             (long long)P.pre_end);
    BP_CHECK(std::isfinite(P.weight), BP_ERR_INVALID_ARG, "projection %d: weight", p);
    BP_CHECK(P.reserved == 0, BP_ERR_INVALID_ARG, "projection %d: reserved must be 0", p);
    if (P.conn == BP_CONN_CSR)
      BP_CHECK(P.pre_end == P.pre_begin || (P.indptr && P.indices), BP_ERR_INVALID_ARG,
               "projection %d: NULL CSR", p);
  }
  BP_CHECK(d->spikes != nullptr && aligned(d->spikes, 4), BP_ERR_INVALID_ARG,
           "spikes NULL/misaligned");
  BP_CHECK(d->params.model == d->model, BP_ERR_INVALID_ARG, "params.model != model");
  BP_CHECK(d->delay_steps >= 0 && d->delay_steps <= kMaxDelay, BP_ERR_INVALID_ARG,
           "delay_steps %d not in [0, %d]", d->delay_steps, kMaxDelay);
  BP_CHECK(d->state.g_kind == d->g_kind, BP_ERR_INVALID_ARG, "state.g_kind != g_kind");
  BP_CHECK(d->exchange == BP_EXCHANGE_CALLER || d->exchange == BP_EXCHANGE_NCCL,
           BP_ERR_INVALID_ARG, "exchange %d", d->exchange);
  BP_CHECK(d->reserved2 == 0, BP_ERR_INVALID_ARG, "reserved2 must be 0");
  if (d->exchange == BP_EXCHANGE_NCCL) {
    BP_CHECK(d->world >= 1 && d->rank >= 0 && d->rank < d->world, BP_ERR_INVALID_ARG,
             "rank %d of world %d", d->rank, d->world);
    BP_CHECK(d->part_len > 0 && d->part_len % 32 == 0, BP_ERR_SHAPE,
             "part_len %lld must be a positive multiple of 32", (long long)d->part_len);
    BP_CHECK(d->part_len * d->world >= d->n, BP_ERR_SHAPE, "world * part_len < n");
    const int64_t lo = d->rank * d->part_len;
    const int64_t hi = std::min<int64_t>(d->n, lo + d->part_len);
    BP_CHECK(d->col_begin == lo && d->col_end == hi, BP_ERR_SHAPE,
             "rank %d must own [%lld, %lld)", d->rank, (long long)lo, (long long)hi);
  }
  BP_CHECK(d->ws != nullptr && aligned(d->ws, 256), BP_ERR_WORKSPACE,
           "workspace NULL or not 256-byte aligned");
  BP_CHECK(d->ws_bytes >= bp_network_workspace_bytes(d), BP_ERR_WORKSPACE,
           "workspace too small");
  return BP_OK;
}

// Weight classes: projections with the same (receptor, weight) share one
// count array.  The standard layout (at most one weight per receptor:
// Listing S3) keeps class 0 = excitatory, class 1 = inhibitory and the
// kernels' one-class-per-receptor fold; anything else uses the general merge
// (up to 4 classes, exact integer sums; fp32 needs weights on the 2^-32 grid).
bp_status assign_classes(bp_network *net) {
  const bp_network_desc &d = net->d;
  float w_rec[2] = {0.f, 0.f};
  int n_w[2] = {0, 0};
  for (int p = 0; p < d.n_proj; ++p) {
    const int r = d.proj[p].receptor;
    if (n_w[r] == 0 || std::memcmp(&w_rec[r], &d.proj[p].weight, sizeof(float)) != 0) {
      if (n_w[r] == 0) w_rec[r] = d.proj[p].weight;
      n_w[r] += (n_w[r] == 0 || std::memcmp(&w_rec[r], &d.proj[p].weight, sizeof(float)) != 0);
    }
  }
  bool standard = n_w[0] <= 1 && n_w[1] <= 1;
  if (const char *env = std::getenv("BP_MERGE_GENERAL")) standard = standard && !std::atoi(env);
  if (standard) {
    net->n_cls = 2;
    net->ncls_kernel = 2;
    net->cls_w[0] = w_rec[0];
    net->cls_w[1] = w_rec[1];
    net->cls_rec[0] = 0;
    net->cls_rec[1] = 1;
    for (int p = 0; p < d.n_proj; ++p) net->proj_cls[p] = d.proj[p].receptor;
    return BP_OK;
  }
  net->n_cls = 0;
  net->ncls_kernel = bp::kMaxCls;
  for (int p = 0; p < d.n_proj; ++p) {
    int c = 0;
    for (; c < net->n_cls; ++c)
      if (net->cls_rec[c] == d.proj[p].receptor &&
          std::memcmp(&net->cls_w[c], &d.proj[p].weight, sizeof(float)) == 0)
        break;
    if (c == net->n_cls) {
      BP_CHECK(net->n_cls < bp::kMaxCls, BP_ERR_UNSUPPORTED,
               "more than %d distinct (receptor, weight) classes", bp::kMaxCls);
      net->cls_w[c] = d.proj[p].weight;
      net->cls_rec[c] = d.proj[p].receptor;
      ++net->n_cls;
    }
    net->proj_cls[p] = c;
  }
  if (d.g_kind == BP_OUT_F32) {
    for (int c = 0; c < net->n_cls; ++c) {
      const double q = static_cast<double>(net->cls_w[c]) * 4294967296.0;
      BP_CHECK(q == std::rint(q) && std::fabs(q) < 9.0e15, BP_ERR_UNSUPPORTED,
               "fp32 merged conductances need weights on the 2^-32 grid (w = %g)",
               static_cast<double>(net->cls_w[c]));
    }
  }
  // the exact int64 sums of one step cannot overflow: rows x |q| summed
  double bound = 0.0;
  for (int p = 0; p < d.n_proj; ++p)
    bound += static_cast<double>(d.proj[p].pre_end - d.proj[p].pre_begin) *
             std::fabs(static_cast<double>(d.proj[p].weight)) * 4294967296.0;
  BP_CHECK(bound < 4.0e18, BP_ERR_UNSUPPORTED, "merged increments may overflow int64");
  return BP_OK;
}

// Build the device projection table and the launch-wide connection args.
bp::ConnArgs make_conn(bp_network *net, std::vector<bp::NetProj> *table) {
  const bp_network_desc &d = net->d;
  bp::ConnArgs c{};
  c.n_proj = d.n_proj;
  c.n_cols = static_cast<uint32_t>(d.n);
  double e_seg = 0.0;      // most expected events of a row in one segment
  uint32_t n_seg_max = 0;
  net->all_jit = true;
  table->assign(d.n_proj, bp::NetProj{});
  for (int p = 0; p < d.n_proj; ++p) {
    const bp_projection &P = d.proj[p];
    bp::NetProj &t = (*table)[p];
    t.pre_begin = static_cast<uint32_t>(P.pre_begin);
    t.pre_end = static_cast<uint32_t>(P.pre_end);
    t.conn = P.conn;
    t.cls = static_cast<uint32_t>(net->proj_cls[p]);
    if (P.conn == BP_CONN_JIT) {
      t.j = jit_side(&P.jit, net->jr[p], BP_LAW_HOMO, P.weight, 0.f, d.col_begin, d.col_end,
                     nullptr);
      // expected events of one row in one segment: L * 2 / (K + 1)
      e_seg = std::max(e_seg, net->jr[p].L * 2.0 / (net->jr[p].K + 1.0));
      n_seg_max = std::max(n_seg_max, t.j.n_seg);
    } else {
      t.c.indptr = P.indptr;
      t.c.indices = P.indices;
      t.c.w = P.weight;
      net->all_jit = false;
    }
  }
  c.all_jit = net->all_jit ? 1 : 0;
  // Binning work split (k_bin_sorted): a whole warp per row and segment
  // (one step regenerates 128 gaps) or 4 lanes per (row, segment) item (16
  // gaps per step, 8 items per warp in flight).  Measured per binning launch
  // (tools/bin_group_ab.sh, B200): ~80 events per item (config 5) 29.6 vs
  // 32.5 us -> warp; ~10 (config 3 with seg_len n/8, an 8-GPU partition)
  // 16.6 vs 37.4 us and 110 vs 143 us per step -> 4 lanes; ~125 (Fig S3B
  // with seg_len n/8) 18.1 vs 21.6 us -> 4 lanes; rows of ~1000 events keep
  // the warp (63 steps of 16 gaps would serialise).
  c.group_lanes = ((e_seg >= 48.0 && e_seg <= 112.0) || e_seg >= 512.0) ? 32 : 4;
  // rows of several long segments (Fig S3B / S3C with seg_len n/8: ~125 and
  // ~500 events per item, a few hundred rows per step): a warp per (row,
  // segment) item, so one row's segments run on different warps instead of
  // in turn (measured, tools/group_env_ab.sh: S3C binning 34.7 -> 20.6 us,
  // 46.1 -> 32.5 us per step; S3B 18.4 -> 18.1 us; config 3's ~10 events
  // per item stay on 4 lanes: 16.5 vs 47 us)
  if (e_seg >= 112.0 && n_seg_max > 1) c.group_lanes = bp::kWarpPerItem;
  // one local segment of ~10 events per row in a LARGE network (an 8-GPU
  // weak-scaling rank: 80 / 8 events, ~190 k rows per step): 2 lanes per
  // item, 16 items per warp in flight -- twice the rows per warp round, the
  // same gaps per item in 2 steps of 8 (emulated rank of 8: 112.6 -> 109.9
  // us per step).  4 lanes stay at ~40 events per item (2 GPUs: 102.3 vs
  // 105.7 us), for config 3's 8 segments per row (30.5 vs 30.8 us) and when
  // the rows are few (config 3 on 8 GPUs, ~8 k rows per step: ~50 per
  // binning block, 25.5 vs 26.3 us; the 2-lane split would leave warps idle)
  // -- tools/group_small_ab.sh.  "Large": >= 16 M neurons in all.
  if (e_seg <= 16.0 && n_seg_max == 1 && d.n >= (int64_t{1} << 24)) c.group_lanes = 2;
  if (const char *g = std::getenv("BP_BIN_GROUP"); g && *g) {
    const int v = std::atoi(g);
    c.group_lanes = (v == 2 || v == 4 || v == bp::kWarpPerItem) ? v : 32;
  }
  c.n_seg_max = n_seg_max;
  return c;
}

bp::BinTarget bin_target(const bp_network *net, int parity) {
  bp::BinTarget b{};
  b.out = net->bk[parity];
  b.cap = net->cap;
  b.n_local = static_cast<uint32_t>(net->n_local);
  b.col_begin = static_cast<uint32_t>(net->d.col_begin);
  return b;
}

// Mean events per postsynaptic neuron per presynaptic spike wave: fan-in.
double fan_in_estimate(const bp_network *net, cudaStream_t st) {
  const bp_network_desc &d = net->d;
  double f = 0.0;
  for (int p = 0; p < d.n_proj; ++p) {
    const bp_projection &P = d.proj[p];
    const int64_t rows = P.pre_end - P.pre_begin;
    if (rows == 0) continue;
    if (P.conn == BP_CONN_JIT) {
      f += static_cast<double>(rows) * net->jr[p].density;
    } else {
      int64_t nnz = 0;
      cudaMemcpyAsync(&nnz, P.indptr + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      f += static_cast<double>(nnz) / static_cast<double>(net->n_local);
    }
  }
  return f;
}

// Buckets sized for 5 % of the presynaptic neurons spiking in one step
// (500 Hz at dt = 0.1 ms); more events spill exactly (step.cuh).  The
// projection table shares the allocation.
bp_status alloc_buckets(bp_network *net, const std::vector<bp::NetProj> &table,
                        cudaStream_t st) {
  net->n_tiles = static_cast<uint32_t>((net->n_local + bp::kTile - 1) / bp::kTile);
  double expect = bp::kTile * fan_in_estimate(net, st) * 0.05;
  uint32_t cap = static_cast<uint32_t>(round_up(static_cast<size_t>(expect) + 1024, 1024));
  if (const char *env = std::getenv("BP_BUCKET_CAP")) cap = static_cast<uint32_t>(std::atoi(env));
  if (cap < 1) cap = 1;
  if (net->dense) cap = 0;               // every event straight into the dense counts
  net->cap = cap;
  const size_t ncls = static_cast<size_t>(net->ncls_kernel);
  const size_t cnt_b = round_up(static_cast<size_t>(net->n_tiles) * bp::kCntStride *
                                    sizeof(int32_t), 256);
  const size_t buf_b = round_up(static_cast<size_t>(net->n_tiles) * cap * sizeof(uint32_t), 256);
  const size_t spill_b = round_up(ncls * static_cast<size_t>(net->n_local) * sizeof(int32_t), 256);
  const size_t per = 2 * cnt_b + buf_b + spill_b;     // cnt, flag, buf, spill
  const size_t small_b = round_up((static_cast<size_t>(net->n_local) + 64) * sizeof(int32_t), 256);
  const size_t table_b = round_up(table.size() * sizeof(bp::NetProj), 256);
  const size_t R = static_cast<size_t>(net->slots);
  net->dev_bytes = R * per + small_b + table_b;
  BP_CUDA(cudaMalloc(&net->bk_mem, net->dev_bytes));
  char *m = static_cast<char *>(net->bk_mem);
  net->small_count = reinterpret_cast<int32_t *>(m + R * per);
  net->small_active = net->small_count + 64;
  net->proj_dev = reinterpret_cast<bp::NetProj *>(m + R * per + small_b);
  BP_CUDA(cudaMemcpyAsync(net->proj_dev, table.data(), table.size() * sizeof(bp::NetProj),
                          cudaMemcpyHostToDevice, st));
  BP_CUDA(cudaMemsetAsync(net->small_count, 0, sizeof(int32_t), st));
  for (int p = 0; p < net->slots; ++p) {
    char *b = m + p * per;
    net->bk[p].cnt = reinterpret_cast<int32_t *>(b);
    net->bk[p].flag = reinterpret_cast<int32_t *>(b + cnt_b);
    net->bk[p].buf = reinterpret_cast<uint32_t *>(b + 2 * cnt_b);
    net->bk[p].spill = reinterpret_cast<int32_t *>(b + 2 * cnt_b + buf_b);
    BP_CUDA(cudaMemsetAsync(b, 0, 2 * cnt_b, st));
    BP_CUDA(cudaMemsetAsync(net->bk[p].spill, 0, spill_b, st));
  }
  // the table copy reads a host vector: finish it before that goes away
  BP_CUDA(cudaStreamSynchronize(st));
  return BP_OK;
}

// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its predecessor drains; it waits (griddepcontrol.wait)
// before reading the predecessor's results (step.cuh).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem,
                       cudaStream_t st, Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = std::getenv("BP_NO_PDL") ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Bin the rows active[0..*count) into bucket parity `par`: block-aggregated
// when the tile table fits in shared memory, else one atomic per event.
bool bin_sorted_fits(const bp_network *net) {
  const size_t smem = (2 * static_cast<size_t>(bp::kBinStage) + 2 * net->n_tiles) * 4;
  return !net->dense && net->n_tiles <= 8192 && smem <= 200 * 1024 &&
         !std::getenv("BP_BIN_PER_EVENT");
}

template <bool WORDS>
bp_status launch_bin_sorted(bp_network *net, const int32_t *active, const int32_t *count,
                            const bp::WordRange &wr, int par, cudaStream_t st) {
  const size_t smem = (2 * static_cast<size_t>(bp::kBinStage) + 2 * net->n_tiles) * 4;
  static std::atomic<uint64_t> attr_set{0};
  if (first_on_device(attr_set)) {
    BP_CUDA(cudaFuncSetAttribute(bp::k_bin_sorted<WORDS>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    if (const char *c = std::getenv("BP_CARVEOUT"); c && *c)
      cudaFuncSetAttribute(bp::k_bin_sorted<WORDS>,
                           cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(c));
  }
  BP_CUDA(launch_pdl(bp::k_bin_sorted<WORDS>, net->sms, bp::kBinThreads, smem, st, net->conn,
                     bin_target(net, par), active, count, wr, net->counters + 1, net->n_tiles));
  return launched();
}

// Bin the rows active[0..*count) into bucket parity `par`: block-aggregated
// when the tile table fits in shared memory, else one atomic per event.
bp_status launch_bin(bp_network *net, const int32_t *active, const int32_t *count, int par,
                     int64_t max_rows, cudaStream_t st) {
  if (bin_sorted_fits(net))
    return launch_bin_sorted<false>(net, active, count, bp::WordRange{}, par, st);
  bp::k_bin_rows<<<grid_for_items(max_rows, net->sms), bp::kScatterThreads, 0, st>>>(
      net->conn, bin_target(net, par), active, count, net->counters + 1);
  return launched();
}

// Bin the events of the spikes in words [w_begin, w_end) of the global
// vector `vec` (neurons [32 w_begin, min(32 w_end, n))) into bucket parity
// `par`.  Words [skip_b, skip_e) (absolute) are skipped: one pass over the
// remote words on both sides of a partition's own range.  When every
// binning block's share is at most one word per thread, the block-aggregated
// binning lists its rows itself (one launch, no count memset); longer
// vectors go through the compaction launch, whose loads are all in flight
// at once.  Measured (emulated ranks, B200, tools/words_ab.sh): config 3 with
// the strong-scaling segments (420-740 words per block) 29.2 -> 27.2 us per
// step at G = 8, 32.2 -> 30.7 at G = 2; the weak-scaling ranks with in-kernel
// listing 99.8 -> 103.7 us (G = 2, 2.6 k words per block) and 109 -> 123 us
// (G = 8, 18 k) -- kept on the compaction.  BP_BIN_COMPACT=0/1 overrides.
bp_status bin_spike_range(bp_network *net, const uint32_t *vec, int64_t w_begin, int64_t w_end,
                          int par, cudaStream_t st, int64_t skip_b = 0, int64_t skip_e = 0) {
  if (w_end <= w_begin) return BP_OK;
  const int64_t first = w_begin * 32;
  const int64_t last = w_end * 32 < net->d.n ? w_end * 32 : net->d.n;
  if (last <= first) return BP_OK;
  const int64_t sb = std::min(std::max(skip_b, w_begin), w_end);
  const int64_t se = std::min(std::max(skip_e, sb), w_end);
  const int64_t words = (sb - w_begin) + (w_end - se);
  bool listing = words <= static_cast<int64_t>(net->sms) * bp::kBinThreads;
  if (const char *e = std::getenv("BP_BIN_COMPACT"); e && *e) listing = std::atoi(e) == 0;
  const bp::WordRange wr{vec, w_begin, w_end, skip_b, skip_e, net->d.n};
  if (listing && bin_sorted_fits(net))
    return launch_bin_sorted<true>(net, nullptr, nullptr, wr, par, st);
  if (listing) {
    // words per warp: spread the range over all resident warps (8 blocks of
    // 8 warps per SM), up to 32
    const int64_t resident = static_cast<int64_t>(net->sms) * 64;
    const int wpw = static_cast<int>(std::min<int64_t>(32, std::max<int64_t>(1, (words + resident - 1) / resident)));
    const int64_t warps = (words + wpw - 1) / wpw;
    bp::k_bin_rows_words<<<grid_for_items(warps, net->sms), bp::kScatterThreads, 0, st>>>(
        net->conn, bin_target(net, par), wr, wpw, net->counters + 1);
    return launched();
  }
  int32_t *active = net->active[0];
  int32_t *count = net->count;
  BP_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t), st));
  launch_compact(vec + w_begin, last - first, active, count, net->sms, st,
                 static_cast<int32_t>(first), skip_b - w_begin, skip_e - w_begin);
  bp_status s = launched();
  if (s != BP_OK) return s;
  return launch_bin(net, active, count, par, last - first, st);
}

// Quantised class weight for the conductance kind (and the general fp32
// merge, which sums at 2^-32).
long long net_q(const bp_network *net, float w) {
  if (net->d.g_kind == BP_OUT_FIX32)
    return llrint(std::ldexp(static_cast<double>(w), net->neuron.frac_bits));
  return llrint(static_cast<double>(w) * 4294967296.0);
}

// The per-network fields of a step (buckets, order and lists set by callers).
bp::StepArgs step_args(bp_network *net) {
  bp::StepArgs a{};
  a.nrn = net->neuron;
  a.nrn.raster = nullptr;
  a.nrn.active = nullptr;
  a.model = net->d.model;
  a.n_cls = net->n_cls;
  for (int c = 0; c < bp::kMaxCls; ++c) {
    const bool used = c < net->n_cls;
    a.w[c] = used ? net->cls_w[c] : 0.f;
    a.q[c] = used ? net_q(net, net->cls_w[c]) : 0;
    a.rec[c] = used ? net->cls_rec[c] : 0;
  }
  a.saturated = net->counters + 2;
  a.n_tiles = net->n_tiles;
  a.events = net->counters + 1;
  a.spikes = net->counters;
  return a;
}

// The gathered spike vector written by step n (NCCL, D >= 2: alternating).
uint32_t *step_vector(const bp_network *net, int64_t step) {
  return net->spk[net->spk[1] ? (step & 1) : 0];
}

template <int MODEL, int KIND, int NCLS>
bp_status launch_k_step(const bp::StepArgs &a, int grid, cudaStream_t st) {
  constexpr int threads = MODEL == 0 ? bp::kStepThreads : 512;
  constexpr size_t smem = static_cast<size_t>(NCLS) * bp::kTile * sizeof(int32_t);
  if (smem > 48 * 1024) {
    static std::atomic<uint64_t> attr{0};
    if (first_on_device(attr))
      BP_CUDA(cudaFuncSetAttribute(bp::k_step<MODEL, KIND, NCLS>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  }
  BP_CUDA(launch_pdl(bp::k_step<MODEL, KIND, NCLS>, grid, threads, smem, st, a));
  return BP_OK;
}

// Persistent k_step (LIF): one resident wave of blocks taking tiles from
// a per-step counter.  Measured (tools/persist_ab.sh, B200): f32 config 5
// (3052 tiles, 5.2 waves) 63.8 -> 61.8 us; but config 3 (977 tiles) 23.5 ->
// 24.9 us and the fixed-point kinds slower (fix32 71.9 -> 79.4, fix64
// 95.9 -> 133.4: the int64 state spills) -- so only fp32 state with at
// least 4 waves of tiles uses it (BP_STEP_PERSIST=0/1 overrides).
template <int KIND, int NCLS>
bp_status launch_k_step_persist(const bp::StepArgs &a, int sms, cudaStream_t st) {
  constexpr size_t smem = static_cast<size_t>(NCLS) * bp::kTile * sizeof(int32_t);
  static std::atomic<uint64_t> attr{0};
  static int per_sm[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (first_on_device(attr)) {
    if (const char *c = std::getenv("BP_CARVEOUT"); c && *c)
      cudaFuncSetAttribute(bp::k_step_persist<0, KIND, NCLS>,
                           cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(c));
    // (the opt-in also covers the kernel's static shared words beyond 48 KB)
    BP_CUDA(cudaFuncSetAttribute(bp::k_step_persist<0, KIND, NCLS>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    int b = 0;
    BP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, bp::k_step_persist<0, KIND, NCLS>,
                                                          bp::kStepThreads, smem));
    per_sm[dev & 63] = b > 0 ? b : 1;
  }
  int grid = sms * per_sm[dev & 63];
  if (grid > static_cast<int>(a.n_tiles)) grid = static_cast<int>(a.n_tiles);
  BP_CUDA(launch_pdl(bp::k_step_persist<0, KIND, NCLS>, grid, bp::kStepThreads, smem, st, a));
  return BP_OK;
}

template <int MODEL, int KIND>
bp_status launch_k_step_n(const bp::StepArgs &a, int ncls, int grid, cudaStream_t st, int sms) {
  const char *env = std::getenv("BP_STEP_PERSIST");
  const bool persist = env ? std::atoi(env) != 0
                           : (KIND == 0 && a.n_tiles >= static_cast<uint32_t>(4 * 4 * sms));
  if (MODEL == 0 && persist)
    return ncls == 2 ? launch_k_step_persist<KIND, 2>(a, sms, st)
                     : launch_k_step_persist<KIND, bp::kMaxCls>(a, sms, st);
  return ncls == 2 ? launch_k_step<MODEL, KIND, 2>(a, grid, st)
                   : launch_k_step<MODEL, KIND, bp::kMaxCls>(a, grid, st);
}

bp_status launch_step(bp_network *net, uint32_t *raster, cudaStream_t st,
                      int32_t *step_spikes = nullptr, cudaEvent_t mid = nullptr,
                      cudaEvent_t mid2 = nullptr) {
  const bp_network_desc &d = net->d;
  bp::StepArgs a = step_args(net);
  a.nrn.raster = raster;
  a.nrn.spikes = step_vector(net, net->steps_done) + d.col_begin / 32;
  const int in_slot = static_cast<int>(net->steps_done % net->slots);
  const int out_slot = static_cast<int>((net->steps_done + net->delay) % net->slots);
  a.in = net->bk[in_slot];
  a.out = bin_target(net, out_slot);
  a.reverse = static_cast<int>(net->steps_done & 1);
  a.step_spikes = step_spikes;
  const int out_par = out_slot;
  // ping-pong list counters: this step appends at count[2 + p] and zeroes
  // count[2 + (p ^ 1)] for the next step (its reader finished last step)
  const int cp = static_cast<int>(net->steps_done & 1);
  a.active = net->active[1];
  a.active_count = net->count + 2 + cp;
  a.zero_count = net->count + 2 + (cp ^ 1);
  a.tile_counter = net->count + 4 + cp;           // k_step_persist's tile scheduler
  a.zero_tile_counter = net->count + 4 + (cp ^ 1);
  const int grid = static_cast<int>(net->n_tiles);
  // dense HH: the update kernel delivers its own spikes (BP_HH_FUSED=0: the
  // separate binning launch)
  const bool fused = net->dense && d.model == BP_MODEL_HH && net->hh_fused;
  if (fused) a.conn = net->conn;
  bp_status s = BP_OK;
  if (net->dense) {
    const int dgrid = static_cast<int>((net->n_local + 4 * bp::kDenseThreads - 1) /
                                       (4 * bp::kDenseThreads));
    if (d.model == BP_MODEL_LIF) {
      if (d.g_kind == BP_OUT_FIX64) BP_CUDA(launch_pdl(bp::k_step_dense<0, 1>, dgrid, bp::kDenseThreads, 0, st, a));
      else if (d.g_kind == BP_OUT_FIX32) BP_CUDA(launch_pdl(bp::k_step_dense<0, 2>, dgrid, bp::kDenseThreads, 0, st, a));
      else BP_CUDA(launch_pdl(bp::k_step_dense<0, 0>, dgrid, bp::kDenseThreads, 0, st, a));
    } else {   // HH: one neuron per thread
      const int64_t per_block = static_cast<int64_t>(bp::kHHThreads) * bp::kHHPerThread;
      const int hgrid = static_cast<int>((net->n_local + per_block - 1) / per_block);
      if (fused) {
        if (d.g_kind == BP_OUT_FIX64) BP_CUDA(launch_pdl(bp::k_hh_dense1<1, true>, hgrid, bp::kHHThreads, 0, st, a));
        else if (d.g_kind == BP_OUT_FIX32) BP_CUDA(launch_pdl(bp::k_hh_dense1<2, true>, hgrid, bp::kHHThreads, 0, st, a));
        else BP_CUDA(launch_pdl(bp::k_hh_dense1<0, true>, hgrid, bp::kHHThreads, 0, st, a));
      } else {
        if (d.g_kind == BP_OUT_FIX64) BP_CUDA(launch_pdl(bp::k_hh_dense1<1>, hgrid, bp::kHHThreads, 0, st, a));
        else if (d.g_kind == BP_OUT_FIX32) BP_CUDA(launch_pdl(bp::k_hh_dense1<2>, hgrid, bp::kHHThreads, 0, st, a));
        else BP_CUDA(launch_pdl(bp::k_hh_dense1<0>, hgrid, bp::kHHThreads, 0, st, a));
      }
    }
  } else if (d.model == BP_MODEL_LIF) {
    if (d.g_kind == BP_OUT_FIX64) s = launch_k_step_n<0, 1>(a, net->ncls_kernel, grid, st, net->sms);
    else if (d.g_kind == BP_OUT_FIX32) s = launch_k_step_n<0, 2>(a, net->ncls_kernel, grid, st, net->sms);
    else s = launch_k_step_n<0, 0>(a, net->ncls_kernel, grid, st, net->sms);
  } else {   // HH is compute-latency-bound: 512 threads per tile
    if (d.g_kind == BP_OUT_FIX64) s = launch_k_step_n<1, 1>(a, net->ncls_kernel, grid, st, net->sms);
    else if (d.g_kind == BP_OUT_FIX32) s = launch_k_step_n<1, 2>(a, net->ncls_kernel, grid, st, net->sms);
    else s = launch_k_step_n<1, 0>(a, net->ncls_kernel, grid, st, net->sms);
  }
  if (s != BP_OK) return s;
  s = launched();
  if (s != BP_OK) return s;
  if (mid) BP_CUDA(cudaEventRecord(mid, st));
  if (mid2) BP_CUDA(cudaEventRecord(mid2, st));
  if (net->debug_nan)
    bp::k_count_nonfinite<<<net->sms * 4, 256, 0, st>>>(d.state.v, net->n_local,
                                                         net->counters + 3);
  if (!fused) {
    s = launch_bin(net, net->active[1], net->count + 2 + cp, out_par, net->n_local, st);
    if (s != BP_OK) return s;
  }
  net->steps_done += 1;
  return BP_OK;
}

}  // namespace

namespace {

template <int MODEL, int KIND>
bp_status launch_small(const bp::SmallArgs &a, cudaStream_t st) {
  const size_t smem = bp::small_net_smem(MODEL, KIND);
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr))
    BP_CUDA(cudaFuncSetAttribute(bp::k_small_net<MODEL, KIND>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  bp::k_small_net<MODEL, KIND><<<1, bp::kSmallThreads, smem, st>>>(a);
  return launched();
}

bp_status small_step(bp_network *net, int64_t n_steps, uint32_t *raster, int32_t *counts_out,
                     cudaStream_t st) {
  const bp_network_desc &d = net->d;
  if (counts_out && n_steps > net->small_steps_cap) {
    if (net->small_steps) cudaFree(net->small_steps);
    net->small_steps = nullptr;
    BP_CUDA(cudaMalloc(&net->small_steps, n_steps * sizeof(int32_t)));
    net->small_steps_cap = n_steps;
  }
  bp::SmallArgs a{};
  a.nrn = net->neuron;
  a.nrn.raster = raster;
  a.conn = net->conn;
  a.w_e = net->cls_w[0];
  a.w_i = net->cls_w[1];
  a.q_e = net_q(net, net->cls_w[0]);
  a.q_i = net_q(net, net->cls_w[1]);
  a.saturated = net->counters + 2;
  a.n_steps = n_steps;
  a.step_counts = counts_out ? net->small_steps : nullptr;
  a.active_io = net->small_active;
  a.count_io = net->small_count;
  a.events = net->counters + 1;
  a.spikes = net->counters;
  cudaEvent_t *ev = nullptr;
  if (net->prof_ev && net->prof_used < net->prof_cap) {
    ev = net->prof_ev + 3 * net->prof_used++;
    net->prof_steps += n_steps;
  }
  if (ev) BP_CUDA(cudaEventRecord(ev[0], st));
  bp_status s;
  if (d.model == BP_MODEL_LIF)
    s = d.g_kind == BP_OUT_FIX64   ? launch_small<0, 1>(a, st)
        : d.g_kind == BP_OUT_FIX32 ? launch_small<0, 2>(a, st)
                                   : launch_small<0, 0>(a, st);
  else
    s = d.g_kind == BP_OUT_FIX64   ? launch_small<1, 1>(a, st)
        : d.g_kind == BP_OUT_FIX32 ? launch_small<1, 2>(a, st)
                                   : launch_small<1, 0>(a, st);
  if (s != BP_OK) return s;
  if (ev) {   // the single launch is the "update" interval; no binning kernel
    BP_CUDA(cudaEventRecord(ev[1], st));
    BP_CUDA(cudaEventRecord(ev[2], st));
  }
  if (counts_out)
    BP_CUDA(cudaMemcpyAsync(counts_out, net->small_steps, n_steps * sizeof(int32_t),
                            cudaMemcpyDefault, st));
  net->steps_done += n_steps;
  return BP_OK;
}

// Remote spikes of step `step` (the words outside this rank's slice of the
// gathered vector) into the slot they are delivered at, step + delay.
bp_status remote_scatter(bp_network *net, int64_t step, cudaStream_t st) {
  if (net->d.exchange == BP_EXCHANGE_NCCL && net->d.world == 1) return BP_OK;
  const int64_t lw0 = net->d.col_begin / 32;
  const int64_t lw1 = (net->d.col_end + 31) / 32;
  const int slot = static_cast<int>((step + net->delay) % net->slots);
  // one compaction + one binning launch for the words on both sides
  return bin_spike_range(net, step_vector(net, step), 0, net->global_words, slot, st, lw0, lw1);
}

// One step of a BP_EXCHANGE_NCCL network:
//   D = 1:  [wait gather(n-1); remote scatter(n-1)] -> k_step(n) -> local bin(n)
//           with gather(n) on the comm stream after k_step (overlaps the bin);
//   D >= 2: k_step(n) -> local bin(n) -> [wait gather(n-1); remote scatter(n-1)]
//           -- gather(n) overlaps local bin(n), remote scatter(n-1) and the
//           whole k_step(n + 1) (vectors alternate per step).
bp_status nccl_step(bp_network *net, uint32_t *raster, int32_t *step_spikes, cudaEvent_t *prof,
                    cudaStream_t st) {
  const int64_t n = net->steps_done;
  bp_status s = BP_OK;
  if (net->delay == 1 && n > 0) {
    BP_CUDA(cudaStreamWaitEvent(st, net->ev_gath[(n - 1) & 1], 0));
    s = remote_scatter(net, n - 1, st);
    if (s != BP_OK) return s;
  }
  // profiling: [0] before k_step, [1] after it, [2] after the local binning
  if (prof) BP_CUDA(cudaEventRecord(prof[0], st));
  s = launch_step(net, raster, st, step_spikes, net->ev_spk,
                  prof ? prof[1] : nullptr);   // steps_done -> n + 1
  if (s != BP_OK) return s;
  if (prof) BP_CUDA(cudaEventRecord(prof[2], st));
  // gather(n): every rank's words of step n into the vector of step n
  uint32_t *vec = step_vector(net, n);
  BP_CUDA(cudaStreamWaitEvent(net->comm_st, net->ev_spk, 0));
  BP_NCCL(g_nccl.all_gather(vec + net->d.rank * net->part_words, vec,
                            static_cast<size_t>(net->part_words), ncclUint32, net->comm,
                            net->comm_st));
  BP_CUDA(cudaEventRecord(net->ev_gath[n & 1], net->comm_st));
  if (net->delay > 1 && n > 0) {
    BP_CUDA(cudaStreamWaitEvent(st, net->ev_gath[(n - 1) & 1], 0));
    s = remote_scatter(net, n - 1, st);
    if (s != BP_OK) return s;
  }
  return BP_OK;
}

bp_status nccl_setup(bp_network *net, cudaStream_t st) {
  bp_status s = nccl_load();
  if (s != BP_OK) return s;
  ncclUniqueId id;
  std::memcpy(&id, net->d.nccl_id, sizeof id);
  BP_CUDA(cudaStreamSynchronize(st));
  BP_NCCL(g_nccl.comm_init_rank(&net->comm, net->d.world, id, net->d.rank));
  BP_CUDA(cudaStreamCreateWithFlags(&net->comm_st, cudaStreamNonBlocking));
  BP_CUDA(cudaEventCreateWithFlags(&net->ev_spk, cudaEventDisableTiming));
  BP_CUDA(cudaEventCreateWithFlags(&net->ev_gath[0], cudaEventDisableTiming));
  BP_CUDA(cudaEventCreateWithFlags(&net->ev_gath[1], cudaEventDisableTiming));
  net->part_words = net->d.part_len / 32;
  net->nccl = true;
  return BP_OK;
}

}  // namespace

extern "C" {

size_t bp_network_workspace_bytes(const bp_network_desc *desc) {
  if (desc == nullptr || desc->n < 0) return 0;
  return network_ws_layout(desc).total;
}

size_t bp_network_device_bytes(const bp_network *net) { return net ? net->dev_bytes : 0; }

bp_status bp_network_describe(const bp_network *net, int32_t *out, int32_t n) {
  BP_CHECK(net != nullptr && out != nullptr && n >= 0, BP_ERR_INVALID_ARG, "bad arguments");
  const int32_t v[8] = {net->small ? 1 : 0, net->dense ? 1 : 0, static_cast<int32_t>(net->n_tiles),
                        static_cast<int32_t>(net->cap), net->ncls_kernel, net->conn.group_lanes,
                        net->nccl ? 1 : 0, net->n_cls};
  for (int32_t i = 0; i < n && i < 8; ++i) out[i] = v[i];
  return BP_OK;
}

bp_status bp_network_create(const bp_network_desc *desc, bp_stream stream,
                            bp_network **out) {
  int sms = 0;
  bp_status s = device_ready(&sms);
  if (s != BP_OK) return s;
  BP_CHECK(out != nullptr, BP_ERR_INVALID_ARG, "out is NULL");
  s = validate_network(desc);
  if (s != BP_OK) return s;
  bp_network *net = new (std::nothrow) bp_network();
  BP_CHECK(net != nullptr, BP_ERR_INVALID_ARG, "out of host memory");
  net->d = *desc;
  net->sms = sms;
  net->delay = desc->delay_steps > 0 ? desc->delay_steps : 1;
  net->slots = net->delay + 1;
  net->debug_nan = std::getenv("BP_DEBUG_NAN") && std::atoi(std::getenv("BP_DEBUG_NAN"));
  if (const char *f = std::getenv("BP_HH_FUSED"); f && *f) net->hh_fused = std::atoi(f) != 0;
  net->n_local = desc->col_end - desc->col_begin;
  net->local_words = (net->n_local + 31) / 32;
  net->global_words = desc->exchange == BP_EXCHANGE_NCCL
                          ? desc->world * (desc->part_len / 32)
                          : (desc->n + 31) / 32;
  for (int p = 0; p < desc->n_proj && s == BP_OK; ++p) {
    const bp_projection &P = desc->proj[p];
    if (P.conn != BP_CONN_JIT) continue;
    s = resolve_jit(&P.jit, desc->n, &net->jr[p]);
    if (s == BP_OK && net->jr[p].geo_c != 0.f)
      s = fail(BP_ERR_UNSUPPORTED,
               "networks use the uniform gap sampler (rule J3); gap_law must be 0");
    if (s == BP_OK && (desc->col_begin % net->jr[p].L ||
                       (desc->col_end != desc->n && desc->col_end % net->jr[p].L)))
      s = fail(BP_ERR_SHAPE, "partition not aligned to seg_len of projection %d", p);
  }
  if (s == BP_OK) s = fill_neuron_args(&desc->params, &desc->state, net->n_local, &net->neuron);
  if (s == BP_OK) s = assign_classes(net);
  if (s != BP_OK) {
    delete net;
    return s;
  }
  // dense delivery for the compute-bound HH model up to 2 M local neurons
  // (counts stay L2-resident; 4096-neuron tiles would leave SMs idle);
  // BP_DENSE=0/1 overrides.  Standard class layout only.
  {
    const char *env = std::getenv("BP_DENSE");
    net->dense = (env ? std::atoi(env) != 0 : dense_delivery(desc->model, net->n_local)) &&
                 net->ncls_kernel == 2;
  }
  const NetWsLayout wl = network_ws_layout(desc);
  char *ws = static_cast<char *>(desc->ws);
  net->counters = reinterpret_cast<unsigned long long *>(ws);
  net->count = reinterpret_cast<int32_t *>(ws + 64);
  net->active[0] = reinterpret_cast<int32_t *>(ws + wl.active0);
  net->active[1] = reinterpret_cast<int32_t *>(ws + wl.active1);
  net->spk[0] = desc->spikes;
  if (wl.total > wl.spk1) net->spk[1] = reinterpret_cast<uint32_t *>(ws + wl.spk1);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(ws, 0, 256, st);
  if (e != cudaSuccess) {
    delete net;
    return fail(BP_ERR_CUDA, "network init: %s", cudaGetErrorString(e));
  }
  // L2 residency of g across steps: evict_last on the fraction of the g
  // lines that fits ~72 % of the L2 (BP_L2_KEEP_MB overrides the budget;
  // 0 disables the hints).
  {
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    double budget = 0.72 * static_cast<double>(l2);
    if (const char *env = std::getenv("BP_L2_KEEP_MB")) budget = std::atof(env) * 1048576.0;
    const double g_bytes = 2.0 * static_cast<double>(net->n_local) *
                           (desc->g_kind == BP_OUT_FIX64 ? 8.0 : 4.0);
    double f = g_bytes > 0 ? budget / g_bytes : 0.0;
    if (f > 1.0) f = 1.0;
    if (f < 0.0) f = 0.0;
    net->keep_frac = static_cast<float>(f);
    net->neuron.keep_frac = net->keep_frac;
  }
  net->neuron.spikes = desc->spikes + desc->col_begin / 32;
  net->neuron.active_base = static_cast<int32_t>(desc->col_begin);
  std::vector<bp::NetProj> table;
  net->conn = make_conn(net, &table);
  s = alloc_buckets(net, table, st);
  net->conn.proj = net->proj_dev;
  if (s == BP_OK && desc->exchange == BP_EXCHANGE_NCCL) s = nccl_setup(net, st);
  // spikes_{-1}: the local part is delivered into the first step; with the
  // library's exchange the caller's initial vector is complete, so its
  // remote part is binned here too; otherwise it arrives through
  // bp_network_scatter
  const int first_slot = (net->delay - 1) % net->slots;
  if (s == BP_OK)
    s = bin_spike_range(net, desc->spikes, desc->col_begin / 32, (desc->col_end + 31) / 32,
                        first_slot, st);
  if (s == BP_OK && net->nccl && desc->world > 1)
    s = bin_spike_range(net, desc->spikes, 0, net->global_words, first_slot, st,
                        desc->col_begin / 32, (desc->col_end + 31) / 32);
  // one device, whole network, state fits one CTA's shared memory: the
  // single-CTA time loop (k_small_net) drives bp_network_step
  net->small = s == BP_OK && desc->col_begin == 0 && desc->col_end == desc->n &&
               desc->n <= bp::kSmallMax && net->delay == 1 && net->ncls_kernel == 2 &&
               !net->nccl && !std::getenv("BP_NO_SMALL_NET");
  if (net->small) {
    launch_compact(desc->spikes, desc->n, net->small_active, net->small_count, sms, st);
    s = launched();
  }
  if (s != BP_OK) {
    bp_network_destroy(net);
    return s;
  }
  *out = net;
  return BP_OK;
}

bp_status bp_network_step(bp_network *net, int64_t n_steps, uint32_t *raster_out,
                          int32_t *counts_out, bp_stream stream) {
  bp_status s = device_ready(nullptr);
  if (s != BP_OK) return s;
  BP_CHECK(net != nullptr && n_steps >= 0, BP_ERR_INVALID_ARG, "bad net/n_steps");
  cudaStream_t st = as_stream(stream);
  if (net->small && n_steps > 0) return small_step(net, n_steps, raster_out, counts_out, st);
  for (int64_t k = 0; k < n_steps; ++k) {
    cudaEvent_t *ev = nullptr;
    if (net->prof_ev && net->prof_used < net->prof_cap) {
      ev = net->prof_ev + 3 * net->prof_used++;
      net->prof_steps += 1;
    }
    uint32_t *row = raster_out ? raster_out + k * net->local_words : nullptr;
    if (counts_out) BP_CUDA(cudaMemsetAsync(net->count + 1, 0, sizeof(int32_t), st));
    if (net->nccl) {
      s = nccl_step(net, row, counts_out ? net->count + 1 : nullptr, ev, st);
    } else {
      if (ev) BP_CUDA(cudaEventRecord(ev[0], st));
      s = launch_step(net, row, st, counts_out ? net->count + 1 : nullptr, ev ? ev[1] : nullptr);
      if (s == BP_OK && ev) BP_CUDA(cudaEventRecord(ev[2], st));
    }
    if (s != BP_OK) return s;
    if (counts_out)
      BP_CUDA(cudaMemcpyAsync(counts_out + k, net->count + 1, sizeof(int32_t),
                              cudaMemcpyDefault, st));
  }
  return BP_OK;
}

bp_status bp_network_profile_begin(bp_network *net, int64_t max_steps) {
  BP_CHECK(net != nullptr && max_steps >= 0, BP_ERR_INVALID_ARG, "bad arguments");
  BP_CHECK(net->prof_ev == nullptr, BP_ERR_INVALID_ARG, "profiling already active");
  net->prof_ev = new (std::nothrow) cudaEvent_t[3 * max_steps + 1];
  BP_CHECK(net->prof_ev != nullptr, BP_ERR_INVALID_ARG, "out of host memory");
  for (int64_t i = 0; i < 3 * max_steps; ++i)
    BP_CUDA(cudaEventCreate(&net->prof_ev[i]));
  net->prof_cap = max_steps;
  net->prof_used = 0;
  net->prof_steps = 0;
  return BP_OK;
}

bp_status bp_network_profile_end(bp_network *net, double *scatter_ms,
                                 double *update_ms, int64_t *steps) {
  BP_CHECK(net != nullptr && net->prof_ev != nullptr, BP_ERR_INVALID_ARG,
           "profiling not active");
  double sc = 0.0, up = 0.0;
  bp_status s = BP_OK;
  for (int64_t k = 0; k < net->prof_used && s == BP_OK; ++k) {
    cudaEvent_t *ev = net->prof_ev + 3 * k;
    float a = 0.f, b = 0.f;
    cudaError_t e = cudaEventSynchronize(ev[2]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&a, ev[0], ev[1]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&b, ev[1], ev[2]);
    if (e != cudaSuccess) s = fail(BP_ERR_CUDA, "profile: %s", cudaGetErrorString(e));
    up += a;   // neuron update (k_step)
    sc += b;   // event regeneration + binning (k_bin_rows)
  }
  for (int64_t i = 0; i < 3 * net->prof_cap; ++i) cudaEventDestroy(net->prof_ev[i]);
  delete[] net->prof_ev;
  net->prof_ev = nullptr;
  if (scatter_ms) *scatter_ms = sc;
  if (update_ms) *update_ms = up;
  if (steps) *steps = net->prof_steps;
  net->prof_cap = net->prof_used = 0;
  net->prof_steps = 0;
  return s;
}

bp_status bp_network_scatter(bp_network *net, bp_stream stream) {
  bp_status s = device_ready(nullptr);
  if (s != BP_OK) return s;
  BP_CHECK(net != nullptr, BP_ERR_INVALID_ARG, "net is NULL");
  BP_CHECK(!net->nccl, BP_ERR_INVALID_ARG, "BP_EXCHANGE_NCCL networks run whole steps");
  // Deliver the spikes of the OTHER partitions (words outside this rank's
  // slice) of step steps_done - 1 into the buckets of their arrival step;
  // local spikes were binned by the update that produced them.
  return remote_scatter(net, net->steps_done - 1, as_stream(stream));
}

bp_status bp_network_update(bp_network *net, uint32_t *raster_row, bp_stream stream) {
  bp_status s = device_ready(nullptr);
  if (s != BP_OK) return s;
  BP_CHECK(net != nullptr, BP_ERR_INVALID_ARG, "net is NULL");
  BP_CHECK(!net->nccl, BP_ERR_INVALID_ARG, "BP_EXCHANGE_NCCL networks run whole steps");
  return launch_step(net, raster_row, as_stream(stream));
}

bp_status bp_network_update_overlap(bp_network *net, uint32_t *raster_row, bp_stream stream,
                                    bp_stream exchange_stream) {
  bp_status s = device_ready(nullptr);
  if (s != BP_OK) return s;
  BP_CHECK(net != nullptr, BP_ERR_INVALID_ARG, "net is NULL");
  BP_CHECK(!net->nccl, BP_ERR_INVALID_ARG, "BP_EXCHANGE_NCCL networks run whole steps");
  if (net->xev == nullptr) BP_CUDA(cudaEventCreateWithFlags(&net->xev, cudaEventDisableTiming));
  // k_step (spike words of this step) -> record xev -> local binning; the
  // exchange stream waits for xev only, so the all-gather overlaps k_bin
  s = launch_step(net, raster_row, as_stream(stream), nullptr, net->xev);
  if (s != BP_OK) return s;
  BP_CUDA(cudaStreamWaitEvent(as_stream(exchange_stream), net->xev, 0));
  return BP_OK;
}

bp_status bp_network_counters(bp_network *net, uint64_t *host_out, bp_stream stream) {
  bp_status s = device_ready(nullptr);
  if (s != BP_OK) return s;
  BP_CHECK(net != nullptr && host_out != nullptr, BP_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = as_stream(stream);
  if (net->nccl) {   // the comm stream's last gather is part of the state
    BP_CUDA(cudaStreamWaitEvent(st, net->ev_gath[(net->steps_done + 1) & 1], 0));
  }
  BP_CUDA(cudaMemcpyAsync(host_out, net->counters, 4 * sizeof(uint64_t),
                          cudaMemcpyDeviceToHost, st));
  BP_CUDA(cudaStreamSynchronize(st));
  return BP_OK;
}

void bp_network_destroy(bp_network *net) {
  if (net == nullptr) return;
  if (net->comm_st) cudaStreamSynchronize(net->comm_st);
  if (net->comm) g_nccl.comm_destroy(net->comm);
  if (net->comm_st) cudaStreamDestroy(net->comm_st);
  if (net->ev_spk) cudaEventDestroy(net->ev_spk);
  for (cudaEvent_t e : net->ev_gath)
    if (e) cudaEventDestroy(e);
  if (net->xev) cudaEventDestroy(net->xev);
  if (net->bk_mem) cudaFree(net->bk_mem);
  if (net->small_steps) cudaFree(net->small_steps);
  if (net->prof_ev) {
    for (int64_t i = 0; i < 3 * net->prof_cap; ++i) cudaEventDestroy(net->prof_ev[i]);
    delete[] net->prof_ev;
  }
  delete net;
}

}  // extern "C"
