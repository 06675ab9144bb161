/*
 * bp.h -- C ABI of the B200-native BrainPy hot path (libbp.so).
 *
 * The operations follow the paper's statement of the operators
 * (arxiv 2311.05106, PAPER.md; "P:n" = line n):
 *   bp_compact_spikes        -- spike vector -> active-row list; "computes only
 *                               at positions where the spike in v is True"
 *                               (App. B)                   [SURVEY 8(a) a1]
 *   bp_event_csrmv           -- brainpy.math.event.csrmv, Listing S1
 *                               (App. B)                         [a2]
 *   bp_jitconn_event_mv_*    -- brainpy.math.jitconn.event_mv_prob_{homo,
 *                               uniform,normal}, Listing S2 (App. C;
 *                               P:192)                       [a3, a4]
 *   bp_neuron_step           -- Expon + COBA + LIF
 *                               or COBA-HH (rule H1, EXTERNAL)   [a5, a6]
 *   bp_network_*             -- Listing S3's update() loop: 1-step
 *                               delayed spikes -> scatter -> neuron update [a7];
 *                               several projections merged per receptor
 *                               (AlignPost); multi-GPU: the library's
 *                               own NCCL spike all-gather or the
 *                               caller-driven halves bp_network_scatter /
 *                               _update(_overlap)                          [a8]
 *   bp_jitconn_mv_*          -- mv_prob_* with a float vector (NEXT 1, MV1)
 *   bp_csrmv_gather,
 *   bp_event_csrmv_grad      -- csrmv(transpose=False) and the reverse mode
 *                               (NEXT 3, G1)
 *   bp_jitconn.gap_law       -- BP_GAP_GEOMETRIC: the Geo(p) sampler the paper
 *                               compares against (NEXT 4, J10)
 * Rule names (J1..J10, J7n, F1, F2, N1, H1, S1, D1, G1, MV1, R-numbered
 * readings) refer to DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every pointer argument is a DEVICE pointer owned by the caller unless
 *    stated otherwise; the library allocates no device memory per call.
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream) and returns after enqueueing.  Arguments are validated
 *    synchronously before any launch.
 *  - Spike vectors are bit-packed: neuron r is bit (r & 31) of 32-bit word
 *    r >> 5, little-endian bit order; bits past the vector length are ignored
 *    on input and written 0 on output.
 *  - CSR rows are PRESYNAPTIC (the event index) and columns POSTSYNAPTIC (the
 *    output index): Listing S1 iterates `events` over rows and scatters into
 *    `outs`.  indptr int64[n_rows+1], indices int32[nnz] sorted
 *    within a row, data float32[nnz] or NULL for one homogeneous weight.
 *  - Output accumulators (bp_out_kind): BP_OUT_F32 = float32 with fp32
 *    atomics (summation order unspecified); BP_OUT_FIX64 = int64 fixed point
 *    with 32 fractional bits, each weight quantised as llrint(w * 2^32)
 *    (rule F1) -- bit-reproducible for any launch configuration.
 *  - Unless BP_ACCUMULATE is set in `flags`, the output is zeroed first.
 *  - Errors: a non-zero bp_status; bp_last_error() gives a thread-local
 *    message.  Faults raised asynchronously by a kernel surface at the
 *    caller's next synchronisation and are reported as BP_ERR_CUDA by the
 *    next call.  The library never aborts the process.
 *  - Only sm_100 devices are supported (BP_ERR_UNSUPPORTED otherwise).
 */
#ifndef BP_H_
#define BP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *bp_stream; /* cudaStream_t */

typedef enum {
  BP_OK = 0,
  BP_ERR_INVALID_ARG = 1, /* null pointer, p outside (0,1], NaN, sigma < 0 ... */
  BP_ERR_SHAPE = 2,       /* sizes <= 0 or >= 2^31, partition not aligned      */
  BP_ERR_UNSUPPORTED = 3, /* not an sm_100 device, K too large for 32-bit pos  */
  BP_ERR_WORKSPACE = 4,   /* workspace NULL, misaligned or too small           */
  BP_ERR_CUDA = 5,        /* a CUDA runtime error (launch or sticky)           */
  BP_ERR_NCCL = 6         /* NCCL missing or an NCCL call failed               */
} bp_status;

/* Output / state accumulator kinds.  BP_OUT_FIX32 is a STATE kind only
 * (network and neuron conductances): int32 with g_frac_bits fractional bits,
 * a step's increments summed exactly and added with saturation (rule F2). */
typedef enum { BP_OUT_F32 = 0, BP_OUT_FIX64 = 1, BP_OUT_FIX32 = 2 } bp_out_kind;

#define BP_ACCUMULATE 1u

typedef enum { BP_LAW_HOMO = 0, BP_LAW_UNIFORM = 1, BP_LAW_NORMAL = 2 } bp_law;
typedef enum { BP_MODEL_LIF = 0, BP_MODEL_HH = 1 } bp_model;
typedef enum { BP_CONN_JIT = 0, BP_CONN_CSR = 1 } bp_conn;

int bp_abi_version(void); /* 2 */
const char *bp_status_string(int status);
const char *bp_last_error(void);

/* Rule J1: K = floor(2/p - 1), snapped to the nearest integer when
 * within 1e-9 relative of it, K >= 1.  Returns 0 when p is not in (0, 1].
 * Host function. */
uint32_t bp_conn_len(double prob);

/* Bytes of caller-provided workspace the stateless scatter calls need for an
 * input of n_rows presynaptic neurons (active-row list + counter).  Host. */
size_t bp_workspace_bytes(int64_t n_rows);

/* Workspace for bp_event_csrmv on an n_rows x n_cols matrix with output
 * kind out_kind: the active list plus, when the output fits a few
 * shared-memory column tiles, the per-CTA partial tiles that make the
 * accumulation atomic-free (>= bp_workspace_bytes(n_rows); with only
 * bp_workspace_bytes(n_rows) bytes the partial tiles are flushed with
 * atomics instead).  Host function (queries the current device). */
size_t bp_csrmv_workspace_bytes(int64_t n_rows, int64_t n_cols, int out_kind);

/* a1: active = { r < n : bit r of spikes set }, written to active[0..count)
 * in unspecified order (a set); *count (device int32) receives its size.
 * active must hold n entries. */
bp_status bp_compact_spikes(const uint32_t *spikes, int64_t n, int32_t *active,
                            int32_t *count, bp_stream stream);

/* a2: event_csrmv, Listing S1 with indices[j] (the listing's indices[i] is a
 * typo):  for r with bit r set, for k in [indptr[r], indptr[r+1]):
 *     out[indices[k]] += (data ? data[k] : w_homo)
 * indices: ascending within each row (canonical CSR); an unsorted row gives
 * wrong sums on the tiled paths but never writes outside `out`.
 * out: n_cols float32 (BP_OUT_F32) or int64 (BP_OUT_FIX64), 16-byte aligned.
 * ws: >= bp_workspace_bytes(n_rows) bytes (bp_csrmv_workspace_bytes for the
 * atomic-free path), 256-byte aligned. */
bp_status bp_event_csrmv(const int64_t *indptr, const int32_t *indices,
                         const float *data, float w_homo, int64_t n_rows,
                         int64_t n_cols, const uint32_t *spikes, void *out,
                         int out_kind, uint32_t flags, void *ws,
                         size_t ws_bytes, bp_stream stream);

/* Gather orientation (BrainPy csrmv(..., transpose=False); SURVEY 8(f)
 * NEXT 3, reading G1): the CSR rows are the OUTPUTS, the column indices the
 * event index:  out[r] (+)= sum_{k in row r} w_k [bit indices[k] of spikes].
 * spikes: ceil(n_cols/32) words; out: n_rows float32 / int64 fixed point.
 * One warp per output row: no atomics, deterministic (fp32: fixed warp-tree
 * order, rule T2 against the sequential sum; homogeneous: fl32(count * w);
 * fixed point exact).  Indices need not be sorted. */
bp_status bp_csrmv_gather(const int64_t *indptr, const int32_t *indices, const float *data,
                          float w_homo, int64_t n_rows, int64_t n_cols, const uint32_t *spikes,
                          void *out, int out_kind, uint32_t flags, bp_stream stream);

/* Reverse mode of the event scatter y = M^T s (bp_event_csrmv; SURVEY 8(f)
 * NEXT 3, reading G1; the paper's differentiability claim) for an
 * upstream gradient gy (n_cols float32):
 *   grad_data[k]   = s[r(k)] * gy[indices[k]]          (nnz, exact)
 *   grad_events[r] = sum_{k in row r} w_k gy[indices[k]] (n_rows; the events
 *                    as real inputs; fp32, fixed warp-tree order)
 *   grad_w         = sum_{r: s[r]} sum_k gy[indices[k]] (fp64 scalar, only
 *                    for homogeneous weights, data == NULL; overwritten)
 * spikes: ceil(n_rows/32) words.  Any output may be NULL. */
bp_status bp_event_csrmv_grad(const int64_t *indptr, const int32_t *indices, const float *data,
                              float w_homo, int64_t n_rows, int64_t n_cols,
                              const uint32_t *spikes, const float *gy, float *grad_data,
                              float *grad_events, double *grad_w, bp_stream stream);

/* a2 with a reusable analysis of a fixed matrix (cf. cuSPARSE's SpMV
 * preprocessing).  bp_event_csrmv splits every active row at the column-tile
 * boundaries of its shared-memory accumulation on each call; for a matrix
 * that is reused (a network's projection, a benchmark's 10,000 calls) the
 * split points of all rows can be computed once:
 *   plan_bytes = bp_csrmv_plan_bytes(n_rows, n_cols, out_kind, data == NULL)
 *     (0: nothing to precompute);
 *   bp_csrmv_plan(...) writes the analysis into the caller's device buffer
 *     `plan` (16-byte aligned) and a host summary into *info (nullable);
 *   bp_event_csrmv_planned(plan, plan_bytes, info, ...) then behaves like
 *     bp_event_csrmv without the per-call split.
 * Heterogeneous weights with an fp32 output (rule T4): given a
 * workspace (ws >= bp_csrmv_workspace_bytes), the analysis also bounds every
 * column's sum of |w| over all rows (one pass of the kernel itself; this
 * call then SYNCHRONISES `stream`) and picks info->f32_fixed_bits = F, so
 * that each call accumulates q = rint(w 2^F) exactly in two independent
 * 32-bit integer words per column (native shared-memory atomics instead of
 * an fp32 compare-and-swap loop) and rounds each column's exact sum to fp32
 * once -- independent of the summation order; the error per column is at
 * most (terms) 2^-(F+1) + 1/2 ulp, within rule T2 unless a column's active
 * terms average below 2^-(F+1) 1e5 in magnitude (T4).  -1: the
 * fp32-atomic path (no workspace, n_rows >= 2^24, unbounded sums, or
 * BP_CSR_NO_T4=1).
 * The plan is valid for the same (indptr, indices, data, n_rows, n_cols,
 * out_kind, homogeneous-or-not) on the same device type; a stale plan gives
 * wrong sums but never reads outside the row.  Requires indices ascending
 * per row. */
typedef struct {
  int32_t n_tiles;          /* column tiles of the accumulation                */
  int32_t f32_fixed_bits;   /* rule T4 scale F (fp32 output, heterogeneous), or -1 */
  double max_col_abs_sum;   /* max over columns of sum |w| (when F >= 0)       */
} bp_csrmv_plan_info;
size_t bp_csrmv_plan_bytes(int64_t n_rows, int64_t n_cols, int out_kind, int homo);
bp_status bp_csrmv_plan(const int64_t *indptr, const int32_t *indices, const float *data,
                        int64_t n_rows, int64_t n_cols, int out_kind, int homo, void *plan,
                        size_t plan_bytes, bp_csrmv_plan_info *info, void *ws,
                        size_t ws_bytes, bp_stream stream);
bp_status bp_event_csrmv_planned(const void *plan, size_t plan_bytes,
                                 const bp_csrmv_plan_info *info, const int64_t *indptr,
                                 const int32_t *indices, const float *data, float w_homo,
                                 int64_t n_rows, int64_t n_cols, const uint32_t *spikes,
                                 void *out, int out_kind, uint32_t flags, void *ws,
                                 size_t ws_bytes, bp_stream stream);

/* JIT connectivity (App. C; the "four scalars (p, mu, sigma, s)"
 * of P:192).  The matrix is a pure function of (seed, K, seg_len, n_rows,
 * n_cols): row r's targets in segment s = [s*L, min((s+1)L, n_cols)) are
 * pos_0 = s*L + a(r,s) (stationary first offset, rule J5) and
 * pos_{e+1} = pos_e + U[1,K](Philox word e), rules J2-J6.  No connectivity
 * memory is used or stored. */
typedef struct {
  uint64_t seed;
  double prob;       /* connection probability p in (0, 1]                  */
  uint32_t conn_len; /* K; 0 => bp_conn_len(prob)                           */
  uint32_t seg_len;  /* L; 0 => n_cols (one segment per row)                */
  int32_t gap_law;   /* bp_gap_law; 0 = the paper's uniform gaps            */
  int32_t reserved;  /* must be 0                                           */
} bp_jitconn;

/* Gap sampler of a JIT matrix.
 * BP_GAP_UNIFORM (the paper's proposal): gaps U[1, K], stationary
 *   first offset (rules J1-J6); connection density 2/(K+1).
 * BP_GAP_GEOMETRIC (the baseline the paper compares against, after
 *   Knight & Nowotny 2020): gaps Geo(p) by CDF
 *   inversion, G = ceil(logf_j10(u) / fl32(log1p(-p))) with u = ((x >> 8) +
 *   1) 2^-24 and the op-for-op specified fp32 log of rule J10,
 *   clamped to [1, L + 1]; first target = segment start + G_0 - 1.  The
 *   targets form a Bernoulli(p) process (density p exactly).  conn_len is
 *   ignored; requires n_cols + 128 (L + 1) < 2^32.  Stateless operators only
 *   (event_mv, mv, row_counts, materialize); networks return
 *   BP_ERR_UNSUPPORTED. */
typedef enum { BP_GAP_UNIFORM = 0, BP_GAP_GEOMETRIC = 1 } bp_gap_law;

/* Workspace for bp_jitconn_event_mv_* over output columns [col_begin,
 * col_end): the active list plus, when the partition fits <= 16 shared-memory
 * column tiles, the per-CTA partial tiles of the tiled path (k_jit_tiled:
 * events accumulate in shared memory instead of one global atomic each).
 * With only bp_workspace_bytes(n_rows) bytes the per-event path runs.  Host
 * function (queries the current device). */
size_t bp_jitconn_workspace_bytes(int64_t n_rows, int64_t col_begin, int64_t col_end,
                                  int out_kind);

/* a3+a4: out[c - col_begin] += sum over active rows r of w_e(r) for every
 * generated edge (r, c) with c in [col_begin, col_end).  col_begin must be a
 * multiple of seg_len and col_end a multiple of seg_len or equal to n_cols
 * (a postsynaptic partition).  Requires
 * n_cols + 128 * K < 2^32 (32-bit positions), else BP_ERR_UNSUPPORTED.
 *   homo    : w_e = weight                                  (Listing S2)
 *   uniform : w_e ~ U[w_low, w_high)                         (rule J7)
 *   normal  : w_e ~ N(w_mu, w_sigma^2), Box-Muller           (rule J7)
 * out: (col_end - col_begin) float32 / int64; ws as for bp_event_csrmv. */
bp_status bp_jitconn_event_mv_homo(const bp_jitconn *spec, float weight,
                                   const uint32_t *spikes, int64_t n_rows,
                                   int64_t n_cols, int64_t col_begin,
                                   int64_t col_end, void *out, int out_kind,
                                   uint32_t flags, void *ws, size_t ws_bytes,
                                   bp_stream stream);
bp_status bp_jitconn_event_mv_uniform(const bp_jitconn *spec, float w_low,
                                      float w_high, const uint32_t *spikes,
                                      int64_t n_rows, int64_t n_cols,
                                      int64_t col_begin, int64_t col_end,
                                      void *out, int out_kind, uint32_t flags,
                                      void *ws, size_t ws_bytes,
                                      bp_stream stream);
bp_status bp_jitconn_event_mv_normal(const bp_jitconn *spec, float w_mu,
                                     float w_sigma, const uint32_t *spikes,
                                     int64_t n_rows, int64_t n_cols,
                                     int64_t col_begin, int64_t col_end,
                                     void *out, int out_kind, uint32_t flags,
                                     void *ws, size_t ws_bytes,
                                     bp_stream stream);

/* Non-event products with the same JIT matrices (brainpy.math.jitconn
 * mv_prob_{homo,uniform,normal}(vector, ...); SURVEY
 * 8(f) NEXT 1), reading MV1:
 *     out[c] (+)= sum_r v[r] * w_e(r)   over the edges (r, e) with pos_e(r) = c,
 * v: n_rows float32 (device); rows with v[r] == 0 are skipped (they add
 * nothing).  Contribution per edge: fl32(v[r] * w) in BP_OUT_F32 (float
 * atomics, order-dependent, rule T2); in BP_OUT_FIX64 the exact fp64 product
 * rounded once to 2^-32 (bit-reproducible).  Connectivity, weights,
 * partition, workspace (bp_jitconn_workspace_bytes) and errors as the event
 * variants.  With v in {0, 1} the result equals the event variant bit for
 * bit in fixed point. */
bp_status bp_jitconn_mv_homo(const bp_jitconn *spec, float weight, const float *v,
                             int64_t n_rows, int64_t n_cols, int64_t col_begin,
                             int64_t col_end, void *out, int out_kind, uint32_t flags,
                             void *ws, size_t ws_bytes, bp_stream stream);
bp_status bp_jitconn_mv_uniform(const bp_jitconn *spec, float w_low, float w_high,
                                const float *v, int64_t n_rows, int64_t n_cols,
                                int64_t col_begin, int64_t col_end, void *out, int out_kind,
                                uint32_t flags, void *ws, size_t ws_bytes, bp_stream stream);
bp_status bp_jitconn_mv_normal(const bp_jitconn *spec, float w_mu, float w_sigma,
                               const float *v, int64_t n_rows, int64_t n_cols,
                               int64_t col_begin, int64_t col_end, void *out, int out_kind,
                               uint32_t flags, void *ws, size_t ws_bytes, bp_stream stream);

/* Debug/inspection: materialise the implied matrix with the KERNEL's own
 * generator.  row_counts: counts[r] = number of edges of row r (int64[n_rows]).
 * materialize: given indptr (exclusive prefix sum of the counts, int64
 * [n_rows+1]) write indices[indptr[r]..) ascending and data (nullable) with
 * the weights of `law` (w0, w1) = (weight, -) | (w_low, w_high) | (mu, sigma). */
bp_status bp_jitconn_row_counts(const bp_jitconn *spec, int64_t n_rows,
                                int64_t n_cols, int64_t *counts,
                                bp_stream stream);
/* indptr (int64[n_rows+1]) of the implied matrix: row counts and their
 * exclusive prefix sum, on the device (the CSR row pointer that
 * bp_jitconn_materialize takes). */
bp_status bp_jitconn_indptr(const bp_jitconn *spec, int64_t n_rows, int64_t n_cols,
                            int64_t *indptr, bp_stream stream);
bp_status bp_jitconn_materialize(const bp_jitconn *spec, int law, float w0,
                                 float w1, int64_t n_rows, int64_t n_cols,
                                 const int64_t *indptr, int32_t *indices,
                                 float *data, bp_stream stream);

/* Neuron parameters.  LIF (rule N1, Listing S3): alpha_v =
 * fl32(exp(-dt/tau)), alpha_e/alpha_i = exp(-dt/tau_syn) in fp64, ref_steps
 * = tau_ref/dt.  HH (rule H1): Traub-Miles COBAHH constants (mV, ms, nS, pF).
 * Both: E_exc/E_inh reversal potentials, i_ext constant input. */
typedef struct {
  int32_t model; /* bp_model */
  int32_t ref_steps;
  float v_rest, v_reset, v_th, r, i_ext, e_exc, e_inh, alpha_v;
  double alpha_e, alpha_i;
  /* HH only */
  float c_m, g_l, e_l, g_na, e_na, g_k, e_k, v_t, dt, v_spike;
} bp_neuron_params;

/* State of n neurons (device arrays of n entries).  g_exc/g_inh are float32
 * or int64 fixed point (g_kind); they hold alpha*g_{n-1} + increments on entry
 * and are pre-decayed on exit (reading R12).  LIF uses v, ref; HH uses v, m,
 * h, n_gate. */
typedef struct {
  float *v;
  void *g_exc;
  void *g_inh;
  int32_t g_kind;      /* bp_out_kind */
  int32_t g_frac_bits; /* BP_OUT_FIX32 only: fractional bits F (0 => 20) */
  uint8_t *ref;
  float *m, *h, *n_gate;
} bp_neuron_state;

/* a5+a6: one step for neurons [0, n).  spikes_out: ceil(n/32) words (bit set
 * = spike).  active_out (nullable, n entries) receives the spiking indices
 * plus `active_base`, appended at *count_out (device int32, which the caller
 * zeroes). */
bp_status bp_neuron_step(const bp_neuron_params *params,
                         const bp_neuron_state *state, int64_t n,
                         uint32_t *spikes_out, int32_t *active_out,
                         int32_t *count_out, int64_t active_base,
                         bp_stream stream);

/* ---------------------------------------------------------------------
 * Network: Listing S3, generalised to up to BP_MAX_PROJ
 * homogeneous projections (AlignPost): projection k
 * takes the spikes of presynaptic neurons [pre_begin, pre_end) (its rows
 * 0 .. pre_end - pre_begin - 1) and adds `weight` per event into the
 * conductance of its receptor at every target among all n neurons
 * (columns).  Projections of one receptor MERGE into that
 * receptor's single conductance per neuron (one g_exc and one g_inh array
 * however many projections: "all synaptic interactions with
 * identical time constants can be converged into a single trace"); their
 * increments of one step are summed exactly (fixed point: integer sum; fp32:
 * the exactly rounded sum, rule N1-f32 -- which requires every fp32 weight
 * of a receptor with several distinct weights to be a multiple of 2^-32,
 * else BP_ERR_UNSUPPORTED).  At most 4 distinct (receptor, weight) pairs.
 * Listing S3 itself is two projections: E rows [0, n_exc) -> g_exc with
 * w_E, I rows [n_exc, n) -> g_inh with w_I.
 *
 * This process owns postsynaptic neurons [col_begin, col_end) (SURVEY
 * 8(e)); col_begin must be a multiple of 32 and of every JIT seg_len.
 * Per step (rule S1): scatter(spikes_{n-D}) into g, neuron update ->
 * spikes_n.
 *
 * Several processes (one per GPU), two ways:
 *  - exchange = BP_EXCHANGE_NCCL: the library owns an NCCL communicator
 *    (created in bp_network_create from nccl_id / rank / world, a
 *    collective call on every rank) and bp_network_step runs the whole
 *    loop, the bit-packed spike all-gather included ("gather only
 *    non-zero spikes", realised as bit packing).  The partition must be
 *    rank-ordered with equal lengths: col_begin = rank * part_len, col_end =
 *    min(n, (rank + 1) * part_len), part_len a multiple of 32; `spikes` holds
 *    world * part_len / 32 words.  The all-gather of step n overlaps the
 *    local binning of step n (delay 1) or the whole update of step n + 1
 *    (delay >= 2; SURVEY 8(e) options (i) and (iii)).  world may be 1.
 *  - exchange = BP_EXCHANGE_CALLER: the caller all-gathers the vector itself
 *    between bp_network_update and the next bp_network_scatter.
 *
 * Memory: the network's event buckets (~5 % of the fan-in x local neurons
 * x 4 B per delay slot, plus 4 B x classes x local neurons of overflow
 * counters) and its projection table are DEVICE memory that
 * bp_network_create allocates and bp_network_destroy frees
 * (bp_network_device_bytes reports the amount); all state arrays, the spike
 * vector and the workspace belong to the caller.
 * --------------------------------------------------------------------- */
#define BP_MAX_PROJ 8
typedef enum { BP_RECEPTOR_EXC = 0, BP_RECEPTOR_INH = 1 } bp_receptor;
typedef enum { BP_EXCHANGE_CALLER = 0, BP_EXCHANGE_NCCL = 1 } bp_exchange;

typedef struct {
  int32_t conn;               /* bp_conn                                        */
  int32_t receptor;           /* bp_receptor: the conductance it adds into      */
  int64_t pre_begin, pre_end; /* presynaptic neurons (global ids)               */
  float weight;               /* homogeneous weight per event                   */
  int32_t reserved;           /* must be 0                                      */
  bp_jitconn jit;             /* conn == BP_CONN_JIT: columns = all n neurons   */
  /* conn == BP_CONN_CSR: column-sliced CSR of this process's columns, indices
   * local to [col_begin, col_end), pre_end - pre_begin rows               */
  const int64_t *indptr;
  const int32_t *indices;
} bp_projection;

typedef struct {
  int32_t model;  /* bp_model */
  int32_t g_kind; /* bp_out_kind of state.g_exc / g_inh */
  int32_t delay_steps; /* synaptic delay D in steps (0 => 1, the paper's one-step
                          VarDelay); spikes of step n are delivered at
                          step n + D (reading D1); <= 16.
                          D > 1 keeps D + 1 bucket slots. */
  int32_t n_proj; /* 1 .. BP_MAX_PROJ */
  int64_t n;
  int64_t col_begin, col_end;
  bp_projection proj[BP_MAX_PROJ];
  bp_neuron_params params;
  bp_neuron_state state; /* local neurons, col_end - col_begin entries     */
  uint32_t *spikes;      /* global bit vector, >= ceil(n/32) words (NCCL:
                            world * part_len / 32); holds spikes_{n-1} on
                            entry to a step                               */
  void *ws;              /* >= bp_network_workspace_bytes(desc), 256-aligned */
  size_t ws_bytes;
  /* multi-process exchange */
  int32_t exchange;      /* bp_exchange                                     */
  int32_t rank, world;   /* BP_EXCHANGE_NCCL: this process / process count  */
  int32_t reserved2;     /* must be 0                                       */
  int64_t part_len;      /* BP_EXCHANGE_NCCL: partition length (see above)  */
  uint8_t nccl_id[128];  /* BP_EXCHANGE_NCCL: ncclUniqueId, the same bytes on
                            every rank (bp_nccl_unique_id on one of them)   */
} bp_network_desc;

typedef struct bp_network bp_network; /* opaque; not thread-safe */

/* ncclUniqueId for BP_EXCHANGE_NCCL (128 bytes into out), to be sent to every
 * rank by the caller's own means.  BP_ERR_NCCL when NCCL cannot be loaded
 * (libbp resolves NCCL at run time: an already loaded libnccl.so.2, else
 * the one the dynamic loader finds; BP_NCCL_LIB overrides the path). */
bp_status bp_nccl_unique_id(uint8_t *out);
/* The NCCL the library resolved (ncclGetVersion code, e.g. 22809), or
 * BP_ERR_NCCL when none can be loaded -- a cheap check every rank can make
 * before the collective bp_network_create. */
bp_status bp_nccl_version(int32_t *version);

size_t bp_network_workspace_bytes(const bp_network_desc *desc);
/* Copies *desc (all buffers stay owned by the caller), initialises the
 * workspace on `stream` from desc->spikes.  With BP_EXCHANGE_NCCL this is a
 * collective: every rank must call it (ncclCommInitRank). */
bp_status bp_network_create(const bp_network_desc *desc, bp_stream stream,
                            bp_network **out);
/* n_steps full steps (with BP_EXCHANGE_NCCL the all-gather included).
 * raster_out (nullable, device): n_steps x ceil((col_end-col_begin)/32)
 * words of local spikes.  counts_out (nullable; device or page-locked host
 * memory): n_steps int32, the number of local spikes emitted in each step
 * (copied asynchronously). */
bp_status bp_network_step(bp_network *net, int64_t n_steps,
                          uint32_t *raster_out, int32_t *counts_out,
                          bp_stream stream);
/* The two halves of a step for BP_EXCHANGE_CALLER multi-process runs. */
bp_status bp_network_scatter(bp_network *net, bp_stream stream);
bp_status bp_network_update(bp_network *net, uint32_t *raster_row,
                            bp_stream stream);
/* bp_network_update, and make `exchange_stream` wait (cudaStreamWaitEvent)
 * only for this step's spike words -- before the local binning kernel -- so
 * the caller's all-gather on exchange_stream overlaps the binning (SURVEY
 * 8(e) overlap option (i)).  The caller must order its next
 * bp_network_scatter on `stream` after the exchange. */
bp_status bp_network_update_overlap(bp_network *net, uint32_t *raster_row,
                                    bp_stream stream, bp_stream exchange_stream);
/* Device counters since create: [0] = local spikes, [1] = synaptic events
 * delivered into local neurons, [2] = saturated BP_OUT_FIX32 conductance
 * updates (0 in a well-scaled run), [3] = non-finite membrane potentials
 * seen after a step (debug check, only with the environment variable
 * BP_DEBUG_NAN=1 at create; else 0).  Copies into host uint64[4];
 * synchronises `stream`. */
bp_status bp_network_counters(bp_network *net, uint64_t *host_out,
                              bp_stream stream);
/* Device memory the network allocated itself (buckets, projection table). */
size_t bp_network_device_bytes(const bp_network *net);
/* The execution plan chosen at create, into out[0 .. n) (host int32, up to
 * 8): [0] single-CTA time loop, [1] dense delivery, [2] tiles, [3] bucket
 * capacity per tile, [4] weight-class fold (2 or 4), [5] JIT binning split
 * (2 or 4 lanes per (row, segment) item, 32 = a warp per row, 64 = a warp
 * per (row, segment) item), [6] library NCCL exchange, [7] weight classes. */
bp_status bp_network_describe(const bp_network *net, int32_t *out, int32_t n);
/* Per-kernel timing of the next bp_network_step calls (at most max_steps
 * steps): CUDA events are recorded on `stream` before the neuron-update
 * kernel, between it and the event-binning kernel, and after the latter
 * (a step without a binning launch -- the dense HH update delivers its own
 * spikes -- records an empty binning interval).
 * _end synchronises and returns the summed device milliseconds of the
 * update kernels (update_ms) and of the binning kernels (scatter_ms) and
 * the number of steps recorded. */
bp_status bp_network_profile_begin(bp_network *net, int64_t max_steps);
bp_status bp_network_profile_end(bp_network *net, double *scatter_ms,
                                 double *update_ms, int64_t *steps);
/* Frees the buckets and, with BP_EXCHANGE_NCCL, destroys the communicator. */
void bp_network_destroy(bp_network *net);

#ifdef __cplusplus
}
#endif
#endif /* BP_H_ */
