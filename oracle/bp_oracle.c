/*
 * bp_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, single-threaded CPU oracle for the hot path of BrainPy
 * (arxiv 2311.05106): event-driven CSR scatter (Listing S1), just-in-time
 * random connectivity (App. C, Listing S2), exponential synapse + COBA + LIF
 * (App. E/F, Listing S3) and the COBA-HH variant (rule H1, EXTERNAL).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * constant table or helper with the CUDA product in paper_2311_05106_b200/.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 *        -o liboracle.so bp_oracle.c -lm
 * -ffp-contract=off: no multiply-add contraction; every FMA below is an
 * explicit fmaf()/fma() call, exactly where rules N1/H1/J7 write one.
 *
 * Citation key: P:n = line n of PAPER.md, S:n = line n of SPEC.md,
 * "rule Xn" = the reading recorded in DESIGN.md section "Readings".
 *
 * Parity pins (tests/test_oracle_*.py): every function here is pinned by
 * something other than itself; see the "pinned by" line of each function.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#define OR_OUT_F64 0   /* accumulate (double)w                               */
#define OR_OUT_FIX 1   /* accumulate llrint(w * 2^32) into int64 (rule F1)   */
#define OR_OUT_F32 2   /* accumulate w in float, sequentially (network f32)  */
#define OR_OUT_FIX32 3 /* accumulate llrint(w * 2^F) into int64 (rule F2)    */

/* ------------------------------------------------------------------------
 * Threads (test-time speed only; default 1).  The loops that may run on
 * several host threads are the ones whose result does not depend on the
 * order: per-neuron updates (or_lif_step, or_hh_step: independent
 * neurons) and event scatters into INTEGER accumulators (fixed point, or
 * fp64 sums of integer-valued weights, exact below 2^53), where every add
 * is an atomic integer/exact add.  Every other call runs the plain
 * sequential loop.  The parallel result is therefore bit-identical to the
 * sequential one (pinned: test_oracle_network.py threaded == sequential).
 * ---------------------------------------------------------------------- */
static int g_threads = 1;
void or_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int or_get_threads(void) { return g_threads; }

/* Rule F2 (32-bit fixed point): F fractional bits, set per run. */
static int g_fix32_bits = 20;
void or_set_fix32_bits(int bits) { g_fix32_bits = bits; }

#define OR_LAW_HOMO 0
#define OR_LAW_UNIFORM 1
#define OR_LAW_NORMAL 2

/* ------------------------------------------------------------------------
 * Rule J2: Philox4x32-10 (Salmon et al., SC'11).  Listing S2 uses Python's
 * global `random`; a counter-based generator keyed by
 * (seed, row, segment, draw) is our reading (reading R5/R7).
 * Pinned by: the three Random123 known-answer vectors (test_oracle_rng.py).
 * ---------------------------------------------------------------------- */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                      uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
    uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* word(tag, row, seg, j) = Philox(ctr=(j>>2, row, seg, tag),
 *                                 key=(lo32(seed), hi32(seed)))[j & 3]
 * Tags: 0 = gaps, 1 = weights, 2 = first offset (rule J2). */
uint32_t or_word(uint64_t seed, uint32_t tag, uint32_t row, uint32_t seg,
                 uint32_t j) {
  uint32_t ctr[4] = {j >> 2, row, seg, tag};
  uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
  uint32_t out[4];
  or_philox4x32_10(ctr, key, out);
  return out[j & 3u];
}

/* Rule J3: integer in [lo, hi] from one 32-bit word by multiply-shift. */
static uint32_t uniform_int(uint32_t lo, uint32_t hi, uint32_t x) {
  uint64_t span = (uint64_t)hi - (uint64_t)lo + 1u;
  return lo + (uint32_t)(((uint64_t)x * span) >> 32);
}

/* ------------------------------------------------------------------------
 * Rule J1: the gap bound K.  App. C: gaps ~ U[1, floor(2/p - 1)]
 * (the text's floor, not Listing S2's ceil at P:350).  Because fp64
 * 2/p - 1 lands a hair below an integer for many p = 80/N (e.g. N = 4M),
 * a result within 1e-9 relative of an integer is snapped to it.
 * Returns 0 if p is not in (0, 1].
 * Pinned by: table test (p in {1e-3,1e-2,2e-2,5e-2} -> {1999,199,99,39},
 * N = 4e6 -> 99999, K = 1 iff p > 2/3), test_oracle_rng.py.
 * ---------------------------------------------------------------------- */
uint32_t or_conn_len(double p) {
  if (!(p > 0.0) || !(p <= 1.0)) return 0;
  double x = 2.0 / p - 1.0;
  double r = nearbyint(x);
  double k;
  double scale = fabs(x) > 1.0 ? fabs(x) : 1.0;
  if (fabs(x - r) <= 1e-9 * scale) k = r; else k = floor(x);
  if (k < 1.0) k = 1.0;
  if (k > 2147483647.0) return 0;
  return (uint32_t)k;
}

/* ------------------------------------------------------------------------
 * Rule J10: the geometric-gap sampler the paper
 * compares against (App. C: "sampled in constant time by inverting
 * the cumulative density function ... log(U[0,1]) / log(1 - P)", after
 * Knight & Nowotny 2020).  Gaps G ~ Geo(p) on {1, 2, ...}:
 *   u = ((x >> 8) + 1) 2^-24 in (0, 1]           (24-bit, exact in fp32)
 *   t = logf_j10(u) / c,   c = fl32(log1p(-p))    (IEEE fp32 division)
 *   G = 1 if ceil(t) < 1;  cap if t >= (float)cap;  else (uint32) ceil(t)
 * P(G >= k) = P(u < (1-p)^(k-1)) = (1-p)^(k-1): the exact geometric law
 * (up to the 24-bit u and fp32 rounding).  Being memoryless, the first
 * target of a segment is seg_begin + G_0 - 1 (G_0 from the tag-2 word 0):
 * every column is connected independently with probability p -- unlike
 * the uniform-gap rule, whose density is 2/(K+1) (reading R4).
 * cap = L + 1 (L = seg_len): any gap that long leaves the segment, so the
 * cap changes no position and keeps positions within 32 bits.
 * logf_j10 is an op-for-op specified fp32 log (the product kernels run the
 * same operations, so both sides draw identical gaps):
 *   u = m 2^e, m in [1, 2); if m > fl32(sqrt 2): m /= 2, e += 1
 *   f = m - 1 (exact), s = f / (2 + f), z = s s,
 *   r = Horner(z; 1/11, 1/9, 1/7, 1/5, 1/3) with fmaf (fl32 coefficients),
 *   log m = fmaf(2s, z r, 2s)   (2 atanh(s) = 2s (1 + z/3 + z^2/5 + ...))
 *   log u = fmaf(e, LN2_HI, fmaf(e, LN2_LO, log m)), LN2_HI = 0.693145751953125
 * Pinned by: <= 2 ulp vs libm logf on (0, 1]; the SPEC example p = 0.5,
 * u = 0.25 -> 2 and u -> 1 -> 1; mean gap 1/p within 1 %;
 * P(first = j) = (1-p)^j p; per-column density p within 4 sigma; row
 * fan-out variance L p (1-p) (Bernoulli process), test_oracle_jit.py.
 * ---------------------------------------------------------------------- */
static float g_geo_c = 0.0f;          /* 0: uniform gaps (rule J3)         */
void or_set_gap_sampler(float c) { g_geo_c = c; }
float or_geo_c(double p) { return (float)log1p(-p); }

float or_logf_j10(float u) {
  uint32_t b;
  memcpy(&b, &u, 4);
  int e = (int)(b >> 23) - 127;
  uint32_t mb = (b & 0x7FFFFFu) | 0x3F800000u;
  float m;
  memcpy(&m, &mb, 4);
  if (m > 1.41421353816986083984375f) { m = m * 0.5f; e += 1; }
  float f = m - 1.0f;
  float s = f / (2.0f + f);
  float z = s * s;
  float r = fmaf(z, 1.0f / 11.0f, 1.0f / 9.0f);
  r = fmaf(z, r, 1.0f / 7.0f);
  r = fmaf(z, r, 1.0f / 5.0f);
  r = fmaf(z, r, 1.0f / 3.0f);
  float zr = z * r;
  float s2 = s + s;
  float lm = fmaf(s2, zr, s2);
  float ef = (float)e;
  return fmaf(ef, 0.693145751953125f, fmaf(ef, 1.428606765330187e-6f, lm));
}

/* ------------------------------------------------------------------------
 * Reading J7n: cos(2 pi u) for u in [0, 1) (24-bit u), op-for-op specified
 * in fp32 (the kernels run the same operations):
 *   v = u - rint(u) in [-1/2, 1/2] (exact);  a = |v|;
 *   a > 1/4:  cos(2 pi a) = -cos(2 pi (1/2 - a));  b = min(a, 1/2 - a) (exact)
 *   b <= 1/8: cos(theta), theta = fl(2 pi b), Taylor to theta^10 (Horner, fmaf)
 *   b >  1/8: sin(theta'), theta' = fl(2 pi (1/4 - b)), Taylor to theta'^9
 * Pinned by: <= 4 ulp vs libm cos on a dense grid of [0, 1) (absolute
 * 2^-24 near the zeros), symmetry and the exact values at u = 0, 1/4, 1/2.
 * ---------------------------------------------------------------------- */
float or_cos2pi_j7(float u) {
  float v = u - rintf(u);
  float a = fabsf(v);
  float sgn = 1.0f;
  if (a > 0.25f) { a = 0.5f - a; sgn = -1.0f; }
  float r;
  if (a <= 0.125f) {
    float t = 6.28318548202514648438f * a;            /* fl32(2 pi) */
    float t2 = t * t;
    float p = fmaf(t2, -2.7557319e-7f, 2.4801587e-5f);   /* -1/10!, 1/8! */
    p = fmaf(t2, p, -1.3888889e-3f);                     /* -1/6! */
    p = fmaf(t2, p, 4.1666668e-2f);                      /* 1/4! */
    p = fmaf(t2, p, -0.5f);
    r = fmaf(t2, p, 1.0f);
  } else {
    float t = 6.28318548202514648438f * (0.25f - a);
    float t2 = t * t;
    float p = fmaf(t2, 2.7557319e-6f, -1.9841270e-4f);  /* 1/9!, -1/7! */
    p = fmaf(t2, p, 8.3333338e-3f);                      /* 1/5! */
    p = fmaf(t2, p, -0.16666667f);                       /* -1/3! */
    r = fmaf(t * t2, p, t);
  }
  return sgn * r;
}

uint32_t or_geo_gap(float c, uint32_t cap, uint32_t x) {
  float u = (float)((x >> 8) + 1u) * 0x1p-24f;
  float t = or_logf_j10(u) / c;
  if (!(t < (float)cap)) return cap;
  float ct = ceilf(t);
  if (ct < 1.0f) return 1u;
  uint32_t g = (uint32_t)ct;
  return g > cap ? cap : g;
}

/* Sampler-cost probe (App. C: uniform gaps are "one order of
 * magnitude faster than sampling from Geo[p]"; SPEC bench_gap_samplers):
 * sum of n gaps drawn from counter-based words with U[1, K] (geometric == 0)
 * or Geo(p) by inversion (geometric != 0, c = fl32(log1p(-p))).  Timed by
 * tests/test_oracle_jit.py; the sums pin both means (K+1)/2 and ~1/p. */
uint64_t or_gap_draws(int geometric, double p, uint64_t n, uint64_t seed) {
  uint32_t K = or_conn_len(p);
  float c = (float)log1p(-p);
  uint64_t sum = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t x = or_word(seed, 0u, (uint32_t)(i >> 20), 0u, (uint32_t)(i & 0xFFFFFu));
    sum += geometric ? or_geo_gap(c, 0x7FFFFFFFu, x) : uniform_int(1u, K, x);
  }
  return sum;
}

/* Offset of the first target of (row, seg) from the segment start: rule J5
 * (uniform gaps) or G_0 - 1 (rule J10). */
static uint32_t first_offset_of(uint64_t seed, uint32_t K, uint32_t L,
                                uint32_t row, uint32_t s) {
  if (g_geo_c != 0.0f)
    return or_geo_gap(g_geo_c, L + 1u, or_word(seed, 2u, row, s, 0u)) - 1u;
  uint32_t a = uniform_int(0u, K - 1u, or_word(seed, 2u, row, s, 0u));
  uint32_t b = uniform_int(0u, K, or_word(seed, 2u, row, s, 1u));
  if (b <= a) a = K - 1u - a;
  return a;
}

/* Gap e of (row, seg): U[1, K] (rule J3/J6) or Geo(p) (rule J10). */
static uint32_t gap_of(uint64_t seed, uint32_t K, uint32_t L, uint32_t row,
                       uint32_t s, uint32_t e) {
  uint32_t x = or_word(seed, 0u, row, s, e);
  if (g_geo_c != 0.0f) return or_geo_gap(g_geo_c, L + 1u, x);
  return uniform_int(1u, K, x);
}

/* Rule F1: fixed-point quantisation q(w) = llrint(w * 2^32) (half-even). */
int64_t or_quantize(float w) {
  return llrint((double)w * 4294967296.0);
}

/* Rule J7: weight of edge e of (row, seg).  Weights use their own stream
 * (tag 1), so the connectivity does not depend on the weight law.
 *   homo    : w0 (Listing S2 caption: "all nonzero elements ... the
 *             same value").
 *   uniform : U[w0, w1) (`mv_prob_uniform(w_low, w_high, ...)`).
 *   normal  : N(mu = w0, sigma = w1) by Box-Muller. */
static float edge_weight(uint64_t seed, int law, float w0, float w1,
                         uint32_t row, uint32_t seg, uint32_t e) {
  if (law == OR_LAW_HOMO) return w0;
  if (law == OR_LAW_UNIFORM) {
    uint32_t x = or_word(seed, 1u, row, seg, e);
    float u = (float)(x >> 8) * 0x1p-24f;              /* [0, 1), exact */
    float span = w1 - w0;                              /* fp32 rounding */
    return fmaf(u, span, w0);
  }
  /* normal: Box-Muller in fp32 with the specified log (rule J10) and
   * cos(2 pi u) (or_cos2pi_j7) -- reading J7n */
  uint32_t x1 = or_word(seed, 1u, row, seg, 2u * e);
  uint32_t x2 = or_word(seed, 1u, row, seg, 2u * e + 1u);
  float u1 = (float)((x1 >> 8) + 1u) * 0x1p-24f;       /* (0, 1], exact */
  float u2 = (float)(x2 >> 8) * 0x1p-24f;              /* [0, 1), exact */
  float radius = sqrtf(-2.0f * or_logf_j10(u1));       /* IEEE sqrt */
  float z = radius * or_cos2pi_j7(u2);
  return fmaf(w1, z, w0);
}

/* ------------------------------------------------------------------------
 * Rules J4-J7: the targets and weights of one row, in order.
 * For each segment s = [s*L, min((s+1)*L, n_cols)) (rule J4):
 *   first offset a (rule J5): a = U[0,K-1](word(2,r,s,0)),
 *       b = U[0,K](word(2,r,s,1)); if b <= a then a = K-1-a;
 *   pos = s*L + a; e = 0
 *   while pos < seg_end: emit (pos, w_e); pos += U[1,K](word(0,r,s,e)); e++
 * This is Listing S2's loop ("post_i += random.randint(1,
 * max_cdist)") with a per-(row, segment) counter stream and the stationary
 * start instead of randint(1, K) (readings R5, R6).
 * Writes at most `cap` entries; returns the full count.
 * Pinned by: K = 1 dense rows, E[fan-out] = n_cols*2/(K+1) within 4 sigma,
 * per-column connection frequency, first-offset histogram
 * 2(K-j)/(K(K+1)), mean gap (K+1)/2 (test_oracle_jit.py).
 * ---------------------------------------------------------------------- */
int64_t or_jit_row(uint64_t seed, uint32_t K, uint32_t L, int64_t n_cols,
                   int law, float w0, float w1, uint32_t row,
                   int64_t seg_first, int64_t seg_last,
                   int32_t *pos_out, float *w_out, int64_t cap) {
  int64_t count = 0;
  for (int64_t s = seg_first; s <= seg_last; ++s) {
    int64_t seg_begin = s * (int64_t)L;
    int64_t seg_end = seg_begin + (int64_t)L;
    if (seg_end > n_cols) seg_end = n_cols;
    int64_t pos = seg_begin + (int64_t)first_offset_of(seed, K, L, row, (uint32_t)s);
    uint32_t e = 0;
    while (pos < seg_end) {
      if (count < cap) {
        pos_out[count] = (int32_t)pos;
        if (w_out) w_out[count] = edge_weight(seed, law, w0, w1, row, (uint32_t)s, e);
      }
      ++count;
      pos += (int64_t)gap_of(seed, K, L, row, (uint32_t)s, e);
      ++e;
    }
  }
  return count;
}

/* The exact-accumulation kinds that may be summed by several threads. */
static int order_free(int out_kind, const double *abs_out, int law, float w0,
                      const float *data) {
  if (g_threads <= 1 || abs_out) return 0;
  if (out_kind == OR_OUT_FIX || out_kind == OR_OUT_FIX32) return 1;
  return out_kind == OR_OUT_F64 && law == OR_LAW_HOMO && !data &&
         w0 == rintf(w0) && fabsf(w0) < 1048576.0f;
}

/* Atomic variant of accumulate() for order_free() kinds. */
static void accumulate_atomic(int out_kind, void *out, int64_t c, float w) {
  if (out_kind == OR_OUT_F64) {
    double *o = (double *)out + c;
#pragma omp atomic
    *o += (double)w;
  } else {
    int64_t q = out_kind == OR_OUT_FIX ? or_quantize(w)
                                       : llrint(ldexp((double)w, g_fix32_bits));
    int64_t *o = (int64_t *)out + c;
#pragma omp atomic
    *o += q;
  }
}

static void accumulate(int out_kind, void *out, double *abs_out, int64_t c,
                       float w) {
  if (out_kind == OR_OUT_F64) {
    ((double *)out)[c] += (double)w;
  } else if (out_kind == OR_OUT_FIX) {
    ((int64_t *)out)[c] += or_quantize(w);
  } else if (out_kind == OR_OUT_FIX32) {
    ((int64_t *)out)[c] += llrint(ldexp((double)w, g_fix32_bits));
  } else {
    ((float *)out)[c] += w;
  }
  if (abs_out) abs_out[c] += fabs((double)w);
}

/* ------------------------------------------------------------------------
 * event_csrmv -- Listing S1 with `indices[j]` (the listing's
 * `indices[i]` is a typo; reading R1):
 *   for i, event in enumerate(events):
 *     if event:
 *       for j in range(indptr[i], indptr[i+1]):
 *         outs[indices[j]] += data[j]
 * data == NULL means the homogeneous weight w_homo.
 * Accumulates into `out` (caller zeroes it).  abs_out (nullable) receives
 * the sum of |w| per output, for the T2 tolerance.
 * Pinned by: dense brute force D^T s in numpy on random tiny instances
 * (exact for integer weights), test_oracle_csr.py.
 * ---------------------------------------------------------------------- */
void or_event_csrmv(const int64_t *indptr, const int32_t *indices,
                    const float *data, float w_homo, int64_t n_rows,
                    const uint8_t *events, int out_kind, void *out,
                    double *abs_out) {
  if (order_free(out_kind, abs_out, OR_LAW_HOMO, w_homo, data)) {
#pragma omp parallel for schedule(dynamic, 64) num_threads(g_threads)
    for (int64_t i = 0; i < n_rows; ++i) {
      if (!events[i]) continue;
      for (int64_t j = indptr[i]; j < indptr[i + 1]; ++j)
        accumulate_atomic(out_kind, out, (int64_t)indices[j], w_homo);
    }
    return;
  }
  for (int64_t i = 0; i < n_rows; ++i) {
    if (!events[i]) continue;
    for (int64_t j = indptr[i]; j < indptr[i + 1]; ++j) {
      float w = data ? data[j] : w_homo;
      accumulate(out_kind, out, abs_out, (int64_t)indices[j], w);
    }
  }
}

/* ------------------------------------------------------------------------
 * jitconn event_mv -- Listing S2, rule J9:
 *   out[c - col_begin] += sum over active rows r of the edges of row r
 *   whose target c lies in [col_begin, col_end).
 * Only the segments that intersect [col_begin, col_end) are generated;
 * the connectivity of a row is the same whichever columns are requested.
 * Pinned by: materialise -> CSR -> or_event_csrmv (an independent path),
 * single-spike probes, K = 1 closed form, test_oracle_jit.py.
 * ---------------------------------------------------------------------- */
void or_jit_event_mv(uint64_t seed, uint32_t K, uint32_t L, int law, float w0,
                     float w1, int64_t n_rows, int64_t n_cols,
                     int64_t col_begin, int64_t col_end,
                     const uint8_t *events, int out_kind, void *out,
                     double *abs_out) {
  if (col_end <= col_begin) return;
  int64_t seg_first = col_begin / (int64_t)L;
  int64_t seg_last = (col_end - 1) / (int64_t)L;
  const int par = order_free(out_kind, abs_out, law, w0, NULL);
#pragma omp parallel for schedule(dynamic, 64) num_threads(g_threads) if (par)
  for (int64_t r = 0; r < n_rows; ++r) {
    if (!events[r]) continue;
    for (int64_t s = seg_first; s <= seg_last; ++s) {
      int64_t seg_begin = s * (int64_t)L;
      int64_t seg_end = seg_begin + (int64_t)L;
      if (seg_end > n_cols) seg_end = n_cols;
      int64_t pos = seg_begin +
                    (int64_t)first_offset_of(seed, K, L, (uint32_t)r, (uint32_t)s);
      uint32_t e = 0;
      while (pos < seg_end) {
        if (pos >= col_begin && pos < col_end) {
          float w = edge_weight(seed, law, w0, w1, (uint32_t)r, (uint32_t)s, e);
          if (par) accumulate_atomic(out_kind, out, pos - col_begin, w);
          else accumulate(out_kind, out, abs_out, pos - col_begin, w);
        }
        pos += (int64_t)gap_of(seed, K, L, (uint32_t)r, (uint32_t)s, e);
        ++e;
      }
    }
  }
}

/* ------------------------------------------------------------------------
 * Gather-orientation event csrmv (BrainPy csrmv(..., transpose=False);
 * SURVEY 8(f) NEXT 3, reading G1): the CSR rows are the OUTPUTS and the
 * column indices the event (spike) index:
 *   out[r] (+)= sum_{k in row r} [events[indices[k]]] * w_k.
 * Pinned by: equals the scatter (Listing S1) of the transposed matrix, bit
 * for bit in fixed point (test_oracle_csr.py).
 * ---------------------------------------------------------------------- */
void or_csrmv_gather(const int64_t *indptr, const int32_t *indices, const float *data,
                     float w_homo, int64_t n_rows, const uint8_t *events, int out_kind,
                     void *out, double *abs_out) {
  for (int64_t r = 0; r < n_rows; ++r)
    for (int64_t k = indptr[r]; k < indptr[r + 1]; ++k)
      if (events[indices[k]]) accumulate(out_kind, out, abs_out, r, data ? data[k] : w_homo);
}

/* ------------------------------------------------------------------------
 * Reverse mode of the event scatter y = M^T s (Listing S1; SURVEY 8(f)
 * NEXT 3, "differentiability", reading G1): with upstream gradient gy
 * (n_cols) of L,
 *   dL/ddata[k] = s[r(k)] * gy[indices[k]]            (grad_data, nnz)
 *   dL/ds[r]    = sum_{k in row r} w_k * gy[indices[k]] (grad_events, n_rows,
 *                 the events read as real numbers: a gather product)
 *   dL/dw       = sum_{r: s[r]} sum_{k in row r} gy[indices[k]]  (homogeneous w)
 * in fp64 (grad_data is exact in fp32).  Any output may be NULL.
 * Pinned by: torch autograd of the dense fp64 product (test_oracle_csr.py).
 * ---------------------------------------------------------------------- */
void or_csrmv_grad(const int64_t *indptr, const int32_t *indices, const float *data,
                   float w_homo, int64_t n_rows, const uint8_t *events, const float *gy,
                   float *grad_data, double *grad_events, double *grad_w) {
  double gw = 0.0;
  for (int64_t r = 0; r < n_rows; ++r) {
    double ge = 0.0;
    for (int64_t k = indptr[r]; k < indptr[r + 1]; ++k) {
      const double g = (double)gy[indices[k]];
      if (grad_data) grad_data[k] = events[r] ? gy[indices[k]] : 0.0f;
      ge += (data ? (double)data[k] : (double)w_homo) * g;
      if (events[r]) gw += g;
    }
    if (grad_events) grad_events[r] = ge;
  }
  if (grad_w) *grad_w = gw;
}

/* ------------------------------------------------------------------------
 * Non-event JIT matrix-vector product, mv_prob_{homo,uniform,normal} (P:94,
 * P:192), reading MV1:
 *   out[c] (+)= sum_r v[r] * w_e(r) over the edges (r, e) with pos_e(r) = c,
 * the same connectivity and weights as rules J1-J9 (orientation as
 * Listing S2: rows = vector index, columns = output).  The product of two
 * fp32 numbers is exact in fp64, so
 *   OR_OUT_F64: (double)v * (double)w   (the reference),
 *   OR_OUT_FIX: llrint(2^32 * (double)v * (double)w)  (one rounding, rule F1),
 *   OR_OUT_F32: fl32(v * w) added in fp32.
 * Rows with v[r] == 0 contribute nothing and are skipped.
 * Pinned by: v in {0, 1} equals or_jit_event_mv bit for bit (fixed point),
 * the dense fp64 D^T v of the materialised matrix, linearity in v
 * (test_oracle_jit.py).
 * ---------------------------------------------------------------------- */
void or_jit_mv(uint64_t seed, uint32_t K, uint32_t L, int law, float w0, float w1,
               int64_t n_rows, int64_t n_cols, int64_t col_begin, int64_t col_end,
               const float *v, int out_kind, void *out, double *abs_out) {
  if (col_end <= col_begin) return;
  int64_t seg_first = col_begin / (int64_t)L;
  int64_t seg_last = (col_end - 1) / (int64_t)L;
  for (int64_t r = 0; r < n_rows; ++r) {
    if (v[r] == 0.0f) continue;
    for (int64_t s = seg_first; s <= seg_last; ++s) {
      int64_t seg_begin = s * (int64_t)L;
      int64_t seg_end = seg_begin + (int64_t)L;
      if (seg_end > n_cols) seg_end = n_cols;
      int64_t pos = seg_begin +
                    (int64_t)first_offset_of(seed, K, L, (uint32_t)r, (uint32_t)s);
      uint32_t e = 0;
      while (pos < seg_end) {
        if (pos >= col_begin && pos < col_end) {
          float w = edge_weight(seed, law, w0, w1, (uint32_t)r, (uint32_t)s, e);
          double prod = (double)v[r] * (double)w;         /* exact */
          int64_t c = pos - col_begin;
          if (out_kind == OR_OUT_F64) ((double *)out)[c] += prod;
          else if (out_kind == OR_OUT_FIX) ((int64_t *)out)[c] += llrint(ldexp(prod, 32));
          else ((float *)out)[c] += v[r] * w;
          if (abs_out) abs_out[c] += fabs(prod);
        }
        pos += (int64_t)gap_of(seed, K, L, (uint32_t)r, (uint32_t)s, e);
        ++e;
      }
    }
  }
}

/* ------------------------------------------------------------------------
 * Rule F2: a step's increments (summed exactly in int64, OR_OUT_FIX32) are
 * added to the int32 conductance with saturation at the int32 range.
 * Returns the number of saturated entries (a diagnostic; 0 in any sane run).
 * Pinned by: fixed-point vs fp64 recursion bound and the saturation test.
 * ---------------------------------------------------------------------- */
int64_t or_fix32_add(int32_t *g, const int64_t *inc, int64_t n) {
  int64_t sat = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t v = (int64_t)g[i] + inc[i];
    if (v > INT32_MAX) { v = INT32_MAX; ++sat; }
    if (v < INT32_MIN) { v = INT32_MIN; ++sat; }
    g[i] = (int32_t)v;
  }
  return sat;
}

/* ------------------------------------------------------------------------
 * Rule N1: one step of exponential synapse (AlignPost) + COBA + LIF with
 * refractory period for neurons [0, n).
 *   LIF: tau dV/dt = -(V - V_rest) + R G;  spike if V > V_th,
 *        then V = V_reset; refractory 5 ms held as an integer countdown.
 *   COBA: G = -sum_j g_j (V - E_j) = g_E(E_E - V) + g_I(E_I - V).
 *   Expon: g(t) = exp(-dt/tau) g(t - dt); g += w on a spike.
 *        g arrives here already holding alpha*g_{n-1} + increments; after
 *        the update it is pre-decayed for the next step (reading R12).
 *   I_ext: step_run(i, 20.) adds 20 every step (reading R19).
 * Integration: exponential Euler with I held over the step (reading R15):
 *   I    = fmaf(gI, E_I - V, fmaf(gE, E_E - V, I_ext))
 *   Vinf = fmaf(R, I, V_rest)
 *   Vc   = fmaf(V - Vinf, alpha_V, Vinf)
 * g_kind 1 (fixed point, rule F1): g = (float)ldexp((double)g_fix, -32);
 *   g_fix' = llrint((double)g_fix * alpha_d).   g_kind 0: g' = g*(float)alpha.
 * g_kind 2 (32-bit fixed point, rule F2): g = (float)ldexp((double)g, -F);
 *   g' = (g * A + 2^31) >> 32 with A = llrint(alpha_d * 2^32).
 * Writes events[i] = 1 for a spike, else 0.
 * Pinned by: subthreshold closed form V_n = V_rest + (V0-V_rest) alpha^n,
 * the 139-step first passage and 189-step period of an unconnected neuron,
 * COBA current I = 36 at E=0, V=-60, g=0.6, decay semigroup
 * (test_oracle_neuron.py).
 * ---------------------------------------------------------------------- */
typedef struct {
  float v_rest, v_reset, v_th, r, i_ext, e_exc, e_inh, alpha_v;
  double alpha_e, alpha_i;
  int32_t ref_steps;
  int32_t pad_;
} or_lif_params;

static float g_read(int g_kind, const void *g, int64_t i) {
  if (g_kind == 1) return (float)ldexp((double)((const int64_t *)g)[i], -32);
  if (g_kind == 2) return (float)ldexp((double)((const int32_t *)g)[i], -g_fix32_bits);
  return ((const float *)g)[i];
}

static void g_decay(int g_kind, void *g, int64_t i, double alpha) {
  if (g_kind == 1) {
    int64_t *gf = (int64_t *)g;
    gf[i] = llrint((double)gf[i] * alpha);
  } else if (g_kind == 2) {
    /* rule F2 decay: A = llrint(alpha * 2^32); g' = (g * A + 2^31) >> 32
     * (integer multiply-shift, round half up; arithmetic shift) */
    int32_t *gf = (int32_t *)g;
    int64_t A = llrint(alpha * 4294967296.0);
    gf[i] = (int32_t)(((int64_t)gf[i] * A + ((int64_t)1 << 31)) >> 32);
  } else {
    float *gs = (float *)g;
    gs[i] = gs[i] * (float)alpha;
  }
}

void or_lif_step(const or_lif_params *p, int64_t n, float *v, void *g_exc,
                 void *g_inh, int g_kind, uint8_t *ref, uint8_t *events) {
  #pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (int64_t i = 0; i < n; ++i) {
    float V = v[i];
    float gE = g_read(g_kind, g_exc, i);
    float gI = g_read(g_kind, g_inh, i);
    float I = fmaf(gI, p->e_inh - V, fmaf(gE, p->e_exc - V, p->i_ext));
    float Vinf = fmaf(p->r, I, p->v_rest);
    float Vc = fmaf(V - Vinf, p->alpha_v, Vinf);
    uint8_t spike = 0;
    if (ref[i] > 0) {
      ref[i] = (uint8_t)(ref[i] - 1);           /* hold V while refractory */
    } else if (Vc > p->v_th) {                  /* strict '>'      */
      v[i] = p->v_reset;
      ref[i] = (uint8_t)p->ref_steps;
      spike = 1;
    } else {
      v[i] = Vc;
    }
    events[i] = spike;
    g_decay(g_kind, g_exc, i, p->alpha_e);
    g_decay(g_kind, g_inh, i, p->alpha_i);
  }
}

/* ------------------------------------------------------------------------
 * Rule H1-exp: the exponential used by the HH update on both sides of the
 * parity test, fixed op-for-op so the two sides agree bit for bit:
 *   x clamped to [-87, 88]; k = rintf(x * log2(e));
 *   r = fmaf(k, -ln2_hi, x); r = fmaf(k, -ln2_lo, r);
 *   p = degree-7 Taylor polynomial of e^r by Horner with fmaf;
 *   result = p * 2^k.
 * Pinned by: |or_expf(x) - exp(x)| <= 2 ulp on a dense grid of [-87, 88]
 * against libm's double exp (test_oracle_neuron.py).
 * ---------------------------------------------------------------------- */
float or_expf(float x) {
  if (x > 88.0f) x = 88.0f;
  if (x < -87.0f) x = -87.0f;
  float t = x * 1.44269502162933349609375f;            /* log2(e) in fp32 */
  float k = rintf(t);
  float r = fmaf(k, -0.693145751953125f, x);            /* ln2 high part   */
  r = fmaf(k, -1.428606765330187045e-06f, r);           /* ln2 low part    */
  float q = 1.98412698412698412e-04f;                   /* 1/5040          */
  q = fmaf(q, r, 1.38888888888888889e-03f);             /* 1/720           */
  q = fmaf(q, r, 8.33333333333333333e-03f);             /* 1/120           */
  q = fmaf(q, r, 4.16666666666666667e-02f);             /* 1/24            */
  q = fmaf(q, r, 1.66666666666666667e-01f);             /* 1/6             */
  q = fmaf(q, r, 0.5f);
  q = fmaf(q, r, 1.0f);
  q = fmaf(q, r, 1.0f);
  int ki = (int)k;
  uint32_t bits = (uint32_t)(ki + 127) << 23;
  float scale;
  memcpy(&scale, &bits, sizeof scale);
  return q * scale;
}

/* u / (exp(u/k) - 1), with its removable singularity at u = 0 replaced by
 * the first-order value k - u/2 when |u| < 1e-4 (rule H1). */
static float efrac(float u, float k) {
  if (fabsf(u) < 1e-4f) return fmaf(-0.5f, u, k);
  return u / (or_expf(u / k) - 1.0f);
}

/* ------------------------------------------------------------------------
 * Rule H1 (EXTERNAL -- the paper only cites the COBA-HH benchmark of
 * Brette et al. 2007 at P:184 / P:177): Traub-Miles HH with COBA synapses,
 * one exponential-Euler step for neurons [0, n).  Units mV, ms, nS, pF.
 *   x = V - V_T
 *   am = 0.32 efrac(13 - x, 4)        bm = 0.28 efrac(x - 40, 5)
 *   ah = 0.128 e^{(17 - x)/18}        bh = 4 / (1 + e^{(40 - x)/5})
 *   an = 0.032 efrac(15 - x, 5)       bn = 0.5 e^{(10 - x)/40}
 *   y' = y_inf + (y - y_inf) e^{-dt (a + b)},   y_inf = a / (a + b)
 *   G  = g_L + g_Na m^3 h + g_K n^4 + g_E + g_I   (old m, h, n)
 *   V_inf = (g_L E_L + g_Na m^3 h E_Na + g_K n^4 E_K + g_E E_E + g_I E_I
 *            + I_ext) / G
 *   V' = V_inf + (V - V_inf) e^{-dt G / C}
 *   spike: V' >= V_spike and V < V_spike (upward crossing of -20 mV).
 * g is read, used, then pre-decayed exactly as in or_lif_step.
 * Pinned by: resting fixed point with no input, single-neuron spike times
 * against an fp64 RK4 reference at dt = 1e-3 ms (test_oracle_neuron.py).
 * ---------------------------------------------------------------------- */
typedef struct {
  float c_m, g_l, e_l, g_na, e_na, g_k, e_k, v_t;
  float e_exc, e_inh, i_ext, dt, v_spike;
  float pad_;
  double alpha_e, alpha_i;
} or_hh_params;

void or_hh_step(const or_hh_params *p, int64_t n, float *v, float *m, float *h,
                float *nk, void *g_exc, void *g_inh, int g_kind,
                uint8_t *events) {
  #pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (int64_t i = 0; i < n; ++i) {
    float V = v[i], M = m[i], H = h[i], Nk = nk[i];
    float gE = g_read(g_kind, g_exc, i);
    float gI = g_read(g_kind, g_inh, i);
    float x = V - p->v_t;
    float am = 0.32f * efrac(13.0f - x, 4.0f);
    float bm = 0.28f * efrac(x - 40.0f, 5.0f);
    float ah = 0.128f * or_expf((17.0f - x) / 18.0f);
    float bh = 4.0f / (1.0f + or_expf((40.0f - x) / 5.0f));
    float an = 0.032f * efrac(15.0f - x, 5.0f);
    float bn = 0.5f * or_expf((10.0f - x) / 40.0f);

    float sm = am + bm, sh = ah + bh, sn = an + bn;
    float m_inf = am / sm, h_inf = ah / sh, n_inf = an / sn;
    float m_new = fmaf(M - m_inf, or_expf(-(p->dt * sm)), m_inf);
    float h_new = fmaf(H - h_inf, or_expf(-(p->dt * sh)), h_inf);
    float n_new = fmaf(Nk - n_inf, or_expf(-(p->dt * sn)), n_inf);

    float g_na = p->g_na * (M * M * M) * H;
    float n2 = Nk * Nk;
    float g_k = p->g_k * (n2 * n2);
    float G = p->g_l + g_na + g_k + gE + gI;
    float num = p->g_l * p->e_l + g_na * p->e_na + g_k * p->e_k +
                gE * p->e_exc + gI * p->e_inh + p->i_ext;
    float Vinf = num / G;
    float V_new = fmaf(V - Vinf, or_expf(-(p->dt * G / p->c_m)), Vinf);

    events[i] = (uint8_t)((V_new >= p->v_spike && V < p->v_spike) ? 1 : 0);
    v[i] = V_new; m[i] = m_new; h[i] = h_new; nk[i] = n_new;
    g_decay(g_kind, g_exc, i, p->alpha_e);
    g_decay(g_kind, g_inh, i, p->alpha_i);
  }
}
