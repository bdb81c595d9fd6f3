/*
 * atk_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference `atk` core for the
 * two-stage approximate top-k hot path.  It is the *checker* for the CUDA
 * product in paper_2506_04165_b200/: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it.  The product never links or calls
 * this file, and there is no CPU fallback path that routes through it.
 *
 * Pinning: tests/test_oracle.py checks every function here against
 *   (a) the reference's own known-answer tests, restated from
 *       proj/tests/test_topk.cpp, test_planner.cpp, test_recall.cpp, and
 *   (b) the reference library itself, compiled from /root/reference sources
 *       into oracle/_ref/libatk_ref.so by oracle/Makefile (outputs committed
 *       as tests/golden/*.npz by tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj/core).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_EINFEASIBLE 3

static const char* g_err = "";
const char* orc_last_error(void) { return g_err; }
static int fail(const char* m) { g_err = m; return ORC_EINVAL; }

/* ---- rng: include/atk/rng.hpp:15-81 ------------------------------------ */
static uint64_t splitmix64_next(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint64_t orc_derive_seed(uint64_t seed, uint64_t stream) { /* rng.hpp:25-32 */
  uint64_t s = seed;
  (void)splitmix64_next(&s);
  s ^= 0x9e3779b97f4a7c15ull * (stream + 1);
  uint64_t a = splitmix64_next(&s);
  uint64_t b = splitmix64_next(&s);
  return a ^ (b >> 1);
}
typedef struct { uint64_t s[4]; } xoshiro;
static void xo_init(xoshiro* x, uint64_t seed) { /* rng.hpp:37-40 */
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) x->s[i] = splitmix64_next(&sm);
}
static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
static uint64_t xo_next(xoshiro* x) { /* rng.hpp:42-52 */
  uint64_t* s = x->s;
  const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
  s[2] ^= t; s[3] = rotl(s[3], 45);
  return r;
}
static double xo_double(xoshiro* x) { return (double)(xo_next(x) >> 11) * 0x1.0p-53; }
static uint64_t xo_below(xoshiro* x, uint64_t bound) { /* rng.hpp:59-73 */
  uint64_t v = xo_next(x);
  unsigned __int128 m = (unsigned __int128)v * bound;
  uint64_t lo = (uint64_t)m;
  if (lo < bound) {
    const uint64_t th = (0 - bound) % bound;
    while (lo < th) { v = xo_next(x); m = (unsigned __int128)v * bound; lo = (uint64_t)m; }
  }
  return (uint64_t)(m >> 64);
}
void orc_xoshiro_fill(uint64_t seed, uint64_t count, uint64_t* out) {
  xoshiro x; xo_init(&x, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = xo_next(&x);
}
void orc_shuffled_iota(uint64_t n, uint64_t seed, float* row) { /* tests/test_topk.cpp:30-39 */
  for (uint64_t i = 0; i < n; ++i) row[i] = (float)(i + 1);
  xoshiro x; xo_init(&x, seed);
  for (uint64_t i = n - 1; i >= 1; --i) {
    uint64_t j = xo_below(&x, i + 1);
    float t = row[i]; row[i] = row[j]; row[j] = t;
  }
}
void orc_uniform_below(uint64_t seed, uint64_t bound, uint64_t count, float* out) {
  xoshiro x; xo_init(&x, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = (float)xo_below(&x, bound);
}

/* ---- seeded normal inputs (the build's input convention) ---
 * A second, independent statement of csrc/datagen.cpp, so the reference arm
 * of bench.py can make its inputs without the product library: block q of
 * 65536 elements draws Box-Muller pairs from xoshiro256++(derive_seed(seed,
 * q)); z = sqrt(-2 ln(1-u1)) (cos, sin)(2 pi u2) in double, rounded once to
 * fp32.  tests/test_oracle.py pins the two byte for byte. */
void orc_fill_normal_range(uint64_t seed, uint64_t start, uint64_t count, float mean, float stddev,
                           float* out) {
  const uint64_t blk = 65536, q0 = start / blk;
  const double two_pi = 6.283185307179586476925286766559;
  for (uint64_t qq = 0; qq * blk < count; ++qq) {
    xoshiro x; xo_init(&x, orc_derive_seed(seed, q0 + qq));
    const uint64_t i0 = qq * blk, i1 = count < i0 + blk ? count : i0 + blk;
    for (uint64_t i = i0; i < i1; i += 2) {
      const double u1 = xo_double(&x), u2 = xo_double(&x);
      const double r = sqrt(-2.0 * log(1.0 - u1)), a = two_pi * u2;
      out[i] = (float)((double)mean + (double)stddev * (r * cos(a)));
      if (i + 1 < i1) out[i + 1] = (float)((double)mean + (double)stddev * (r * sin(a)));
    }
  }
}
/* round-to-nearest-even fp32 -> bf16 -> fp32 (the bf16 configs' exact values) */
void orc_round_bf16(const float* in, uint64_t count, float* out, uint16_t* bits) {
  for (uint64_t i = 0; i < count; ++i) {
    uint32_t u;
    memcpy(&u, &in[i], 4);
    uint16_t h;
    if ((u & 0x7fffffffu) > 0x7f800000u) h = (uint16_t)((u >> 16) | 0x40u);
    else h = (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
    if (bits) bits[i] = h;
    const uint32_t v = (uint32_t)h << 16;
    memcpy(&out[i], &v, 4);
  }
}

/* ---- params validation: src/topk.cpp:54-67 ------------------------------ */
int orc_validate(uint64_t n, uint64_t b, uint32_t kp, uint32_t k, uint32_t lane) {
  if (n == 0) return fail("n must be >= 1");
  if (n > 0xffffffffull) return fail("n exceeds the 32-bit index range");
  if (b == 0) return fail("num_buckets must be >= 1");
  if (n % b != 0) return fail("num_buckets must divide n");
  if (lane == 0) return fail("lane_multiple must be >= 1");
  if (b % lane != 0) return fail("num_buckets must be a multiple of lane_multiple");
  if (kp == 0) return fail("local_k must be >= 1");
  if (k == 0) return fail("global_k must be >= 1");
  if (k > n) return fail("global_k must not exceed n");
  if (b * (uint64_t)kp < k) return fail("num_buckets * local_k must be >= global_k");
  return ORC_OK;
}

/* ---- Alg. 1: src/topk.cpp:80-102 -------------------- */
void orc_update_bucket(float* v, uint32_t* ix, uint32_t kp, float value, uint32_t index) {
  const int take = value >= v[kp - 1];
  if (take) { v[kp - 1] = value; ix[kp - 1] = index; }
  for (uint32_t k = kp - 1; k >= 1; --k) {
    const int up = value > v[k - 1];
    if (up) {
      float tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
      uint32_t ti = ix[k]; ix[k] = ix[k - 1]; ix[k - 1] = ti;
    }
  }
}

static int has_nan(const float* x, uint64_t n) { /* src/topk.cpp:22-28 */
  int bad = 0;
  for (uint64_t i = 0; i < n; ++i) bad |= (x[i] != x[i]);
  return bad;
}

/* Stage1Accumulator: src/topk.cpp:114-172.  The reference vectorises over
 * bucket-aligned runs; per element it is exactly Alg. 1 on bucket g % B in
 * index order, which is what this streaming restatement does.  grid layout is
 * bucket-minor [kp][B] (topk.hpp:59-67). */
void orc_stage1_init(uint64_t b, uint32_t kp, float* vals, uint32_t* idx) {
  for (uint64_t s = 0; s < b * kp; ++s) { vals[s] = -INFINITY; idx[s] = 0; }
}
int orc_stage1_consume(uint64_t n, uint64_t b, uint32_t kp, float* vals, uint32_t* idx,
                       uint64_t consumed, const float* block, uint64_t len) {
  if (consumed + len > n) return fail("stage 1 fed more than n elements");
  if (has_nan(block, len)) return fail("input contains NaN");
  float* lv = (float*)malloc(sizeof(float) * kp);
  uint32_t* li = (uint32_t*)malloc(sizeof(uint32_t) * kp);
  for (uint64_t j = 0; j < len; ++j) {
    const uint64_t g = consumed + j;
    const uint64_t bk = g % b;
    for (uint32_t k = 0; k < kp; ++k) { lv[k] = vals[k * b + bk]; li[k] = idx[k * b + bk]; }
    orc_update_bucket(lv, li, kp, block[j], (uint32_t)g);
    for (uint32_t k = 0; k < kp; ++k) { vals[k * b + bk] = lv[k]; idx[k * b + bk] = li[k]; }
  }
  free(lv); free(li);
  return ORC_OK;
}
/* stage1_partial_reduce: src/topk.cpp:178-186 */
int orc_stage1(const float* in, uint64_t n, uint64_t b, uint32_t kp, uint32_t lane,
               float* vals, uint32_t* idx) {
  int rc = orc_validate(n, b, kp, 1, lane);
  if (rc) return rc;
  orc_stage1_init(b, kp, vals, idx);
  return orc_stage1_consume(n, b, kp, vals, idx, 0, in, n);
}

/* ---- rank keys: src/topk.cpp:30-50 -------------------------------------- */
static uint64_t rank_key(float value, uint32_t index) {
  uint32_t bits; memcpy(&bits, &value, 4);
  if (bits == 0x80000000u) bits = 0;
  const uint32_t asc = (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
  return ((uint64_t)(~asc) << 32) | index;
}
static float key_value(uint64_t key) {
  const uint32_t asc = (uint32_t)~(key >> 32);
  const uint32_t bits = (asc & 0x80000000u) ? (asc & 0x7fffffffu) : ~asc;
  float f; memcpy(&f, &bits, 4);
  return f;
}
static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}
static void top_k_from_keys(uint64_t* keys, uint64_t count, uint32_t k,
                            float* ov, uint32_t* oi) { /* topk.cpp:192-202 */
  qsort(keys, count, sizeof(uint64_t), cmp_u64);
  for (uint32_t i = 0; i < k; ++i) { ov[i] = key_value(keys[i]); oi[i] = (uint32_t)keys[i]; }
}

/* select_top_k_candidates: src/topk.cpp:219-236 */
int orc_select_candidates(const float* v, const uint32_t* ix, uint64_t count, uint32_t k,
                          uint64_t index_limit, float* ov, uint32_t* oi) {
  if (k == 0) return fail("k must be >= 1");
  if (has_nan(v, count)) return fail("input contains NaN");
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (count ? count : 1));
  uint64_t m = 0;
  for (uint64_t i = 0; i < count; ++i)
    if (ix[i] < index_limit) keys[m++] = rank_key(v[i], ix[i]);
  if (m < k) { free(keys); return fail("fewer candidates than k"); }
  top_k_from_keys(keys, m, k, ov, oi);
  free(keys);
  return ORC_OK;
}

/* exact_top_k: src/topk.cpp:206-217 */
int orc_exact_top_k(const float* in, uint64_t n, uint32_t k, float* ov, uint32_t* oi) {
  if (k == 0) return fail("k must be >= 1");
  if (n > 0xffffffffull + 1) return fail("input exceeds the 32-bit index range");
  if (k > n) return fail("k must not exceed the input length");
  if (has_nan(in, n)) return fail("input contains NaN");
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < n; ++i) keys[i] = rank_key(in[i], (uint32_t)i);
  top_k_from_keys(keys, n, k, ov, oi);
  free(keys);
  return ORC_OK;
}

/* approx_top_k: src/topk.cpp:238-258 */
int orc_approx_top_k(const float* in, uint64_t n, uint64_t b, uint32_t kp, uint32_t k,
                     uint32_t lane, float* ov, uint32_t* oi) {
  int rc = orc_validate(n, b, kp, k, lane);
  if (rc) return rc;
  float* gv = (float*)malloc(sizeof(float) * b * kp);
  uint32_t* gi = (uint32_t*)malloc(sizeof(uint32_t) * b * kp);
  orc_stage1_init(b, kp, gv, gi);
  rc = orc_stage1_consume(n, b, kp, gv, gi, 0, in, n);
  if (!rc) {
    const uint64_t s = n / b;
    const uint64_t filled = kp < s ? kp : s;
    rc = orc_select_candidates(gv, gi, filled * b, k, UINT64_MAX, ov, oi);
  }
  free(gv); free(gi);
  return rc;
}

/* approx_top_k_batch: src/topk.cpp:260-273 (single-threaded here; the
 * reference's result is thread-count invariant, threads.hpp:13-17) */
int orc_approx_top_k_batch(const float* rows, uint64_t row_count, uint64_t n, uint64_t b,
                           uint32_t kp, uint32_t k, uint32_t lane, float* ov, uint32_t* oi) {
  int rc = orc_validate(n, b, kp, k, lane);
  if (rc) return rc;
  for (uint64_t r = 0; r < row_count; ++r) {
    rc = orc_approx_top_k(rows + r * n, n, b, kp, k, lane, ov + r * k, oi + r * k);
    if (rc) return rc;
  }
  return ORC_OK;
}

/* measure_recall: src/topk.cpp:275-297 */
static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}
int orc_measure_recall(const uint32_t* approx, const uint32_t* exact, uint64_t k, double* out) {
  if (k == 0) return fail("recall of empty results is undefined");
  uint32_t* a = (uint32_t*)malloc(4 * k);
  uint32_t* e = (uint32_t*)malloc(4 * k);
  memcpy(a, approx, 4 * k); memcpy(e, exact, 4 * k);
  qsort(a, k, 4, cmp_u32); qsort(e, k, 4, cmp_u32);
  uint64_t hits = 0, i = 0, j = 0;
  while (i < k && j < k) {
    if (a[i] < e[j]) ++i; else if (e[j] < a[i]) ++j; else { ++hits; ++i; ++j; }
  }
  free(a); free(e);
  *out = (double)hits / (double)k;
  return ORC_OK;
}

/* ---- recall analysis: src/hypergeom.cpp, src/recall.cpp ----------------- */
static double log_choose(uint64_t n, uint64_t k) { /* hypergeom.cpp:10-15 */
  if (k > n) return -INFINITY;
  return lgamma((double)n + 1.0) - lgamma((double)k + 1.0) - lgamma((double)(n - k) + 1.0);
}
typedef struct { uint64_t pop, succ, draws; } hyper;
static uint64_t hg_min(hyper h) { uint64_t miss = h.pop - h.succ; return h.draws > miss ? h.draws - miss : 0; }
static uint64_t hg_max(hyper h) { return h.succ < h.draws ? h.succ : h.draws; }
static double hg_mean(hyper h) { return (double)h.draws * (double)h.succ / (double)h.pop; }
static double hg_std(hyper h) { /* hypergeom.cpp:40-47 */
  if (h.pop <= 1) return 0.0;
  const double n = (double)h.pop, p = (double)h.succ / n, s = (double)h.draws;
  const double var = s * p * (1.0 - p) * (n - s) / (n - 1.0);
  return var > 0.0 ? sqrt(var) : 0.0;
}
static double hg_logpmf(hyper h, uint64_t r) { /* hypergeom.cpp:49-55 */
  if (r < hg_min(h) || r > hg_max(h)) return -INFINITY;
  return log_choose(h.succ, r) + log_choose(h.pop - h.succ, h.draws - r) - log_choose(h.pop, h.draws);
}

/* bucket_excess_mean: recall.cpp:33-56 (Kahan summation) */
static double bucket_excess_mean(uint64_t n, uint64_t k, uint64_t s, uint32_t kp) {
  hyper h = {n, k, s};
  const uint64_t rmax = hg_max(h);
  if (kp >= rmax) return 0.0;
  uint64_t rmin = hg_min(h);
  if ((uint64_t)kp + 1 > rmin) rmin = (uint64_t)kp + 1;
  const double lden = log_choose(n, s);
  const double mode = ((double)s + 1.0) * ((double)k + 1.0) / ((double)n + 2.0);
  double sum = 0.0, c = 0.0;
  for (uint64_t r = rmin; r <= rmax; ++r) {
    const double lterm = log_choose(k, r) + log_choose(n - k, s - r) - lden;
    const double term = (double)(r - kp) * exp(lterm);
    const double y = term - c;
    const double t = sum + y;
    c = (t - sum) - y;
    sum = t;
    if ((double)r > mode + 2.0 && term <= sum * 1e-18) break;
  }
  return sum;
}
static int validate_analysis(uint64_t n, uint64_t b, uint32_t kp, uint32_t k) { /* topk.cpp:69-76 */
  if (n == 0) return fail("n must be >= 1");
  if (b == 0) return fail("num_buckets must be >= 1");
  if (b > n) return fail("num_buckets must not exceed n");
  if (kp == 0) return fail("local_k must be >= 1");
  if (k == 0) return fail("global_k must be >= 1");
  if (k > n) return fail("global_k must not exceed n");
  return ORC_OK;
}
static double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }
/* exact_expected_recall: recall.cpp:76-100 (Theorem 1) */
int orc_exact_expected_recall(uint64_t n, uint64_t b, uint32_t kp, uint32_t k, double* out) {
  int rc = validate_analysis(n, b, kp, k);
  if (rc) return rc;
  const uint64_t s_lo = n / b, hi = n % b, lo = b - hi;
  double excess = 0.0;
  if (lo > 0) excess += (double)lo * bucket_excess_mean(n, k, s_lo, kp);
  if (hi > 0) excess += (double)hi * bucket_excess_mean(n, k, s_lo + 1, kp);
  *out = clamp01(1.0 - excess / (double)k);
  return ORC_OK;
}

/* HypergeometricSampler: hypergeom.cpp:61-103 */
typedef struct { uint64_t lo; uint64_t len; double* cdf; } sampler;
static void sampler_init(sampler* sp, hyper h) {
  const uint64_t smin = hg_min(h), smax = hg_max(h);
  const double mu = hg_mean(h), sigma = hg_std(h), span = 60.0 * sigma + 2.0;
  uint64_t lo = smin, hi = smax;
  if (mu - span > (double)smin) lo = (uint64_t)(mu - span);
  if (mu + span < (double)smax) hi = (uint64_t)(mu + span) + 1;
  if (hi < lo) hi = lo;
  sp->lo = lo; sp->len = hi - lo + 1;
  sp->cdf = (double*)malloc(sizeof(double) * sp->len);
  const double n = (double)h.pop, k = (double)h.succ, s = (double)h.draws;
  double p = exp(hg_logpmf(h, lo)), cum = 0.0;
  for (uint64_t r = lo; r <= hi; ++r) {
    cum += p;
    sp->cdf[r - lo] = cum;
    const double rr = (double)r;
    const double num = (k - rr) * (s - rr);
    const double den = (rr + 1.0) * (n - k - s + rr + 1.0);
    p = den > 0.0 ? p * (num / den) : 0.0;
  }
}
static uint64_t sampler_draw(const sampler* sp, xoshiro* x) {
  const double u = xo_double(x);
  /* upper_bound: first cdf > u */
  uint64_t lo = 0, hi = sp->len;
  while (lo < hi) { uint64_t mid = (lo + hi) / 2; if (sp->cdf[mid] > u) hi = mid; else lo = mid + 1; }
  if (lo == sp->len) return sp->lo + sp->len - 1;
  return sp->lo + lo;
}
/* mc_expected_recall: recall.cpp:102-154 */
int orc_mc_expected_recall(uint64_t n, uint64_t b, uint32_t kp, uint32_t k, uint64_t trials,
                           uint64_t seed, double* mean_out, double* se_out) {
  int rc = validate_analysis(n, b, kp, k);
  if (rc) return rc;
  if (trials < 2) return fail("mc_expected_recall needs trials >= 2");
  const uint64_t s_lo = n / b, chi = n % b, clo = b - chi;
  const double kd = (double)k;
  hyper hl = {n, k, s_lo}, hh = {n, k, chi > 0 ? s_lo + 1 : s_lo};
  sampler sl, sh;
  sampler_init(&sl, hl);
  sampler_init(&sh, hh);
  xoshiro x; xo_init(&x, seed);
  double mean = 0.0, m2 = 0.0;
  for (uint64_t t = 0; t < trials; ++t) {
    double excess = 0.0;
    if (clo > 0) { uint64_t v = sampler_draw(&sl, &x); if (v > kp) excess += (double)clo * (double)(v - kp); }
    if (chi > 0) { uint64_t v = sampler_draw(&sh, &x); if (v > kp) excess += (double)chi * (double)(v - kp); }
    const double rec = 1.0 - excess / kd;
    const double d = rec - mean;
    mean += d / (double)(t + 1);
    m2 += d * (rec - mean);
  }
  free(sl.cdf); free(sh.cdf);
  const double var = m2 / (double)(trials - 1);
  *mean_out = mean;
  *se_out = sqrt((var > 0.0 ? var : 0.0) / (double)trials);
  return ORC_OK;
}
/* mc_expected_recall_adaptive: recall.cpp:156-165 */
int orc_mc_adaptive(uint64_t n, uint64_t b, uint32_t kp, uint32_t k, uint64_t seed,
                    double* mean, double* se, uint64_t* trials_out) {
  uint64_t trials = 4096;
  for (uint64_t attempt = 0;; ++attempt) {
    int rc = orc_mc_expected_recall(n, b, kp, k, trials, orc_derive_seed(seed, attempt), mean, se);
    if (rc) return rc;
    if (3.0 * *se <= 0.005) { *trials_out = trials; return ORC_OK; }
    trials *= 2;
  }
}

/* legal_bucket_counts: planner.cpp:59-77 (returns count; out may be NULL) */
static int cmp_u64_desc(const void* a, const void* b) { return -cmp_u64(a, b); }
uint64_t orc_legal_bucket_counts(uint64_t n, uint64_t lane, uint64_t* out, uint64_t cap) {
  if (n == 0 || lane == 0 || n % lane != 0) return 0;
  const uint64_t m = n / lane;
  uint64_t cnt = 0;
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * 4096);
  for (uint64_t d = 1; d * d <= m; ++d) {
    if (m % d) continue;
    tmp[cnt++] = d * lane;
    if (d != m / d) tmp[cnt++] = (m / d) * lane;
  }
  qsort(tmp, cnt, sizeof(uint64_t), cmp_u64_desc);
  if (out) for (uint64_t i = 0; i < cnt && i < cap; ++i) out[i] = tmp[i];
  free(tmp);
  return cnt;
}

/* select_parameters: planner.cpp:79-147 */
int orc_select_parameters(uint64_t n, uint64_t k, double target, const uint32_t* kps_in,
                          uint32_t nkps, uint32_t lane, uint64_t seed, uint32_t* kp_out,
                          uint64_t* b_out, double* recall_out, int* exact_out, int* warn_out) {
  if (n == 0) return fail("plan: n must be >= 1");
  if (k == 0 || k > n) return fail("plan: k must satisfy 1 <= k <= n");
  if (k > 0xffffffffull) return fail("plan: k exceeds the 32-bit result size");
  if (!(target > 0.0) || !(target < 1.0)) return fail("plan: recall_target must be in (0, 1)");
  if (nkps == 0) return fail("plan: allowed_local_k must not be empty");
  for (uint32_t i = 0; i < nkps; ++i) if (kps_in[i] == 0) return fail("plan: allowed_local_k entries must be >= 1");
  if (lane == 0) return fail("plan: lane_multiple must be >= 1");

  uint64_t nb = orc_legal_bucket_counts(n, lane, NULL, 0);
  uint64_t* buckets = (uint64_t*)malloc(sizeof(uint64_t) * (nb ? nb : 1));
  orc_legal_bucket_counts(n, lane, buckets, nb);
  /* sorted unique local_k */
  uint32_t kps[64]; uint32_t nk = 0;
  for (uint32_t i = 0; i < nkps && nk < 64; ++i) {
    uint32_t v = kps_in[i], dup = 0;
    for (uint32_t j = 0; j < nk; ++j) dup |= (kps[j] == v);
    if (!dup) kps[nk++] = v;
  }
  for (uint32_t i = 1; i < nk; ++i) for (uint32_t j = i; j > 0 && kps[j - 1] > kps[j]; --j) {
    uint32_t t = kps[j]; kps[j] = kps[j - 1]; kps[j - 1] = t; }

  typedef struct { uint32_t kp; uint64_t b; double est; } cand;
  cand* pass = (cand*)malloc(sizeof(cand) * (nb * nk + 1));
  uint64_t np = 0;
  for (uint32_t a = 0; a < nk; ++a) {
    const uint32_t kp = kps[a];
    const uint64_t kseed = orc_derive_seed(seed, kp);
    for (uint64_t i = 0; i < nb; ++i) {
      const uint64_t b = buckets[i];
      if (b * kp < k) break;
      double mean, se; uint64_t tr;
      orc_mc_adaptive(n, b, kp, (uint32_t)k, orc_derive_seed(kseed, b), &mean, &se, &tr);
      if (!(mean >= target)) break;
      pass[np].kp = kp; pass[np].b = b; pass[np].est = mean; ++np;
    }
  }
  free(buckets);
  if (np == 0) { free(pass); g_err = "no legal (local_k, num_buckets) configuration meets the recall target"; return ORC_EINFEASIBLE; }
  /* stable sort by (elements, kp): insertion sort is stable */
  for (uint64_t i = 1; i < np; ++i) {
    for (uint64_t j = i; j > 0; --j) {
      const uint64_t ea = pass[j - 1].b * pass[j - 1].kp, eb = pass[j].b * pass[j].kp;
      const int less = (eb < ea) || (eb == ea && pass[j].kp < pass[j - 1].kp);
      if (!less) break;
      cand t = pass[j]; pass[j] = pass[j - 1]; pass[j - 1] = t;
    }
  }
  for (uint64_t i = 0; i < np; ++i) {
    double est = pass[i].est; int exact = 0;
    const uint64_t nb_ = n / pass[i].b;
    if ((k < nb_ ? k : nb_) <= 10000) {
      orc_exact_expected_recall(n, pass[i].b, pass[i].kp, (uint32_t)k, &est);
      exact = 1;
      if (est < target) continue;
    }
    *kp_out = pass[i].kp; *b_out = pass[i].b; *recall_out = est; *exact_out = exact;
    *warn_out = target >= 0.995;
    free(pass);
    return ORC_OK;
  }
  free(pass);
  g_err = "every MC-passing configuration failed exact re-validation";
  return ORC_EINFEASIBLE;
}

/* ---- MIPS scorer: src/mips.cpp:57-95 (compiled with -ffp-contract=off) -- */
void orc_score_block(const float* queries, uint64_t b, const float* database, uint64_t d,
                     uint64_t c0, uint64_t c1, float* out, uint64_t out_stride) {
  enum { LANES = 8, TILE = 512 };
  const uint64_t groups = (b + LANES - 1) / LANES;
  float* tile = (float*)malloc(sizeof(float) * d * LANES);
  for (uint64_t ct = c0; ct < c1; ct += TILE) {
    const uint64_t ce = c1 < ct + TILE ? c1 : ct + TILE;
    for (uint64_t g = 0; g < groups; ++g) {
      const uint64_t q0 = g * LANES;
      const uint64_t live = (b - q0) < LANES ? (b - q0) : LANES;
      for (uint64_t j = 0; j < d; ++j)
        for (uint64_t l = 0; l < LANES; ++l)
          tile[j * LANES + l] = l < live ? queries[(q0 + l) * d + j] : 0.0f;
      for (uint64_t c = ct; c < ce; ++c) {
        const float* w = database + c * d;
        float acc[LANES] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint64_t j = 0; j < d; ++j) {
          const float wj = w[j];
          const float* qj = &tile[j * LANES];
          for (uint64_t l = 0; l < LANES; ++l) acc[l] += qj[l] * wj;
        }
        for (uint64_t l = 0; l < live; ++l) out[(q0 + l) * out_stride + (c - c0)] = acc[l];
      }
    }
  }
  free(tile);
}
