/* TEST INFRASTRUCTURE ONLY — the parity oracle, never the product.
 *
 * Plain-C restatement of the reference BSC truncated-EM step. Each function
 * cites the reference lines it follows (paths relative to
 * /root/reference/proj/src). Summation orders follow the reference compiled
 * against oracle/eigen_shim; tests/test_oracle.py checks this file bit for
 * bit against oracle/_ref/libprsp_ref.so (the reference sources themselves)
 * and against the SPEC.md known answers.
 */
#define _GNU_SOURCE
#include "bsc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, E_CONFIG = 2, E_DATA = 3, E_NUMERIC = 4, E_INTERNAL = 5 };

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* bsc_last_error(void) { return g_err; }

#define K_LOG_2PI 1.8378770664093454836 /* linear_discrete.cpp:24 */
#define K_MIN_SIGMA2 1e-12              /* model.hpp:32 */
#define K_MIN_PI 1e-6                   /* model.hpp:33 */

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* ------------------------------------------------------------------ RNG */
/* std::mt19937_64 (the engine pinned by core.hpp:129-150). */
typedef struct {
  uint64_t mt[312];
  int idx;
} rng_t;

static void rng_seed(rng_t* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = 312;
}

static uint64_t rng_next(rng_t* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) |
                   (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* splitmix64 mix, core.cpp:50-57; RngStream::derived core.cpp:59-61. */
static uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

static void rng_derived(rng_t* r, uint64_t base, uint64_t index) {
  rng_seed(r, mix64(mix64(base) ^ mix64(index + 1)));
}

/* core.cpp:63-66 */
static double rng_uniform01(rng_t* r) {
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}

/* core.cpp:68-76 (Box-Muller on the stream's own uniforms). */
static double rng_normal(rng_t* r) {
  double u1 = rng_uniform01(r);
  while (u1 <= 0.0) u1 = rng_uniform01(r);
  const double u2 = rng_uniform01(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* core.cpp:78 */
static int rng_bernoulli(rng_t* r, double p) { return rng_uniform01(r) < p; }

int bsc_rng_normals(uint64_t base_seed, uint64_t index, int derived, uint64_t n,
                    double* out) {
  rng_t r;
  if (derived)
    rng_derived(&r, base_seed, index);
  else
    rng_seed(&r, base_seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_normal(&r);
  return OK;
}

int bsc_rng_uniforms(uint64_t seed, uint64_t n, double* out) {
  rng_t r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_uniform01(&r);
  return OK;
}

/* ------------------------------------------------------------- fixtures */
/* bars.cpp:20-31 (dictionary) and :33-65 (draw order: 2R Bernoullis, then
 * one normal per pixel). */
int bsc_make_bars(uint32_t size, uint64_t n, double prob, double amplitude,
                  double noise, int max_mode, uint64_t seed, double* y_out,
                  double* truth_out) {
  if (size == 0) return fail(E_CONFIG, "bars: size must be >= 1");
  if (n == 0) return fail(E_CONFIG, "bars: need at least one data point");
  if (amplitude <= 0.0) return fail(E_CONFIG, "bars: amplitude must be > 0");
  if (noise < 0.0) return fail(E_CONFIG, "bars: noise must be >= 0");
  const uint32_t nb = 2 * size;
  const double p = prob > 0.0 ? prob : 2.0 / (double)nb;
  if (p >= 1.0) return fail(E_CONFIG, "bars: prob must lie in (0,1)");
  const size_t d = (size_t)size * size;
  double* w = calloc(d * nb, sizeof(double));
  uint32_t* act = malloc(nb * sizeof(uint32_t));
  for (uint32_t k = 0; k < size; ++k)
    for (uint32_t j = 0; j < size; ++j) {
      w[((size_t)k * size + j) * nb + k] = amplitude;
      w[((size_t)j * size + k) * nb + size + k] = amplitude;
    }
  rng_t r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t na = 0;
    for (uint32_t b = 0; b < nb; ++b)
      if (rng_bernoulli(&r, p)) act[na++] = b;
    for (size_t px = 0; px < d; ++px) {
      double v = 0.0;
      for (uint32_t a = 0; a < na; ++a) {
        const double wv = w[px * nb + act[a]];
        v = max_mode ? dmax(v, wv) : v + wv;
      }
      y_out[i * d + px] = v + noise * rng_normal(&r);
    }
  }
  if (truth_out) memcpy(truth_out, w, d * nb * sizeof(double));
  free(w);
  free(act);
  return OK;
}

static int validate_params(uint32_t d, uint32_t h, const double* w, double pi,
                           double sigma2) {
  for (size_t i = 0; i < (size_t)d * h; ++i)
    if (!isfinite(w[i])) return fail(E_NUMERIC, "bsc: non-finite dictionary");
  if (!(sigma2 > 0.0) || !isfinite(sigma2))
    return fail(E_CONFIG, "bsc: sigma2 must be positive");
  if (!(pi > 0.0 && pi < 1.0)) return fail(E_CONFIG, "bsc: pi must lie in (0,1)");
  return OK;
}

/* LinearDiscreteModel::generate, linear_discrete.cpp:452-479 (BSC): H
 * Bernoullis, mean = W s (left-to-right; s_j = 0 terms add an exact zero and
 * are skipped, s_j = 1 terms add W exactly), then D normals. */
int bsc_generate(uint32_t d, uint32_t h, const double* w, double pi,
                 double sigma2, uint64_t n, uint64_t seed, double* y_out) {
  int rc = validate_params(d, h, w, pi, sigma2);
  if (rc) return rc;
  const double noise_std = sqrt(sigma2);
  uint32_t* act = malloc(h * sizeof(uint32_t));
  rng_t r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t na = 0;
    for (uint32_t j = 0; j < h; ++j)
      if (rng_bernoulli(&r, pi)) act[na++] = j;
    for (uint32_t di = 0; di < d; ++di) {
      double acc = 0.0;
      const double* row = w + (size_t)di * h;
      for (uint32_t a = 0; a < na; ++a) acc += row[act[a]];
      y_out[i * d + di] = acc + noise_std * rng_normal(&r);
    }
  }
  free(act);
  return OK;
}

/* Ground-truth dictionary for BASELINE configs c2-c4:
 * W_dh ~ N(0,1) from RngStream::derived(seed, 0x77747275 "wtru") in
 * row-major order, each column scaled to unit L2 norm, then times `scale`. */
int bsc_random_dictionary(uint32_t d, uint32_t h, uint64_t seed, double scale,
                          double* w_out) {
  rng_t r;
  rng_derived(&r, seed, 0x77747275ULL);
  for (size_t i = 0; i < (size_t)d * h; ++i) w_out[i] = rng_normal(&r);
  for (uint32_t j = 0; j < h; ++j) {
    double acc = 0.0;
    for (uint32_t i = 0; i < d; ++i) acc += w_out[(size_t)i * h + j] * w_out[(size_t)i * h + j];
    const double nrm = sqrt(acc);
    for (uint32_t i = 0; i < d; ++i)
      w_out[(size_t)i * h + j] = w_out[(size_t)i * h + j] / nrm * scale;
  }
  return OK;
}

/* model.cpp:187-199 (data_column_means, data_mean_variance). */
static void column_means(const double* y, uint64_t n, uint32_t d, double* means) {
  for (uint32_t j = 0; j < d; ++j) means[j] = 0.0;
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < d; ++j) means[j] += y[i * d + j];
  for (uint32_t j = 0; j < d; ++j) means[j] /= (double)n;
}

static double mean_variance(const double* y, uint64_t n, uint32_t d,
                            const double* means) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < d; ++j) {
      const double c = y[i * d + j] - means[j];
      acc += c * c;
    }
  return acc / (double)(n * d);
}

int bsc_data_mean_variance(const double* y, uint64_t n, uint32_t d, double* out) {
  double* m = malloc(d * sizeof(double));
  column_means(y, n, d, m);
  *out = mean_variance(y, n, d, m);
  free(m);
  return OK;
}

/* BASELINE.json init recipe as pinned in SURVEY.md §8(d):
 * W0[d,h] = mean_d + 0.25*std_d*z (z: RngStream::derived(seed, 0x696e6974),
 * row-major (d,h)); std_d the per-pixel population std; pi0 = 1/H;
 * sigma2_0 = data_mean_variance (model.cpp:187-199). */
int bsc_baseline_init(uint32_t d, uint32_t h, const double* y, uint64_t n,
                      uint64_t seed, double* w_out, double* pi_out,
                      double* sigma2_out) {
  if (n < 2) return fail(E_DATA, "init requires at least two data points");
  double* m = malloc(d * sizeof(double));
  double* sd = malloc(d * sizeof(double));
  column_means(y, n, d, m);
  for (uint32_t j = 0; j < d; ++j) sd[j] = 0.0;
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < d; ++j) {
      const double c = y[i * d + j] - m[j];
      sd[j] += c * c;
    }
  for (uint32_t j = 0; j < d; ++j) sd[j] = sqrt(sd[j] / (double)n);
  rng_t r;
  rng_derived(&r, seed, 0x696e6974ULL);
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j)
      w_out[(size_t)i * h + j] = m[i] + 0.25 * sd[i] * rng_normal(&r);
  *pi_out = 1.0 / (double)h;
  *sigma2_out = dmax(mean_variance(y, n, d, m), K_MIN_SIGMA2);
  free(m);
  free(sd);
  return OK;
}

/* LinearDiscreteModel::standard_init, linear_discrete.cpp:129-148 with
 * detail::init_weights, model.cpp:201-220 (RngStream(seed)). */
int bsc_standard_init(uint32_t d, uint32_t h, uint32_t hprime, const double* y,
                      uint64_t n, uint64_t seed, double* w_out, double* pi_out,
                      double* sigma2_out) {
  if (n < 2) return fail(E_DATA, "standard_init requires at least two data points");
  double* m = malloc(d * sizeof(double));
  column_means(y, n, d, m);
  const double var = mean_variance(y, n, d, m);
  const double sd = var > 0.0 ? sqrt(var / h) : 0.0;
  rng_t r;
  rng_seed(&r, seed);
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j) w_out[(size_t)i * h + j] = m[i] + sd * rng_normal(&r);
  *sigma2_out = dmax(var, K_MIN_SIGMA2);
  const double hp = (double)(hprime < h ? hprime : h);
  *pi_out = hp / (2.0 * (double)h);
  free(m);
  return OK;
}

/* ----------------------------------------------------------- truncation */
/* core.cpp:36-45 */
static int lse(const double* v, size_t n, double* out) {
  if (n == 0) return fail(E_NUMERIC, "log_sum_exp: empty support");
  double m = -INFINITY;
  for (size_t i = 0; i < n; ++i) m = dmax(m, v[i]);
  if (isinf(m) && m < 0) return fail(E_NUMERIC, "log_sum_exp: empty support");
  if (n == 1) {
    *out = v[0];
    return OK;
  }
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += exp(v[i] - m);
  *out = m + log(acc);
  return OK;
}

int bsc_log_sum_exp(const double* v, uint64_t n, double* out) {
  return lse(v, (size_t)n, out);
}

typedef struct {
  const double* s;
  uint32_t i;
} keyed_t;

/* Descending score, equal scores keep the lower index (stable_sort semantics
 * of truncation.cpp:48-53 with `>` as the strict order). */
static int cmp_desc(const void* a, const void* b) {
  const keyed_t* x = a;
  const keyed_t* y = b;
  const double sx = x->s[x->i], sy = y->s[y->i];
  if (sx > sy) return -1;
  if (sy > sx) return 1;
  return (x->i < y->i) ? -1 : (x->i > y->i);
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x < y) ? -1 : (x > y);
}

/* truncation.cpp:38-57, with a caller-provided scratch of h entries. */
static int select_cands(const double* scores, uint32_t h, uint32_t hprime,
                        uint32_t* out, keyed_t* scratch) {
  if (hprime == 0 || hprime > h)
    return fail(E_CONFIG, "select_candidates: hprime out of range");
  for (uint32_t i = 0; i < h; ++i)
    if (!isfinite(scores[i]))
      return fail(E_CONFIG, "select_candidates: scores must be finite");
  for (uint32_t i = 0; i < h; ++i) scratch[i] = (keyed_t){scores, i};
  qsort(scratch, h, sizeof(keyed_t), cmp_desc);
  for (uint32_t i = 0; i < hprime; ++i) out[i] = scratch[i].i;
  qsort(out, hprime, sizeof(uint32_t), cmp_u32);
  return OK;
}

int bsc_select_candidates(const double* scores, uint32_t h, uint32_t hprime,
                          uint32_t* out) {
  keyed_t* k = malloc((h ? h : 1) * sizeof(keyed_t));
  int rc = select_cands(scores, h, hprime, out, k);
  free(k);
  return rc;
}

/* truncation.cpp:23-30 */
static int validate_trunc(uint32_t h, uint32_t hprime, uint32_t gamma) {
  if (h == 0) return fail(E_CONFIG, "truncation: latents must be >= 1");
  if (hprime == 0 || hprime > h)
    return fail(E_CONFIG, "truncation: hprime must satisfy 1 <= hprime <= latents");
  if (gamma == 0 || gamma > hprime)
    return fail(E_CONFIG, "truncation: gamma must satisfy 1 <= gamma <= hprime");
  return OK;
}

/* ------------------------------------------------------- value tables */
/* LinearDiscreteModel::value_table, linear_discrete.cpp:71-97: the non-zero
 * alphabet with its log-probabilities and log P(s = 0). family 0 = bsc,
 * 1 = tsc, 2 = dsc (alphabet ascending with 0, probabilities aligned). */
#define LD_MAX_V 8
typedef struct {
  uint32_t family, nalpha;
  const double* alpha;
  const double* probs;
  double pi;
} prior_t;

typedef struct {
  uint32_t nv;
  double values[LD_MAX_V];
  double log_probs[LD_MAX_V];
  double log_p0;
} vtab_t;

static const char* family_name(uint32_t f) { return f == 0 ? "bsc" : f == 1 ? "tsc" : "dsc"; }

static int value_table(const prior_t* pr, vtab_t* t) {
  t->nv = 0;
  switch (pr->family) {
    case 0:
      t->nv = 1;
      t->values[0] = 1.0;
      t->log_probs[0] = log(pr->pi);
      t->log_p0 = log(1.0 - pr->pi);
      break;
    case 1:
      t->nv = 2;
      t->values[0] = -1.0;
      t->values[1] = 1.0;
      t->log_probs[0] = log(pr->pi / 2.0);
      t->log_probs[1] = log(pr->pi / 2.0);
      t->log_p0 = log(1.0 - pr->pi);
      break;
    case 2:
      for (uint32_t k = 0; k < pr->nalpha; ++k) {
        if (pr->alpha[k] == 0.0) {
          t->log_p0 = log(pr->probs[k]);
        } else {
          if (t->nv == LD_MAX_V) return fail(E_CONFIG, "oracle: more than %d non-zero values", LD_MAX_V);
          t->values[t->nv] = pr->alpha[k];
          t->log_probs[t->nv] = log(pr->probs[k]);
          t->nv++;
        }
      }
      break;
    default:
      return fail(E_CONFIG, "oracle: unknown family %u", pr->family);
  }
  return OK;
}

/* LinearDiscreteModel::validate, linear_discrete.cpp:99-127. */
static int validate_ld(uint32_t d, uint32_t h, const double* w, double sigma2, const prior_t* pr) {
  const char* nm = family_name(pr->family);
  for (size_t i = 0; i < (size_t)d * h; ++i)
    if (!isfinite(w[i])) return fail(E_NUMERIC, "%s: non-finite dictionary", nm);
  if (!(sigma2 > 0.0) || !isfinite(sigma2)) return fail(E_CONFIG, "%s: sigma2 must be positive", nm);
  if (pr->family == 2) {
    if (pr->nalpha < 2) return fail(E_CONFIG, "dsc: values/probs size mismatch");
    for (uint32_t k = 1; k < pr->nalpha; ++k)
      if (pr->alpha[k] < pr->alpha[k - 1]) return fail(E_CONFIG, "dsc: values must be ascending");
    int zero = 0;
    for (uint32_t k = 0; k < pr->nalpha; ++k) zero |= pr->alpha[k] == 0.0;
    if (!zero) return fail(E_CONFIG, "dsc: alphabet must contain 0");
    double total = 0.0;
    for (uint32_t k = 0; k < pr->nalpha; ++k) {
      if (!(pr->probs[k] > 0.0)) return fail(E_CONFIG, "dsc: probabilities must be positive");
      total += pr->probs[k];
    }
    if (fabs(total - 1.0) > 1e-6) return fail(E_CONFIG, "dsc: probabilities must sum to 1");
  } else if (!(pr->pi > 0.0 && pr->pi < 1.0)) {
    return fail(E_CONFIG, "%s: pi must lie in (0,1)", nm);
  }
  return OK;
}

/* truncation.cpp:61-93, saturating. */
static uint64_t sat_mul(uint64_t a, uint64_t b) {
  if (a != 0 && b > UINT64_MAX / a) return UINT64_MAX;
  return a * b;
}
static uint64_t sat_add(uint64_t a, uint64_t b) {
  return (UINT64_MAX - a < b) ? UINT64_MAX : a + b;
}
static uint64_t binom(uint64_t n, uint64_t k) {
  if (k > n) return 0;
  if (n - k < k) k = n - k;
  uint64_t r = 1;
  for (uint64_t i = 1; i <= k; ++i) {
    r = sat_mul(r, n - k + i);
    r /= i;
  }
  return r;
}
static uint64_t state_count_v(uint32_t h, uint32_t hprime, uint32_t gamma, uint32_t nv) {
  uint64_t total = sat_add(1, sat_mul(h, nv));
  uint64_t vpow = nv;
  for (uint32_t k = 2; k <= gamma; ++k) {
    vpow = sat_mul(vpow, nv);
    total = sat_add(total, sat_mul(binom(hprime, k), vpow));
  }
  return total;
}

int bsc_state_count(uint32_t h, uint32_t hprime, uint32_t gamma, uint64_t* out) {
  int rc = validate_trunc(h, hprime, gamma);
  if (rc) return rc;
  *out = state_count_v(h, hprime, gamma, 1);
  return OK;
}

int ld_state_count(uint32_t h, uint32_t hprime, uint32_t gamma, uint32_t nv, uint64_t* out) {
  int rc = validate_trunc(h, hprime, gamma);
  if (rc) return rc;
  *out = state_count_v(h, hprime, gamma, nv);
  return OK;
}

/* StateTemplate multi-active patterns, truncation.cpp:95-151: depth-first
 * over candidate positions (supports of size 2..gamma, lexicographic,
 * prefixes first); within a support the value odometer runs, last slot
 * fastest. Patterns are stored as (position, value index) lists. */
typedef struct {
  uint32_t hprime, gamma, nv;
  size_t count;
  uint8_t* len;  /* [count] */
  uint8_t* pos;  /* [count * gamma] */
  uint8_t* vix;  /* [count * gamma] */
} tmpl_t;

static void emit_values(tmpl_t* t, const uint8_t* support, uint32_t k) {
  uint8_t vi[256];
  memset(vi, 0, k);
  for (;;) {
    t->len[t->count] = (uint8_t)k;
    memcpy(t->pos + t->count * t->gamma, support, k);
    memcpy(t->vix + t->count * t->gamma, vi, k);
    t->count++;
    uint32_t i = k; /* advance the odometer, last slot fastest */
    for (;;) {
      if (i == 0) return;
      --i;
      if (++vi[i] < t->nv) break;
      vi[i] = 0;
      if (i == 0) return;
    }
  }
}

static void dfs(tmpl_t* t, uint8_t* support, uint32_t depth, uint32_t next) {
  if (depth >= 2) emit_values(t, support, depth);
  if (depth == t->gamma) return;
  for (uint32_t p = next; p < t->hprime; ++p) {
    support[depth] = (uint8_t)p;
    dfs(t, support, depth + 1, p + 1);
  }
}

static int tmpl_build(tmpl_t* t, uint32_t h, uint32_t hprime, uint32_t gamma, uint32_t nv,
                      uint64_t cap) {
  int rc = validate_trunc(h, hprime, gamma);
  if (rc) return rc;
  const uint64_t total = state_count_v(h, hprime, gamma, nv);
  if (total > cap)
    return fail(E_CONFIG, "state explosion: %llu states per data point exceeds cap of %llu",
                (unsigned long long)total, (unsigned long long)cap);
  if (hprime > 255) return fail(E_CONFIG, "oracle: hprime > 255 unsupported");
  t->hprime = hprime;
  t->gamma = gamma;
  t->nv = nv;
  t->count = 0;
  const size_t np = (size_t)(total - 1 - (uint64_t)h * nv);
  t->len = malloc(np ? np : 1);
  t->pos = malloc((np ? np : 1) * gamma);
  t->vix = malloc((np ? np : 1) * gamma);
  uint8_t support[256];
  if (gamma >= 2) dfs(t, support, 0, 0);
  return OK;
}

static void tmpl_free(tmpl_t* t) {
  free(t->len);
  free(t->pos);
  free(t->vix);
}

/* StateTemplate::instantiate, truncation.cpp:153-169, as (count, units,
 * values) lists: zero state, the (h, v) singletons over all H, then the
 * patterns mapped through the candidates. */
typedef struct {
  size_t n;
  uint8_t* len;   /* [n] */
  uint32_t* act;  /* [n * stride] ascending unit indices */
  uint8_t* vix;   /* [n * stride] value indices */
  uint32_t stride;
} states_t;

static void states_alloc(states_t* s, size_t total, uint32_t gamma) {
  s->stride = gamma;
  s->len = malloc(total);
  s->act = malloc(total * gamma * sizeof(uint32_t));
  s->vix = malloc(total * gamma);
}

static void states_free(states_t* s) {
  free(s->len);
  free(s->act);
  free(s->vix);
}

static void instantiate(const tmpl_t* t, uint32_t h, const uint32_t* cand, states_t* s) {
  size_t k = 0;
  s->len[k++] = 0;
  for (uint32_t u = 0; u < h; ++u)
    for (uint32_t v = 0; v < t->nv; ++v) {
      s->len[k] = 1;
      s->act[k * s->stride] = u;
      s->vix[k * s->stride] = (uint8_t)v;
      ++k;
    }
  for (size_t p = 0; p < t->count; ++p) {
    s->len[k] = t->len[p];
    for (uint32_t a = 0; a < t->len[p]; ++a) {
      s->act[k * s->stride + a] = cand[t->pos[p * t->gamma + a]];
      s->vix[k * s->stride + a] = t->vix[p * t->gamma + a];
    }
    ++k;
  }
  s->n = k;
}

int bsc_enumerate_binary(const uint32_t* cand, uint32_t hprime, uint32_t h,
                         uint32_t gamma, double* out, uint64_t* count) {
  for (uint32_t i = 1; i < hprime; ++i)
    if (cand[i] <= cand[i - 1])
      return fail(E_CONFIG, "enumerate states: candidate set must be ascending");
  for (uint32_t i = 0; i < hprime; ++i)
    if (cand[i] >= h)
      return fail(E_CONFIG, "enumerate states: candidate index out of range");
  tmpl_t t;
  int rc = tmpl_build(&t, h, hprime, gamma, 1, 1000000);
  if (rc) return rc;
  states_t s;
  states_alloc(&s, 1 + h + t.count, gamma);
  instantiate(&t, h, cand, &s);
  *count = s.n;
  if (out) {
    memset(out, 0, s.n * h * sizeof(double));
    for (size_t i = 0; i < s.n; ++i)
      for (uint32_t a = 0; a < s.len[i]; ++a) out[i * h + s.act[i * s.stride + a]] = 1.0;
  }
  states_free(&s);
  tmpl_free(&t);
  return OK;
}

/* ---------------------------------------------------------------- model */
static double gauss_log_norm(size_t dim, double sigma2) { /* :26-28 */
  return -0.5 * (double)dim * (K_LOG_2PI + log(sigma2));
}

/* log_prior :150-166 + log_joint :168-178. */
static int log_joint_v(uint32_t d, uint32_t h, const double* w, double sigma2, const vtab_t* vt,
                       const char* nm, const double* y, const double* s, double* out) {
  double prior = 0.0;
  for (uint32_t j = 0; j < h; ++j) {
    if (s[j] == 0.0) {
      prior += vt->log_p0;
      continue;
    }
    uint32_t k = 0;
    while (k < vt->nv && vt->values[k] != s[j]) ++k;
    if (k == vt->nv) return fail(E_CONFIG, "%s: latent value outside the alphabet", nm);
    prior += vt->log_probs[k];
  }
  double resid = 0.0;
  for (uint32_t i = 0; i < d; ++i) {
    double acc = 0.0;
    for (uint32_t j = 0; j < h; ++j) acc += w[(size_t)i * h + j] * s[j];
    const double r = y[i] - acc;
    resid += r * r;
  }
  *out = prior + gauss_log_norm(d, sigma2) - resid / (2.0 * sigma2);
  return OK;
}

int bsc_log_joint(uint32_t d, uint32_t h, const double* w, double pi,
                  double sigma2, const double* y, const double* s, double* out) {
  const prior_t pr = {0, 0, NULL, NULL, pi};
  vtab_t vt;
  value_table(&pr, &vt);
  return log_joint_v(d, h, w, sigma2, &vt, "bsc", y, s, out);
}

/* Per-shard accumulators in the field order of linear_discrete.cpp:211-217. */
typedef struct {
  double *sum_s, *sum_ssT, *sum_y_sT;
  double counts[LD_MAX_V];
  double sum_y2, log_partition;
  uint64_t points;
} stats_t;

typedef struct {
  uint32_t d, h, hprime, gamma;
  const double* w;
  double sigma2, temperature;
  vtab_t vt;
  const double* y;
  const double* gram; /* W^T W, left-to-right over d (linear_discrete.cpp:220) */
  const double* wt;   /* W^T, H x D */
  const tmpl_t* tmpl;
} ctx_t;

static void stats_alloc(stats_t* s, uint32_t d, uint32_t h) {
  s->sum_s = calloc(h, sizeof(double));
  s->sum_ssT = calloc((size_t)h * h, sizeof(double));
  s->sum_y_sT = calloc((size_t)d * h, sizeof(double));
  for (int k = 0; k < LD_MAX_V; ++k) s->counts[k] = 0.0;
  s->sum_y2 = s->log_partition = 0.0;
  s->points = 0;
}

static void stats_free(stats_t* s) {
  free(s->sum_s);
  free(s->sum_ssT);
  free(s->sum_y_sT);
}

static void gram_of(const double* w, uint32_t d, uint32_t h, double* wt, double* gram) {
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j) wt[(size_t)j * d + i] = w[(size_t)i * h + j];
  for (uint32_t i = 0; i < h; ++i)
    for (uint32_t j = 0; j < h; ++j) {
      double acc = 0.0;
      for (uint32_t t = 0; t < d; ++t) acc += wt[(size_t)i * d + t] * w[(size_t)t * h + j];
      gram[(size_t)i * h + j] = acc;
    }
}

/* Selection scores, linear_discrete.cpp:244-252: max over the non-zero
 * alphabet of log p_v + (2 v b − v² G_uu)·inv2s. */
static void scores_of(const vtab_t* vt, const double* b, const double* gram, uint32_t h, double inv2s,
                      double* scores) {
  for (uint32_t u = 0; u < h; ++u) {
    double best = -INFINITY;
    for (uint32_t k = 0; k < vt->nv; ++k) {
      const double v = vt->values[k];
      best = dmax(best, vt->log_probs[k] + (2.0 * v * b[u] - v * v * gram[(size_t)u * h + u]) * inv2s);
    }
    scores[u] = best;
  }
}

/* LinearDiscreteModel::estep_impl, linear_discrete.cpp:202-325. If
 * `map_states` is non-NULL the inference readout of :313-322 is written too. */
static int estep_rows(const ctx_t* c, uint64_t row_begin, uint64_t row_end,
                      stats_t* st, double* map_states, double* map_mass,
                      double* expected) {
  const uint32_t d = c->d, h = c->h;
  const vtab_t* vt = &c->vt;
  const double inv2s = 1.0 / (2.0 * c->sigma2);
  const double norm_const = gauss_log_norm(d, c->sigma2);
  double dlp[LD_MAX_V];
  for (uint32_t k = 0; k < vt->nv; ++k) dlp[k] = vt->log_probs[k] - vt->log_p0;
  const double zero_prior = (double)h * vt->log_p0;

  const size_t total = 1 + (size_t)h * vt->nv + c->tmpl->count;
  states_t s;
  states_alloc(&s, total, c->gamma);
  double* b = malloc(h * sizeof(double));
  double* scores = malloc(h * sizeof(double));
  double* es = malloc(h * sizeof(double));
  double* lj = malloc(total * sizeof(double));
  double* q = malloc(total * sizeof(double));
  uint32_t* cand = malloc(c->hprime * sizeof(uint32_t));
  keyed_t* scratch = malloc(h * sizeof(keyed_t));
  int rc = OK;

  for (uint64_t n = row_begin; n < row_end; ++n) {
    const double* y = c->y + n * d;
    for (uint32_t u = 0; u < h; ++u) { /* :241, b = W^T y */
      double acc = 0.0;
      for (uint32_t t = 0; t < d; ++t) acc += c->wt[(size_t)u * d + t] * y[t];
      b[u] = acc;
    }
    double y2 = 0.0; /* :242 */
    for (uint32_t t = 0; t < d; ++t) y2 += y[t] * y[t];
    scores_of(vt, b, c->gram, h, inv2s, scores); /* :244-252 */
    rc = select_cands(scores, h, c->hprime, cand, scratch); /* :253 */
    if (rc) break;
    instantiate(c->tmpl, h, cand, &s); /* :254 */

    const double base = zero_prior + norm_const - y2 * inv2s; /* :256 */
    for (size_t i = 0; i < s.n; ++i) {                      /* :257-270 */
      const uint32_t* act = s.act + i * s.stride;
      const uint8_t* vix = s.vix + i * s.stride;
      double prior = 0.0, lin = 0.0, quad = 0.0;
      for (uint32_t a = 0; a < s.len[i]; ++a) {
        const uint32_t ha = act[a];
        const double va = vt->values[vix[a]];
        prior += dlp[vix[a]];
        lin += va * b[ha];
        quad += va * va * c->gram[(size_t)ha * h + ha];
        for (uint32_t cc = a + 1; cc < s.len[i]; ++cc)
          quad += 2.0 * va * vt->values[vix[cc]] * c->gram[(size_t)ha * h + act[cc]];
      }
      lj[i] = base + prior + (2.0 * lin - quad) * inv2s;
    }

    double lse1;
    rc = lse(lj, s.n, &lse1); /* :272 */
    if (rc) break;
    if (c->temperature == 1.0) { /* :273-276 */
      for (size_t i = 0; i < s.n; ++i) q[i] = exp(lj[i] - lse1);
    } else { /* :277-286 */
      double m = lj[0];
      for (size_t i = 0; i < s.n; ++i) m = dmax(m, lj[i]);
      double acc = 0.0;
      for (size_t i = 0; i < s.n; ++i) {
        q[i] = exp((lj[i] - m) / c->temperature);
        acc += q[i];
      }
      for (size_t i = 0; i < s.n; ++i) q[i] /= acc;
    }

    for (uint32_t j = 0; j < h; ++j) es[j] = 0.0; /* :288-303 */
    for (size_t i = 0; i < s.n; ++i) {
      const double qi = q[i];
      const uint32_t* act = s.act + i * s.stride;
      const uint8_t* vix = s.vix + i * s.stride;
      for (uint32_t a = 0; a < s.len[i]; ++a) {
        const uint32_t ha = act[a];
        const double va = vt->values[vix[a]];
        es[ha] += qi * va;
        st->counts[vix[a]] += qi;
        st->sum_ssT[(size_t)ha * h + ha] += qi * va * va;
        for (uint32_t cc = a + 1; cc < s.len[i]; ++cc) {
          const double cross = qi * va * vt->values[vix[cc]];
          st->sum_ssT[(size_t)ha * h + act[cc]] += cross;
          st->sum_ssT[(size_t)act[cc] * h + ha] += cross;
        }
      }
    }
    for (uint32_t j = 0; j < h; ++j) st->sum_s[j] += es[j]; /* :304 */
    for (uint32_t i = 0; i < d; ++i) {                       /* :305-308 */
      const double yi = y[i];
      double* row = st->sum_y_sT + (size_t)i * h;
      for (uint32_t j = 0; j < h; ++j) row[j] += yi * es[j];
    }
    st->sum_y2 += y2; /* :309-311 */
    st->log_partition += lse1;
    st->points++;

    if (map_states) { /* :313-322 */
      size_t best = 0;
      for (size_t i = 1; i < s.n; ++i)
        if (q[i] > q[best]) best = i;
      map_mass[n] = q[best];
      for (uint32_t a = 0; a < s.len[best]; ++a)
        map_states[n * h + s.act[best * s.stride + a]] = vt->values[s.vix[best * s.stride + a]];
      for (uint32_t j = 0; j < h; ++j) expected[n * h + j] = es[j];
    }
  }
  states_free(&s);
  free(b);
  free(scores);
  free(es);
  free(lj);
  free(q);
  free(cand);
  free(scratch);
  return rc;
}

static int ctx_init(ctx_t* c, tmpl_t* t, uint32_t d, uint32_t h, uint32_t hprime,
                    uint32_t gamma, const double* w, const prior_t* pr, double sigma2,
                    double temperature, const double* y) {
  int rc = validate_ld(d, h, w, sigma2, pr);
  if (rc) return rc;
  vtab_t vt;
  rc = value_table(pr, &vt);
  if (rc) return rc;
  rc = tmpl_build(t, h, hprime, gamma, vt.nv, 1000000);
  if (rc) return rc;
  double* wt = malloc((size_t)d * h * sizeof(double));
  double* gram = malloc((size_t)h * h * sizeof(double));
  gram_of(w, d, h, wt, gram);
  *c = (ctx_t){d, h, hprime, gamma, w, sigma2, temperature, vt, y, gram, wt, t};
  return OK;
}

static void ctx_free(ctx_t* c, tmpl_t* t) {
  free((void*)c->gram);
  free((void*)c->wt);
  tmpl_free(t);
}

static void stats_out(const stats_t* st, uint32_t d, uint32_t h, uint32_t nv, double* sum_s,
                      double* sum_ssT, double* sum_y_sT, double* value_counts,
                      double* scalars) {
  if (sum_s) memcpy(sum_s, st->sum_s, h * sizeof(double));
  if (sum_ssT) memcpy(sum_ssT, st->sum_ssT, (size_t)h * h * sizeof(double));
  if (sum_y_sT) memcpy(sum_y_sT, st->sum_y_sT, (size_t)d * h * sizeof(double));
  if (value_counts) memcpy(value_counts, st->counts, nv * sizeof(double));
  if (scalars) {
    scalars[0] = st->sum_y2;
    scalars[1] = st->log_partition;
    scalars[2] = (double)st->points;
  }
}

/* estep_stats, linear_discrete.cpp:327-334 */
int ld_estep_stats(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
                   double pi, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                   const double* w, double sigma2, double temperature, const double* y,
                   uint64_t n, uint64_t row_begin, uint64_t row_end, double* sum_s,
                   double* sum_ssT, double* sum_y_sT, double* value_counts, double* scalars) {
  if (row_end < row_begin || row_end > n) return fail(E_CONFIG, "bad row range");
  const prior_t pr = {family, nalpha, alpha, probs, pi};
  ctx_t c;
  tmpl_t t;
  int rc = ctx_init(&c, &t, d, h, hprime, gamma, w, &pr, sigma2, temperature, y);
  if (rc) return rc;
  stats_t st;
  stats_alloc(&st, d, h);
  rc = estep_rows(&c, row_begin, row_end, &st, NULL, NULL, NULL);
  if (!rc) stats_out(&st, d, h, c.vt.nv, sum_s, sum_ssT, sum_y_sT, value_counts, scalars);
  stats_free(&st);
  ctx_free(&c, &t);
  return rc;
}

int bsc_estep_stats(uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                    const double* w, double pi, double sigma2,
                    double temperature, const double* y, uint64_t n,
                    uint64_t row_begin, uint64_t row_end, double* sum_s,
                    double* sum_ssT, double* sum_y_sT, double* value_counts,
                    double* scalars) {
  return ld_estep_stats(0, NULL, NULL, 0, pi, d, h, hprime, gamma, w, sigma2, temperature, y, n,
                        row_begin, row_end, sum_s, sum_ssT, sum_y_sT, value_counts, scalars);
}

/* Left-looking Cholesky + per-column substitution, the order fixed by
 * oracle/eigen_shim (Eigen::LLT usage at linear_discrete.cpp:354-357). */
static int cholesky(const double* a, size_t n, double* l) {
  memset(l, 0, n * n * sizeof(double));
  for (size_t j = 0; j < n; ++j) {
    double s = a[j * n + j];
    for (size_t k = 0; k < j; ++k) s -= l[j * n + k] * l[j * n + k];
    if (!(s > 0.0) || !isfinite(s)) return 1;
    const double dd = sqrt(s);
    l[j * n + j] = dd;
    for (size_t i = j + 1; i < n; ++i) {
      double t = a[i * n + j];
      for (size_t k = 0; k < j; ++k) t -= l[i * n + k] * l[j * n + k];
      l[i * n + j] = t / dd;
    }
  }
  return 0;
}

static void chol_solve(const double* l, size_t n, double* v) {
  for (size_t i = 0; i < n; ++i) {
    double s = v[i];
    for (size_t k = 0; k < i; ++k) s -= l[i * n + k] * v[k];
    v[i] = s / l[i * n + i];
  }
  for (size_t ii = n; ii-- > 0;) {
    double s = v[ii];
    for (size_t k = ii + 1; k < n; ++k) s -= l[k * n + ii] * v[k];
    v[ii] = s / l[ii * n + ii];
  }
}

#define K_MIN_CATEGORICAL 1e-9 /* model.hpp:34 */

/* LinearDiscreteModel::mstep, linear_discrete.cpp:336-408 (family branches
 * :371-405). `probs_out` (dsc) is aligned with the alphabet. */
int ld_mstep(uint32_t family, const double* alpha, uint32_t nalpha, uint32_t d, uint32_t h,
             const double* w_prev, const double* sum_s, const double* sum_ssT,
             const double* sum_y_sT, const double* value_counts, const double* scalars,
             double* w_out, double* pi_out, double* probs_out, double* sigma2_out) {
  (void)sum_s;
  const uint64_t points = (uint64_t)scalars[2];
  const double n = (double)points, dd = (double)d, nh = n * (double)h;
  if (points == 0) return fail(E_CONFIG, "%s: mstep without data", family_name(family));
  if (w_out != w_prev) memcpy(w_out, w_prev, (size_t)d * h * sizeof(double));

  double trace = 0.0; /* :349 */
  for (uint32_t i = 0; i < h; ++i) trace += sum_ssT[(size_t)i * h + i];
  if (trace > 0.0) {
    double* bm = malloc((size_t)h * h * sizeof(double));
    double* l = malloc((size_t)h * h * sizeof(double));
    memcpy(bm, sum_ssT, (size_t)h * h * sizeof(double));
    const double ridge = 1e-9 * trace / (double)h; /* :352-353 */
    for (uint32_t i = 0; i < h; ++i) bm[(size_t)i * h + i] += ridge;
    if (cholesky(bm, h, l) == 0) { /* :354-360 */
      double* col = malloc(h * sizeof(double));
      for (uint32_t c = 0; c < d; ++c) {
        for (uint32_t i = 0; i < h; ++i) col[i] = sum_y_sT[(size_t)c * h + i];
        chol_solve(l, h, col);
        for (uint32_t i = 0; i < h; ++i) w_out[(size_t)c * h + i] = col[i];
      }
      free(col);
    }
    free(bm);
    free(l);
  }

  const double t1 = scalars[0]; /* :366-369 */
  double t2 = 0.0;
  for (size_t i = 0; i < (size_t)d * h; ++i) t2 += w_out[i] * sum_y_sT[i];
  double t3 = 0.0;
  for (uint32_t i = 0; i < h; ++i)
    for (uint32_t j = 0; j < h; ++j) {
      double acc = 0.0;
      for (uint32_t t = 0; t < d; ++t) acc += w_out[(size_t)t * h + i] * w_out[(size_t)t * h + j];
      t3 += acc * sum_ssT[(size_t)i * h + j];
    }
  *sigma2_out = dmax((t1 - 2.0 * t2 + t3) / (n * dd), K_MIN_SIGMA2);

  switch (family) {
    case 0: /* :373-376 */
      if (pi_out) *pi_out = dmin(dmax(value_counts[0] / nh, K_MIN_PI), 1.0 - K_MIN_PI);
      break;
    case 1: /* :377-381 */
      if (pi_out) *pi_out = dmin(dmax((value_counts[0] + value_counts[1]) / nh, K_MIN_PI), 1.0 - K_MIN_PI);
      break;
    default: { /* :382-404 */
      double nonzero_mass = 0.0;
      uint32_t k = 0;
      for (uint32_t i = 0; i < nalpha; ++i) {
        if (alpha[i] == 0.0) continue;
        probs_out[i] = value_counts[k] / nh;
        nonzero_mass += probs_out[i];
        ++k;
      }
      for (uint32_t i = 0; i < nalpha; ++i)
        if (alpha[i] == 0.0) probs_out[i] = 1.0 - nonzero_mass;
      int floored = 0;
      for (uint32_t i = 0; i < nalpha; ++i)
        if (probs_out[i] < K_MIN_CATEGORICAL) {
          probs_out[i] = K_MIN_CATEGORICAL;
          floored = 1;
        }
      if (floored) {
        double tot = 0.0;
        for (uint32_t i = 0; i < nalpha; ++i) tot += probs_out[i];
        for (uint32_t i = 0; i < nalpha; ++i) probs_out[i] /= tot;
      }
      break;
    }
  }
  return OK;
}

int bsc_mstep(uint32_t d, uint32_t h, const double* w_prev, double pi_prev,
              double sigma2_prev, const double* sum_s, const double* sum_ssT,
              const double* sum_y_sT, const double* value_counts,
              const double* scalars, double* w_out, double* pi_out,
              double* sigma2_out) {
  (void)pi_prev;
  (void)sigma2_prev;
  return ld_mstep(0, NULL, 0, d, h, w_prev, sum_s, sum_ssT, sum_y_sT, value_counts, scalars, w_out,
                  pi_out, NULL, sigma2_out);
}

/* ------------------------------------------------- map_reduce over shards */
typedef struct {
  const ctx_t* c;
  uint64_t n, shards;
  stats_t* partial;
  int* rc;
  char (*err)[512];
  uint64_t next;
  pthread_mutex_t mu;
} pool_t;

static void shard_range(uint64_t n, uint64_t shards, uint64_t i, uint64_t* b,
                        uint64_t* e) { /* ShardPlan::with_shards, parallel.cpp:27-43 */
  const uint64_t base = n / shards, extra = n % shards;
  *b = i * base + (i < extra ? i : extra);
  *e = *b + base + (i < extra ? 1 : 0);
}

static void* pool_worker(void* arg) {
  pool_t* p = arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    const uint64_t i = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (i >= p->shards) return NULL;
    uint64_t b, e;
    shard_range(p->n, p->shards, i, &b, &e);
    p->rc[i] = estep_rows(p->c, b, e, &p->partial[i], NULL, NULL, NULL);
    if (p->rc[i]) snprintf(p->err[i], 512, "shard %llu: %s", (unsigned long long)i, g_err);
  }
}

/* LinearDiscreteModel::step (:410-427) via map_reduce (parallel.cpp:109-158):
 * per-shard stats, ordered fold (SuffStats::combine, :89-107), then mstep. */
int ld_step(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
            double pi, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
            const double* w, double sigma2, double temperature, const double* y, uint64_t n,
            uint32_t shards, uint32_t workers, double* w_out, double* pi_out,
            double* probs_out, double* sigma2_out, double* free_energy) {
  if (shards == 0 || workers == 0) return fail(E_CONFIG, "shard plan: shards and workers must be >= 1");
  const prior_t pr = {family, nalpha, alpha, probs, pi};
  ctx_t c;
  tmpl_t t;
  int rc = ctx_init(&c, &t, d, h, hprime, gamma, w, &pr, sigma2, temperature, y);
  if (rc) return rc;
  pool_t p;
  p.c = &c;
  p.n = n;
  p.shards = shards;
  p.partial = malloc(shards * sizeof(stats_t));
  p.rc = calloc(shards, sizeof(int));
  p.err = calloc(shards, 512);
  p.next = 0;
  pthread_mutex_init(&p.mu, NULL);
  for (uint32_t i = 0; i < shards; ++i) stats_alloc(&p.partial[i], d, h);
  const uint32_t threads = workers < shards ? workers : shards;
  if (threads <= 1) {
    pool_worker(&p);
  } else {
    pthread_t* th = malloc(threads * sizeof(pthread_t));
    for (uint32_t i = 0; i < threads; ++i) pthread_create(&th[i], NULL, pool_worker, &p);
    for (uint32_t i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    free(th);
  }
  for (uint32_t i = 0; i < shards && !rc; ++i)
    if (p.rc[i]) rc = fail(p.rc[i], "%s", p.err[i]);
  if (!rc) {
    stats_t* tot = &p.partial[0];
    for (uint32_t i = 1; i < shards; ++i) {
      const stats_t* o = &p.partial[i];
      for (uint32_t j = 0; j < h; ++j) tot->sum_s[j] += o->sum_s[j];
      for (size_t j = 0; j < (size_t)h * h; ++j) tot->sum_ssT[j] += o->sum_ssT[j];
      for (size_t j = 0; j < (size_t)d * h; ++j) tot->sum_y_sT[j] += o->sum_y_sT[j];
      for (uint32_t k = 0; k < c.vt.nv; ++k) tot->counts[k] += o->counts[k];
      tot->sum_y2 += o->sum_y2;
      tot->log_partition += o->log_partition;
      tot->points += o->points;
    }
    double scal[3] = {tot->sum_y2, tot->log_partition, (double)tot->points};
    rc = ld_mstep(family, alpha, nalpha, d, h, w, tot->sum_s, tot->sum_ssT, tot->sum_y_sT,
                  tot->counts, scal, w_out, pi_out, probs_out, sigma2_out);
    *free_energy = tot->log_partition;
  }
  for (uint32_t i = 0; i < shards; ++i) stats_free(&p.partial[i]);
  free(p.partial);
  free(p.rc);
  free(p.err);
  pthread_mutex_destroy(&p.mu);
  ctx_free(&c, &t);
  return rc;
}

int bsc_step(uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
             const double* w, double pi, double sigma2, double temperature,
             const double* y, uint64_t n, uint32_t shards, uint32_t workers,
             double* w_out, double* pi_out, double* sigma2_out,
             double* free_energy) {
  return ld_step(0, NULL, NULL, 0, pi, d, h, hprime, gamma, w, sigma2, temperature, y, n, shards,
                 workers, w_out, pi_out, NULL, sigma2_out, free_energy);
}

/* Per-point candidate sets exactly as estep_impl selects them (:240-253). */
int ld_candidates(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
                  double pi, uint32_t d, uint32_t h, uint32_t hprime, const double* w,
                  double sigma2, const double* y, uint64_t n, uint32_t* out) {
  const prior_t pr = {family, nalpha, alpha, probs, pi};
  int rc = validate_ld(d, h, w, sigma2, &pr);
  if (rc) return rc;
  vtab_t vt;
  rc = value_table(&pr, &vt);
  if (rc) return rc;
  double* wt = malloc((size_t)d * h * sizeof(double));
  double* gram = malloc((size_t)h * h * sizeof(double));
  double* b = malloc(h * sizeof(double));
  double* scores = malloc(h * sizeof(double));
  keyed_t* scratch = malloc(h * sizeof(keyed_t));
  gram_of(w, d, h, wt, gram);
  const double inv2s = 1.0 / (2.0 * sigma2);
  for (uint64_t i = 0; i < n && !rc; ++i) {
    const double* yy = y + i * d;
    for (uint32_t u = 0; u < h; ++u) {
      double acc = 0.0;
      for (uint32_t t = 0; t < d; ++t) acc += wt[(size_t)u * d + t] * yy[t];
      b[u] = acc;
    }
    scores_of(&vt, b, gram, h, inv2s, scores);
    rc = select_cands(scores, h, hprime, out + i * hprime, scratch);
  }
  free(wt);
  free(gram);
  free(b);
  free(scores);
  free(scratch);
  return rc;
}

int bsc_candidates(uint32_t d, uint32_t h, uint32_t hprime, const double* w,
                   double pi, double sigma2, const double* y, uint64_t n,
                   uint32_t* out) {
  return ld_candidates(0, NULL, NULL, 0, pi, d, h, hprime, w, sigma2, y, n, out);
}

/* LinearDiscreteModel::inference, linear_discrete.cpp:429-450 (T = 1). */
int ld_inference(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
                 double pi, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                 const double* w, double sigma2, const double* y, uint64_t n,
                 double* map_states, double* map_mass, double* expected) {
  const prior_t pr = {family, nalpha, alpha, probs, pi};
  ctx_t c;
  tmpl_t t;
  int rc = ctx_init(&c, &t, d, h, hprime, gamma, w, &pr, sigma2, 1.0, y);
  if (rc) return rc;
  memset(map_states, 0, n * h * sizeof(double));
  stats_t st;
  stats_alloc(&st, d, h);
  rc = estep_rows(&c, 0, n, &st, map_states, map_mass, expected);
  stats_free(&st);
  ctx_free(&c, &t);
  return rc;
}

int bsc_inference(uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                  const double* w, double pi, double sigma2, const double* y,
                  uint64_t n, double* map_states, double* map_mass,
                  double* expected) {
  return ld_inference(0, NULL, NULL, 0, pi, d, h, hprime, gamma, w, sigma2, y, n, map_states,
                      map_mass, expected);
}

/* exact_log_likelihood, linear_discrete.cpp:481-508: the full state space is
 * the truncated enumeration with hprime = gamma = H. */
int ld_exact_log_likelihood(uint32_t family, const double* alpha, const double* probs,
                            uint32_t nalpha, double pi, uint32_t d, uint32_t h,
                            const double* w, double sigma2, const double* y, uint64_t n,
                            double* out) {
  const prior_t pr = {family, nalpha, alpha, probs, pi};
  int rc = validate_ld(d, h, w, sigma2, &pr);
  if (rc) return rc;
  vtab_t vt;
  rc = value_table(&pr, &vt);
  if (rc) return rc;
  const uint64_t count = state_count_v(h, h, h, vt.nv);
  if (count > (1u << 22))
    return fail(E_CONFIG, "%s: state space too large for exact evaluation", family_name(family));
  uint32_t* all = malloc(h * sizeof(uint32_t));
  for (uint32_t i = 0; i < h; ++i) all[i] = i;
  tmpl_t t;
  rc = tmpl_build(&t, h, h, h, vt.nv, 1u << 22);
  if (rc) {
    free(all);
    return rc;
  }
  states_t s;
  states_alloc(&s, count, h);
  instantiate(&t, h, all, &s);
  double* dense = malloc(h * sizeof(double));
  double* lj = malloc(count * sizeof(double));
  double total = 0.0;
  for (uint64_t i = 0; i < n && !rc; ++i) {
    for (size_t k = 0; k < s.n && !rc; ++k) {
      memset(dense, 0, h * sizeof(double));
      for (uint32_t a = 0; a < s.len[k]; ++a)
        dense[s.act[k * s.stride + a]] = vt.values[s.vix[k * s.stride + a]];
      rc = log_joint_v(d, h, w, sigma2, &vt, family_name(family), y + i * d, dense, &lj[k]);
    }
    double l;
    if (!rc) rc = lse(lj, s.n, &l);
    if (!rc) total += l;
  }
  *out = total;
  free(all);
  free(dense);
  free(lj);
  states_free(&s);
  tmpl_free(&t);
  return rc;
}

int bsc_exact_log_likelihood(uint32_t d, uint32_t h, const double* w, double pi,
                             double sigma2, const double* y, uint64_t n,
                             double* out) {
  return ld_exact_log_likelihood(0, NULL, NULL, 0, pi, d, h, w, sigma2, y, n, out);
}

/* LinearDiscreteModel::generate, linear_discrete.cpp:452-479 (TSC / DSC
 * draws; BSC is bsc_generate). mean = W s summed left to right over h. */
static uint32_t rng_categorical(rng_t* r, const double* probs, uint32_t k) {
  /* RngStream::categorical, core.cpp:80-91 */
  double total = 0.0;
  for (uint32_t i = 0; i < k; ++i) total += probs[i];
  const double u = rng_uniform01(r) * total;
  double acc = 0.0;
  for (uint32_t i = 0; i + 1 < k; ++i) {
    acc += probs[i];
    if (u < acc) return i;
  }
  return k - 1;
}

int ld_generate(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
                double pi, uint32_t d, uint32_t h, const double* w, double sigma2, uint64_t n,
                uint64_t seed, double* y_out) {
  if (family == 0) return bsc_generate(d, h, w, pi, sigma2, n, seed, y_out);
  const prior_t pr = {family, nalpha, alpha, probs, pi};
  int rc = validate_ld(d, h, w, sigma2, &pr);
  if (rc) return rc;
  const double noise_std = sqrt(sigma2);
  double* s = malloc(h * sizeof(double));
  rng_t r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) {
    for (uint32_t j = 0; j < h; ++j) {
      if (family == 1)
        s[j] = rng_bernoulli(&r, pi) ? (rng_bernoulli(&r, 0.5) ? 1.0 : -1.0) : 0.0;
      else
        s[j] = alpha[rng_categorical(&r, probs, nalpha)];
    }
    for (uint32_t di = 0; di < d; ++di) {
      double acc = 0.0;
      const double* row = w + (size_t)di * h;
      for (uint32_t j = 0; j < h; ++j) acc += row[j] * s[j];
      y_out[i * d + di] = acc + noise_std * rng_normal(&r);
    }
  }
  free(s);
  return OK;
}

/* ============================================================ max causes */
/* MaxCausesModel (max_causes.cpp): binary latents, the data mean at each
 * dimension is the dictionary entry of the winning active unit (largest W, or
 * largest |W| in absmax mode; ties keep the lowest unit). mode 0 = mca (kMax),
 * 1 = mmca (kAbsMax). */
#define K_MIN_MCA_WEIGHT 1e-8 /* model.hpp:36 */
#define K_EVIDENCE_FLOOR 1e-9 /* model.hpp:37 */

typedef struct {
  uint32_t mode;
  double rho; /* soft winner exponent (mca only), 0 = hard winners */
} mca_cfg_t;

/* winner_at, max_causes.cpp:27-41 */
static uint32_t mca_winner(const double* w, uint32_t h, size_t d, const uint32_t* act, uint32_t k,
                           uint32_t mode) {
  uint32_t best = act[0];
  double best_key = mode == 0 ? w[d * h + act[0]] : fabs(w[d * h + act[0]]);
  for (uint32_t i = 1; i < k; ++i) {
    const double key = mode == 0 ? w[d * h + act[i]] : fabs(w[d * h + act[i]]);
    if (key > best_key) {
      best_key = key;
      best = act[i];
    }
  }
  return best;
}

static int mca_validate(uint32_t d, uint32_t h, const double* w, double pi, double sigma2, uint32_t mode) {
  const char* nm = mode == 0 ? "mca" : "mmca";
  for (size_t i = 0; i < (size_t)d * h; ++i)
    if (!isfinite(w[i])) return fail(E_NUMERIC, "%s: non-finite dictionary", nm);
  if (mode == 0)
    for (size_t i = 0; i < (size_t)d * h; ++i)
      if (w[i] < K_MIN_MCA_WEIGHT) return fail(E_CONFIG, "mca: dictionary entries must be >= the weight floor");
  if (!(pi > 0.0 && pi < 1.0)) return fail(E_CONFIG, "%s: pi must lie in (0,1)", nm);
  if (!(sigma2 > 0.0)) return fail(E_CONFIG, "%s: sigma2 must be positive", nm);
  return OK;
}

/* selection scores, max_causes.cpp:174-176: (2 w_h·y − ‖w_h‖²)·inv2s */
static void mca_scores(const double* wt, uint32_t d, uint32_t h, const double* y, double inv2s, double* scores) {
  for (uint32_t u = 0; u < h; ++u) {
    const double* col = wt + (size_t)u * d;
    double dot = 0.0, sq = 0.0;
    for (uint32_t t = 0; t < d; ++t) dot += col[t] * y[t];
    for (uint32_t t = 0; t < d; ++t) sq += col[t] * col[t];
    scores[u] = (2.0 * dot - sq) * inv2s;
  }
}

typedef struct {
  double *num, *den; /* winner_num, winner_den (D×H) */
  double sum_act, log_partition;
  uint64_t points;
  double residual; /* residual pass */
} mca_stats_t;

/* Per-point states, log-joints (and winners) under W: the shared core of
 * estep_impl (:180-250) and residual_impl (:283-350). */
static int mca_point(const double* w, const double* wt, uint32_t d, uint32_t h, uint32_t hprime,
                     const tmpl_t* tmpl, uint32_t mode, double pi, double sigma2, const double* y,
                     states_t* s, uint32_t* cand, double* scores, keyed_t* scratch, double* lj,
                     uint32_t* winners, double* resid_out) {
  const double lp1 = log(pi), lp0 = log(1.0 - pi);
  const double norm_const = -0.5 * (double)d * (K_LOG_2PI + log(sigma2));
  const double inv2s = 1.0 / (2.0 * sigma2);
  mca_scores(wt, d, h, y, inv2s, scores);
  int rc = select_cands(scores, h, hprime, cand, scratch);
  if (rc) return rc;
  instantiate(tmpl, h, cand, s);
  for (size_t i = 0; i < s->n; ++i) {
    const uint32_t k = s->len[i];
    const uint32_t* act = s->act + i * s->stride;
    double resid = 0.0;
    if (k == 0) {
      for (uint32_t t = 0; t < d; ++t) resid += y[t] * y[t];
    } else {
      for (uint32_t t = 0; t < d; ++t) {
        const uint32_t win = mca_winner(w, h, t, act, k, mode);
        if (winners) winners[i * d + t] = win;
        const double r = y[t] - w[(size_t)t * h + win];
        resid += r * r;
      }
    }
    if (resid_out) resid_out[i] = resid;
    const double kk = (double)k;
    lj[i] = kk * lp1 + ((double)h - kk) * lp0 + norm_const - resid * inv2s;
  }
  return OK;
}

typedef struct {
  uint32_t d, h, hprime, gamma, mode;
  double rho, pi, sigma2, temperature;
  const double *w, *wt, *y;
  const double *w_new; /* residual pass: the updated dictionary (NULL in the E pass) */
  const tmpl_t* tmpl;
} mca_ctx_t;

static int mca_rows(const mca_ctx_t* c, uint64_t rb, uint64_t re, mca_stats_t* st, double* map_states,
                    double* map_mass, double* expected) {
  const uint32_t d = c->d, h = c->h;
  const size_t total = 1 + h + c->tmpl->count;
  states_t s;
  states_alloc(&s, total, c->gamma);
  double* scores = malloc(h * sizeof(double));
  double* lj = malloc(total * sizeof(double));
  double* q = malloc(total * sizeof(double));
  double* es = malloc(h * sizeof(double));
  double* rnew = malloc(total * sizeof(double));
  uint32_t* winners = malloc(total * d * sizeof(uint32_t));
  uint32_t* cand = malloc(c->hprime * sizeof(uint32_t));
  keyed_t* scratch = malloc(h * sizeof(keyed_t));
  int rc = OK;
  for (uint64_t n = rb; n < re && !rc; ++n) {
    const double* y = c->y + n * d;
    rc = mca_point(c->w, c->wt, d, h, c->hprime, c->tmpl, c->mode, c->pi, c->sigma2, y, &s, cand, scores,
                   scratch, lj, c->w_new ? NULL : winners, NULL);
    if (rc) break;
    if (c->w_new) { /* residual_impl :315-349: q at T (max/sum), resid under W' */
      for (size_t i = 0; i < s.n; ++i) {
        const uint32_t k = s.len[i];
        const uint32_t* act = s.act + i * s.stride;
        double r = 0.0;
        if (k == 0) {
          for (uint32_t t = 0; t < d; ++t) r += y[t] * y[t];
        } else {
          for (uint32_t t = 0; t < d; ++t) {
            const double b = y[t] - c->w_new[(size_t)t * h + mca_winner(c->w_new, h, t, act, k, c->mode)];
            r += b * b;
          }
        }
        rnew[i] = r;
      }
      double m = lj[0];
      for (size_t i = 0; i < s.n; ++i) m = dmax(m, lj[i]);
      double acc = 0.0;
      for (size_t i = 0; i < s.n; ++i) {
        q[i] = exp((lj[i] - m) / c->temperature);
        acc += q[i];
      }
      double pr = 0.0;
      for (size_t i = 0; i < s.n; ++i) pr += q[i] / acc * rnew[i];
      st->residual += pr;
      st->points++;
      continue;
    }
    double lse1;
    rc = lse(lj, s.n, &lse1);
    if (rc) break;
    if (c->temperature == 1.0) {
      for (size_t i = 0; i < s.n; ++i) q[i] = exp(lj[i] - lse1);
    } else {
      double m = lj[0];
      for (size_t i = 0; i < s.n; ++i) m = dmax(m, lj[i]);
      double acc = 0.0;
      for (size_t i = 0; i < s.n; ++i) {
        q[i] = exp((lj[i] - m) / c->temperature);
        acc += q[i];
      }
      for (size_t i = 0; i < s.n; ++i) q[i] /= acc;
    }
    for (uint32_t j = 0; j < h; ++j) es[j] = 0.0; /* :226-259 */
    for (size_t i = 0; i < s.n; ++i) {
      const double qi = q[i];
      const uint32_t k = s.len[i];
      const uint32_t* act = s.act + i * s.stride;
      if (k == 0) continue;
      st->sum_act += qi * (double)k;
      for (uint32_t a = 0; a < k; ++a) es[act[a]] += qi;
      if (c->rho > 0.0) {
        for (uint32_t t = 0; t < d; ++t) {
          double wmax = 0.0;
          for (uint32_t a = 0; a < k; ++a) wmax = dmax(wmax, c->w[(size_t)t * h + act[a]]);
          double tot = 0.0;
          for (uint32_t a = 0; a < k; ++a) tot += pow(c->w[(size_t)t * h + act[a]] / wmax, c->rho);
          for (uint32_t a = 0; a < k; ++a) {
            const double share = pow(c->w[(size_t)t * h + act[a]] / wmax, c->rho) / tot;
            st->num[(size_t)t * h + act[a]] += qi * share * y[t];
            st->den[(size_t)t * h + act[a]] += qi * share;
          }
        }
      } else {
        for (uint32_t t = 0; t < d; ++t) {
          const uint32_t win = winners[i * d + t];
          st->num[(size_t)t * h + win] += qi * y[t];
          st->den[(size_t)t * h + win] += qi;
        }
      }
    }
    st->log_partition += lse1;
    st->points++;
    if (map_states) {
      size_t best = 0;
      for (size_t i = 1; i < s.n; ++i)
        if (q[i] > q[best]) best = i;
      map_mass[n] = q[best];
      for (uint32_t a = 0; a < s.len[best]; ++a) map_states[n * h + s.act[best * s.stride + a]] = 1.0;
      for (uint32_t j = 0; j < h; ++j) expected[n * h + j] = es[j];
    }
  }
  states_free(&s);
  free(scores);
  free(lj);
  free(q);
  free(es);
  free(rnew);
  free(winners);
  free(cand);
  free(scratch);
  return rc;
}

static int mca_ctx_init(mca_ctx_t* c, tmpl_t* t, uint32_t mode, double rho, uint32_t d, uint32_t h,
                        uint32_t hprime, uint32_t gamma, const double* w, double pi, double sigma2,
                        double temperature, const double* y) {
  int rc = mca_validate(d, h, w, pi, sigma2, mode);
  if (rc) return rc;
  if (rho < 0.0) return fail(E_CONFIG, "%s: soft winner exponent must be >= 0", mode == 0 ? "mca" : "mmca");
  if (rho > 0.0 && mode != 0) return fail(E_CONFIG, "soft winners require the non-negative max mode");
  rc = tmpl_build(t, h, hprime, gamma, 1, 1000000);
  if (rc) return rc;
  double* wt = malloc((size_t)d * h * sizeof(double));
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j) wt[(size_t)j * d + i] = w[(size_t)i * h + j];
  *c = (mca_ctx_t){d, h, hprime, gamma, mode, rho, pi, sigma2, temperature, w, wt, y, NULL, t};
  return OK;
}

/* MaxCausesModel::estep_stats (:384-391). scalars = {sum_act, log_partition, points}. */
int mca_estep_stats(uint32_t mode, double rho, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                    const double* w, double pi, double sigma2, double temperature, const double* y, uint64_t n,
                    uint64_t row_begin, uint64_t row_end, double* winner_num, double* winner_den,
                    double* scalars) {
  if (row_end < row_begin || row_end > n) return fail(E_CONFIG, "bad row range");
  mca_ctx_t c;
  tmpl_t t;
  int rc = mca_ctx_init(&c, &t, mode, rho, d, h, hprime, gamma, w, pi, sigma2, temperature, y);
  if (rc) return rc;
  mca_stats_t st = {calloc((size_t)d * h, 8), calloc((size_t)d * h, 8), 0.0, 0.0, 0, 0.0};
  rc = mca_rows(&c, row_begin, row_end, &st, NULL, NULL, NULL);
  if (!rc) {
    memcpy(winner_num, st.num, (size_t)d * h * 8);
    memcpy(winner_den, st.den, (size_t)d * h * 8);
    scalars[0] = st.sum_act;
    scalars[1] = st.log_partition;
    scalars[2] = (double)st.points;
  }
  free(st.num);
  free(st.den);
  free((void*)c.wt);
  tmpl_free(&t);
  return rc;
}

/* MaxCausesModel::mstep_fixedpoint (:393-414). */
int mca_mstep_fixedpoint(uint32_t mode, uint32_t d, uint32_t h, const double* w_prev, const double* winner_num,
                         const double* winner_den, const double* scalars, double* w_out, double* pi_out) {
  const uint64_t points = (uint64_t)scalars[2];
  if (points == 0) return fail(E_CONFIG, "%s: mstep without data", mode == 0 ? "mca" : "mmca");
  const double nh = (double)points * (double)h;
  if (w_out != w_prev) memcpy(w_out, w_prev, (size_t)d * h * 8);
  for (size_t i = 0; i < (size_t)d * h; ++i)
    if (winner_den[i] >= K_EVIDENCE_FLOOR) {
      double v = winner_num[i] / winner_den[i];
      if (mode == 0) v = dmax(v, K_MIN_MCA_WEIGHT);
      w_out[i] = v;
    }
  *pi_out = dmin(dmax(scalars[0] / nh, K_MIN_PI), 1.0 - K_MIN_PI);
  return OK;
}

/* ------------- map_reduce for the two passes of MaxCausesModel::step */
typedef struct {
  const mca_ctx_t* c;
  uint64_t n, shards;
  mca_stats_t* partial;
  int* rc;
  char (*err)[512];
  uint64_t next;
  pthread_mutex_t mu;
} mca_pool_t;

static void* mca_worker(void* arg) {
  mca_pool_t* p = arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    const uint64_t i = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (i >= p->shards) return NULL;
    uint64_t b, e;
    shard_range(p->n, p->shards, i, &b, &e);
    p->rc[i] = mca_rows(p->c, b, e, &p->partial[i], NULL, NULL, NULL);
    if (p->rc[i]) snprintf(p->err[i], 512, "shard %llu: %s", (unsigned long long)i, g_err);
  }
}

static int mca_map_reduce(const mca_ctx_t* c, uint64_t n, uint32_t shards, uint32_t workers, mca_stats_t* tot) {
  mca_pool_t p;
  p.c = c;
  p.n = n;
  p.shards = shards;
  p.partial = malloc(shards * sizeof(mca_stats_t));
  p.rc = calloc(shards, sizeof(int));
  p.err = calloc(shards, 512);
  p.next = 0;
  pthread_mutex_init(&p.mu, NULL);
  const size_t dh = (size_t)c->d * c->h;
  for (uint32_t i = 0; i < shards; ++i)
    p.partial[i] = (mca_stats_t){calloc(dh, 8), calloc(dh, 8), 0.0, 0.0, 0, 0.0};
  const uint32_t threads = workers < shards ? workers : shards;
  if (threads <= 1) {
    mca_worker(&p);
  } else {
    pthread_t* th = malloc(threads * sizeof(pthread_t));
    for (uint32_t i = 0; i < threads; ++i) pthread_create(&th[i], NULL, mca_worker, &p);
    for (uint32_t i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    free(th);
  }
  int rc = OK;
  for (uint32_t i = 0; i < shards && !rc; ++i)
    if (p.rc[i]) rc = fail(p.rc[i], "%s", p.err[i]);
  if (!rc) { /* SuffStats::combine: ordered fold, fields in insertion order */
    *tot = p.partial[0];
    p.partial[0].num = p.partial[0].den = NULL;
    for (uint32_t i = 1; i < shards; ++i) {
      const mca_stats_t* o = &p.partial[i];
      for (size_t j = 0; j < dh; ++j) tot->num[j] += o->num[j];
      for (size_t j = 0; j < dh; ++j) tot->den[j] += o->den[j];
      tot->sum_act += o->sum_act;
      tot->log_partition += o->log_partition;
      tot->residual += o->residual;
      tot->points += o->points;
    }
  }
  for (uint32_t i = 0; i < shards; ++i) {
    free(p.partial[i].num);
    free(p.partial[i].den);
  }
  free(p.partial);
  free(p.rc);
  free(p.err);
  pthread_mutex_destroy(&p.mu);
  return rc;
}

/* MaxCausesModel::step (:416-446): E pass, fixed-point M-step, then the
 * residual pass for sigma2 (posterior held at the incoming params). */
int mca_step(uint32_t mode, double rho, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
             const double* w, double pi, double sigma2, double temperature, const double* y, uint64_t n,
             uint32_t shards, uint32_t workers, double* w_out, double* pi_out, double* sigma2_out,
             double* free_energy) {
  if (shards == 0 || workers == 0) return fail(E_CONFIG, "shard plan: shards and workers must be >= 1");
  mca_ctx_t c;
  tmpl_t t;
  int rc = mca_ctx_init(&c, &t, mode, rho, d, h, hprime, gamma, w, pi, sigma2, temperature, y);
  if (rc) return rc;
  mca_stats_t st = {0};
  rc = mca_map_reduce(&c, n, shards, workers, &st);
  double* wn = malloc((size_t)d * h * 8);
  double pin = pi;
  if (!rc) {
    double sc[3] = {st.sum_act, st.log_partition, (double)st.points};
    rc = mca_mstep_fixedpoint(mode, d, h, w, st.num, st.den, sc, wn, &pin);
  }
  if (!rc) {
    mca_ctx_t c2 = c;
    c2.w_new = wn;
    mca_stats_t rs = {0};
    rc = mca_map_reduce(&c2, n, shards, workers, &rs);
    if (!rc) {
      memcpy(w_out, wn, (size_t)d * h * 8);
      *pi_out = pin;
      *sigma2_out = dmax(rs.residual / ((double)st.points * (double)d), K_MIN_SIGMA2);
      *free_energy = st.log_partition;
    }
    free(rs.num);
    free(rs.den);
  }
  free(wn);
  free(st.num);
  free(st.den);
  free((void*)c.wt);
  tmpl_free(&t);
  return rc;
}

int mca_candidates(uint32_t mode, uint32_t d, uint32_t h, uint32_t hprime, const double* w, double pi,
                   double sigma2, const double* y, uint64_t n, uint32_t* out) {
  int rc = mca_validate(d, h, w, pi, sigma2, mode);
  if (rc) return rc;
  double* wt = malloc((size_t)d * h * 8);
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j) wt[(size_t)j * d + i] = w[(size_t)i * h + j];
  double* scores = malloc(h * 8);
  keyed_t* scratch = malloc(h * sizeof(keyed_t));
  for (uint64_t i = 0; i < n && !rc; ++i) {
    mca_scores(wt, d, h, y + i * d, 1.0 / (2.0 * sigma2), scores);
    rc = select_cands(scores, h, hprime, out + i * hprime, scratch);
  }
  free(wt);
  free(scores);
  free(scratch);
  return rc;
}

/* MaxCausesModel::inference (:448-468). */
int mca_inference(uint32_t mode, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma, const double* w,
                  double pi, double sigma2, const double* y, uint64_t n, double* map_states, double* map_mass,
                  double* expected) {
  mca_ctx_t c;
  tmpl_t t;
  int rc = mca_ctx_init(&c, &t, mode, 0.0, d, h, hprime, gamma, w, pi, sigma2, 1.0, y);
  if (rc) return rc;
  memset(map_states, 0, n * h * 8);
  mca_stats_t st = {calloc((size_t)d * h, 8), calloc((size_t)d * h, 8), 0.0, 0.0, 0, 0.0};
  rc = mca_rows(&c, 0, n, &st, map_states, map_mass, expected);
  free(st.num);
  free(st.den);
  free((void*)c.wt);
  tmpl_free(&t);
  return rc;
}

/* MaxCausesModel::log_joint (:132-153). */
int mca_log_joint(uint32_t mode, uint32_t d, uint32_t h, const double* w, double pi, double sigma2,
                  const double* y, const double* s, double* out) {
  uint32_t* act = malloc((h ? h : 1) * sizeof(uint32_t));
  uint32_t k = 0;
  for (uint32_t j = 0; j < h; ++j) {
    if (s[j] == 1.0)
      act[k++] = j;
    else if (s[j] != 0.0) {
      free(act);
      return fail(E_CONFIG, "max causes: latent configuration must be binary");
    }
  }
  double resid = 0.0;
  for (uint32_t t = 0; t < d; ++t) {
    const double wb = k ? w[(size_t)t * h + mca_winner(w, h, t, act, k, mode)] : 0.0;
    const double r = y[t] - wb;
    resid += r * r;
  }
  free(act);
  const double prior = (double)k * log(pi) + (double)(h - k) * log(1.0 - pi);
  *out = prior - 0.5 * (double)d * (K_LOG_2PI + log(sigma2)) - resid / (2.0 * sigma2);
  return OK;
}

/* MaxCausesModel::exact_log_likelihood (:454-474): all 2^H masks. */
int mca_exact_log_likelihood(uint32_t mode, uint32_t d, uint32_t h, const double* w, double pi, double sigma2,
                             const double* y, uint64_t n, double* out) {
  int rc = mca_validate(d, h, w, pi, sigma2, mode);
  if (rc) return rc;
  if (h > 22) return fail(E_CONFIG, "%s: state space too large for exact evaluation", mode == 0 ? "mca" : "mmca");
  const uint64_t ns = 1ull << h;
  double* lj = malloc(ns * 8);
  double* s = malloc(h * 8);
  double total = 0.0;
  for (uint64_t i = 0; i < n && !rc; ++i) {
    for (uint64_t m = 0; m < ns && !rc; ++m) {
      for (uint32_t j = 0; j < h; ++j) s[j] = (m >> j) & 1 ? 1.0 : 0.0;
      rc = mca_log_joint(mode, d, h, w, pi, sigma2, y + i * d, s, &lj[m]);
    }
    double l;
    if (!rc) rc = lse(lj, ns, &l);
    if (!rc) total += l;
  }
  *out = total;
  free(lj);
  free(s);
  return rc;
}

/* MaxCausesModel::generate (:430-452). */
int mca_generate(uint32_t mode, uint32_t d, uint32_t h, const double* w, double pi, double sigma2, uint64_t n,
                 uint64_t seed, double* y_out) {
  int rc = mca_validate(d, h, w, pi, sigma2, mode);
  if (rc) return rc;
  const double noise_std = sqrt(sigma2);
  uint32_t* act = malloc((h ? h : 1) * sizeof(uint32_t));
  rng_t r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t k = 0;
    for (uint32_t j = 0; j < h; ++j)
      if (rng_bernoulli(&r, pi)) act[k++] = j;
    for (uint32_t t = 0; t < d; ++t) {
      const double wb = k ? w[(size_t)t * h + mca_winner(w, h, t, act, k, mode)] : 0.0;
      y_out[i * d + t] = wb + noise_std * rng_normal(&r);
    }
  }
  free(act);
  return OK;
}

/* MaxCausesModel::standard_init (:121-130) with detail::init_weights
 * (model.cpp:201-220, take_abs in mca mode). */
int mca_standard_init(uint32_t mode, uint32_t d, uint32_t h, uint32_t hprime, const double* y, uint64_t n,
                      uint64_t seed, double* w_out, double* pi_out, double* sigma2_out) {
  if (n < 2) return fail(E_DATA, "standard_init requires at least two data points");
  double* m = malloc(d * sizeof(double));
  column_means(y, n, d, m);
  const double var = mean_variance(y, n, d, m);
  const double sd = var > 0.0 ? sqrt(var / h) : 0.0;
  rng_t r;
  rng_seed(&r, seed);
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j) {
      double v = m[i] + sd * rng_normal(&r);
      if (mode == 0) v = dmax(fabs(v), K_MIN_MCA_WEIGHT);
      w_out[(size_t)i * h + j] = v;
    }
  *sigma2_out = dmax(var, K_MIN_SIGMA2);
  *pi_out = (double)(hprime < h ? hprime : h) / (2.0 * (double)h);
  free(m);
  return OK;
}
