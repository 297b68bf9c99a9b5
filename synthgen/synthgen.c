/*
 * synthgen.c — seeded synthetic EHR-shaped irregular sparse tensors for COPA.
 *
 * This module is INPUT SYNTHESIS ONLY. It holds none of the method's arithmetic
 * (no projection, no SVD, no MTTKRP, no ADMM). It is the one module shared by the
 * oracle (oracle/) and the CUDA path (paper_1803_04572_b200/): both read the arrays
 * it writes, neither imports the other.
 *
 * Randomness is counter-based: every patient k draws from its own splitmix64
 * streams keyed by (seed, stream id, k), so
 *   - output is independent of thread count / scheduling (OpenMP over patients),
 *   - any patient range [k0, k1) can be generated on its own and is bit-identical
 *     to the same patients of the full workload (used for bounded oracle samples
 *     and for per-rank shards).
 *
 * Distributions (BASELINE.json configs; readings listed in DESIGN.md §3):
 *   I_k      : uniform int [lo,hi] | geometric(p) on {1,2,..} clipped | lognormal(median, sigma)
 *              rounded half-even, clipped  (DESIGN.md R-gen-1..3)
 *   row size : Poisson(lambda) + 1, capped at J
 *   features : distinct within a row; uniform over J, or Zipf(s): P(j) ∝ (j+1)^-s (j = 0 most frequent);
 *              drawn by inverse CDF with rejection of duplicates; stored sorted ascending
 *   values   : uniform int {1..5} | 1 + Poisson(1) | constant 1.0
 *   times    : I_k iid uniforms on [0, 36.5·I_k] days, sorted, strictly increasing
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t K;
  int32_t J;
  int32_t ik_dist;   /* 0 uniform [ik_lo, ik_hi]; 1 geometric(p = ik_a); 2 lognormal(median ik_a, sigma ik_b) */
  double ik_a, ik_b;
  int32_t ik_lo, ik_hi;
  double row_lambda; /* row size = Poisson(row_lambda) + 1 */
  double zipf_s;     /* <= 0: uniform features */
  int32_t val_dist;  /* 0: uniform int 1..5; 1: 1 + Poisson(1); 2: constant 1 */
  int32_t times;     /* 1: generate visit times */
  uint64_t seed;
} gen_config;

enum { ST_IK = 1, ST_ROWS = 2, ST_FEAT = 3, ST_VAL = 4, ST_TIME = 5 };

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct { uint64_t s; } rng_t;

static inline rng_t rng_make(uint64_t seed, uint64_t stream, uint64_t k) {
  rng_t r;
  r.s = mix64(mix64(seed ^ 0xC0FFEE1234567ull) ^ mix64((stream << 48) ^ 0x5DEECE66Dull) ^ mix64(k + 0x1234ull));
  return r;
}
static inline uint64_t rng_next(rng_t* r) {
  r->s += 0x9E3779B97F4A7C15ull;
  uint64_t z = r->s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
/* uniform in [0,1) with 53 random bits */
static inline double rng_u01(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
/* uniform in (0,1] */
static inline double rng_u01_open0(rng_t* r) { return ((double)(rng_next(r) >> 11) + 1.0) * 0x1.0p-53; }

static int32_t poisson_inv(double lambda, double u) {
  double p = exp(-lambda), F = p;
  int32_t k = 0;
  while (u > F && k < 1000) {
    ++k;
    p *= lambda / k;
    F += p;
  }
  return k;
}

static int32_t draw_ik(const gen_config* c, int64_t k) {
  rng_t r = rng_make(c->seed, ST_IK, (uint64_t)k);
  int64_t v;
  if (c->ik_dist == 0) {
    uint64_t span = (uint64_t)(c->ik_hi - c->ik_lo + 1);
    v = c->ik_lo + (int64_t)(rng_next(&r) % span);
  } else if (c->ik_dist == 1) {
    double u = rng_u01_open0(&r);
    double g = ceil(log(u) / log1p(-c->ik_a));
    if (g < 1) g = 1;
    if (g > 1e9) g = 1e9;
    v = (int64_t)g;
  } else {
    double u1 = rng_u01_open0(&r), u2 = rng_u01(&r);
    double z = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
    double x = exp(log(c->ik_a) + c->ik_b * z);
    if (x > 1e9) x = 1e9;
    v = (int64_t)nearbyint(x); /* default rounding mode: half-even */
  }
  if (v < c->ik_lo) v = c->ik_lo;
  if (v > c->ik_hi) v = c->ik_hi;
  return (int32_t)v;
}

/* Phase 1: rows per patient for k in [k0, k1). */
void gen_patient_rows(const gen_config* c, int64_t k0, int64_t k1, int32_t* I_out) {
#pragma omp parallel for schedule(static)
  for (int64_t k = k0; k < k1; ++k) I_out[k - k0] = draw_ik(c, k);
}

/* Phase 2: nnz per row. patient_row_ptr is local ([k1-k0+1], starting at 0). */
void gen_row_sizes(const gen_config* c, int64_t k0, int64_t k1, const int64_t* patient_row_ptr, int32_t* row_nnz) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t k = k0; k < k1; ++k) {
    rng_t r = rng_make(c->seed, ST_ROWS, (uint64_t)k);
    int64_t a = patient_row_ptr[k - k0], b = patient_row_ptr[k - k0 + 1];
    for (int64_t i = a; i < b; ++i) {
      int32_t s = poisson_inv(c->row_lambda, rng_u01(&r)) + 1;
      if (s > c->J) s = c->J;
      row_nnz[i] = s;
    }
  }
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}
static int cmp_f64(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

static int32_t draw_feature(const gen_config* c, const double* cdf, rng_t* r) {
  if (c->zipf_s <= 0) return (int32_t)(rng_next(r) % (uint64_t)c->J);
  double u = rng_u01(r) * cdf[c->J - 1];
  int32_t lo = 0, hi = c->J - 1; /* first index with cdf[idx] > u */
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    if (cdf[mid] > u) hi = mid; else lo = mid + 1;
  }
  return lo;
}

/* Phase 3: columns, values and (optionally) times.
 * patient_row_ptr: local [k1-k0+1]; row_ptr: local [rows+1] (nnz offsets, starting at 0). */
void gen_fill(const gen_config* c, int64_t k0, int64_t k1, const int64_t* patient_row_ptr, const int64_t* row_ptr,
              int32_t* col, double* val, double* times) {
  double* cdf = NULL;
  if (c->zipf_s > 0) {
    cdf = (double*)malloc(sizeof(double) * (size_t)c->J);
    double acc = 0;
    for (int32_t j = 0; j < c->J; ++j) {
      acc += pow((double)(j + 1), -c->zipf_s);
      cdf[j] = acc;
    }
  }
#pragma omp parallel
  {
    unsigned char* seen = (unsigned char*)calloc((size_t)c->J, 1);
    double* tbuf = NULL;
    int64_t tcap = 0;
#pragma omp for schedule(dynamic, 64)
    for (int64_t k = k0; k < k1; ++k) {
      rng_t rf = rng_make(c->seed, ST_FEAT, (uint64_t)k);
      rng_t rv = rng_make(c->seed, ST_VAL, (uint64_t)k);
      int64_t a = patient_row_ptr[k - k0], b = patient_row_ptr[k - k0 + 1];
      for (int64_t i = a; i < b; ++i) {
        int64_t p0 = row_ptr[i], p1 = row_ptr[i + 1];
        int64_t n = 0;
        while (p0 + n < p1) {
          int32_t j = draw_feature(c, cdf, &rf);
          if (seen[j]) continue; /* distinct within the row: reject duplicates */
          seen[j] = 1;
          col[p0 + n] = j;
          ++n;
        }
        for (int64_t p = p0; p < p1; ++p) seen[col[p]] = 0;
        qsort(col + p0, (size_t)(p1 - p0), sizeof(int32_t), cmp_i32);
        for (int64_t p = p0; p < p1; ++p) {
          double v;
          if (c->val_dist == 0) v = (double)(1 + (int64_t)(rng_next(&rv) % 5u));
          else if (c->val_dist == 1) v = (double)(1 + poisson_inv(1.0, rng_u01(&rv)));
          else v = 1.0;
          val[p] = v;
        }
      }
      if (c->times && times) {
        int64_t n = b - a;
        if (n > tcap) {
          free(tbuf);
          tcap = n;
          tbuf = (double*)malloc(sizeof(double) * (size_t)n);
        }
        rng_t rt = rng_make(c->seed, ST_TIME, (uint64_t)k);
        double span = 36.5 * (double)n;
        for (int64_t i = 0; i < n; ++i) tbuf[i] = rng_u01(&rt) * span;
        qsort(tbuf, (size_t)n, sizeof(double), cmp_f64);
        for (int64_t i = 1; i < n; ++i)
          if (!(tbuf[i] > tbuf[i - 1])) tbuf[i] = nextafter(tbuf[i - 1], INFINITY);
        memcpy(times + a, tbuf, sizeof(double) * (size_t)n);
      }
    }
    free(seen);
    free(tbuf);
  }
  free(cdf);
}

/* Dense uniform [0,1) block for initial factors: out[i] = U(seed, stream, first + i). */
void gen_uniform(uint64_t seed, uint64_t stream, int64_t first, int64_t n, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    rng_t r = rng_make(seed, 100 + stream, (uint64_t)(first + i));
    out[i] = rng_u01(&r);
  }
}
