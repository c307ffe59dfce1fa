/*
 * mpsgen.c -- seeded synthetic inputs for the five BASELINE.json configs.
 *
 * Shared by the parity tests and bench.py (it is neither the product nor the
 * oracle).  The reference measures on SuiteSparse matrices;
 * there is no network here, so these seeded generators stand in for them with
 * the shapes, sizes and value distributions BASELINE.json names.
 *
 * Determinism: every row / element draws from its own counter-seeded
 * splitmix64 stream, so output is independent of the OpenMP thread count.
 * Only IEEE +,-,*,/ and sqrt are used (own log/exp below, no libm
 * transcendental), so results are bit-identical on any x86-64 host.
 *
 * Configs:
 *   1  2D 5-point Laplacian g x g, values 4 / -1 (lower components 0)
 *   2  n rows, L_i = max(1, Poisson(lambda)), row i holds i plus L_i-1
 *      distinct uniform columns, sorted; values N(0,1)-style
 *   3  banded, half-bandwidth hb, complex (independent re / im planes)
 *   4  n rows, L_i = min(clip, max(1, Zipf(s))), uniform sorted distinct
 *      columns; values U[-1,1]-style
 *   5  3D 7-point Laplacian g^3, diagonal fl(6.001), off-diagonal -1
 * Value styles (lower component j = previous * 2^-53 * U[-1,1]):
 *   VAL_UNIFORM  hi ~ U[-1,1]
 *   VAL_NORMAL   hi ~ N(0,1)
 *   VAL_UNIFORM0 hi ~ U[-1,1], lower components 0 (CG x_true)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define API __attribute__((visibility("default")))

enum { VAL_UNIFORM = 0, VAL_NORMAL = 1, VAL_UNIFORM0 = 2 };

/* ------------------------------------------------------------ RNG ------ */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
typedef struct {
  uint64_t s;
} rng_t;
static inline rng_t rng_make(uint64_t seed, uint64_t tag, uint64_t idx) {
  rng_t r;
  r.s = mix64(mix64(seed ^ 0x6d70737061727365ull) ^ mix64(tag * 0x9e3779b97f4a7c15ull + 1) ^
              (idx * 0xd1b54a32d192ed03ull));
  return r;
}
static inline uint64_t rng_next(rng_t *r) {
  r->s += 0x9e3779b97f4a7c15ull;
  return mix64(r->s);
}
/* [0,1) on the 2^-53 grid */
static inline double u01(rng_t *r) { return (double)(rng_next(r) >> 11) * 0x1p-53; }
/* (0,1] */
static inline double u01_open0(rng_t *r) { return (double)((rng_next(r) >> 11) + 1) * 0x1p-53; }
/* [-1,1) exactly representable */
static inline double usym(rng_t *r) { return 2.0 * u01(r) - 1.0; }
static inline uint64_t uint_below(rng_t *r, uint64_t n) {
  return (uint64_t)(((__uint128_t)rng_next(r) * n) >> 64);
}

/* ------------------------------------------ deterministic log / exp --- */
static const double LN2 = 0.6931471805599453094;
/* natural log for x > 0 finite: x = m 2^e, m in [sqrt(.5), sqrt(2)) */
static double dlog(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  int e = (int)((b >> 52) & 0x7ff);
  if (e == 0) { /* subnormal: scale up */
    x *= 0x1p64;
    memcpy(&b, &x, 8);
    e = (int)((b >> 52) & 0x7ff) - 64;
  }
  e -= 1023;
  b = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &b, 8);
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  double s = (m - 1.0) / (m + 1.0), s2 = s * s, term = s, acc = 0.0;
  for (int k = 1; k <= 41; k += 2) {
    acc += term / (double)k;
    term *= s2;
  }
  return (double)e * LN2 + 2.0 * acc;
}
/* exp for moderate y (|y| < 700) */
static double dexp(double y) {
  double nf = y / LN2;
  int n = (int)(nf < 0 ? nf - 0.5 : nf + 0.5);
  double r = y - (double)n * LN2, term = 1.0, acc = 1.0;
  for (int k = 1; k <= 27; ++k) {
    term = term * r / (double)k;
    acc += term;
  }
  uint64_t b = (uint64_t)(n + 1023) << 52;
  double p;
  memcpy(&p, &b, 8);
  return acc * p;
}

/* N(0,1) via Marsaglia's polar method on the deterministic log */
static double normal(rng_t *r) {
  for (;;) {
    double u = usym(r), v = usym(r), s = u * u + v * v;
    if (s > 0.0 && s < 1.0) {
      double f = -2.0 * dlog(s) / s;
      /* sqrt is correctly rounded (IEEE) */
      return u * __builtin_sqrt(f);
    }
  }
}

static void draw_value(rng_t *r, int style, int K, double *out) {
  double hi = (style == VAL_NORMAL) ? normal(r) : usym(r);
  out[0] = hi;
  for (int j = 1; j < K; ++j)
    out[j] = (style == VAL_UNIFORM0) ? 0.0 : out[j - 1] * 0x1p-53 * usym(r);
}

/* ------------------------------------------------------ row lengths --- */
static int poisson(rng_t *r, double lambda) {
  /* Knuth's product method; exp(-lambda) from the deterministic dexp */
  double L = dexp(-lambda), p = 1.0;
  int k = 0;
  do {
    ++k;
    p *= u01_open0(r);
  } while (p > L);
  return k - 1;
}

typedef struct {
  double s;
  int64_t clip;
  double *cdf; /* cdf[k-1] = P(X <= k), k = 1..clip-1 */
} zipf_t;
static zipf_t *zipf_build(double s, int64_t clip) {
  zipf_t *z = malloc(sizeof(zipf_t));
  z->s = s;
  z->clip = clip;
  z->cdf = malloc(sizeof(double) * (size_t)clip);
  double acc = 0.0;
  for (int64_t k = 1; k < clip; ++k) {
    acc += dexp(-s * dlog((double)k));
    z->cdf[k - 1] = acc;
  }
  /* tail sum_{k>=clip} k^-s by the midpoint integral (K-1/2)^(1-s)/(s-1) */
  double tail = dexp((1.0 - s) * dlog((double)clip - 0.5)) / (s - 1.0);
  double Z = acc + tail;
  for (int64_t k = 1; k < clip; ++k) z->cdf[k - 1] /= Z;
  return z;
}
static int64_t zipf_draw(const zipf_t *z, rng_t *r) {
  double u = u01(r);
  int64_t lo = 0, hi = z->clip - 1; /* first index with cdf > u, or clip-1 */
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (z->cdf[mid] > u)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo + 1; /* lo == clip-1 means the clipped tail */
}

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* L distinct uniform columns of [0,n) that include `must` (if >= 0), sorted */
static void distinct_cols(rng_t *r, int64_t n, int64_t L, int64_t must, int64_t *out) {
  int64_t have = 0;
  if (must >= 0) out[have++] = must;
  while (have < L) {
    int64_t start = have;
    for (int64_t i = start; i < L; ++i) out[i] = (int64_t)uint_below(r, (uint64_t)n);
    qsort(out, (size_t)L, sizeof(int64_t), cmp_i64);
    int64_t w = 0;
    for (int64_t i = 0; i < L; ++i)
      if (w == 0 || out[i] != out[w - 1]) out[w++] = out[i];
    have = w;
  }
}

/* ------------------------------------------------------------ API ------ */
enum { TAG_LEN = 1, TAG_COL = 2, TAG_RE = 3, TAG_IM = 4, TAG_VEC = 5, TAG_VEC_IM = 6 };

/* Number of rows of a config instance (p1 = g for grids, else n). */
API int64_t gen_nrows(int cfg, int64_t p1) {
  if (cfg == 1) return p1 * p1;
  if (cfg == 5) return p1 * p1 * p1;
  return p1;
}

/* Fills indptr[0..n] and returns nnz.  p2: Poisson mean (cfg 2), half
 * bandwidth (cfg 3), Zipf clip (cfg 4); p3: Zipf exponent (cfg 4). */
API int64_t gen_indptr(int cfg, int64_t p1, double p2, double p3, uint64_t seed, int64_t *indptr) {
  int64_t n = gen_nrows(cfg, p1);
  zipf_t *z = (cfg == 4) ? zipf_build(p3, (int64_t)p2) : NULL;
  indptr[0] = 0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t L = 0;
    if (cfg == 1) {
      int64_t g = p1, a = i / g, b = i % g;
      L = 1 + (a > 0) + (a < g - 1) + (b > 0) + (b < g - 1);
    } else if (cfg == 5) {
      int64_t g = p1, a = i / (g * g), b = (i / g) % g, c = i % g;
      L = 1 + (a > 0) + (a < g - 1) + (b > 0) + (b < g - 1) + (c > 0) + (c < g - 1);
    } else if (cfg == 2) {
      rng_t r = rng_make(seed, TAG_LEN, (uint64_t)i);
      L = poisson(&r, p2);
      if (L < 1) L = 1;
      if (L > n) L = n;
    } else if (cfg == 3) {
      int64_t hb = (int64_t)p2, lo = i - hb < 0 ? 0 : i - hb, hi = i + hb > n - 1 ? n - 1 : i + hb;
      L = hi - lo + 1;
    } else if (cfg == 4) {
      rng_t r = rng_make(seed, TAG_LEN, (uint64_t)i);
      L = zipf_draw(z, &r);
      if (L > n) L = n;
    }
    indptr[i + 1] = L;
  }
  for (int64_t i = 0; i < n; ++i) indptr[i + 1] += indptr[i];
  if (z) {
    free(z->cdf);
    free(z);
  }
  return indptr[n];
}

/* Fills indices and K value planes.  planes: [K][nnz] (re), followed by
 * [K][nnz] (im) when cfg == 3. */
API void gen_fill(int cfg, int64_t p1, double p2, uint64_t seed, int K, const int64_t *indptr,
                  int64_t *indices, double *planes) {
  int64_t n = gen_nrows(cfg, p1);
  int64_t nnz = indptr[n];
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) {
    int64_t b = indptr[i], L = indptr[i + 1] - b;
    int64_t *col = indices + b;
    if (cfg == 1 || cfg == 5) {
      int64_t g = p1, gg = (cfg == 5) ? g * g : 0, w = 0;
      int64_t a = (cfg == 5) ? i / gg : 0;
      int64_t bb = (cfg == 5) ? (i / g) % g : i / g;
      int64_t c = i % g;
      if (cfg == 5 && a > 0) col[w++] = i - gg;
      if (bb > 0) col[w++] = i - g;
      if (c > 0) col[w++] = i - 1;
      col[w++] = i;
      if (c < g - 1) col[w++] = i + 1;
      if (bb < g - 1) col[w++] = i + g;
      if (cfg == 5 && a < g - 1) col[w++] = i + gg;
      for (int64_t k = 0; k < L; ++k) {
        double v = (col[k] == i) ? (cfg == 1 ? 4.0 : 6.001) : -1.0;
        planes[b + k] = v;
        for (int j = 1; j < K; ++j) planes[(int64_t)j * nnz + b + k] = 0.0;
      }
      continue;
    }
    if (cfg == 3) {
      int64_t hb = (int64_t)p2, lo = i - hb < 0 ? 0 : i - hb;
      for (int64_t k = 0; k < L; ++k) col[k] = lo + k;
    } else {
      rng_t r = rng_make(seed, TAG_COL, (uint64_t)i);
      distinct_cols(&r, n, L, cfg == 2 ? i : -1, col);
    }
    int style = (cfg == 4) ? VAL_UNIFORM : VAL_NORMAL;
    rng_t rr = rng_make(seed, TAG_RE, (uint64_t)i);
    rng_t ri = rng_make(seed, TAG_IM, (uint64_t)i);
    double v[4];
    for (int64_t k = 0; k < L; ++k) {
      draw_value(&rr, style, K, v);
      for (int j = 0; j < K; ++j) planes[(int64_t)j * nnz + b + k] = v[j];
      if (cfg == 3) {
        draw_value(&ri, style, K, v);
        for (int j = 0; j < K; ++j) planes[(int64_t)(K + j) * nnz + b + k] = v[j];
      }
    }
  }
}

/* Vector of n K-component values, AoS [n][K]; `imag` selects the second
 * independent stream (imaginary part of a complex vector). */
API void gen_vector(int style, int64_t n, uint64_t seed, int K, int imag, double *aos) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    rng_t r = rng_make(seed, imag ? TAG_VEC_IM : TAG_VEC, (uint64_t)i);
    draw_value(&r, style, K, aos + i * K);
  }
}
