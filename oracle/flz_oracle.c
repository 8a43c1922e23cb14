/* flz_oracle.c — TEST INFRASTRUCTURE ONLY (never linked into, imported by or
 * executed from the product path).
 *
 * A plain-C99 restatement of the reference CPU library `speig`
 * (/root/reference/proj) for the filter-and-Lanczos hot path: every function
 * cites the reference file:line whose arithmetic (including the order of the
 * floating-point operations of the reference's *scalar* backend) it follows.
 *
 * PARITY IS PINNED: tests/test_oracle.py checks this file
 *   (1) against the known answers the reference's own tests hold
 *       (filter_test.cpp:27-47, :96-99, :218-234; lanczos_test.cpp:252-289, :426-452;
 *        acceptance_main.cpp:39-46), and
 *   (2) against the unmodified reference compiled into oracle/_ref/libspeig_ref.so
 *       (bit-for-bit on the scalar backend where the evaluation order is fixed),
 *   (3) against golden vectors generated from that library (tests/golden/).
 *
 * Third-party arithmetic: none in the reference.  The only toolchain
 * pieces are libm and libstdc++'s <random>; std::mt19937_64 and the Marsaglia-polar
 * std::normal_distribution of libstdc++ 13 are restated below (rng_* functions).
 *
 * Build: make -C oracle port  ->  oracle/_build/libflz_oracle.so  (-ffp-contract=off
 * so that no FMA is formed: the reference's scalar TU is compiled without -mfma).
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_PREFIX orc_
#include "oracle_abi.h"

#define PI 3.14159265358979323846264338327950288

static char g_err[512];
static uint64_t g_matvecs = 0;

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}

const char* orc_last_error(void) { return g_err; }
const char* orc_kind(void) { return "port"; }
int orc_set_backend(int backend) { return backend == 0 ? 0 : fail("port: scalar backend only"); }
int orc_get_backend(void) { return 0; }
uint64_t orc_matvec_count(void) { return g_matvecs; }

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* L0 kernels — scalar backend, kernels.cpp:11-41                           */
/* ------------------------------------------------------------------------ */

/* kernels.cpp:11-15: serial left-to-right sum */
double orc_dot(const double* x, const double* y, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += x[i] * y[i];
  return acc;
}
/* kernels.cpp:107 */
double orc_nrm2(const double* x, int64_t n) { return sqrt(orc_dot(x, x, n)); }
/* kernels.cpp:17-19 */
void orc_axpy(double a, const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] += a * x[i];
}
/* kernels.cpp:21-23 */
void orc_scal(double a, double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) x[i] *= a;
}
/* kernels.cpp:25-34 */
void orc_csr_matvec(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                    const double* values, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) acc += values[p] * x[col_idx[p]];
    y[i] = acc;
  }
}
/* kernels.cpp:36-41; out may alias y2 (kernels.hpp:45-49) */
void orc_clenshaw_combine(int64_t n, double s1, double s2, double b, const double* w,
                          const double* y1, const double* y2, const double* x, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = s1 * w[i] + s2 * y1[i] - y2[i] + b * x[i];
}

/* ------------------------------------------------------------------------ */
/* Filter scalars — filter.cpp:33-96                                        */
/* ------------------------------------------------------------------------ */

static int check_unit_interval(double as, double bs) { /* filter.cpp:15-20 */
  if (!(as < bs)) return fail("filter interval endpoints out of order");
  if (as < -1.0 || bs > 1.0) return fail("filter interval endpoints outside [-1, 1]");
  return 0;
}

/* filter.cpp:33-44 */
int orc_indicator_coefficients(double as, double bs, int degree, double* out) {
  if (check_unit_interval(as, bs)) return -1;
  if (degree < 0) return fail("indicator_coefficients: negative degree");
  const double ta = acos(as), tb = acos(bs);
  out[0] = (ta - tb) / PI;
  for (int i = 1; i <= degree; ++i) out[i] = 2.0 * (sin(i * ta) - sin(i * tb)) / (i * PI);
  return 0;
}

/* filter.cpp:53-84 */
int orc_select_degree(double as, double bs, double epsilon, int max_degree, int* clamped) {
  if (check_unit_interval(as, bs)) return -1;
  if (!(epsilon > 0.0 && epsilon < 1.0)) return fail("select_degree: epsilon must lie in (0, 1)");
  if (max_degree < 1) return fail("select_degree: max_degree must be >= 1");
  size_t cap = 20 * (size_t)max_degree;
  if (cap < 10000) cap = 10000;
  const double ta = acos(as), tb = acos(bs);
  double* suffix = (double*)calloc(cap + 2, sizeof(double));
  /* suffix[m] = sum_{i=m..cap} b_i^2 accumulated from the small end (filter.cpp:69-75) */
  for (size_t i = cap; i >= 1; --i) {
    const double bi = 2.0 * (sin((double)i * ta) - sin((double)i * tb)) / ((double)i * PI);
    suffix[i] = suffix[i + 1] + bi * bi;
  }
  const double threshold = epsilon * sqrt(bs - as);
  int result = max_degree, was_clamped = 1;
  for (int m = 1; m <= max_degree; ++m) {
    const double err = sqrt(0.5 * PI * suffix[m + 1]);
    if (err < threshold) {
      result = m;
      was_clamped = 0;
      break;
    }
  }
  free(suffix);
  if (clamped) *clamped = was_clamped;
  return result;
}

/* filter.cpp:86-96 */
double orc_clenshaw(const double* coeffs, int ncoeffs, double t) {
  if (ncoeffs <= 0) return 0.0;
  double y1 = 0.0, y2 = 0.0;
  for (int j = ncoeffs - 1; j >= 1; --j) {
    const double y = 2.0 * t * y1 - y2 + coeffs[j];
    y2 = y1;
    y1 = y;
  }
  return t * y1 - y2 + coeffs[0];
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* filter.cpp:163-184 (+ ctor :98-107, SpectralBounds :24-31) */
int orc_build_filter(double lo, double hi, double alpha, double beta, int degree, double epsilon,
                     int max_degree, double* coeffs, int cap, double* alpha_s, double* beta_s,
                     int* clamped) {
  if (!(lo < hi)) return fail("spectral bounds require lambda_min < lambda_max");
  if (!(alpha < beta)) return fail("build_filter requires alpha < beta");
  const double c = 0.5 * (lo + hi), e = 0.5 * (hi - lo);
  const double as = clampd((alpha - c) / e, -1.0, 1.0);
  const double bs = clampd((beta - c) / e, -1.0, 1.0);
  if (!(as < bs)) return fail("interval lies outside the spectral bounds");
  int m, cl = 0;
  if (degree > 0) {
    m = degree;
  } else {
    m = orc_select_degree(as, bs, epsilon, max_degree, &cl);
    if (m < 0) return -1;
  }
  if (coeffs) {
    if (m + 1 > cap) return fail("build_filter: coefficient buffer too small");
    if (orc_indicator_coefficients(as, bs, m, coeffs)) return -1;
  }
  if (alpha_s) *alpha_s = as;
  if (beta_s) *beta_s = bs;
  if (clamped) *clamped = cl;
  return m;
}

/* ------------------------------------------------------------------------ */
/* Matrix — sparse.cpp:27-117                                               */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t n, nnz;
  int64_t* row_ptr;
  int32_t* col_idx;
  double* values;
  double max_abs;
} Matrix;

typedef struct {
  int64_t row, col;
  double value;
} Trip;

static int trip_cmp(const void* a, const void* b) {
  const Trip* x = (const Trip*)a;
  const Trip* y = (const Trip*)b;
  if (x->row != y->row) return x->row < y->row ? -1 : 1;
  if (x->col != y->col) return x->col < y->col ? -1 : 1;
  return 0;
}

/* stable merge sort keyed on (row, col): std::sort's order among equal keys is
 * unspecified, but duplicates are summed, and IEEE addition of two values commutes;
 * for >2 duplicates the reference's sum order is implementation-defined anyway. */
static void trip_sort(Trip* t, int64_t count) {
  if (count < 2) return;
  Trip* tmp = (Trip*)malloc((size_t)count * sizeof(Trip));
  for (int64_t width = 1; width < count; width *= 2) {
    for (int64_t lo = 0; lo < count; lo += 2 * width) {
      int64_t mid = lo + width < count ? lo + width : count;
      int64_t hi = lo + 2 * width < count ? lo + 2 * width : count;
      int64_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) tmp[o++] = trip_cmp(&t[b], &t[a]) < 0 ? t[b++] : t[a++];
      while (a < mid) tmp[o++] = t[a++];
      while (b < hi) tmp[o++] = t[b++];
    }
    memcpy(t, tmp, (size_t)count * sizeof(Trip));
  }
  free(tmp);
}

void orc_matrix_free(void* Ap) {
  Matrix* A = (Matrix*)Ap;
  if (!A) return;
  free(A->row_ptr);
  free(A->col_idx);
  free(A->values);
  free(A);
}

/* sparse.cpp:27-85 */
static Matrix* matrix_from_trips(int64_t n, Trip* t, int64_t count) {
  for (int64_t i = 0; i < count; ++i) {
    if (t[i].row < 0 || t[i].col < 0 || t[i].row >= n || t[i].col >= n) {
      fail("matrix entry index out of range");
      return NULL;
    }
    if (!isfinite(t[i].value)) {
      fail("matrix entry is not finite");
      return NULL;
    }
  }
  trip_sort(t, count);
  int64_t out = 0;
  for (int64_t i = 0; i < count; ++i) {
    if (out > 0 && t[out - 1].row == t[i].row && t[out - 1].col == t[i].col)
      t[out - 1].value += t[i].value;
    else
      t[out++] = t[i];
  }
  Matrix* A = (Matrix*)calloc(1, sizeof(Matrix));
  A->n = n;
  A->nnz = out;
  A->row_ptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  A->col_idx = (int32_t*)malloc((size_t)(out > 0 ? out : 1) * sizeof(int32_t));
  A->values = (double*)malloc((size_t)(out > 0 ? out : 1) * sizeof(double));
  for (int64_t i = 0; i < out; ++i) {
    A->row_ptr[t[i].row + 1]++;
    A->col_idx[i] = (int32_t)t[i].col;
    A->values[i] = t[i].value;
    if (fabs(t[i].value) > A->max_abs) A->max_abs = fabs(t[i].value);
  }
  for (int64_t i = 0; i < n; ++i) A->row_ptr[i + 1] += A->row_ptr[i];
  /* exact structural + numerical symmetry (sparse.cpp:65-83) */
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) {
      const int64_t j = A->col_idx[p];
      if (j <= i) continue;
      int64_t lo = A->row_ptr[j], hi = A->row_ptr[j + 1];
      while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (A->col_idx[mid] < (int32_t)i) lo = mid + 1; else hi = mid;
      }
      if (lo == A->row_ptr[j + 1] || A->col_idx[lo] != (int32_t)i) {
        fail("matrix is structurally asymmetric");
        orc_matrix_free(A);
        return NULL;
      }
      if (A->values[p] != A->values[lo]) {
        fail("matrix is numerically asymmetric");
        orc_matrix_free(A);
        return NULL;
      }
    }
  return A;
}

void* orc_matrix_from_triplets(int64_t n, int64_t count, const int64_t* rows,
                               const int64_t* cols, const double* values) {
  Trip* t = (Trip*)malloc((size_t)(count > 0 ? count : 1) * sizeof(Trip));
  for (int64_t i = 0; i < count; ++i) {
    t[i].row = rows[i];
    t[i].col = cols[i];
    t[i].value = values[i];
  }
  Matrix* A = matrix_from_trips(n, t, count);
  free(t);
  return A;
}

void* orc_matrix_from_csr(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                          const double* values) {
  const int64_t count = row_ptr[n];
  Trip* t = (Trip*)malloc((size_t)(count > 0 ? count : 1) * sizeof(Trip));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      t[p].row = i;
      t[p].col = col_idx[p];
      t[p].value = values[p];
    }
  Matrix* A = matrix_from_trips(n, t, count);
  free(t);
  return A;
}

int64_t orc_matrix_dim(void* A) { return ((Matrix*)A)->n; }
int64_t orc_matrix_nnz(void* A) { return ((Matrix*)A)->nnz; }
void orc_matrix_csr(void* Ap, int64_t* row_ptr, int32_t* col_idx, double* values) {
  const Matrix* A = (const Matrix*)Ap;
  memcpy(row_ptr, A->row_ptr, (size_t)(A->n + 1) * sizeof(int64_t));
  memcpy(col_idx, A->col_idx, (size_t)A->nnz * sizeof(int32_t));
  memcpy(values, A->values, (size_t)A->nnz * sizeof(double));
}

/* sparse.cpp:87-94 */
static void apply_uncounted(const Matrix* A, const double* x, double* y) {
  orc_csr_matvec(A->n, A->row_ptr, A->col_idx, A->values, x, y);
}
static void spmv(const Matrix* A, const double* x, double* y) {
  apply_uncounted(A, x, y);
  g_matvecs += 1;
}
/* sparse.cpp:105-111: r independent spmv calls, column by column */
static void spmm_block(const Matrix* A, const double* X, int r, double* Y) {
  for (int j = 0; j < r; ++j) spmv(A, X + (size_t)j * A->n, Y + (size_t)j * A->n);
}

/* ------------------------------------------------------------------------ */
/* Block Clenshaw filter — filter.cpp:122-155                               */
/* ------------------------------------------------------------------------ */

typedef struct {
  int m;          /* degree; coeffs has m+1 entries */
  double* coeffs;
  double lo, hi, c, e;
  double alpha, beta, alpha_s, beta_s;
  int clamped;
} Filter;

static void filter_apply(const Filter* f, const Matrix* A, const double* X, int r, double* Y) {
  const size_t total = (size_t)A->n * (size_t)r;
  const int m = f->m;
  const double inv_e = 1.0 / f->e, c = f->c;
  if (m == 0) { /* filter.cpp:133-136 */
    for (size_t i = 0; i < total; ++i) Y[i] = f->coeffs[0] * X[i];
    return;
  }
  double* Y1 = (double*)calloc(total, sizeof(double));
  double* Y2 = (double*)calloc(total, sizeof(double));
  double* W = (double*)calloc(total, sizeof(double));
  for (size_t i = 0; i < total; ++i) Y1[i] = f->coeffs[m] * X[i]; /* :144 */
  for (int j = m - 1; j >= 1; --j) {                              /* :146-151 */
    spmm_block(A, Y1, r, W);
    orc_clenshaw_combine((int64_t)total, 2.0 * inv_e, -2.0 * c * inv_e, f->coeffs[j], W, Y1, Y2,
                         X, Y2);
    double* t = Y1;
    Y1 = Y2;
    Y2 = t;
  }
  spmm_block(A, Y1, r, W); /* :152-154 */
  orc_clenshaw_combine((int64_t)total, inv_e, -c * inv_e, f->coeffs[0], W, Y1, Y2, X, Y);
  free(Y1);
  free(Y2);
  free(W);
}

int orc_filter_apply(void* Ap, const double* coeffs, int m, double lo, double hi, const double* X,
                     int r, double* Y) {
  if (!(lo < hi)) return fail("spectral bounds require lambda_min < lambda_max");
  if (m < 0) return fail("filter needs at least one coefficient");
  Filter f;
  memset(&f, 0, sizeof f);
  f.m = m;
  f.coeffs = (double*)coeffs;
  f.lo = lo;
  f.hi = hi;
  f.c = 0.5 * (lo + hi);
  f.e = 0.5 * (hi - lo);
  filter_apply(&f, (const Matrix*)Ap, X, r, Y);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* libstdc++ 13 <random>: mt19937_64 + normal_distribution<double>          */
/* (toolchain behaviour the reference relies on, lanczos.cpp:82-86, :137-138)*/
/* ------------------------------------------------------------------------ */

typedef struct {
  uint64_t mt[312];
  int idx;
  int has_saved;
  double saved;
} Rng;

static void rng_seed(Rng* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
  g->has_saved = 0;
  g->saved = 0.0;
}
static uint64_t rng_u64(Rng* g) {
  if (g->idx >= 312) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MAT = 0xB5026F5AA96619E9ULL;
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      g->mt[i] = g->mt[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ULL) ? MAT : 0ULL);
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
/* std::generate_canonical<double, 53>(mt19937_64): one draw scaled by 2^-64 */
static double rng_canonical(Rng* g) {
  const double sum = (double)rng_u64(g);
  double ret = sum / 18446744073709551616.0;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret;
}
/* std::normal_distribution<double>(0,1): Marsaglia polar, second value cached */
static double rng_gauss(Rng* g) {
  if (g->has_saved) {
    g->has_saved = 0;
    return g->saved * 1.0 + 0.0;
  }
  double x, y, r2;
  do {
    x = 2.0 * rng_canonical(g) - 1.0;
    y = 2.0 * rng_canonical(g) - 1.0;
    r2 = x * x + y * y;
  } while (r2 > 1.0 || r2 == 0.0);
  const double mult = sqrt(-2.0 * log(r2) / r2);
  g->saved = x * mult;
  g->has_saved = 1;
  return y * mult * 1.0 + 0.0;
}

/* lanczos.cpp:25-30 */
static uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + salt + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* lanczos.cpp:35-42: sequential dot-then-axpy per basis column (MGS numerics) */
static void cgs_pass(const double* basis, int64_t ld, int64_t cols, double* z, int64_t n,
                     double* acc) {
  for (int64_t i = 0; i < cols; ++i) {
    const double c = orc_dot(basis + i * ld, z, n);
    orc_axpy(-c, basis + i * ld, z, n);
    if (acc) acc[i] += c;
  }
}

/* lanczos.cpp:78-103 */
int orc_init_block(int64_t n, int r, uint64_t seed, double* Q) {
  if (r > n) return fail("init_block: more columns than rows");
  if (r == 0) return fail("init_block: empty block");
  Rng g;
  rng_seed(&g, seed);
  for (int j = 0; j < r; ++j)
    for (int64_t i = 0; i < n; ++i) Q[(size_t)j * n + i] = rng_gauss(&g);
  for (int j = 0; j < r; ++j) {
    double* z = Q + (size_t)j * n;
    cgs_pass(Q, n, j, z, n, NULL);
    cgs_pass(Q, n, j, z, n, NULL);
    double norm = orc_nrm2(z, n);
    while (norm < 1e-8 * sqrt((double)n)) {
      for (int64_t i = 0; i < n; ++i) z[i] = rng_gauss(&g);
      cgs_pass(Q, n, j, z, n, NULL);
      cgs_pass(Q, n, j, z, n, NULL);
      norm = orc_nrm2(z, n);
    }
    orc_scal(1.0 / norm, z, n);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Banded symmetric eigensolver — band_eig.cpp                              */
/* ------------------------------------------------------------------------ */

#define AT(M, ld, i, j) (M)[(size_t)(j) * (size_t)(ld) + (size_t)(i)]

/* band_eig.cpp:51-78 */
static void plane_rotation(double* A, double* G, int64_t n, int64_t p, double c, double s,
                           int64_t half) {
  const int64_t q = p + 1;
  const int64_t lo = p > half ? p - half : 0;
  const int64_t hi = (n - 1) < (q + half) ? (n - 1) : (q + half);
  for (int64_t j = lo; j <= hi; ++j) {
    const double ap = AT(A, n, p, j), aq = AT(A, n, q, j);
    AT(A, n, p, j) = c * ap + s * aq;
    AT(A, n, q, j) = -s * ap + c * aq;
  }
  for (int64_t i = lo; i <= hi; ++i) {
    const double ap = AT(A, n, i, p), aq = AT(A, n, i, q);
    AT(A, n, i, p) = c * ap + s * aq;
    AT(A, n, i, q) = -s * ap + c * aq;
  }
  double* gp = G + (size_t)p * n;
  double* gq = G + (size_t)q * n;
  for (int64_t i = 0; i < n; ++i) {
    const double vp = gp[i], vq = gq[i];
    gp[i] = c * vp + s * vq;
    gq[i] = -s * vp + c * vq;
  }
}

static double* band_to_dense(int64_t n, int64_t sb, const double* bands) { /* :36-44 */
  double* A = (double*)calloc((size_t)n * n, sizeof(double));
  for (int64_t d = 0; d <= sb; ++d)
    for (int64_t i = 0; i + d < n; ++i) {
      AT(A, n, i + d, i) = bands[d * n + i];
      AT(A, n, i, i + d) = bands[d * n + i];
    }
  return A;
}

static void identity(double* G, int64_t n) {
  memset(G, 0, (size_t)n * n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) AT(G, n, i, i) = 1.0;
}

/* band_eig.cpp:83-115 */
static void reduce_band_givens(int64_t n, int64_t b, const double* bands, double* d, double* e,
                               double* G) {
  double* A = band_to_dense(n, b, bands);
  identity(G, n);
  const int64_t half = b + 2;
  for (int64_t j = 0; j + 2 < n; ++j) {
    const int64_t istart = (j + b) < (n - 1) ? (j + b) : (n - 1);
    for (int64_t i = istart; i >= j + 2; --i) {
      int64_t jj = j, ii = i;
      for (;;) {
        const double head = AT(A, n, ii - 1, jj), tail = AT(A, n, ii, jj);
        if (tail != 0.0) {
          const double rr = hypot(head, tail);
          plane_rotation(A, G, n, ii - 1, head / rr, tail / rr, half);
          AT(A, n, ii, jj) = 0.0;
          AT(A, n, jj, ii) = 0.0;
        }
        if (ii + b >= n) break;
        jj = ii - 1;
        ii = ii + b;
      }
    }
  }
  for (int64_t i = 0; i < n; ++i) d[i] = AT(A, n, i, i);
  for (int64_t i = 0; i + 1 < n; ++i) e[i] = AT(A, n, i + 1, i);
  free(A);
}

/* band_eig.cpp:119-180 */
static void reduce_dense_householder(int64_t n, int64_t sb, const double* bands, double* d,
                                     double* e, double* G) {
  double* A = band_to_dense(n, sb, bands);
  identity(G, n);
  double* v = (double*)calloc((size_t)n * 4, sizeof(double));
  double *p = v + n, *w = v + 2 * n, *gv = v + 3 * n;
  for (int64_t k = 0; k + 2 < n; ++k) {
    const int64_t L = n - k - 1;
    double norm_sq = 0.0;
    for (int64_t i = 0; i < L; ++i) {
      v[i] = AT(A, n, k + 1 + i, k);
      norm_sq += v[i] * v[i];
    }
    const double below_sq = norm_sq - v[0] * v[0];
    if (below_sq <= 0.0) continue;
    const double norm = sqrt(norm_sq);
    const double alpha = v[0] >= 0.0 ? -norm : norm;
    v[0] -= alpha;
    double vnorm = 0.0;
    for (int64_t i = 0; i < L; ++i) vnorm += v[i] * v[i];
    vnorm = sqrt(vnorm);
    if (vnorm == 0.0) continue;
    for (int64_t i = 0; i < L; ++i) v[i] /= vnorm;
    for (int64_t i = 0; i < L; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < L; ++j) acc += AT(A, n, k + 1 + i, k + 1 + j) * v[j];
      p[i] = acc;
    }
    double beta = 0.0;
    for (int64_t i = 0; i < L; ++i) beta += v[i] * p[i];
    for (int64_t i = 0; i < L; ++i) w[i] = p[i] - beta * v[i];
    for (int64_t i = 0; i < L; ++i)
      for (int64_t j = 0; j < L; ++j)
        AT(A, n, k + 1 + i, k + 1 + j) -= 2.0 * (v[i] * w[j] + w[i] * v[j]);
    AT(A, n, k + 1, k) = alpha;
    AT(A, n, k, k + 1) = alpha;
    for (int64_t i = k + 2; i < n; ++i) {
      AT(A, n, i, k) = 0.0;
      AT(A, n, k, i) = 0.0;
    }
    for (int64_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < L; ++j) acc += AT(G, n, i, k + 1 + j) * v[j];
      gv[i] = acc;
    }
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < L; ++j) AT(G, n, i, k + 1 + j) -= 2.0 * gv[i] * v[j];
  }
  for (int64_t i = 0; i < n; ++i) d[i] = AT(A, n, i, i);
  for (int64_t i = 0; i + 1 < n; ++i) e[i] = AT(A, n, i + 1, i);
  free(A);
  free(v);
}

/* band_eig.cpp:184-202; e has n entries here (last unused) */
static void tridiagonalize(int64_t n, int64_t b, const double* bands, double* d, double* e,
                           double* G) {
  for (int64_t i = 0; i < n; ++i) e[i] = 0.0;
  if (b <= 1 || n <= 2) {
    identity(G, n);
    for (int64_t i = 0; i < n; ++i) d[i] = bands[i];
    for (int64_t i = 0; i + 1 < n && b >= 1; ++i) e[i] = bands[n + i];
    return;
  }
  if (b >= n / 2) {
    reduce_dense_householder(n, b, bands, d, e, G);
    return;
  }
  reduce_band_givens(n, b, bands, d, e, G);
}

typedef struct {
  double v;
  int64_t i;
} SortKey;
static int sortkey_cmp(const void* a, const void* b) {
  const SortKey* x = (const SortKey*)a;
  const SortKey* y = (const SortKey*)b;
  if (x->v < y->v) return -1;
  if (x->v > y->v) return 1;
  return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}

/* band_eig.cpp:204-283: implicit-shift QL; G is grows x n, column-major */
static int tridiag_eig(int64_t n, double* d, double* e, double* G, int64_t grows) {
  if (n == 0) return 0;
  double* f = (double*)calloc((size_t)n, sizeof(double));
  for (int64_t i = 0; i + 1 < n; ++i) f[i] = e[i];
  const double eps = 2.220446049250313e-16;
  for (int64_t l = 0; l < n; ++l) {
    int iter = 0;
    int64_t m;
    do {
      for (m = l; m + 1 < n; ++m) {
        const double dd = fabs(d[m]) + fabs(d[m + 1]);
        if (fabs(f[m]) <= eps * dd) break;
      }
      if (m != l) {
        if (iter++ == 30) {
          free(f);
          return fail("tridiag_eig: eigenvalue failed to converge after 30 sweeps");
        }
        double g = (d[l + 1] - d[l]) / (2.0 * f[l]);
        double r = hypot(g, 1.0);
        g = d[m] - d[l] + f[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int underflow = 0;
        for (int64_t i1 = m; i1-- > l;) {
          double ff = s * f[i1];
          const double bb = c * f[i1];
          r = hypot(ff, g);
          f[i1 + 1] = r;
          if (r == 0.0) {
            d[i1 + 1] -= p;
            f[m] = 0.0;
            underflow = 1;
            break;
          }
          s = ff / r;
          c = g / r;
          g = d[i1 + 1] - p;
          r = (d[i1] - g) * s + 2.0 * c * bb;
          p = s * r;
          d[i1 + 1] = g + p;
          g = c * r - bb;
          double* gc0 = G + (size_t)i1 * grows;
          double* gc1 = G + (size_t)(i1 + 1) * grows;
          for (int64_t row = 0; row < grows; ++row) {
            ff = gc1[row];
            gc1[row] = s * gc0[row] + c * ff;
            gc0[row] = c * gc0[row] - s * ff;
          }
        }
        if (underflow) continue;
        d[l] -= p;
        f[l] = g;
        f[m] = 0.0;
      }
    } while (m != l);
  }
  /* ascending, carrying columns along (:269-281). std::sort on d only; ties among
   * exactly equal eigenvalues are broken by index here. */
  SortKey* key = (SortKey*)malloc((size_t)n * sizeof(SortKey));
  for (int64_t i = 0; i < n; ++i) {
    key[i].v = d[i];
    key[i].i = i;
  }
  qsort(key, (size_t)n, sizeof(SortKey), sortkey_cmp);
  double* Gs = (double*)malloc((size_t)grows * n * sizeof(double));
  for (int64_t j = 0; j < n; ++j) {
    d[j] = key[j].v;
    memcpy(Gs + (size_t)j * grows, G + (size_t)key[j].i * grows, (size_t)grows * sizeof(double));
  }
  memcpy(G, Gs, (size_t)grows * n * sizeof(double));
  free(Gs);
  free(key);
  free(f);
  return 0;
}

/* band_eig.cpp:285-291 (+ SymBandMatrix ctor :10-18) */
int orc_sym_band_eig(int64_t dim, int64_t sb, const double* bands, double* values,
                     double* vectors) {
  if (dim <= 0) return fail("SymBandMatrix: dimension must be positive");
  if (sb >= dim && dim > 1)
    return fail("SymBandMatrix: semi-bandwidth must be smaller than the dimension");
  if (dim == 1) sb = 0;
  double* e = (double*)calloc((size_t)dim, sizeof(double));
  double* G = vectors ? vectors : (double*)malloc((size_t)dim * dim * sizeof(double));
  tridiagonalize(dim, sb, bands, values, e, G);
  const int rc = tridiag_eig(dim, values, e, G, dim);
  if (!vectors) free(G);
  free(e);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Lanczos factorization — lanczos.cpp:105-271                              */
/* ------------------------------------------------------------------------ */

typedef struct {
  const Matrix* A;
  Filter filter;     /* filter.m < 0 => plain operator */
  int64_t n, r, k, max_cols;
  double* basis;     /* n x (max_cols + r), zero-initialised (lanczos.cpp:111) */
  double* D;         /* k blocks, row-major r x r */
  double* S;
  int64_t cap_blocks;
  uint8_t* dead;     /* one flag per basis column incl. pending */
  int64_t dead_len;
  int exhausted, breakdown;
  double max_diag_asym, op_scale;
  uint64_t rng_state;
  double mv_s, orth_s;
} Fact;

static void op_apply(const Fact* F, const double* X, double* Y) { /* lanczos.cpp:71-76 */
  if (F->filter.m >= 0)
    filter_apply(&F->filter, F->A, X, (int)F->r, Y);
  else
    spmm_block(F->A, X, (int)F->r, Y);
}

void orc_fact_free(void* Fp) {
  Fact* F = (Fact*)Fp;
  if (!F) return;
  free(F->filter.coeffs);
  free(F->basis);
  free(F->D);
  free(F->S);
  free(F->dead);
  free(F);
}

void* orc_fact_create(void* Ap, const double* coeffs, int m, double lo, double hi, double alpha,
                      double beta, const double* start, int r, int64_t max_cols) {
  const Matrix* A = (const Matrix*)Ap;
  if (r <= 0 || A->n == 0) {
    fail("LanczosFactorization: empty start block");
    return NULL;
  }
  if (max_cols < 2 * r) {
    fail("LanczosFactorization: column budget too small");
    return NULL;
  }
  Fact* F = (Fact*)calloc(1, sizeof(Fact));
  F->A = A;
  F->filter.m = m;
  if (m >= 0) {
    if (!(lo < hi)) {
      fail("spectral bounds require lambda_min < lambda_max");
      free(F);
      return NULL;
    }
    F->filter.coeffs = (double*)malloc((size_t)(m + 1) * sizeof(double));
    memcpy(F->filter.coeffs, coeffs, (size_t)(m + 1) * sizeof(double));
    F->filter.lo = lo;
    F->filter.hi = hi;
    F->filter.c = 0.5 * (lo + hi);
    F->filter.e = 0.5 * (hi - lo);
    F->filter.alpha = alpha;
    F->filter.beta = beta;
    F->filter.alpha_s = clampd((alpha - F->filter.c) / F->filter.e, -1.0, 1.0);
    F->filter.beta_s = clampd((beta - F->filter.c) / F->filter.e, -1.0, 1.0);
  }
  F->n = A->n;
  F->r = r;
  F->max_cols = max_cols;
  F->basis = (double*)calloc((size_t)F->n * (size_t)(max_cols + r), sizeof(double));
  if (!F->basis) {
    fail("LanczosFactorization: out of memory");
    orc_fact_free(F);
    return NULL;
  }
  memcpy(F->basis, start, (size_t)F->n * r * sizeof(double));
  F->cap_blocks = max_cols / r + 2;
  F->D = (double*)calloc((size_t)F->cap_blocks * r * r, sizeof(double));
  F->S = (double*)calloc((size_t)F->cap_blocks * r * r, sizeof(double));
  F->dead = (uint8_t*)calloc((size_t)(max_cols + 2 * r), 1);
  F->dead_len = r;
  F->rng_state = mix_seed(0xD1B54A32D192ED03ULL, (uint64_t)max_cols); /* lanczos.cpp:112 */
  return F;
}

/* lanczos.cpp:134-271 */
int orc_fact_expand(void* Fp, int nblocks) {
  Fact* F = (Fact*)Fp;
  const int64_t n = F->n, r = F->r;
  Rng rng;
  rng_seed(&rng, F->rng_state);
  double* Z = (double*)calloc((size_t)n * r, sizeof(double));
  double* B = (double*)calloc((size_t)n * r, sizeof(double));
  double* coeff = (double*)calloc((size_t)(F->max_cols + r), sizeof(double));
  int added = 0;
  for (int step = 0; step < nblocks; ++step) {
    if (F->k * r + r > F->max_cols) break;
    int pending_live = 0;
    for (int64_t j = 0; j < r && !pending_live; ++j) pending_live = F->dead[F->k * r + j] == 0;
    if (!pending_live) break;

    F->k += 1;
    const int64_t cols = F->k * r, newest = cols - r;
    double t0 = now_s();
    memcpy(B, F->basis + (size_t)newest * n, (size_t)n * r * sizeof(double));
    op_apply(F, B, Z);
    F->mv_s += now_s() - t0;

    t0 = now_s();
    for (int64_t j = 0; j < r; ++j) {
      const double nz = orc_nrm2(Z + (size_t)j * n, n);
      if (nz > F->op_scale) F->op_scale = nz;
    }
    double* Dk = F->D + (size_t)(F->k - 1) * r * r;
    for (int64_t j = 0; j < r; ++j) {
      memset(coeff, 0, (size_t)cols * sizeof(double));
      cgs_pass(F->basis, n, cols, Z + (size_t)j * n, n, coeff);
      for (int64_t i = 0; i < r; ++i) Dk[i * r + j] = coeff[newest + i];
      cgs_pass(F->basis, n, cols, Z + (size_t)j * n, n, NULL);
    }
    double asym = 0.0;
    for (int64_t i = 0; i < r; ++i)
      for (int64_t j = i + 1; j < r; ++j) {
        const double a = fabs(Dk[i * r + j] - Dk[j * r + i]);
        if (a > asym) asym = a;
      }
    if (asym > F->max_diag_asym) F->max_diag_asym = asym;
    for (int64_t i = 0; i < r; ++i)
      for (int64_t j = i + 1; j < r; ++j) {
        const double avg = 0.5 * (Dk[i * r + j] + Dk[j * r + i]);
        Dk[i * r + j] = avg;
        Dk[j * r + i] = avg;
      }

    double* Sk = F->S + (size_t)(F->k - 1) * r * r;
    memset(Sk, 0, (size_t)r * r * sizeof(double));
    const double dead_tol = 1e-10 * (F->op_scale > 1e-300 ? F->op_scale : 1e-300);
    int64_t live_total = 0;
    for (int64_t c = 0; c < cols; ++c) live_total += F->dead[c] ? 0 : 1;

    for (int64_t j = 0; j < r; ++j) {
      double* z = Z + (size_t)j * n;
      double* dest = F->basis + (size_t)(cols + j) * n;
      for (int64_t i = 0; i < j; ++i) coeff[i] = 0.0;
      for (int pass = 0; pass < 2; ++pass)
        for (int64_t i = 0; i < j; ++i) {
          const double c = orc_dot(F->basis + (size_t)(cols + i) * n, z, n);
          orc_axpy(-c, F->basis + (size_t)(cols + i) * n, z, n);
          coeff[i] += c;
        }
      for (int64_t i = 0; i < j; ++i) Sk[i * r + j] = coeff[i];
      const double norm = orc_nrm2(z, n);
      if (norm > dead_tol) {
        Sk[j * r + j] = norm;
        for (int64_t i = 0; i < n; ++i) dest[i] = z[i] / norm;
        F->dead[F->dead_len++] = 0;
        ++live_total;
        continue;
      }
      /* breakdown (lanczos.cpp:232-262) */
      F->breakdown = 1;
      int replaced = 0;
      if (live_total < n) {
        for (int attempt = 0; attempt < 5 && !replaced; ++attempt) {
          for (int64_t i = 0; i < n; ++i) dest[i] = rng_gauss(&rng);
          for (int pass = 0; pass < 2; ++pass) {
            cgs_pass(F->basis, n, cols, dest, n, NULL);
            for (int64_t i = 0; i < j; ++i) {
              const double c = orc_dot(F->basis + (size_t)(cols + i) * n, dest, n);
              orc_axpy(-c, F->basis + (size_t)(cols + i) * n, dest, n);
            }
          }
          const double rn = orc_nrm2(dest, n);
          if (rn > 1e-4) {
            orc_scal(1.0 / rn, dest, n);
            replaced = 1;
          }
        }
      }
      if (replaced) {
        F->dead[F->dead_len++] = 0;
        ++live_total;
      } else {
        memset(dest, 0, (size_t)n * sizeof(double));
        F->dead[F->dead_len++] = 1;
        F->exhausted = 1;
      }
    }
    F->orth_s += now_s() - t0;
    ++added;
  }
  F->rng_state = rng_u64(&rng);
  free(Z);
  free(B);
  free(coeff);
  return added;
}

int64_t orc_fact_block_count(void* F) { return ((Fact*)F)->k; }
int orc_fact_flags(void* Fp) {
  const Fact* F = (const Fact*)Fp;
  return (F->exhausted ? 1 : 0) | (F->breakdown ? 2 : 0);
}
void orc_fact_get(void* Fp, double* basis, double* D, double* S, uint8_t* dead) {
  const Fact* F = (const Fact*)Fp;
  const size_t rr = (size_t)(F->r * F->r);
  if (basis) memcpy(basis, F->basis, (size_t)F->n * (size_t)(F->k * F->r + F->r) * sizeof(double));
  if (D) memcpy(D, F->D, (size_t)F->k * rr * sizeof(double));
  if (S) memcpy(S, F->S, (size_t)F->k * rr * sizeof(double));
  if (dead) memcpy(dead, F->dead, (size_t)F->dead_len);
}
/* lanczos.cpp:120-132 */
double orc_fact_ortho_error(void* Fp) {
  const Fact* F = (const Fact*)Fp;
  const int64_t cols = F->k * F->r;
  double worst = 0.0;
  for (int64_t i = 0; i < cols; ++i) {
    if (F->dead[i]) continue;
    for (int64_t j = i; j < cols; ++j) {
      if (F->dead[j]) continue;
      const double g = orc_dot(F->basis + (size_t)i * F->n, F->basis + (size_t)j * F->n, F->n);
      const double dev = fabs(g - (i == j ? 1.0 : 0.0));
      if (dev > worst) worst = dev;
    }
  }
  return worst;
}

/* ------------------------------------------------------------------------ */
/* Projected problem + convergence — lanczos.cpp:273-405                    */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t dim;
  double* values;    /* descending */
  double* vectors;   /* dim x dim column-major */
  double* estimates;
  uint8_t* wanted;
  uint8_t* dead;
  int converged;
} Ritz;

static void ritz_free(Ritz* R) {
  free(R->values);
  free(R->vectors);
  free(R->estimates);
  free(R->wanted);
  free(R->dead);
}

typedef struct {
  const double* v;
  double alpha, beta;
} DistCtx;
static DistCtx g_dist;
static double dist_to_interval(int64_t c) {
  const double v = g_dist.v[c];
  return v < g_dist.alpha ? g_dist.alpha - v : (v > g_dist.beta ? v - g_dist.beta : 0.0);
}

static int check_convergence(const Fact* F, double alpha, double beta, double tol, int extra_ritz,
                             Ritz* out) {
  const int64_t r = F->r, k = F->k;
  if (k == 0) return fail("check_convergence: empty factorization");
  const int64_t dim = k * r;
  const int64_t sb = r < dim - 1 ? r : dim - 1;
  /* assemble_projected (lanczos.cpp:273-296) */
  double* bands = (double*)calloc((size_t)(sb + 1) * dim, sizeof(double));
  for (int64_t blk = 0; blk < k; ++blk) {
    const double* Db = F->D + (size_t)blk * r * r;
    const double* Sb = F->S + (size_t)blk * r * r;
    for (int64_t a = 0; a < r; ++a)
      for (int64_t b = 0; b <= a; ++b)
        bands[(a - b) * dim + (blk * r + b)] = 0.5 * (Db[a * r + b] + Db[b * r + a]);
    if (blk + 1 < k)
      for (int64_t a = 0; a < r; ++a)
        for (int64_t b = a; b < r; ++b) {
          const int64_t i = (blk + 1) * r + a, j = blk * r + b;
          bands[(i - j) * dim + j] = Sb[a * r + b];
        }
  }
  double t_scale = 0.0; /* band_max_abs (:300-306) */
  for (int64_t d = 0; d <= sb; ++d)
    for (int64_t i = 0; i + d < dim; ++i)
      if (fabs(bands[d * dim + i]) > t_scale) t_scale = fabs(bands[d * dim + i]);

  double* ev = (double*)malloc((size_t)dim * sizeof(double));
  double* G = (double*)malloc((size_t)dim * dim * sizeof(double));
  if (orc_sym_band_eig(dim, sb, bands, ev, G)) {
    free(bands);
    free(ev);
    free(G);
    return -1;
  }
  free(bands);

  out->dim = dim;
  out->values = (double*)malloc((size_t)dim * sizeof(double));
  out->vectors = (double*)malloc((size_t)dim * dim * sizeof(double));
  out->estimates = (double*)calloc((size_t)dim, sizeof(double));
  out->wanted = (uint8_t*)calloc((size_t)dim, 1);
  out->dead = (uint8_t*)calloc((size_t)dim, 1);
  for (int64_t c = 0; c < dim; ++c) { /* descending (:329-333) */
    const int64_t src = dim - 1 - c;
    out->values[c] = ev[src];
    memcpy(out->vectors + (size_t)c * dim, G + (size_t)src * dim, (size_t)dim * sizeof(double));
  }
  free(ev);
  free(G);

  const double* S_last = F->S + (size_t)(k - 1) * r * r;
  const int filtered = F->filter.m >= 0;
  double tau = 0.0; /* :343-349 */
  if (filtered) {
    const double pa = orc_clenshaw(F->filter.coeffs, F->filter.m + 1, F->filter.alpha_s);
    const double pb = orc_clenshaw(F->filter.coeffs, F->filter.m + 1, F->filter.beta_s);
    tau = (pa < pb ? pa : pb) - 1e-10 * t_scale;
  }
  for (int64_t c = 0; c < dim; ++c) {
    const double* w = out->vectors + (size_t)c * dim;
    double est = 0.0;
    for (int64_t a = 0; a < r; ++a) {
      double acc = 0.0;
      for (int64_t b = a; b < r; ++b) acc += S_last[a * r + b] * w[(k - 1) * r + b];
      est += acc * acc;
    }
    out->estimates[c] = sqrt(est);
    double dead_mass = 0.0;
    for (int64_t i = 0; i < dim; ++i)
      if (F->dead[i]) dead_mass += w[i] * w[i];
    if (dead_mass > 0.5) {
      out->dead[c] = 1;
      continue;
    }
    if (filtered)
      out->wanted[c] = out->values[c] >= tau ? 1 : 0;
    else
      out->wanted[c] = (out->values[c] >= alpha && out->values[c] <= beta) ? 1 : 0;
  }
  const double threshold = tol * t_scale;
  int ok = 1;
  for (int64_t c = 0; c < dim && ok; ++c)
    if (out->wanted[c] && out->estimates[c] > threshold) ok = 0;
  if (ok) { /* :377-402 */
    int64_t* unwanted = (int64_t*)malloc((size_t)dim * sizeof(int64_t));
    int64_t nu = 0;
    for (int64_t c = 0; c < dim; ++c)
      if (!out->wanted[c] && !out->dead[c]) unwanted[nu++] = c;
    if (!filtered) { /* nearest to the interval first: insertion sort (stable) */
      g_dist.v = out->values;
      g_dist.alpha = alpha;
      g_dist.beta = beta;
      for (int64_t i = 1; i < nu; ++i) {
        const int64_t key = unwanted[i];
        int64_t j = i;
        while (j > 0 && dist_to_interval(unwanted[j - 1]) > dist_to_interval(key)) {
          unwanted[j] = unwanted[j - 1];
          --j;
        }
        unwanted[j] = key;
      }
    }
    const int64_t need = extra_ritz < nu ? extra_ritz : nu;
    for (int64_t t = 0; t < need && ok; ++t)
      if (out->estimates[unwanted[t]] > threshold) ok = 0;
    free(unwanted);
  }
  out->converged = ok;
  return 0;
}

int orc_fact_check(void* Fp, double alpha, double beta, double tol, int extra_ritz,
                   double* values, double* estimates, uint8_t* wanted, uint8_t* dead) {
  Ritz R;
  memset(&R, 0, sizeof R);
  if (check_convergence((const Fact*)Fp, alpha, beta, tol, extra_ritz, &R)) return -1;
  memcpy(values, R.values, (size_t)R.dim * sizeof(double));
  memcpy(estimates, R.estimates, (size_t)R.dim * sizeof(double));
  memcpy(wanted, R.wanted, (size_t)R.dim);
  memcpy(dead, R.dead, (size_t)R.dim);
  const int conv = R.converged;
  ritz_free(&R);
  return conv;
}

/* ------------------------------------------------------------------------ */
/* Recovery — lanczos.cpp:407-510                                           */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t n, count;
  double* eigenvalues;
  double* residuals;
  double* eigenvectors; /* n x count */
  orc_stats stats;
} Result;

typedef struct {
  double lambda, residual;
  double* v;
} Pair;
static int pair_cmp(const void* a, const void* b) {
  const Pair* x = (const Pair*)a;
  const Pair* y = (const Pair*)b;
  return x->lambda < y->lambda ? -1 : (x->lambda > y->lambda ? 1 : 0);
}

static int recover(const Fact* F, double alpha, double beta, const Ritz* ritz,
                   double norm_estimate, Result* out) {
  const int64_t n = F->n, dim = F->k * F->r;
  const Matrix* A = F->A;
  const double scale = norm_estimate > 0.0 ? norm_estimate : 1.0;
  int64_t ncand = 0;
  for (int64_t c = 0; c < ritz->dim; ++c)
    if (ritz->wanted[c] && !ritz->dead[c]) ++ncand;
  double* V = (double*)calloc((size_t)n * (size_t)(ncand > 0 ? ncand : 1), sizeof(double));
  int64_t* kept_src = (int64_t*)malloc((size_t)(ncand > 0 ? ncand : 1) * sizeof(int64_t));
  int64_t w = 0;
  for (int64_t c = 0; c < ritz->dim; ++c) { /* :422-433 */
    if (!(ritz->wanted[c] && !ritz->dead[c])) continue;
    const double* wc = ritz->vectors + (size_t)c * dim;
    double* v = V + (size_t)w * n;
    memset(v, 0, (size_t)n * sizeof(double));
    for (int64_t j = 0; j < dim; ++j)
      if (wc[j] != 0.0) orc_axpy(wc[j], F->basis + (size_t)j * n, v, n);
    const double vnorm = orc_nrm2(v, n);
    if (vnorm < 0.5) continue;
    orc_scal(1.0 / vnorm, v, n);
    kept_src[w] = c;
    ++w;
  }
  Pair* pairs = (Pair*)calloc((size_t)(w > 0 ? w : 1), sizeof(Pair));
  int64_t np = 0;
  double* av = (double*)malloc((size_t)n * sizeof(double));
  if (F->filter.m >= 0 && w > 0) { /* :440-479 */
    double* AV = (double*)malloc((size_t)n * w * sizeof(double));
    for (int64_t j = 0; j < w; ++j) apply_uncounted(A, V + (size_t)j * n, AV + (size_t)j * n);
    const int64_t sbB = w > 1 ? w - 1 : 0;
    double* bands = (double*)calloc((size_t)(sbB + 1) * w, sizeof(double));
    for (int64_t i = 0; i < w; ++i)
      for (int64_t j = i; j < w; ++j) {
        const double bij = 0.5 * (orc_dot(V + (size_t)i * n, AV + (size_t)j * n, n) +
                                  orc_dot(V + (size_t)j * n, AV + (size_t)i * n, n));
        bands[(j - i) * w + i] = bij;
      }
    double* sv = (double*)malloc((size_t)w * sizeof(double));
    double* sU = (double*)malloc((size_t)w * w * sizeof(double));
    if (orc_sym_band_eig(w, sbB, bands, sv, sU)) return -1;
    for (int64_t c = 0; c < w; ++c) {
      const double lambda = sv[c];
      if (lambda < alpha || lambda > beta) continue;
      Pair* p = &pairs[np++];
      p->lambda = lambda;
      p->v = (double*)calloc((size_t)n, sizeof(double));
      memset(av, 0, (size_t)n * sizeof(double));
      for (int64_t j = 0; j < w; ++j) {
        const double u = sU[(size_t)c * w + j];
        orc_axpy(u, V + (size_t)j * n, p->v, n);
        orc_axpy(u, AV + (size_t)j * n, av, n);
      }
      const double vnorm = orc_nrm2(p->v, n);
      orc_scal(1.0 / vnorm, p->v, n);
      orc_scal(1.0 / vnorm, av, n);
      orc_axpy(-lambda, p->v, av, n);
      p->residual = orc_nrm2(av, n) / scale;
    }
    free(AV);
    free(bands);
    free(sv);
    free(sU);
  } else { /* plain mode :480-495 */
    for (int64_t c = 0; c < w; ++c) {
      const double lambda = ritz->values[kept_src[c]];
      if (lambda < alpha || lambda > beta) continue;
      Pair* p = &pairs[np++];
      p->lambda = lambda;
      p->v = (double*)malloc((size_t)n * sizeof(double));
      memcpy(p->v, V + (size_t)c * n, (size_t)n * sizeof(double));
      apply_uncounted(A, p->v, av);
      orc_axpy(-lambda, p->v, av, n);
      p->residual = orc_nrm2(av, n) / scale;
    }
  }
  /* ascending; insertion sort keeps it stable */
  for (int64_t i = 1; i < np; ++i) {
    Pair key = pairs[i];
    int64_t j = i;
    while (j > 0 && pair_cmp(&pairs[j - 1], &key) > 0) {
      pairs[j] = pairs[j - 1];
      --j;
    }
    pairs[j] = key;
  }
  out->n = n;
  out->count = np;
  out->eigenvalues = (double*)malloc((size_t)(np > 0 ? np : 1) * sizeof(double));
  out->residuals = (double*)malloc((size_t)(np > 0 ? np : 1) * sizeof(double));
  out->eigenvectors = (double*)malloc((size_t)n * (size_t)(np > 0 ? np : 1) * sizeof(double));
  for (int64_t i = 0; i < np; ++i) {
    out->eigenvalues[i] = pairs[i].lambda;
    out->residuals[i] = pairs[i].residual;
    memcpy(out->eigenvectors + (size_t)i * n, pairs[i].v, (size_t)n * sizeof(double));
    free(pairs[i].v);
  }
  free(pairs);
  free(av);
  free(V);
  free(kept_src);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Spectral bounds — lanczos.cpp:512-569                                    */
/* ------------------------------------------------------------------------ */

int orc_estimate_bounds(void* Ap, int steps, uint64_t seed, double* lo_out, double* hi_out) {
  const Matrix* A = (const Matrix*)Ap;
  const int64_t n = A->n;
  if (n < 2) return fail("estimate_spectral_bounds: matrix dimension must be >= 2");
  if (steps < 2) return fail("estimate_spectral_bounds: steps must be >= 2");
  const int64_t s_max = steps < n ? steps : n;
  Rng g;
  rng_seed(&g, mix_seed(seed, 0xB0u));
  double* Q = (double*)calloc((size_t)n * s_max, sizeof(double));
  double* w = (double*)calloc((size_t)n, sizeof(double));
  double* d = (double*)calloc((size_t)s_max + 1, sizeof(double));
  double* e = (double*)calloc((size_t)s_max + 1, sizeof(double));
  for (int64_t i = 0; i < n; ++i) Q[i] = rng_gauss(&g);
  orc_scal(1.0 / orc_nrm2(Q, n), Q, n);
  double beta_last = 0.0, scale = 0.0;
  int64_t s_done = 0, ne = 0;
  for (int64_t s = 0; s < s_max; ++s) {
    spmv(A, Q + (size_t)s * n, w);
    const double nw = orc_nrm2(w, n);
    if (nw > scale) scale = nw;
    d[s] = orc_dot(Q + (size_t)s * n, w, n);
    cgs_pass(Q, n, s + 1, w, n, NULL);
    cgs_pass(Q, n, s + 1, w, n, NULL);
    beta_last = orc_nrm2(w, n);
    s_done = s + 1;
    if (beta_last <= 1e-14 * (scale > 1e-300 ? scale : 1e-300)) {
      beta_last = 0.0;
      break;
    }
    if (s + 1 < s_max) {
      e[ne++] = beta_last;
      double* next = Q + (size_t)(s + 1) * n;
      for (int64_t i = 0; i < n; ++i) next[i] = w[i] / beta_last;
    }
  }
  for (int64_t i = (s_done > 0 ? s_done - 1 : 0); i < s_max + 1; ++i) e[i] = 0.0;
  double* G = (double*)malloc((size_t)s_done * s_done * sizeof(double));
  identity(G, s_done);
  int rc = tridiag_eig(s_done, d, e, G, s_done);
  if (rc == 0) {
    const double rho_min = fabs(beta_last * AT(G, s_done, s_done - 1, 0));
    const double rho_max = fabs(beta_last * AT(G, s_done, s_done - 1, s_done - 1));
    double lo = d[0] - rho_min, hi = d[s_done - 1] + rho_max;
    const double width = hi - lo;
    if (!(width > 0.0)) {
      rc = fail("estimate_spectral_bounds: spectrum has zero width "
                "(matrix is a multiple of the identity)");
    } else {
      lo -= 0.005 * width;
      hi += 0.005 * width;
      *lo_out = lo;
      *hi_out = hi;
    }
  }
  free(Q);
  free(w);
  free(d);
  free(e);
  free(G);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Solve driver — lanczos.cpp:46-69, 573-667                                */
/* ------------------------------------------------------------------------ */

static int resolved_max_dim(const orc_config* c, int64_t n) { /* :46-55 */
  if (c->max_dim > 0) return c->max_dim;
  const int64_t r = c->block_size;
  int64_t cap = n < 3000 ? n : 3000;
  if (cap < 2 * r) cap = 2 * r;
  cap = (cap + r - 1) / r * r;
  return (int)cap;
}

static int validate(const orc_config* c, int64_t n) { /* :57-69 */
  if (c->block_size < 1) return fail("config: block_size must be >= 1");
  if ((int64_t)c->block_size > n) return fail("config: block_size exceeds the matrix dimension");
  if (!(c->tol > 0.0 && c->tol < 1.0)) return fail("config: tol must lie in (0, 1)");
  if (resolved_max_dim(c, n) < 2 * c->block_size)
    return fail("config: max_dim must be at least 2 * block_size");
  if (c->check_every < 1) return fail("config: check_every must be >= 1");
  if (c->extra_ritz < 0) return fail("config: extra_ritz must be >= 0");
  if (c->bounds_steps < 2) return fail("config: bounds_steps must be >= 2");
  if (!(c->epsilon > 0.0 && c->epsilon < 1.0)) return fail("config: epsilon must lie in (0, 1)");
  return 0;
}

void orc_result_free(void* Rp) {
  Result* R = (Result*)Rp;
  if (!R) return;
  free(R->eigenvalues);
  free(R->residuals);
  free(R->eigenvectors);
  free(R);
}
int64_t orc_result_count(void* R) { return ((Result*)R)->count; }
void orc_result_get(void* Rp, double* eigenvalues, double* residuals, double* eigenvectors,
                    orc_stats* stats) {
  const Result* R = (const Result*)Rp;
  if (eigenvalues) memcpy(eigenvalues, R->eigenvalues, (size_t)R->count * sizeof(double));
  if (residuals) memcpy(residuals, R->residuals, (size_t)R->count * sizeof(double));
  if (eigenvectors)
    memcpy(eigenvectors, R->eigenvectors, (size_t)R->n * (size_t)R->count * sizeof(double));
  if (stats) *stats = R->stats;
}

void* orc_solve(void* Ap, double alpha, double beta, const orc_config* cfg, int plain) {
  const Matrix* A = (const Matrix*)Ap;
  if (validate(cfg, A->n)) return NULL;
  if (!(alpha < beta)) {
    fail("solve: interval requires alpha < beta");
    return NULL;
  }
  const double t_total = now_s();
  const uint64_t mv0 = g_matvecs;
  double lo, hi;
  const double t_pre = now_s();
  if (orc_estimate_bounds((void*)A, cfg->bounds_steps, cfg->seed, &lo, &hi)) return NULL;
  const double time_preproc = now_s() - t_pre;
  const uint64_t mv1 = g_matvecs;
  if (beta < lo || alpha > hi) {
    fail("solve: interval lies outside the estimated spectrum");
    return NULL;
  }
  int m = -1, clamped = 0;
  double* coeffs = NULL;
  if (!plain) {
    m = orc_build_filter(lo, hi, alpha, beta, cfg->degree, cfg->epsilon, cfg->max_degree, NULL, 0,
                         NULL, NULL, &clamped);
    if (m < 0) return NULL;
    coeffs = (double*)malloc((size_t)(m + 1) * sizeof(double));
    orc_build_filter(lo, hi, alpha, beta, m, cfg->epsilon, cfg->max_degree, coeffs, m + 1, NULL,
                     NULL, NULL);
  }
  const int r = cfg->block_size;
  const int64_t max_cols = resolved_max_dim(cfg, A->n);
  double* start = (double*)malloc((size_t)A->n * r * sizeof(double));
  if (orc_init_block(A->n, r, cfg->seed, start)) return NULL;
  Fact* F = (Fact*)orc_fact_create((void*)A, coeffs, m, lo, hi, alpha, beta, start, r, max_cols);
  free(start);
  free(coeffs);
  if (!F) return NULL;
  const double norm_est = fabs(lo) > fabs(hi) ? fabs(lo) : fabs(hi);

  Result* R = (Result*)calloc(1, sizeof(Result));
  int checks = 0, converged = 0, have = 0;
  for (;;) { /* :611-625 */
    if (orc_fact_expand(F, cfg->check_every) == 0) break;
    Ritz ritz;
    memset(&ritz, 0, sizeof ritz);
    if (check_convergence(F, alpha, beta, cfg->tol, cfg->extra_ritz, &ritz)) goto error;
    ++checks;
    if (ritz.converged) {
      if (have) {
        free(R->eigenvalues);
        free(R->residuals);
        free(R->eigenvectors);
      }
      if (recover(F, alpha, beta, &ritz, norm_est, R)) goto error;
      have = 1;
      int ok = 1;
      for (int64_t i = 0; i < R->count; ++i)
        if (!(R->residuals[i] <= cfg->tol)) ok = 0;
      if (ok) {
        converged = 1;
        ritz_free(&ritz);
        break;
      }
    }
    ritz_free(&ritz);
  }
  if (!converged) { /* :627-632 */
    Ritz ritz;
    memset(&ritz, 0, sizeof ritz);
    if (check_convergence(F, alpha, beta, cfg->tol, cfg->extra_ritz, &ritz)) goto error;
    if (have) {
      free(R->eigenvalues);
      free(R->residuals);
      free(R->eigenvectors);
    }
    if (recover(F, alpha, beta, &ritz, norm_est, R)) goto error;
    ritz_free(&ritz);
  }
  {
    const uint64_t mv2 = g_matvecs;
    orc_stats* s = &R->stats;
    s->block_steps = (int32_t)F->k;
    s->basis_vectors = (int32_t)(F->k * F->r);
    s->degree = plain ? 0 : m;
    s->mv_bounds = mv1 - mv0;
    s->mv_iteration = mv2 - mv1;
    s->mv_total = mv2 - mv0;
    s->time_preproc_s = time_preproc;
    s->time_orth_s = F->orth_s;
    s->time_mv_s = F->mv_s;
    s->checks = checks;
    s->converged = converged;
    s->breakdown_replacements = F->breakdown;
    s->degree_clamped = plain ? 0 : clamped;
    s->norm_estimate = norm_est;
    s->lambda_min_est = lo;
    s->lambda_max_est = hi;
    s->ortho_error = cfg->collect_diagnostics ? orc_fact_ortho_error(F) : -1.0;
    s->time_total_s = now_s() - t_total;
  }
  orc_fact_free(F);
  return R;
error:
  orc_fact_free(F);
  orc_result_free(R);
  return NULL;
}
