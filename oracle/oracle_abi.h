/* oracle_abi.h — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * One C ABI, two implementations, selected by the symbol prefix ORC_PREFIX:
 *   ref_*  oracle/ref_shim.cpp   — thin wrappers around the UNMODIFIED reference
 *                                  library compiled from /root/reference/proj/src
 *                                  (built only into oracle/_ref/, never copied).
 *   orc_*  oracle/flz_oracle.c   — a plain-C restatement of the same algorithms
 *                                  (each function cites the reference file:line).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load either library.
 *
 * All dense blocks are column-major (reference DenseBlock, dense_block.hpp:11-40),
 * CSR uses int64 row_ptr / int32 col_idx / f64 values (sparse.hpp:28-33).
 */
#ifndef FLZ_ORACLE_ABI_H
#define FLZ_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef ORC_PREFIX
#error "define ORC_PREFIX (ref_ or orc_) before including oracle_abi.h"
#endif
#define ORC_CAT2(a, b) a##b
#define ORC_CAT(a, b) ORC_CAT2(a, b)
#define ORC(name) ORC_CAT(ORC_PREFIX, name)

/* Mirrors speig::LanczosConfig (lanczos.hpp:14-29). degree <= 0 means auto. */
typedef struct {
  int32_t block_size;
  double tol;
  int32_t max_dim;
  int32_t check_every;
  uint64_t seed;
  int32_t extra_ritz;
  int32_t bounds_steps;
  int32_t degree;
  double epsilon;
  int32_t max_degree;
  int32_t collect_diagnostics;
} orc_config;

/* Mirrors speig::SolveStats (lanczos.hpp:136-155). */
typedef struct {
  int32_t block_steps, basis_vectors, degree;
  uint64_t mv_iteration, mv_bounds, mv_total;
  double time_total_s, time_preproc_s, time_orth_s, time_mv_s;
  int32_t checks, converged, breakdown_replacements, degree_clamped;
  double norm_estimate, lambda_min_est, lambda_max_est, ortho_error;
} orc_stats;

const char* ORC(last_error)(void);
const char* ORC(kind)(void); /* "reference" or "port" */

/* backend: 0 scalar, 1 avx2 (kernels.hpp:15-27). The port only has scalar. */
int ORC(set_backend)(int backend);
int ORC(get_backend)(void);

/* ---- L0 kernels (kernels.hpp:29-49) ---- */
double ORC(dot)(const double* x, const double* y, int64_t n);
double ORC(nrm2)(const double* x, int64_t n);
void ORC(axpy)(double a, const double* x, double* y, int64_t n);
void ORC(scal)(double a, double* x, int64_t n);
void ORC(csr_matvec)(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                     const double* values, const double* x, double* y);
void ORC(clenshaw_combine)(int64_t n, double s1, double s2, double b, const double* w,
                           const double* y1, const double* y2, const double* x, double* out);

/* ---- filter scalars (filter.hpp:36-57) ---- */
int ORC(indicator_coefficients)(double alpha_s, double beta_s, int degree, double* out);
int ORC(select_degree)(double alpha_s, double beta_s, double epsilon, int max_degree,
                       int* clamped);
double ORC(clenshaw)(const double* coeffs, int ncoeffs, double t);

/* ---- matrix handle: SparseSymMatrix::from_entries semantics (sparse.cpp:27-85) ---- */
void* ORC(matrix_from_csr)(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                           const double* values);
void* ORC(matrix_from_triplets)(int64_t n, int64_t count, const int64_t* rows,
                                const int64_t* cols, const double* values);
void ORC(matrix_free)(void* A);
int64_t ORC(matrix_dim)(void* A);
int64_t ORC(matrix_nnz)(void* A);
void ORC(matrix_csr)(void* A, int64_t* row_ptr, int32_t* col_idx, double* values);
uint64_t ORC(matvec_count)(void);

/* Y = p((A - c I)/e) X with explicit coefficients b[0..m] (filter.cpp:122-155). */
int ORC(filter_apply)(void* A, const double* coeffs, int m, double lambda_min,
                      double lambda_max, const double* X, int r, double* Y);
/* build_filter (filter.cpp:163-184): returns degree, fills coeffs (cap entries),
 * mapped endpoints and the clamped flag; degree<=0 selects automatically. */
int ORC(build_filter)(double lambda_min, double lambda_max, double alpha, double beta,
                      int degree, double epsilon, int max_degree, double* coeffs, int cap,
                      double* alpha_s, double* beta_s, int* clamped);

/* init_block (lanczos.cpp:78-103), estimate_spectral_bounds (:512-569). */
int ORC(init_block)(int64_t n, int r, uint64_t seed, double* Q);
int ORC(estimate_bounds)(void* A, int steps, uint64_t seed, double* lo, double* hi);

/* sym_band_eig (band_eig.cpp:285-291). bands[d*dim+i] = M(i+d,i), d=0..sb.
 * values ascending, vectors column-major dim x dim. */
int ORC(sym_band_eig)(int64_t dim, int64_t sb, const double* bands, double* values,
                      double* vectors);

/* ---- factorization handle: LanczosFactorization + expand (lanczos.cpp:105-271) ---- */
/* filtered when m >= 0 (coeffs b[0..m], bounds lo/hi, interval alpha/beta), plain when m < 0 */
void* ORC(fact_create)(void* A, const double* coeffs, int m, double lambda_min,
                       double lambda_max, double alpha, double beta, const double* start,
                       int r, int64_t max_cols);
void ORC(fact_free)(void* F);
int ORC(fact_expand)(void* F, int nblocks);
int64_t ORC(fact_block_count)(void* F);
/* copies: basis n x (k*r + r) (completed + pending), D and S as k row-major r x r blocks */
void ORC(fact_get)(void* F, double* basis, double* D, double* S, uint8_t* dead);
double ORC(fact_ortho_error)(void* F);
int ORC(fact_flags)(void* F); /* bit0 exhausted, bit1 breakdown */
/* check_convergence (lanczos.cpp:310-405): fills values[dim] (descending),
 * residual_estimates[dim], wanted[dim], dead[dim]; returns converged (0/1) or <0. */
int ORC(fact_check)(void* F, double alpha, double beta, double tol, int extra_ritz,
                    double* values, double* estimates, uint8_t* wanted, uint8_t* dead);

/* ---- full solve (lanczos.cpp:573-667) ---- */
void* ORC(solve)(void* A, double alpha, double beta, const orc_config* cfg, int plain);
void ORC(result_free)(void* R);
int64_t ORC(result_count)(void* R);
void ORC(result_get)(void* R, double* eigenvalues, double* residuals, double* eigenvectors,
                     orc_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
