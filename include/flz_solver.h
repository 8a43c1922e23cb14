/* flz_solver.h — C ABI of the HOST solver layer of libflz.so (the C++ facade in
 * the include/flz/ headers, flattened for FFI callers: ctypes, cgo, JNI ...).
 *
 * include/flz.h is the device layer (kernels behind plain pointers); this header is the
 * solver the reference exposes as speig::filtered_lanczos & friends.  Each entry point
 * cites the reference interface it replaces.  Same conventions as flz.h: status codes,
 * flz_last_error(), column-major dense blocks, no exceptions across the boundary.
 */
#ifndef FLZ_SOLVER_H
#define FLZ_SOLVER_H

#include "flz.h"

#ifdef __cplusplus
extern "C" {
#endif

/* speig::LanczosConfig (lanczos.hpp:14-29); degree <= 0 selects the automatic degree. */
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
  /* extension (not in the reference): 0 = keep the eigenvectors on the device side of the
   * recovery and return only eigenvalues and residuals (large runs: n x count doubles need
   * not cross PCIe); flz_config_default sets 1 */
  int32_t return_vectors;
  /* extension: != 0 multiplies the filter coefficients by the Jackson kernel factors on the
   * host (off by default: the reference has no damping) */
  int32_t jackson_damping;
} flz_config;

/* speig::SolveStats (lanczos.hpp:136-155) + the GPU build's host buckets. */
typedef struct {
  int32_t block_steps, basis_vectors, degree;
  uint64_t mv_iteration, mv_bounds, mv_total;
  double time_total_s, time_preproc_s, time_orth_s, time_mv_s;
  int32_t checks, converged, breakdown_replacements, degree_clamped;
  double norm_estimate, lambda_min_est, lambda_max_est, ortho_error;
  double time_check_s, time_recover_s, time_upload_s;
  uint64_t gpu_launches;
} flz_stats;

typedef struct flz_hostmatrix flz_hostmatrix; /* speig::SparseSymMatrix (sparse.hpp:21-60) */
typedef struct flz_result flz_result;         /* speig::EigenResult (lanczos.hpp:157-162)  */
typedef struct flz_fact flz_fact;             /* speig::LanczosFactorization + its operator */

void flz_config_default(flz_config* cfg); /* lanczos.hpp:14-29 defaults */

/* The host layer runs on the process-wide default context; adopt a caller-made one
 * (e.g. a distributed context) with this call.  ctx == NULL restores the lazy default. */
int flz_set_default_ctx(flz_ctx* ctx);
/* TESTS ONLY: the calling THREAD's host-layer calls run on `ctx` (NULL: back to the
 * process-wide one) — the ranks of a loopback run (flz_ctx_create_loopback) are threads. */
int flz_set_thread_ctx(flz_ctx* ctx);
/* The context the host layer is using (created on first use). */
int flz_default_ctx(flz_ctx** out);

/* ---- SparseSymMatrix: from_entries (sparse.cpp:27-85), Matrix Market (:172-331) ---- */
int flz_hostmatrix_from_triplets(int64_t n, int64_t count, const int64_t* rows,
                                 const int64_t* cols, const double* values,
                                 flz_hostmatrix** out);
int flz_hostmatrix_from_csr(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                            const double* values, int check_symmetry, flz_hostmatrix** out);
/* Distributed construction: this rank's rows [row_begin,row_end) (row_ptr starts at 0, global
 * column ids); the row range must be the context's block n*rank/size .. n*(rank+1)/size. */
int flz_hostmatrix_from_local_rows(int64_t n_global, int64_t row_begin, int64_t row_end,
                                   const int64_t* row_ptr, const int32_t* col_idx,
                                   const double* values, flz_hostmatrix** out);
int flz_hostmatrix_load_mm(const char* path, flz_hostmatrix** out);
int flz_hostmatrix_save_mm(const flz_hostmatrix* A, const char* path);
/* binary CSR image (extension; csrc/host/mmio.cpp): header + row_ptr + col_idx + values.
 * flz_hostmatrix_load_mm keeps such images itself when FLZ_MM_CACHE names a directory. */
int flz_hostmatrix_save_bin(const flz_hostmatrix* A, const char* path);
int flz_hostmatrix_load_bin(const char* path, flz_hostmatrix** out);
void flz_hostmatrix_free(flz_hostmatrix* A);
int flz_hostmatrix_dims(const flz_hostmatrix* A, int64_t* n, int64_t* nnz);
/* device layout of the matrix (uploads it when it is not resident yet): bytes of the
 * index-compressed copy one fused Clenshaw step streams, true nonzeros at uniform positions */
int flz_hostmatrix_layout(const flz_hostmatrix* A, int64_t* matrix_bytes,
                          int64_t* uniform_entries);
/* flz_matrix_k1_info of the resident matrix (uploads it when needed) */
int flz_hostmatrix_k1_info(const flz_hostmatrix* A, int r, int64_t* info, char* kernel, int cap);
int flz_hostmatrix_csr(const flz_hostmatrix* A, int64_t* row_ptr, int32_t* col_idx,
                       double* values);
/* SparseSymMatrix::spmm_block / ChebyshevFilter::apply through the C++ facade */
/* X is rows x r; rows != dim(A) is rejected with FLZ_EDIM (speig::DimensionError) */
int flz_hostmatrix_spmm(const flz_hostmatrix* A, const double* X, int64_t rows, int r,
                        double* Y);
int flz_hostmatrix_filter_apply(const flz_hostmatrix* A, const double* coeffs, int m,
                                double lambda_min, double lambda_max, const double* X,
                                int64_t rows, int r, double* Y);

/* ---- filter scalars (filter.cpp:33-96, :163-184); host arithmetic ---- */
int flz_indicator_coefficients(double alpha_s, double beta_s, int degree, double* out);
/* Jackson kernel factors g_0..g_degree (extension; flz/chebyshev.hpp) */
int flz_jackson_factors(int degree, double* out);
int flz_select_degree(double alpha_s, double beta_s, double epsilon, int max_degree,
                      int* clamped); /* returns the degree, < 0 on error */
double flz_clenshaw(const double* coeffs, int ncoeffs, double t);
int flz_build_filter(double lambda_min, double lambda_max, double alpha, double beta, int degree,
                     double epsilon, int max_degree, double* coeffs, int cap, double* alpha_s,
                     double* beta_s, int* clamped); /* returns the degree, < 0 on error */

/* ---- init_block (lanczos.cpp:78-103), estimate_spectral_bounds (:512-569) ---- */
int flz_init_block(int64_t n, int r, uint64_t seed, double* Q);
int flz_estimate_bounds(const flz_hostmatrix* A, int steps, uint64_t seed, double* lo,
                        double* hi);

/* ---- projected eigenproblem (band_eig.cpp); bands[d*dim+i] = M(i+d,i) ---- */
int flz_sym_band_eig(int64_t dim, int64_t sb, const double* bands, double* values,
                     double* vectors /* dim x dim column-major or NULL */);
/* eigenvalues + selected rows of the eigenvector matrix: out_rows is nrows x dim col-major */
int flz_band_ritz_rows(int64_t dim, int64_t sb, const double* bands, int64_t nrows,
                       const int64_t* rows, double* values, double* out_rows);
/* selected eigenvectors by banded inverse iteration; vectors dim x npick column-major */
int flz_band_eigenvectors(int64_t dim, int64_t sb, const double* bands, const double* values,
                          int64_t npick, const int64_t* pick, double* vectors,
                          double* max_residual, double* max_ortho);

/* ---- LanczosFactorization + expand + check_convergence (lanczos.cpp:105-405) ---- */
/* m >= 0: filtered operator with coefficients b[0..m]; m < 0: plain A */
int flz_fact_create(const flz_hostmatrix* A, const double* coeffs, int m, double lambda_min,
                    double lambda_max, double alpha, double beta, const double* start, int r,
                    int64_t max_cols, flz_fact** out);
void flz_fact_free(flz_fact* F);
int flz_fact_expand(flz_fact* F, int nblocks); /* returns blocks added, < 0 on error */
int64_t flz_fact_block_count(const flz_fact* F);
/* basis: n x (k*r + r) incl. the pending block; D, S: k row-major r x r blocks */
int flz_fact_get(const flz_fact* F, double* basis, double* D, double* S, uint8_t* dead);
int flz_fact_ortho_error(const flz_fact* F, double* out);
int flz_fact_flags(const flz_fact* F); /* bit0 exhausted, bit1 breakdown */
/* returns converged (0/1), < 0 on error */
int flz_fact_check(const flz_fact* F, double alpha, double beta, double tol, int extra_ritz,
                   double* values, double* estimates, uint8_t* wanted, uint8_t* dead);

/* ---- filtered_lanczos / plain_lanczos (lanczos.hpp:183-186, lanczos.cpp:573-667) ---- */
int flz_solve(const flz_hostmatrix* A, double alpha, double beta, const flz_config* cfg,
              int plain, flz_result** out);
void flz_result_free(flz_result* R);
int64_t flz_result_count(const flz_result* R);
/* the result's own eigenvector storage (n x count column-major, valid until flz_result_free):
 * lets a binding wrap the vectors without a second host copy */
const double* flz_result_vectors(const flz_result* result);
int64_t flz_result_rows(const flz_result* result); /* rows of that storage (local rows) */
/* any output pointer may be NULL; eigenvectors is n x count column-major */
int flz_result_get(const flz_result* R, double* eigenvalues, double* residuals,
                   double* eigenvectors, flz_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* FLZ_SOLVER_H */
