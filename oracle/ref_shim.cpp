// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// C-ABI wrappers (prefix ref_) around the UNMODIFIED reference library `speig`,
// compiled by oracle/Makefile straight from /root/reference/proj/src into
// oracle/_ref/libspeig_ref.so.  No reference source is copied into this repo: this
// file only *calls* the reference's public API (include/speig/*.hpp).
//
// It is the pin for the plain-C restatement (oracle/flz_oracle.c) and the
// "reference" arm of bench.py / the parity tests.

#include <algorithm>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "speig/band_eig.hpp"
#include "speig/filter.hpp"
#include "speig/kernels.hpp"
#include "speig/lanczos.hpp"
#include "speig/sparse.hpp"

#define ORC_PREFIX ref_
#include "oracle_abi.h"

using namespace speig;

namespace {

thread_local std::string g_err;

struct Fact {
  const SparseSymMatrix* A = nullptr;
  std::optional<ChebyshevFilter> filter;
  std::optional<BlockOperator> op;
  std::unique_ptr<LanczosFactorization> st;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

LanczosConfig to_cfg(const orc_config& c) {
  LanczosConfig k;
  k.block_size = c.block_size;
  k.tol = c.tol;
  k.max_dim = c.max_dim;
  k.check_every = c.check_every;
  k.seed = c.seed;
  k.extra_ritz = c.extra_ritz;
  k.bounds_steps = c.bounds_steps;
  if (c.degree > 0) k.degree = c.degree;
  k.epsilon = c.epsilon;
  k.max_degree = c.max_degree;
  k.collect_diagnostics = c.collect_diagnostics != 0;
  return k;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
const char* ref_kind(void) { return "reference"; }

int ref_set_backend(int backend) {
  return guard([&] {
    kernels::set_backend(backend == 1 ? kernels::Backend::avx2 : kernels::Backend::scalar);
  });
}
int ref_get_backend(void) { return kernels::active_backend() == kernels::Backend::avx2 ? 1 : 0; }

double ref_dot(const double* x, const double* y, int64_t n) { return kernels::dot(x, y, n); }
double ref_nrm2(const double* x, int64_t n) { return kernels::nrm2(x, n); }
void ref_axpy(double a, const double* x, double* y, int64_t n) { kernels::axpy(a, x, y, n); }
void ref_scal(double a, double* x, int64_t n) { kernels::scal(a, x, n); }
void ref_csr_matvec(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                    const double* values, const double* x, double* y) {
  kernels::csr_matvec(n, row_ptr, col_idx, values, x, y);
}
void ref_clenshaw_combine(int64_t n, double s1, double s2, double b, const double* w,
                          const double* y1, const double* y2, const double* x, double* out) {
  kernels::clenshaw_combine(n, s1, s2, b, w, y1, y2, x, out);
}

int ref_indicator_coefficients(double as, double bs, int degree, double* out) {
  return guard([&] {
    const auto b = indicator_coefficients(as, bs, degree);
    std::copy(b.begin(), b.end(), out);
  });
}
int ref_select_degree(double as, double bs, double eps, int max_degree, int* clamped) {
  int m = -1;
  if (guard([&] {
        const auto sel = select_degree(as, bs, eps, max_degree);
        m = sel.degree;
        if (clamped) *clamped = sel.clamped ? 1 : 0;
      }))
    return -1;
  return m;
}
double ref_clenshaw(const double* coeffs, int ncoeffs, double t) {
  return clenshaw(std::span<const double>(coeffs, ncoeffs), t);
}

void* ref_matrix_from_triplets(int64_t n, int64_t count, const int64_t* rows,
                               const int64_t* cols, const double* values) {
  SparseSymMatrix* out = nullptr;
  if (guard([&] {
        std::vector<Triplet> t(count);
        for (int64_t i = 0; i < count; ++i) t[i] = {rows[i], cols[i], values[i]};
        out = new SparseSymMatrix(SparseSymMatrix::from_entries(n, std::move(t)));
      }))
    return nullptr;
  return out;
}
void* ref_matrix_from_csr(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                          const double* values) {
  SparseSymMatrix* out = nullptr;
  if (guard([&] {
        std::vector<Triplet> t;
        t.reserve(row_ptr[n]);
        for (int64_t i = 0; i < n; ++i)
          for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            t.push_back({i, col_idx[p], values[p]});
        out = new SparseSymMatrix(SparseSymMatrix::from_entries(n, std::move(t)));
      }))
    return nullptr;
  return out;
}
// reference-only extra (not part of oracle_abi.h): the reference's own Matrix Market loader
// (sparse.cpp:172-291), the yardstick of the product's multi-threaded loader
void* ref_matrix_load_mm(const char* path) {
  SparseSymMatrix* out = nullptr;
  if (guard([&] { out = new SparseSymMatrix(load_matrix_market(path)); })) return nullptr;
  return out;
}
void ref_matrix_free(void* A) { delete static_cast<SparseSymMatrix*>(A); }
int64_t ref_matrix_dim(void* A) { return static_cast<SparseSymMatrix*>(A)->dim(); }
int64_t ref_matrix_nnz(void* A) { return static_cast<SparseSymMatrix*>(A)->nnz(); }
void ref_matrix_csr(void* Ap, int64_t* row_ptr, int32_t* col_idx, double* values) {
  const auto* A = static_cast<SparseSymMatrix*>(Ap);
  std::copy(A->row_ptr().begin(), A->row_ptr().end(), row_ptr);
  std::copy(A->col_idx().begin(), A->col_idx().end(), col_idx);
  std::copy(A->values().begin(), A->values().end(), values);
}
uint64_t ref_matvec_count(void) { return matvec_count(); }

int ref_filter_apply(void* Ap, const double* coeffs, int m, double lo, double hi,
                     const double* X, int r, double* Y) {
  return guard([&] {
    const auto* A = static_cast<SparseSymMatrix*>(Ap);
    const SpectralBounds bounds(lo, hi);
    const auto f = ChebyshevFilter::from_coefficients(
        bounds, lo, hi, std::vector<double>(coeffs, coeffs + m + 1));
    const std::size_t n = A->dim();
    DenseBlock Xb(n, r), Yb(n, r);
    std::copy(X, X + n * r, Xb.data());
    f.apply(*A, Xb, Yb);
    std::copy(Yb.data(), Yb.data() + n * r, Y);
  });
}

int ref_build_filter(double lo, double hi, double alpha, double beta, int degree,
                     double epsilon, int max_degree, double* coeffs, int cap, double* alpha_s,
                     double* beta_s, int* clamped) {
  int m = -1;
  if (guard([&] {
        const SpectralBounds bounds(lo, hi);
        const ChebyshevFilter f =
            build_filter(bounds, alpha, beta,
                         degree > 0 ? std::optional<int>(degree) : std::nullopt, epsilon,
                         max_degree);
        m = f.degree();
        if (coeffs) {
          if (m + 1 > cap) throw Error("build_filter: coefficient buffer too small");
          std::copy(f.coefficients().begin(), f.coefficients().end(), coeffs);
        }
        if (alpha_s) *alpha_s = f.alpha_mapped();
        if (beta_s) *beta_s = f.beta_mapped();
        if (clamped) *clamped = f.degree_clamped() ? 1 : 0;
      }))
    return -1;
  return m;
}

int ref_init_block(int64_t n, int r, uint64_t seed, double* Q) {
  return guard([&] {
    const DenseBlock B = init_block(n, r, seed);
    std::copy(B.data(), B.data() + B.size(), Q);
  });
}

int ref_estimate_bounds(void* Ap, int steps, uint64_t seed, double* lo, double* hi) {
  return guard([&] {
    const SpectralBounds b =
        estimate_spectral_bounds(*static_cast<SparseSymMatrix*>(Ap), steps, seed);
    *lo = b.lambda_min();
    *hi = b.lambda_max();
  });
}

int ref_sym_band_eig(int64_t dim, int64_t sb, const double* bands, double* values,
                     double* vectors) {
  return guard([&] {
    SymBandMatrix M(dim, sb);
    for (int64_t d = 0; d <= static_cast<int64_t>(M.semi_bandwidth()); ++d)
      for (int64_t i = 0; i + d < dim; ++i) M.set(i + d, i, bands[d * dim + i]);
    const SymEig e = sym_band_eig(M);
    std::copy(e.values.begin(), e.values.end(), values);
    if (vectors) std::copy(e.vectors.data(), e.vectors.data() + dim * dim, vectors);
  });
}

void* ref_fact_create(void* Ap, const double* coeffs, int m, double lo, double hi, double alpha,
                      double beta, const double* start, int r, int64_t max_cols) {
  Fact* F = new Fact;
  if (guard([&] {
        F->A = static_cast<SparseSymMatrix*>(Ap);
        if (m >= 0) {
          F->filter = ChebyshevFilter::from_coefficients(
              SpectralBounds(lo, hi), alpha, beta, std::vector<double>(coeffs, coeffs + m + 1));
          F->op = BlockOperator::filtered(*F->A, *F->filter);
        } else {
          F->op = BlockOperator::plain(*F->A);
        }
        const std::size_t n = F->A->dim();
        DenseBlock S(n, r);
        std::copy(start, start + n * r, S.data());
        F->st = std::make_unique<LanczosFactorization>(*F->op, std::move(S), max_cols);
      })) {
    delete F;
    return nullptr;
  }
  return F;
}
void ref_fact_free(void* F) { delete static_cast<Fact*>(F); }
int ref_fact_expand(void* Fp, int nblocks) {
  int added = -1;
  if (guard([&] { added = expand(*static_cast<Fact*>(Fp)->st, nblocks, nullptr); })) return -1;
  return added;
}
int64_t ref_fact_block_count(void* Fp) { return static_cast<Fact*>(Fp)->st->block_count(); }
void ref_fact_get(void* Fp, double* basis, double* D, double* S, uint8_t* dead) {
  const auto& st = *static_cast<Fact*>(Fp)->st;
  const std::size_t n = st.n(), r = st.block_size(), k = st.block_count();
  if (basis)
    for (std::size_t j = 0; j < k * r + r; ++j)
      std::copy(st.basis_col(j), st.basis_col(j) + n, basis + j * n);
  for (std::size_t b = 0; b < k; ++b) {
    if (D) std::copy(st.diag_blocks()[b].begin(), st.diag_blocks()[b].end(), D + b * r * r);
    if (S) std::copy(st.sub_blocks()[b].begin(), st.sub_blocks()[b].end(), S + b * r * r);
  }
  if (dead) std::copy(st.dead_cols().begin(), st.dead_cols().end(), dead);
}
double ref_fact_ortho_error(void* Fp) { return static_cast<Fact*>(Fp)->st->ortho_error(); }
int ref_fact_flags(void* Fp) {
  const auto& st = *static_cast<Fact*>(Fp)->st;
  return (st.space_exhausted() ? 1 : 0) | (st.had_breakdown() ? 2 : 0);
}
int ref_fact_check(void* Fp, double alpha, double beta, double tol, int extra_ritz,
                   double* values, double* estimates, uint8_t* wanted, uint8_t* dead) {
  int conv = -1;
  if (guard([&] {
        const RitzSet rs =
            check_convergence(*static_cast<Fact*>(Fp)->st, alpha, beta, tol, extra_ritz);
        std::copy(rs.values.begin(), rs.values.end(), values);
        std::copy(rs.residual_estimates.begin(), rs.residual_estimates.end(), estimates);
        std::copy(rs.wanted.begin(), rs.wanted.end(), wanted);
        std::copy(rs.dead.begin(), rs.dead.end(), dead);
        conv = rs.converged ? 1 : 0;
      }))
    return -1;
  return conv;
}

void* ref_solve(void* Ap, double alpha, double beta, const orc_config* cfg, int plain) {
  EigenResult* R = nullptr;
  if (guard([&] {
        const auto& A = *static_cast<SparseSymMatrix*>(Ap);
        const LanczosConfig k = to_cfg(*cfg);
        R = new EigenResult(plain ? plain_lanczos(A, alpha, beta, k)
                                  : filtered_lanczos(A, alpha, beta, k));
      }))
    return nullptr;
  return R;
}
void ref_result_free(void* R) { delete static_cast<EigenResult*>(R); }
int64_t ref_result_count(void* R) { return static_cast<EigenResult*>(R)->eigenvalues.size(); }
void ref_result_get(void* Rp, double* eigenvalues, double* residuals, double* eigenvectors,
                    orc_stats* s) {
  const auto& R = *static_cast<EigenResult*>(Rp);
  if (eigenvalues) std::copy(R.eigenvalues.begin(), R.eigenvalues.end(), eigenvalues);
  if (residuals) std::copy(R.residuals.begin(), R.residuals.end(), residuals);
  if (eigenvectors)
    std::copy(R.eigenvectors.data(), R.eigenvectors.data() + R.eigenvectors.size(),
              eigenvectors);
  if (s) {
    const SolveStats& t = R.stats;
    s->block_steps = t.block_steps;
    s->basis_vectors = t.basis_vectors;
    s->degree = t.degree;
    s->mv_iteration = t.mv_iteration;
    s->mv_bounds = t.mv_bounds;
    s->mv_total = t.mv_total;
    s->time_total_s = t.time_total_s;
    s->time_preproc_s = t.time_preproc_s;
    s->time_orth_s = t.time_orth_s;
    s->time_mv_s = t.time_mv_s;
    s->checks = t.checks;
    s->converged = t.converged;
    s->breakdown_replacements = t.breakdown_replacements;
    s->degree_clamped = t.degree_clamped;
    s->norm_estimate = t.norm_estimate;
    s->lambda_min_est = t.lambda_min_est;
    s->lambda_max_est = t.lambda_max_est;
    s->ortho_error = t.ortho_error;
  }
}

}  // extern "C"
