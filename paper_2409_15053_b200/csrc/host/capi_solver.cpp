// host/capi_solver.cpp — flattens the C++ facade (include/flz/*.hpp) into the C ABI of
// include/flz_solver.h.  No arithmetic lives here.

#include <algorithm>
#include <cstring>
#include <memory>
#include <optional>
#include <cstdlib>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "flz/solver.hpp"
#include "flz_solver.h"

namespace flz {
void set_last_error(const std::string& msg);  // capi.cu
}

using namespace flz;

struct flz_hostmatrix {
  SparseSymMatrix A;
};
struct flz_result {
  EigenResult R;
  std::size_t n = 0;
};
struct flz_fact {
  const SparseSymMatrix* A = nullptr;
  std::optional<ChebyshevFilter> filter;
  std::optional<BlockOperator> op;
  std::unique_ptr<LanczosFactorization> st;
};

namespace {

template <class F>
int wrap(F&& f) {
  try {
    f();
    return FLZ_OK;
  } catch (const ParseError& e) {
    set_last_error(e.what());
    return FLZ_EPARSE;
  } catch (const IntervalError& e) {
    set_last_error(e.what());
    return FLZ_EINTERVAL;
  } catch (const DimensionError& e) {
    set_last_error(e.what());
    return FLZ_EDIM;
  } catch (const DeviceError& e) {
    set_last_error(e.what());
    return FLZ_ECUDA;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return FLZ_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FLZ_EINVAL;
  }
}

LanczosConfig to_config(const flz_config& c) {
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
  k.return_vectors = c.return_vectors != 0;
  k.jackson_damping = c.jackson_damping != 0;
  return k;
}

SymBandMatrix band_from_flat(std::int64_t dim, std::int64_t sb, const double* bands) {
  SymBandMatrix M(static_cast<std::size_t>(dim), static_cast<std::size_t>(sb));
  for (std::size_t d = 0; d <= M.semi_bandwidth(); ++d)
    for (std::size_t i = 0; i + d < M.dim(); ++i) M.set(i + d, i, bands[d * dim + i]);
  return M;
}

}  // namespace

namespace {
// Copy of a caller's array.  A fresh 100 MB vector costs more in page faults than in bytes
// moved when one thread touches it first (~2.5 GB/s), so the pages of the reserved storage
// are faulted in by several threads before the copy.
template <class T>
std::vector<T> copy_of(const T* src, std::size_t count) {
  std::vector<T> v;
  v.reserve(count);
  constexpr std::size_t kPage = 4096 / sizeof(T);
  const std::size_t pages = count / kPage;
  unsigned workers = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (const char* e = std::getenv("FLZ_HOST_THREADS")) workers = std::max(1, std::atoi(e));
  if (pages >= 4096 && workers > 1) {
    T* raw = v.data();   // reserved, not yet constructed: trivially constructible T only
    static_assert(std::is_trivially_copyable<T>::value, "copy_of: trivial element types only");
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < workers; ++t)
      pool.emplace_back([=] {
        for (std::size_t p = pages * t / workers; p < pages * (t + 1) / workers; ++p)
          reinterpret_cast<volatile unsigned char*>(raw + p * kPage)[0] = 0;
      });
    for (auto& th : pool) th.join();
  }
  v.assign(src, src + count);
  return v;
}
}  // namespace

extern "C" {

void flz_config_default(flz_config* cfg) {
  const LanczosConfig k;
  cfg->block_size = k.block_size;
  cfg->tol = k.tol;
  cfg->max_dim = k.max_dim;
  cfg->check_every = k.check_every;
  cfg->seed = k.seed;
  cfg->extra_ritz = k.extra_ritz;
  cfg->bounds_steps = k.bounds_steps;
  cfg->degree = 0;
  cfg->epsilon = k.epsilon;
  cfg->max_degree = k.max_degree;
  cfg->collect_diagnostics = 0;
  cfg->return_vectors = 1;
  cfg->jackson_damping = 0;
}

int flz_set_default_ctx(flz_ctx* ctx) {
  return wrap([&] {
    if (ctx)
      Device::adopt(ctx);
    else
      Device::shutdown();
  });
}

int flz_set_thread_ctx(flz_ctx* ctx) {
  return wrap([&] { Device::adopt_thread(ctx); });
}

int flz_default_ctx(flz_ctx** out) {
  return wrap([&] { *out = Device::context(); });
}

int flz_hostmatrix_from_triplets(int64_t n, int64_t count, const int64_t* rows,
                                 const int64_t* cols, const double* values,
                                 flz_hostmatrix** out) {
  return wrap([&] {
    std::vector<Triplet> t(static_cast<std::size_t>(count));
    for (int64_t i = 0; i < count; ++i) t[i] = {rows[i], cols[i], values[i]};
    *out = new flz_hostmatrix{SparseSymMatrix::from_entries(static_cast<std::size_t>(n),
                                                            std::move(t))};
  });
}
int flz_hostmatrix_from_csr(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                            const double* values, int check_symmetry, flz_hostmatrix** out) {
  return wrap([&] {
    const std::size_t nnz = static_cast<std::size_t>(row_ptr[n]);
    *out = new flz_hostmatrix{SparseSymMatrix::from_csr(
        static_cast<std::size_t>(n), copy_of(row_ptr, static_cast<std::size_t>(n) + 1),
        copy_of(col_idx, nnz), copy_of(values, nnz), check_symmetry != 0)};
  });
}
int flz_hostmatrix_from_local_rows(int64_t n_global, int64_t row_begin, int64_t row_end,
                                   const int64_t* row_ptr, const int32_t* col_idx,
                                   const double* values, flz_hostmatrix** out) {
  return wrap([&] {
    const int64_t nl = row_end - row_begin;
    const std::size_t nnz = static_cast<std::size_t>(row_ptr[nl]);
    *out = new flz_hostmatrix{SparseSymMatrix::from_local_rows(
        static_cast<std::size_t>(n_global), static_cast<std::size_t>(row_begin),
        std::vector<std::int64_t>(row_ptr, row_ptr + nl + 1),
        std::vector<std::int32_t>(col_idx, col_idx + nnz),
        std::vector<double>(values, values + nnz))};
  });
}
int flz_hostmatrix_load_mm(const char* path, flz_hostmatrix** out) {
  return wrap([&] { *out = new flz_hostmatrix{load_matrix_market(path)}; });
}
int flz_hostmatrix_save_mm(const flz_hostmatrix* A, const char* path) {
  return wrap([&] { save_matrix_market(A->A, path); });
}
int flz_hostmatrix_save_bin(const flz_hostmatrix* A, const char* path) {
  return wrap([&] { save_binary_csr(A->A, path); });
}
int flz_hostmatrix_load_bin(const char* path, flz_hostmatrix** out) {
  return wrap([&] { *out = new flz_hostmatrix{load_binary_csr(path)}; });
}
void flz_hostmatrix_free(flz_hostmatrix* A) { delete A; }
int flz_hostmatrix_dims(const flz_hostmatrix* A, int64_t* n, int64_t* nnz) {
  if (n) *n = static_cast<int64_t>(A->A.dim());
  if (nnz) *nnz = static_cast<int64_t>(A->A.nnz());
  return FLZ_OK;
}
int flz_hostmatrix_layout(const flz_hostmatrix* A, int64_t* matrix_bytes,
                          int64_t* uniform_entries) {
  return wrap([&] {
    throw_status(flz_matrix_layout(A->A.device(), matrix_bytes, uniform_entries));
  });
}
int flz_hostmatrix_k1_info(const flz_hostmatrix* A, int r, int64_t* info, char* kernel, int cap) {
  return wrap([&] { throw_status(flz_matrix_k1_info(A->A.device(), r, info, kernel, cap)); });
}
int flz_hostmatrix_csr(const flz_hostmatrix* A, int64_t* row_ptr, int32_t* col_idx,
                       double* values) {
  std::copy(A->A.row_ptr().begin(), A->A.row_ptr().end(), row_ptr);
  std::copy(A->A.col_idx().begin(), A->A.col_idx().end(), col_idx);
  std::copy(A->A.values().begin(), A->A.values().end(), values);
  return FLZ_OK;
}
int flz_hostmatrix_spmm(const flz_hostmatrix* A, const double* X, int64_t rows, int r,
                        double* Y) {
  return wrap([&] {
    const std::size_t n = static_cast<std::size_t>(rows);
    DenseBlock Xb(n, r), Yb;
    std::copy(X, X + n * r, Xb.data());
    A->A.spmm_block(Xb, Yb);
    std::copy(Yb.data(), Yb.data() + n * r, Y);
  });
}
int flz_hostmatrix_filter_apply(const flz_hostmatrix* A, const double* coeffs, int m,
                                double lambda_min, double lambda_max, const double* X,
                                int64_t rows, int r, double* Y) {
  return wrap([&] {
    const std::size_t n = static_cast<std::size_t>(rows);
    const auto f = ChebyshevFilter::from_coefficients(
        SpectralBounds(lambda_min, lambda_max), lambda_min, lambda_max,
        std::vector<double>(coeffs, coeffs + std::max(m, -1) + 1));
    DenseBlock Xb(n, r), Yb;
    std::copy(X, X + n * r, Xb.data());
    f.apply(A->A, Xb, Yb);
    std::copy(Yb.data(), Yb.data() + n * r, Y);
  });
}

int flz_indicator_coefficients(double alpha_s, double beta_s, int degree, double* out) {
  return wrap([&] {
    const auto b = indicator_coefficients(alpha_s, beta_s, degree);
    std::copy(b.begin(), b.end(), out);
  });
}
int flz_jackson_factors(int degree, double* out) {
  return wrap([&] {
    const auto g = jackson_factors(degree);
    std::copy(g.begin(), g.end(), out);
  });
}
int flz_select_degree(double alpha_s, double beta_s, double epsilon, int max_degree,
                      int* clamped) {
  int m = -1;
  const int rc = wrap([&] {
    const DegreeSelection s = select_degree(alpha_s, beta_s, epsilon, max_degree);
    m = s.degree;
    if (clamped) *clamped = s.clamped ? 1 : 0;
  });
  return rc == FLZ_OK ? m : rc;
}
double flz_clenshaw(const double* coeffs, int ncoeffs, double t) {
  return clenshaw(std::span<const double>(coeffs, static_cast<std::size_t>(ncoeffs)), t);
}
int flz_build_filter(double lambda_min, double lambda_max, double alpha, double beta, int degree,
                     double epsilon, int max_degree, double* coeffs, int cap, double* alpha_s,
                     double* beta_s, int* clamped) {
  int m = -1;
  const int rc = wrap([&] {
    const ChebyshevFilter f =
        build_filter(SpectralBounds(lambda_min, lambda_max), alpha, beta,
                     degree > 0 ? std::optional<int>(degree) : std::nullopt, epsilon, max_degree);
    m = f.degree();
    if (coeffs) {
      if (m + 1 > cap) throw Error("build_filter: coefficient buffer too small");
      std::copy(f.coefficients().begin(), f.coefficients().end(), coeffs);
    }
    if (alpha_s) *alpha_s = f.alpha_mapped();
    if (beta_s) *beta_s = f.beta_mapped();
    if (clamped) *clamped = f.degree_clamped() ? 1 : 0;
  });
  return rc == FLZ_OK ? m : rc;
}

int flz_init_block(int64_t n, int r, uint64_t seed, double* Q) {
  return wrap([&] {
    const DenseBlock B = init_block(static_cast<std::size_t>(n), static_cast<std::size_t>(r), seed);
    std::copy(B.data(), B.data() + B.size(), Q);
  });
}
int flz_estimate_bounds(const flz_hostmatrix* A, int steps, uint64_t seed, double* lo,
                        double* hi) {
  return wrap([&] {
    const SpectralBounds b = estimate_spectral_bounds(A->A, steps, seed);
    *lo = b.lambda_min();
    *hi = b.lambda_max();
  });
}

int flz_sym_band_eig(int64_t dim, int64_t sb, const double* bands, double* values,
                     double* vectors) {
  return wrap([&] {
    const SymEig e = sym_band_eig(band_from_flat(dim, sb, bands));
    std::copy(e.values.begin(), e.values.end(), values);
    if (vectors) std::copy(e.vectors.data(), e.vectors.data() + e.vectors.size(), vectors);
  });
}
int flz_band_ritz_rows(int64_t dim, int64_t sb, const double* bands, int64_t nrows,
                       const int64_t* rows, double* values, double* out_rows) {
  return wrap([&] {
    std::vector<std::size_t> rr(rows, rows + nrows);
    const SymEig e = band_ritz_rows(band_from_flat(dim, sb, bands), rr);
    std::copy(e.values.begin(), e.values.end(), values);
    if (out_rows) std::copy(e.vectors.data(), e.vectors.data() + e.vectors.size(), out_rows);
  });
}
int flz_band_eigenvectors(int64_t dim, int64_t sb, const double* bands, const double* values,
                          int64_t npick, const int64_t* pick, double* vectors,
                          double* max_residual, double* max_ortho) {
  return wrap([&] {
    std::vector<std::size_t> pk(pick, pick + npick);
    const DenseBlock W = band_eigenvectors(band_from_flat(dim, sb, bands),
                                           std::vector<double>(values, values + dim), pk,
                                           max_residual, max_ortho);
    std::copy(W.data(), W.data() + W.size(), vectors);
  });
}

int flz_fact_create(const flz_hostmatrix* A, const double* coeffs, int m, double lambda_min,
                    double lambda_max, double alpha, double beta, const double* start, int r,
                    int64_t max_cols, flz_fact** out) {
  return wrap([&] {
    auto F = std::make_unique<flz_fact>();
    F->A = &A->A;
    if (m >= 0) {
      F->filter = ChebyshevFilter::from_coefficients(SpectralBounds(lambda_min, lambda_max),
                                                     alpha, beta,
                                                     std::vector<double>(coeffs, coeffs + m + 1));
      F->op = BlockOperator::filtered(*F->A, *F->filter);
    } else {
      F->op = BlockOperator::plain(*F->A);
    }
    const std::size_t n = F->A->dim();
    DenseBlock S(n, r);
    std::copy(start, start + n * r, S.data());
    F->st = std::make_unique<LanczosFactorization>(*F->op, std::move(S),
                                                   static_cast<std::size_t>(max_cols));
    *out = F.release();
  });
}
void flz_fact_free(flz_fact* F) { delete F; }
int flz_fact_expand(flz_fact* F, int nblocks) {
  int added = -1;
  const int rc = wrap([&] { added = expand(*F->st, nblocks, nullptr); });
  return rc == FLZ_OK ? added : rc;
}
int64_t flz_fact_block_count(const flz_fact* F) {
  return static_cast<int64_t>(F->st->block_count());
}
int flz_fact_get(const flz_fact* F, double* basis, double* D, double* S, uint8_t* dead) {
  return wrap([&] {
    const auto& st = *F->st;
    const std::size_t n = st.n(), r = st.block_size(), k = st.block_count();
    if (basis) {
      const DenseBlock Q = st.basis_block(0, k * r + r);
      std::copy(Q.data(), Q.data() + n * (k * r + r), basis);
    }
    for (std::size_t b = 0; b < k; ++b) {
      if (D) std::copy(st.diag_blocks()[b].begin(), st.diag_blocks()[b].end(), D + b * r * r);
      if (S) std::copy(st.sub_blocks()[b].begin(), st.sub_blocks()[b].end(), S + b * r * r);
    }
    if (dead) std::copy(st.dead_cols().begin(), st.dead_cols().end(), dead);
  });
}
int flz_fact_ortho_error(const flz_fact* F, double* out) {
  return wrap([&] { *out = F->st->ortho_error(); });
}
int flz_fact_flags(const flz_fact* F) {
  return (F->st->space_exhausted() ? 1 : 0) | (F->st->had_breakdown() ? 2 : 0);
}
int flz_fact_check(const flz_fact* F, double alpha, double beta, double tol, int extra_ritz,
                   double* values, double* estimates, uint8_t* wanted, uint8_t* dead) {
  int conv = -1;
  const int rc = wrap([&] {
    const RitzSet rs = check_convergence(*F->st, alpha, beta, tol, extra_ritz);
    std::copy(rs.values.begin(), rs.values.end(), values);
    std::copy(rs.residual_estimates.begin(), rs.residual_estimates.end(), estimates);
    std::copy(rs.wanted.begin(), rs.wanted.end(), wanted);
    std::copy(rs.dead.begin(), rs.dead.end(), dead);
    conv = rs.converged ? 1 : 0;
  });
  return rc == FLZ_OK ? conv : rc;
}

int flz_solve(const flz_hostmatrix* A, double alpha, double beta, const flz_config* cfg,
              int plain, flz_result** out) {
  return wrap([&] {
    flz_config def;
    if (!cfg) {
      flz_config_default(&def);
      cfg = &def;
    }
    const LanczosConfig k = to_config(*cfg);
    auto R = std::make_unique<flz_result>();
    R->n = A->A.dim();
    R->R = plain ? plain_lanczos(A->A, alpha, beta, k) : filtered_lanczos(A->A, alpha, beta, k);
    *out = R.release();
  });
}
void flz_result_free(flz_result* R) { delete R; }
int64_t flz_result_count(const flz_result* R) {
  return static_cast<int64_t>(R->R.eigenvalues.size());
}
const double* flz_result_vectors(const flz_result* R) { return R->R.eigenvectors.data(); }
int64_t flz_result_rows(const flz_result* R) {
  return static_cast<int64_t>(R->R.eigenvectors.rows());
}
int flz_result_get(const flz_result* Rp, double* eigenvalues, double* residuals,
                   double* eigenvectors, flz_stats* s) {
  const EigenResult& R = Rp->R;
  if (eigenvalues) std::copy(R.eigenvalues.begin(), R.eigenvalues.end(), eigenvalues);
  if (residuals) std::copy(R.residuals.begin(), R.residuals.end(), residuals);
  if (eigenvectors)
    std::copy(R.eigenvectors.data(), R.eigenvectors.data() + R.eigenvectors.size(), eigenvectors);
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
    s->time_check_s = t.time_check_s;
    s->time_recover_s = t.time_recover_s;
    s->time_upload_s = t.time_upload_s;
    s->gpu_launches = t.gpu_launches;
  }
  return FLZ_OK;
}

}  // extern "C"
