// host/solver.cpp — host driver of the filtered block-Lanczos solve.
//
// Behavioural contract: src/lanczos.cpp — config :46-69, BlockOperator::apply :71-76,
// init_block :78-103, LanczosFactorization :105-132, expand :134-271, assemble_projected
// :273-296, check_convergence :298-405, recover_eigenpairs :407-510,
// estimate_spectral_bounds :512-569, run_solve :573-667.
//
// What runs where: every O(n) operation (operator application, Gram-Schmidt sweeps,
// intra-block QR, Ritz lift, Rayleigh-Ritz products, residuals) is a device call through
// include/flz.h; this file keeps what the north star leaves on the host — random start
// vectors (libstdc++ mt19937_64 + normal_distribution, so they are the reference's),
// breakdown policy, T_k assembly, the banded eigensolve and the convergence logic.

#include "flz/solver.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <future>
#include <memory>
#include <random>
#include <thread>

#include "flz.h"

namespace flz {

namespace {

class WallClock {
 public:
  WallClock() : t0_(std::chrono::steady_clock::now()) {}
  double seconds() const {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
  }

 private:
  std::chrono::steady_clock::time_point t0_;
};

// FLZ_TRACE=1: phase timings of the host driver on stderr (diagnostics only)
bool trace_on() {
  static const bool on = std::getenv("FLZ_TRACE") != nullptr;
  return on;
}
void trace(const char* what, const WallClock& clk) {
  if (trace_on()) std::fprintf(stderr, "[flz] %-28s %9.3f ms\n", what, clk.seconds() * 1e3);
}

// splitmix64 finaliser; same stream derivation as the reference (lanczos.cpp:25-30)
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t salt) {
  std::uint64_t z = seed + salt + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double host_dot(const double* x, const double* y, std::size_t n) {
  double s = 0.0;
  for (std::size_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}

// z -= Q[:, :cols] (Q[:, :cols]^T z), one column at a time (host; start block only)
void host_mgs(const DenseBlock& Q, std::size_t cols, double* z, std::size_t n) {
  for (std::size_t i = 0; i < cols; ++i) {
    const double c = host_dot(Q.col(i), z, n);
    const double* q = Q.col(i);
    for (std::size_t t = 0; t < n; ++t) z[t] -= c * q[t];
  }
}

// Rows [b, e) of a column-major block (identity when the context owns all rows).
DenseBlock local_rows(const DenseBlock& X, std::size_t n_global) {
  std::size_t b = 0, e = n_global;
  Device::row_range(n_global, b, e);
  if (b == 0 && e == X.rows()) return X;
  DenseBlock L(e - b, X.cols());
  for (std::size_t j = 0; j < X.cols(); ++j) std::copy(X.col(j) + b, X.col(j) + e, L.col(j));
  return L;
}

}  // namespace

// ------------------------------------------------------------------ config
int LanczosConfig::resolved_max_dim(std::size_t n) const {
  if (max_dim > 0) return max_dim;
  const auto r = static_cast<std::size_t>(block_size);
  std::size_t cap = std::max(std::min<std::size_t>(n, 3000), 2 * r);
  cap = (cap + r - 1) / r * r;  // whole blocks
  return static_cast<int>(cap);
}

void LanczosConfig::validate(std::size_t n) const {
  if (block_size < 1) throw Error("config: block_size must be >= 1");
  if (static_cast<std::size_t>(block_size) > n)
    throw Error("config: block_size exceeds the matrix dimension");
  if (!(tol > 0.0 && tol < 1.0)) throw Error("config: tol must lie in (0, 1)");
  if (resolved_max_dim(n) < 2 * block_size)
    throw Error("config: max_dim must be at least 2 * block_size");
  if (check_every < 1) throw Error("config: check_every must be >= 1");
  if (extra_ritz < 0) throw Error("config: extra_ritz must be >= 0");
  if (bounds_steps < 2) throw Error("config: bounds_steps must be >= 2");
  if (degree && *degree < 1) throw Error("config: degree must be >= 1");
  if (!(epsilon > 0.0 && epsilon < 1.0)) throw Error("config: epsilon must lie in (0, 1)");
}

void BlockOperator::apply(const DenseBlock& X, DenseBlock& Y) const {
  if (filter_)
    filter_->apply(*matrix_, X, Y);
  else
    matrix_->spmm_block(X, Y);
}

// -------------------------------------------------------------- start block
DenseBlock init_block(std::size_t n, std::size_t r, std::uint64_t seed) {
  if (r > n) throw Error("init_block: more columns than rows");
  if (r == 0) throw Error("init_block: empty block");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  DenseBlock Q(n, r);
  for (std::size_t j = 0; j < r; ++j) {
    double* q = Q.col(j);
    for (std::size_t i = 0; i < n; ++i) q[i] = gauss(rng);
  }
  const double tiny = 1e-8 * std::sqrt(static_cast<double>(n));
  for (std::size_t j = 0; j < r; ++j) {
    double* z = Q.col(j);
    double norm;
    while (true) {
      host_mgs(Q, j, z, n);
      host_mgs(Q, j, z, n);
      norm = std::sqrt(host_dot(z, z, n));
      if (!(norm < tiny)) break;
      for (std::size_t i = 0; i < n; ++i) z[i] = gauss(rng);  // redraw a degenerate column
    }
    const double inv = 1.0 / norm;
    for (std::size_t i = 0; i < n; ++i) z[i] *= inv;
  }
  return Q;
}

// ----------------------------------------------------------- factorization
LanczosFactorization::LanczosFactorization(const BlockOperator& op, DenseBlock start,
                                           std::size_t max_cols)
    : op_(&op),
      n_(start.rows()),
      r_(start.cols()),
      max_cols_(max_cols),
      rng_state_(mix_seed(0xD1B54A32D192ED03ULL, max_cols)) {
  if (r_ == 0 || n_ == 0) throw Error("LanczosFactorization: empty start block");
  if (max_cols_ < 2 * r_) throw Error("LanczosFactorization: column budget too small");
  {
    std::size_t b = 0, e = op.matrix().dim();
    Device::row_range(op.matrix().dim(), b, e);
    if (n_ != e - b)
      throw DimensionError("LanczosFactorization: start block rows do not match the matrix");
  }
  throw_status(flz_basis_create(Device::context(), op.matrix().device(),
                                static_cast<std::int64_t>(max_cols_), static_cast<int>(r_),
                                start.data(), &dev_));
  dead_.assign(r_, 0);
}

LanczosFactorization::~LanczosFactorization() { flz_basis_destroy(dev_); }

const double* LanczosFactorization::basis_col(std::size_t j) const {
  col_cache_.resize(n_);
  throw_status(flz_basis_get(Device::context(), dev_, static_cast<std::int64_t>(j), 1,
                             col_cache_.data()));
  return col_cache_.data();
}

DenseBlock LanczosFactorization::basis_block(std::size_t j0, std::size_t count) const {
  DenseBlock out(n_, count);
  if (count)
    throw_status(flz_basis_get(Device::context(), dev_, static_cast<std::int64_t>(j0),
                               static_cast<std::int64_t>(count), out.data()));
  return out;
}

double LanczosFactorization::ortho_error() const {
  double worst = 0.0;
  throw_status(flz_basis_ortho_error(Device::context(), dev_, dead_.data(), &worst));
  return worst;
}

int expand(LanczosFactorization& st, int nblocks, ExpandTimes* times) {
  // n: global dimension (random replacement vectors are drawn for all n rows on every rank so
  // that the stream equals the single-GPU one; each rank keeps its slab)
  const std::size_t n = st.op_->matrix().dim(), r = st.r_;
  std::size_t row_b = 0, row_e = n;
  Device::row_range(n, row_b, row_e);
  flz_ctx* ctx = Device::context();
  const BlockOperator& op = *st.op_;
  const ChebyshevFilter* f = op.filter();
  std::mt19937_64 rng(st.rng_state_);
  std::normal_distribution<double> gauss(0.0, 1.0);

  double mv0 = 0.0, orth0 = 0.0;
  flz_basis_times(st.dev_, &mv0, &orth0);

  std::vector<double> Dk(r * r), Sk(r * r), fresh;
  std::vector<std::uint8_t> dead(r);
  int added = 0;
  for (int step = 0; step < nblocks; ++step) {
    if (st.basis_size() + r > st.max_cols_) break;
    bool pending_live = false;  // nothing to promote once every pending direction has died
    for (std::size_t j = 0; j < r && !pending_live; ++j)
      pending_live = st.dead_[st.basis_size() + j] == 0;
    if (!pending_live) break;

    throw_status(flz_lanczos_step(ctx, op.matrix().device(), st.dev_,
                                  f ? f->coefficients().data() : nullptr, f ? f->degree() : -1,
                                  f ? f->bounds().center() : 0.0,
                                  f ? f->bounds().half_width() : 1.0, Dk.data(), Sk.data(),
                                  &st.op_scale_, dead.data()));
    st.k_ += 1;
    const std::size_t cols = st.basis_size();

    // D_k: first-sweep coefficients; record the asymmetry, then symmetrise (:183-194)
    double asym = 0.0;
    for (std::size_t i = 0; i < r; ++i)
      for (std::size_t j = i + 1; j < r; ++j) {
        asym = std::max(asym, std::abs(Dk[i * r + j] - Dk[j * r + i]));
        const double mean = 0.5 * (Dk[i * r + j] + Dk[j * r + i]);
        Dk[i * r + j] = Dk[j * r + i] = mean;
      }
    st.max_diag_asym_ = std::max(st.max_diag_asym_, asym);
    st.D_.push_back(Dk);

    std::size_t live_total = 0;
    for (std::size_t c = 0; c < cols; ++c) live_total += st.dead_[c] ? 0u : 1u;
    for (std::size_t j = 0; j < r; ++j) {
      if (!dead[j]) {
        st.dead_.push_back(0);
        ++live_total;
        continue;
      }
      // breakdown: try fresh random directions while the space is not spanned (:232-262)
      st.breakdown_ = true;
      bool replaced = false;
      if (live_total < n) {
        fresh.resize(n);
        for (int attempt = 0; attempt < 5 && !replaced; ++attempt) {
          for (std::size_t i = 0; i < n; ++i) fresh[i] = gauss(rng);
          double rn = 0.0;
          double* mine = fresh.data() + row_b;  // this rank's rows; rn is the global norm
          // against ALL cols + r columns: the device has already finished the intra-block QR
          // of the live pending columns j+1.., so the replacement must be made orthogonal to
          // them too (the reference removes the replacement from those columns instead,
          // lanczos.cpp:208-218; either way the pending block ends up orthonormal).  Dead
          // columns that are not replaced yet are exactly zero and contribute nothing.
          throw_status(flz_orthogonalize_column(ctx, st.dev_, static_cast<std::int64_t>(cols),
                                                static_cast<int>(r), mine, &rn));
          if (rn > 1e-4) {
            const double inv = 1.0 / rn;
            for (std::size_t i = 0; i < row_e - row_b; ++i) mine[i] *= inv;
            throw_status(flz_basis_set(ctx, st.dev_, static_cast<std::int64_t>(cols + j), mine));
            replaced = true;
          }
        }
      }
      if (replaced) {
        st.dead_.push_back(0);
        ++live_total;
      } else {
        st.dead_.push_back(1);  // the device left the column exactly zero
        st.exhausted_ = true;
      }
    }
    st.S_.push_back(Sk);
    ++added;
  }
  st.rng_state_ = rng();
  if (times) {
    double mv1 = 0.0, orth1 = 0.0;
    flz_basis_times(st.dev_, &mv1, &orth1);
    times->mv_s += mv1 - mv0;
    times->orth_s += orth1 - orth0;
  }
  return added;
}

LanczosFactorization::Snapshot LanczosFactorization::snapshot() const {
  Snapshot s;
  s.r = r_;
  s.k = k_;
  s.D = D_;
  s.S = S_;
  s.dead = dead_;
  s.kind = op_->kind();
  s.filter = op_->filter();
  s.exhausted = exhausted_;
  s.breakdown = breakdown_;
  s.max_diag_asym = max_diag_asym_;
  s.op_scale = op_scale_;
  s.rng_state = rng_state_;
  return s;
}

void LanczosFactorization::rollback(const Snapshot& snap) {
  if (snap.k > k_) throw Error("rollback: snapshot is ahead of the factorization");
  const std::size_t undone = k_ - snap.k;
  if (undone == 0) return;
  throw_status(flz_basis_truncate(Device::context(), dev_, static_cast<std::int64_t>(snap.k),
                                  snap.op_scale));
  const ChebyshevFilter* f = op_->filter();
  flz_matvec_sub(static_cast<std::uint64_t>(undone) * r_ * (f ? f->degree() : 1));
  k_ = snap.k;
  D_ = snap.D;
  S_ = snap.S;
  dead_ = snap.dead;
  exhausted_ = snap.exhausted;
  breakdown_ = snap.breakdown;
  max_diag_asym_ = snap.max_diag_asym;
  op_scale_ = snap.op_scale;
  rng_state_ = snap.rng_state;
}

// -------------------------------------------------------- projected problem
SymBandMatrix assemble_projected(const LanczosFactorization& st) {
  return assemble_projected(st.snapshot());
}

SymBandMatrix assemble_projected(const LanczosFactorization::Snapshot& st) {
  const std::size_t r = st.r, k = st.k;
  if (k == 0) throw Error("assemble_projected: empty factorization");
  const std::size_t dim = k * r;
  SymBandMatrix T(dim, std::min(r, dim - 1));
  for (std::size_t blk = 0; blk < k; ++blk) {
    const auto& D = st.D[blk];
    for (std::size_t a = 0; a < r; ++a)
      for (std::size_t b = 0; b <= a; ++b)
        T.set(blk * r + a, blk * r + b, 0.5 * (D[a * r + b] + D[b * r + a]));
    if (blk + 1 == k) break;  // S_k of the pending block is not part of T_k
    const auto& S = st.S[blk];
    for (std::size_t a = 0; a < r; ++a)
      for (std::size_t b = a; b < r; ++b) T.set((blk + 1) * r + a, blk * r + b, S[a * r + b]);
  }
  return T;
}

RitzSet check_convergence(const LanczosFactorization& st, double alpha, double beta, double tol,
                          int extra_ritz, bool want_vectors) {
  return check_convergence(st.snapshot(), alpha, beta, tol, extra_ritz, want_vectors);
}

RitzSet check_convergence(const LanczosFactorization::Snapshot& st, double alpha, double beta,
                          double tol, int extra_ritz, bool want_vectors) {
  const std::size_t r = st.r, k = st.k;
  if (k == 0) throw Error("check_convergence: empty factorization");
  const std::size_t dim = k * r;
  const SymBandMatrix T = assemble_projected(st);
  const double t_scale = T.max_abs();
  const auto& dead_cols = st.dead;

  // Rows of the eigenvector matrix the classification reads: the last block (residual
  // estimates, :354-361) and the rows of dead columns (dead mass, :363-369).
  std::vector<std::size_t> rows;
  for (std::size_t b = 0; b < r; ++b) rows.push_back((k - 1) * r + b);
  for (std::size_t i = 0; i < dim; ++i)
    if (dead_cols[i] && i < (k - 1) * r) rows.push_back(i);

  SymEig eig = want_vectors ? sym_band_eig(T) : band_ritz_rows(T, rows);
  auto entry = [&](std::size_t t, std::size_t src) {  // W(rows[t], src)
    return want_vectors ? eig.vectors(rows[t], src) : eig.vectors(t, src);
  };

  RitzSet out;
  out.values.resize(dim);
  out.residual_estimates.assign(dim, 0.0);
  out.wanted.assign(dim, 0);
  out.dead.assign(dim, 0);
  if (want_vectors) out.vectors = DenseBlock(dim, dim);

  double tau = 0.0;  // filtered-mode cut at the clipped mapped endpoints (:343-349)
  const bool filtered = st.kind == OperatorKind::filtered;
  if (filtered) {
    const ChebyshevFilter* f = st.filter;
    tau = std::min(clenshaw(f->coefficients(), f->alpha_mapped()),
                   clenshaw(f->coefficients(), f->beta_mapped())) -
          1e-10 * t_scale;
  }
  const auto& S_last = st.S[k - 1];
  for (std::size_t c = 0; c < dim; ++c) {
    const std::size_t src = dim - 1 - c;  // descending order
    out.values[c] = eig.values[src];
    if (want_vectors)
      std::copy(eig.vectors.col(src), eig.vectors.col(src) + dim, out.vectors.col(c));
    double est = 0.0;  // || S_k (E_k^T w) ||
    for (std::size_t a = 0; a < r; ++a) {
      double acc = 0.0;
      for (std::size_t b = a; b < r; ++b) acc += S_last[a * r + b] * entry(b, src);
      est += acc * acc;
    }
    out.residual_estimates[c] = std::sqrt(est);
    double dead_mass = 0.0;
    for (std::size_t t = 0; t < rows.size(); ++t)
      if (dead_cols[rows[t]]) dead_mass += entry(t, src) * entry(t, src);
    if (dead_mass > 0.5) {
      out.dead[c] = 1;
      continue;
    }
    out.wanted[c] = filtered ? (out.values[c] >= tau)
                             : (out.values[c] >= alpha && out.values[c] <= beta);
  }

  const double threshold = tol * t_scale;
  bool ok = true;
  for (std::size_t c = 0; c < dim && ok; ++c)
    ok = !(out.wanted[c] && out.residual_estimates[c] > threshold);
  if (ok) {  // the nearest unwanted pairs must have settled too (:377-402)
    std::vector<std::size_t> unwanted;
    for (std::size_t c = 0; c < dim; ++c)
      if (!out.wanted[c] && !out.dead[c]) unwanted.push_back(c);
    if (!filtered) {
      auto dist = [&](std::size_t c) {
        const double v = out.values[c];
        return v < alpha ? alpha - v : (v > beta ? v - beta : 0.0);
      };
      std::sort(unwanted.begin(), unwanted.end(),
                [&](std::size_t a, std::size_t b) { return dist(a) < dist(b); });
    }
    const std::size_t need = std::min<std::size_t>(extra_ritz, unwanted.size());
    for (std::size_t t = 0; t < need && ok; ++t)
      ok = out.residual_estimates[unwanted[t]] <= threshold;
  }
  out.converged = ok;
  return out;
}

// ----------------------------------------------------------------- recovery
EigenResult recover_eigenpairs(const LanczosFactorization& st, const SparseSymMatrix& A,
                               double alpha, double beta, const RitzSet& ritz,
                               double norm_estimate, bool return_vectors) {
  const std::size_t n = st.n(), dim = st.basis_size();
  const double scale = norm_estimate > 0.0 ? norm_estimate : 1.0;
  flz_ctx* ctx = Device::context();

  std::vector<std::size_t> candidates;
  for (std::size_t c = 0; c < ritz.values.size(); ++c)
    if (ritz.wanted[c] && !ritz.dead[c]) candidates.push_back(c);
  const std::size_t w = candidates.size();
  EigenResult out;
  if (w == 0) {
    out.eigenvectors = DenseBlock(n, 0);
    return out;
  }

  // host storage of the eigenvectors (page-locked or pre-faulted): prepared on a second
  // thread while the device lifts the Ritz vectors; at most w columns are needed
  std::future<DenseBlock> storage;
  if (return_vectors)
    storage = std::async(std::launch::async, [n, w, ctx = Device::context()] {
      // a new host thread starts on device 0: bind it to the rank's device before it
      // page-locks memory, or every rank would create a context on GPU 0
      throw_status(flz_ctx_make_current(ctx));
      return DenseBlock::pinned(n, w);
    });

  // Ritz vectors of T_k for the candidates only.
  const WallClock t_w;
  DenseBlock W(dim, w);
  if (ritz.vectors.size() == dim * dim && dim > 0) {
    for (std::size_t t = 0; t < w; ++t)
      std::copy(ritz.vectors.col(candidates[t]), ritz.vectors.col(candidates[t]) + dim, W.col(t));
  } else {
    const SymBandMatrix T = assemble_projected(st);
    std::vector<double> ascending(ritz.values.rbegin(), ritz.values.rend());
    std::vector<std::size_t> pick(w);
    for (std::size_t t = 0; t < w; ++t) pick[t] = dim - 1 - candidates[t];
    // ascending picks keep clusters adjacent
    std::vector<std::size_t> order(w);
    for (std::size_t t = 0; t < w; ++t) order[t] = w - 1 - t;  // candidates are descending
    std::vector<std::size_t> pick_sorted(w);
    for (std::size_t t = 0; t < w; ++t) pick_sorted[t] = pick[order[t]];
    double res = 0.0, ortho = 0.0;
    DenseBlock Ws = band_eigenvectors(T, ascending, pick_sorted, &res, &ortho);
    if (res <= 1e-13 && ortho <= 1e-11) {
      for (std::size_t t = 0; t < w; ++t)
        std::copy(Ws.col(t), Ws.col(t) + dim, W.col(order[t]));
    } else {  // inverse iteration not clean enough: full QL, as the reference does
      const SymEig full = sym_band_eig(T);
      for (std::size_t t = 0; t < w; ++t)
        std::copy(full.vectors.col(pick[t]), full.vectors.col(pick[t]) + dim, W.col(t));
    }
  }

  trace("recover: T_k eigenvectors", t_w);
  std::vector<double> vnorm(w), Bm(w * w);
  std::vector<std::uint8_t> keep(w);
  int w_kept = 0;
  const WallClock t_lift;
  throw_status(flz_ritz_lift(ctx, A.device(), st.device(), static_cast<std::int64_t>(dim),
                             W.data(), static_cast<int>(w), vnorm.data(), keep.data(), &w_kept,
                             Bm.data()));
  trace("recover: lift + A V + V'AV", t_lift);
  std::vector<std::size_t> kept_src;
  for (std::size_t t = 0; t < w; ++t)
    if (keep[t]) kept_src.push_back(candidates[t]);
  const std::size_t wk = static_cast<std::size_t>(w_kept);

  std::vector<double> lambdas;
  if (st.kind() == OperatorKind::filtered && wk > 0) {
    // Rayleigh-Ritz of A on the lifted subspace (:440-479): B = sym(V^T A V), B = U L U^T
    SymBandMatrix B(wk, wk > 1 ? wk - 1 : 0);
    for (std::size_t i = 0; i < wk; ++i)
      for (std::size_t j = i; j < wk; ++j) B.set(j, i, Bm[i * wk + j]);
    const WallClock t_b;
    const SymEig small = sym_band_eig(B);
    trace("recover: eig of V'AV", t_b);
    std::vector<std::size_t> sel;
    for (std::size_t c = 0; c < wk; ++c)
      if (small.values[c] >= alpha && small.values[c] <= beta) sel.push_back(c);
    DenseBlock U(wk, sel.size());
    for (std::size_t t = 0; t < sel.size(); ++t) {
      std::copy(small.vectors.col(sel[t]), small.vectors.col(sel[t]) + wk, U.col(t));
      lambdas.push_back(small.values[sel[t]]);
    }
    out.eigenvalues = lambdas;  // already ascending
    out.residuals.assign(sel.size(), 0.0);
    if (return_vectors) {
      out.eigenvectors = storage.get();
      out.eigenvectors.shrink_cols(sel.size());
    } else {
      out.eigenvectors = DenseBlock(n, 0);
    }
    const WallClock t_rot;
    if (!sel.empty())
      throw_status(flz_ritz_rotate(ctx, st.device(), U.data(), lambdas.data(),
                                   static_cast<int>(sel.size()), scale, out.residuals.data(),
                                   return_vectors ? out.eigenvectors.data() : nullptr));
    trace("recover: rotate + residuals + D2H", t_rot);
  } else if (wk > 0) {
    // plain mode: Ritz values are the eigenvalue estimates (:480-495)
    std::vector<double> lam(wk), res(wk);
    for (std::size_t c = 0; c < wk; ++c) lam[c] = ritz.values[kept_src[c]];
    DenseBlock V = return_vectors ? storage.get() : DenseBlock(n, 0);
    if (return_vectors) V.shrink_cols(wk);
    throw_status(flz_ritz_plain(ctx, A.device(), st.device(), lam.data(), static_cast<int>(wk),
                                scale, res.data(), return_vectors ? V.data() : nullptr));
    std::vector<std::size_t> sel;
    for (std::size_t c = 0; c < wk; ++c)
      if (lam[c] >= alpha && lam[c] <= beta) sel.push_back(c);
    std::stable_sort(sel.begin(), sel.end(),
                     [&](std::size_t a, std::size_t b) { return lam[a] < lam[b]; });
    out.eigenvectors = DenseBlock(n, return_vectors ? sel.size() : 0);
    for (std::size_t t = 0; t < sel.size(); ++t) {
      out.eigenvalues.push_back(lam[sel[t]]);
      out.residuals.push_back(res[sel[t]]);
      if (return_vectors) std::copy(V.col(sel[t]), V.col(sel[t]) + n, out.eigenvectors.col(t));
    }
  } else {
    out.eigenvectors = DenseBlock(n, 0);
  }
  return out;
}

// ---------------------------------------------------------- spectral bounds
SpectralBounds estimate_spectral_bounds(const SparseSymMatrix& A, int steps, std::uint64_t seed) {
  const std::size_t n = A.dim();
  if (n < 2) throw Error("estimate_spectral_bounds: matrix dimension must be >= 2");
  if (steps < 2) throw Error("estimate_spectral_bounds: steps must be >= 2");
  const std::size_t s_max = std::min<std::size_t>(steps, n);

  std::mt19937_64 rng(mix_seed(seed, 0xB0u));
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::vector<double> q0(n);
  for (std::size_t i = 0; i < n; ++i) q0[i] = gauss(rng);
  const double inv = 1.0 / std::sqrt(host_dot(q0.data(), q0.data(), n));
  for (double& v : q0) v *= inv;

  std::vector<double> d(s_max, 0.0), e(s_max, 0.0);
  double beta_last = 0.0;
  int done = 0;
  std::size_t row_b = 0, row_e = n;
  Device::row_range(n, row_b, row_e);
  throw_status(flz_bounds_lanczos(Device::context(), A.device(), static_cast<int>(s_max),
                                  q0.data() + row_b, d.data(), e.data(), &beta_last, &done));
  const auto s_done = static_cast<std::size_t>(done);
  d.resize(s_done);
  e.resize(s_done > 0 ? s_done - 1 : 0);
  DenseBlock G = DenseBlock::identity(s_done);
  tridiag_eig(d, e, G);

  // Ritz extremes widened by their residual estimates and 0.5 % of the width (:558-567)
  const double rho_min = std::abs(beta_last * G(s_done - 1, 0));
  const double rho_max = std::abs(beta_last * G(s_done - 1, s_done - 1));
  double lo = d.front() - rho_min, hi = d.back() + rho_max;
  const double width = hi - lo;
  if (!(width > 0.0))
    throw Error("estimate_spectral_bounds: spectrum has zero width "
                "(matrix is a multiple of the identity)");
  lo -= 0.005 * width;
  hi += 0.005 * width;
  return SpectralBounds(lo, hi);
}

// ------------------------------------------------------------------- solve
namespace {

EigenResult run_solve(const SparseSymMatrix& A, double alpha, double beta,
                      const LanczosConfig& cfg, OperatorKind kind) {
  cfg.validate(A.dim());
  if (!(alpha < beta)) throw IntervalError("solve: interval requires alpha < beta");

  const WallClock total;
  flz_ctx* ctx = Device::context();
  const std::uint64_t launches0 = flz_ctx_launch_count(ctx);
  const WallClock upload;
  (void)A.device();  // CSR -> SELL + H2D when not resident yet
  const double time_upload = upload.seconds();

  // the start block is host work (the reference's libstdc++ random stream, lanczos.cpp:78-103)
  // that depends on nothing else: it runs beside the device-side bounds estimate
  const auto r = static_cast<std::size_t>(cfg.block_size);
  std::future<DenseBlock> start_block = std::async(
      std::launch::async, [&A, r, seed = cfg.seed] { return init_block(A.dim(), r, seed); });

  const std::uint64_t mv0 = matvec_count();
  const WallClock pre;
  const SpectralBounds bounds = estimate_spectral_bounds(A, cfg.bounds_steps, cfg.seed);
  const double time_preproc = pre.seconds();
  const std::uint64_t mv1 = matvec_count();

  if (beta < bounds.lambda_min() || alpha > bounds.lambda_max())
    throw IntervalError("solve: interval [" + std::to_string(alpha) + ", " +
                        std::to_string(beta) + "] lies outside the estimated spectrum [" +
                        std::to_string(bounds.lambda_min()) + ", " +
                        std::to_string(bounds.lambda_max()) + "]");

  std::optional<ChebyshevFilter> filter;
  if (kind == OperatorKind::filtered) {
    filter = build_filter(bounds, alpha, beta, cfg.degree, cfg.epsilon, cfg.max_degree);
    if (cfg.jackson_damping) filter = filter->damped();   // opt-in, host side only
  }
  const BlockOperator op =
      filter ? BlockOperator::filtered(A, *filter) : BlockOperator::plain(A);

  const auto max_cols = static_cast<std::size_t>(cfg.resolved_max_dim(A.dim()));
  trace("solve: upload + bounds + filter", total);
  const WallClock t_init;
  DenseBlock start = local_rows(start_block.get(), A.dim());
  trace("solve: init_block (host)", t_init);
  const WallClock t_fact;
  LanczosFactorization st(op, std::move(start), max_cols);
  trace("solve: factorization setup", t_fact);
  const double norm_est = std::max(std::abs(bounds.lambda_min()), std::abs(bounds.lambda_max()));

  ExpandTimes times;
  EigenResult result;
  int checks = 0;
  bool converged = false;
  double time_check = 0.0, time_recover = 0.0;
  // The reference alternates expand(check_every) and check_convergence (lanczos.cpp:611-625).
  // Here the host-side checks run on worker threads, each on a snapshot of the state it
  // belongs to, while the device keeps taking block steps; checks are resolved strictly in
  // order, and the first one that reports convergence rolls the factorization back to its
  // snapshot (LanczosFactorization::rollback) before the eigenpairs are recovered.  Every
  // decision is therefore taken on exactly the state the reference would see: results, block
  // counts and matvec counts do not depend on the overlap (scripts/sync_vs_overlap.py).
  struct PendingCheck {
    LanczosFactorization::Snapshot snap;
    std::future<RitzSet> ritz;
  };
  std::deque<std::unique_ptr<PendingCheck>> queue;
  // (row-partitioned runs keep the sequential order: how far the device gets ahead of a
  // check depends on timing, and every rank must issue the same collectives)
  const bool overlap =
      std::getenv("FLZ_SYNC_CHECK") == nullptr && flz_ctx_nranks(Device::context()) == 1;
  // checks in flight: one per host core up to 16 (C1, 174 checks of up to 1 740 x 1 740
  // projected problems on a 16-core host: 2 -> 1.98 s, 4 -> 1.37, 8 -> 0.98, 12 -> 0.89,
  // 16 -> 0.89 s per solve)
  std::size_t max_depth =
      overlap ? std::max(1u, std::min(16u, std::thread::hardware_concurrency())) : 0;
  if (const char* e = std::getenv("FLZ_CHECK_DEPTH"))   // experiments: checks in flight
    if (overlap && std::atoi(e) > 0) max_depth = static_cast<std::size_t>(std::atoi(e));
  auto enqueue = [&] {
    auto p = std::make_unique<PendingCheck>();
    p->snap = st.snapshot();
    const LanczosFactorization::Snapshot* snap = &p->snap;
    p->ritz = std::async(overlap ? std::launch::async : std::launch::deferred, [=, &cfg] {
      return check_convergence(*snap, alpha, beta, cfg.tol, cfg.extra_ritz);
    });
    queue.push_back(std::move(p));
  };
  bool can_expand = true;
  int since_check = 0;
  double waited = 0.0;
  while (!converged && (can_expand || !queue.empty())) {
    // resolve finished checks, oldest first; block on the oldest when nothing else can be done
    while (!queue.empty()) {
      PendingCheck& front = *queue.front();
      const bool must_wait = !can_expand || queue.size() > max_depth;
      if (!must_wait &&
          front.ritz.wait_for(std::chrono::seconds(0)) != std::future_status::ready)
        break;
      const WallClock w;
      const RitzSet ritz = front.ritz.get();
      waited += w.seconds();
      ++checks;
      const LanczosFactorization::Snapshot snap = std::move(front.snap);
      queue.pop_front();
      if (!ritz.converged) continue;
      queue.clear();  // younger checks belong to states that are rolled back now
      st.rollback(snap);
      can_expand = true;
      since_check = 0;
      const WallClock rec;
      result = recover_eigenpairs(st, A, alpha, beta, ritz, norm_est, cfg.return_vectors);
      time_recover += rec.seconds();
      // accept only when every TRUE residual meets the tolerance (:617-623)
      converged = std::all_of(result.residuals.begin(), result.residuals.end(),
                              [&](double res) { return res <= cfg.tol; });
      if (converged) break;
    }
    if (converged || !can_expand) continue;
    if (expand(st, 1, &times) == 0) {
      can_expand = false;  // budget or space exhausted
      if (since_check > 0) enqueue();
      since_check = 0;
    } else if (++since_check == cfg.check_every) {
      enqueue();
      since_check = 0;
    }
  }
  queue.clear();
  time_check = waited;
  if (!converged) {  // budget or space exhausted: best pairs of the final state (:627-632)
    const WallClock chk;
    const RitzSet ritz = check_convergence(st, alpha, beta, cfg.tol, cfg.extra_ritz);
    time_check += chk.seconds();
    const WallClock rec;
    result = recover_eigenpairs(st, A, alpha, beta, ritz, norm_est, cfg.return_vectors);
    time_recover += rec.seconds();
  }

  trace("solve: total", total);
  const std::uint64_t mv2 = matvec_count();
  SolveStats& s = result.stats;
  s.block_steps = static_cast<int>(st.block_count());
  s.basis_vectors = static_cast<int>(st.basis_size());
  s.degree = filter ? filter->degree() : 0;
  s.mv_bounds = mv1 - mv0;
  s.mv_iteration = mv2 - mv1;
  s.mv_total = mv2 - mv0;
  s.time_preproc_s = time_preproc;
  s.time_orth_s = times.orth_s;
  s.time_mv_s = times.mv_s;
  s.checks = checks;
  s.converged = converged;
  s.breakdown_replacements = st.had_breakdown();
  s.degree_clamped = filter ? filter->degree_clamped() : false;
  s.norm_estimate = norm_est;
  s.lambda_min_est = bounds.lambda_min();
  s.lambda_max_est = bounds.lambda_max();
  if (cfg.collect_diagnostics) s.ortho_error = st.ortho_error();
  s.time_check_s = time_check;
  s.time_recover_s = time_recover;
  s.time_upload_s = time_upload;
  s.gpu_launches = flz_ctx_launch_count(ctx) - launches0;
  s.time_total_s = total.seconds();
  return result;
}

}  // namespace

EigenResult filtered_lanczos(const SparseSymMatrix& A, double alpha, double beta,
                             const LanczosConfig& config) {
  return run_solve(A, alpha, beta, config, OperatorKind::filtered);
}

EigenResult plain_lanczos(const SparseSymMatrix& A, double alpha, double beta,
                          const LanczosConfig& config) {
  return run_solve(A, alpha, beta, config, OperatorKind::plain);
}

}  // namespace flz
