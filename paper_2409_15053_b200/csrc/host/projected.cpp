// host/projected.cpp — banded symmetric eigenproblem of the projected matrix T_k (host).
//
// Behavioural contract: src/band_eig.cpp — SymBandMatrix :10-44, Givens band reduction
// :51-115, dense Householder reduction :119-180, dispatch :184-202, implicit-shift QL with
// a 30-sweep cap and ascending sort :204-283, sym_band_eig :285-291.
//
// Restructured for the GPU build: every orthogonal transformation is
// applied to an accumulator with an ARBITRARY number of rows.  With all `dim` rows this is
// the reference's full eigenvector computation; with the last r rows (+ rows of dead
// columns) it is all the periodic convergence check needs, at O(dim^2 r) instead of
// O(dim^3).  The band reduction works on a compact (2b+7)-wide window instead of a dense
// dim x dim embedding.

#include "flz/projected.hpp"
#include "spin_barrier.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <numeric>
#include <thread>

namespace flz {

namespace {
// Rows of an accumulator are independent under column transformations (rotations, reflectors):
// a recorded sequence applied to disjoint row ranges on several threads gives bit-identical
// results to the sequential order.  body(r0, r1) handles rows [r0, r1).
template <class F>
void parallel_rows(std::size_t rows, std::size_t work_per_row, F&& body) {
  unsigned threads = 1;
  if (rows >= 32 && rows * work_per_row >= (std::size_t)1 << 21) {
    unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (const char* e = std::getenv("FLZ_HOST_THREADS")) hw = (unsigned)std::max(1, std::atoi(e));
    threads = (unsigned)std::min<std::size_t>(hw, rows / 8);
  }
  if (threads <= 1) {
    body((std::size_t)0, rows);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&, t] { body(rows * t / threads, rows * (t + 1) / threads); });
  for (auto& th : pool) th.join();
}
}  // namespace

// ------------------------------------------------------------ SymBandMatrix
SymBandMatrix::SymBandMatrix(std::size_t dim, std::size_t semi_bandwidth)
    : dim_(dim), sb_(semi_bandwidth) {
  if (dim == 0) throw Error("SymBandMatrix: dimension must be positive");
  if (sb_ >= dim_ && dim_ > 1)
    throw Error("SymBandMatrix: semi-bandwidth must be smaller than the dimension");
  if (dim_ == 1) sb_ = 0;
  band_.assign((sb_ + 1) * dim_, 0.0);
}

double SymBandMatrix::get(std::size_t i, std::size_t j) const {
  const std::size_t lo = std::min(i, j), d = std::max(i, j) - lo;
  return d > sb_ ? 0.0 : band_[d * dim_ + lo];
}

void SymBandMatrix::set(std::size_t i, std::size_t j, double v) {
  const std::size_t lo = std::min(i, j), d = std::max(i, j) - lo;
  if (d > sb_) throw Error("SymBandMatrix::set outside the band");
  band_[d * dim_ + lo] = v;
}

DenseBlock SymBandMatrix::to_dense() const {
  DenseBlock A(dim_, dim_);
  for (std::size_t d = 0; d <= sb_; ++d)
    for (std::size_t i = 0; i + d < dim_; ++i) A(i + d, i) = A(i, i + d) = band_[d * dim_ + i];
  return A;
}

double SymBandMatrix::max_abs() const {
  double m = 0.0;
  for (std::size_t d = 0; d <= sb_; ++d)
    for (std::size_t i = 0; i + d < dim_; ++i) m = std::max(m, std::abs(band_[d * dim_ + i]));
  return m;
}

namespace {

// Right-multiplies the accumulator by a plane rotation of columns (p, p+1).
inline void rotate_columns(DenseBlock& G, std::size_t p, double c, double s) {
  double* gp = G.col(p);
  double* gq = G.col(p + 1);
  const std::size_t rows = G.rows();
  for (std::size_t i = 0; i < rows; ++i) {
    const double a = gp[i], b = gq[i];
    gp[i] = c * a + s * b;
    gq[i] = c * b - s * a;
  }
}

// Symmetric matrix restricted to |i-j| <= hw, both triangles stored explicitly.
class Window {
 public:
  Window(std::size_t n, std::size_t hw) : n_(n), hw_(hw), w_(2 * hw + 1), a_(n * w_, 0.0) {}
  double& at(std::size_t i, std::size_t j) { return a_[i * w_ + (j + hw_ - i)]; }

 private:
  std::size_t n_, hw_, w_;
  std::vector<double> a_;
};

// Rutishauser / Schwarz band reduction by Givens rotations with bulge chasing.
void reduce_band(const SymBandMatrix& M, std::vector<double>& d, std::vector<double>& e,
                 DenseBlock& G) {
  const std::size_t n = M.dim(), b = M.semi_bandwidth();
  const std::size_t half = b + 2, hw = b + 3;
  Window A(n, hw);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = i > b ? i - b : 0; j <= std::min(n - 1, i + b); ++j)
      A.at(i, j) = M.get(i, j);

  auto rotate = [&](std::size_t p, double c, double s) {
    const std::size_t q = p + 1;
    const std::size_t lo = p > half ? p - half : 0, hi = std::min(n - 1, q + half);
    for (std::size_t j = lo; j <= hi; ++j) {  // rows p, q
      const double x = A.at(p, j), y = A.at(q, j);
      A.at(p, j) = c * x + s * y;
      A.at(q, j) = c * y - s * x;
    }
    for (std::size_t i = lo; i <= hi; ++i) {  // columns p, q
      const double x = A.at(i, p), y = A.at(i, q);
      A.at(i, p) = c * x + s * y;
      A.at(i, q) = c * y - s * x;
    }
    rotate_columns(G, p, c, s);
  };

  for (std::size_t col = 0; col + 2 < n; ++col)
    for (std::size_t row = std::min(col + b, n - 1); row >= col + 2; --row) {
      // zero A(row, col) against A(row-1, col), then chase the bulge it creates b rows down
      std::size_t jj = col, ii = row;
      while (true) {
        const double head = A.at(ii - 1, jj), tail = A.at(ii, jj);
        if (tail != 0.0) {
          const double h = std::hypot(head, tail);
          rotate(ii - 1, head / h, tail / h);
          A.at(ii, jj) = 0.0;
          A.at(jj, ii) = 0.0;
        }
        if (ii + b >= n) break;
        jj = ii - 1;
        ii += b;
      }
    }
  d.resize(n);
  e.assign(n > 1 ? n - 1 : 0, 0.0);
  for (std::size_t i = 0; i < n; ++i) d[i] = A.at(i, i);
  for (std::size_t i = 0; i + 1 < n; ++i) e[i] = A.at(i + 1, i);
}

// Householder tridiagonalization of the dense embedding (wide bands).
void reduce_householder(const SymBandMatrix& M, std::vector<double>& d, std::vector<double>& e,
                        DenseBlock& G) {
  const std::size_t n = M.dim();
  DenseBlock A = M.to_dense();
  std::vector<double> v(n), p(n), w(n), vstore;
  std::vector<std::size_t> reflectors;
  vstore.reserve(n * n / 2 + n);
  // The trailing block's two passes per reflector (p = A22 v, then the rank-2 update) are split
  // over the columns of A22 by a team of threads: every element is computed by exactly the
  // operations of the sequential loops, so the result does not depend on the team size.
  unsigned team = 1;
  if (n >= 192) {
    unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    if (const char* env = std::getenv("FLZ_HOST_THREADS")) hw = (unsigned)std::max(1, std::atoi(env));
    team = std::min(hw, 8u);
  }
  SpinBarrier barrier(team);
  // shared per-reflector state, written by member 0 between barriers
  struct Step {
    std::size_t len = 0;
    double alpha = 0.0;
    bool apply = false, done = false;
  } step;
  auto member = [&](unsigned me) {
    for (std::size_t k = 0; k + 2 < n; ++k) {
      const std::size_t len = n - k - 1;
      if (me == 0) {
        step.len = len;
        step.apply = false;
        double sq = 0.0;
        for (std::size_t i = 0; i < len; ++i) {
          v[i] = A(k + 1 + i, k);
          sq += v[i] * v[i];
        }
        if (sq - v[0] * v[0] > 0.0) {  // something below the sub-diagonal
          const double norm = std::sqrt(sq);
          const double alpha = v[0] >= 0.0 ? -norm : norm;
          v[0] -= alpha;
          double vn = 0.0;
          for (std::size_t i = 0; i < len; ++i) vn += v[i] * v[i];
          vn = std::sqrt(vn);
          if (vn != 0.0) {
            for (std::size_t i = 0; i < len; ++i) v[i] /= vn;
            step.alpha = alpha;
            step.apply = true;
          }
        }
      }
      if (team > 1) barrier.wait();   // v and step are published
      if (!step.apply) {
        if (team > 1) barrier.wait();   // nobody reads `step` while member 0 rewrites it
        continue;
      }
      const std::size_t c0 = len * me / team, c1 = len * (me + 1) / team;
      // trailing block: A22 <- H A22 H with H = I - 2 v v^T
      for (std::size_t i = c0; i < c1; ++i) {
        double acc = 0.0;
        // A22 stays bitwise symmetric under the rank-2 update below, so row i is read as the
        // (contiguous) column i: same values, same summation order
        for (std::size_t j = 0; j < len; ++j) acc += A(k + 1 + j, k + 1 + i) * v[j];
        p[i] = acc;
      }
      if (team > 1) barrier.wait();   // p complete
      double vp = 0.0;                // every member: the same sum in the same order
      for (std::size_t i = 0; i < len; ++i) vp += v[i] * p[i];
      if (me == 0)
        for (std::size_t i = 0; i < len; ++i) w[i] = p[i] - vp * v[i];
      if (team > 1) barrier.wait();   // w complete
      for (std::size_t j = c0; j < c1; ++j)
        for (std::size_t i = 0; i < len; ++i)
          A(k + 1 + i, k + 1 + j) -= 2.0 * (v[i] * w[j] + w[i] * v[j]);
      if (team > 1) barrier.wait();   // update complete: member 0 may touch column k and v
      if (me == 0) {
        A(k + 1, k) = A(k, k + 1) = step.alpha;
        for (std::size_t i = k + 2; i < n; ++i) A(i, k) = A(k, i) = 0.0;
        reflectors.push_back(k);
        vstore.insert(vstore.end(), v.begin(), v.begin() + len);
      }
    }
  };
  if (team <= 1) {
    member(0);
  } else {
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < team; ++t) pool.emplace_back(member, t);
    member(0);
    for (auto& th : pool) th.join();
  }
  {
    // accumulator: G <- G diag(I, H), applied after the loop (rows in parallel)
    const std::size_t rows = G.rows();
    parallel_rows(rows, n * n, [&](std::size_t r0, std::size_t r1) {
      std::vector<double> gv(r1 - r0);
      std::size_t off = 0;
      for (std::size_t k : reflectors) {
        const std::size_t len = n - k - 1;
        const double* vk = vstore.data() + off;
        off += len;
        std::fill(gv.begin(), gv.end(), 0.0);
        for (std::size_t j = 0; j < len; ++j) {
          const double* gc = G.col(k + 1 + j);
          for (std::size_t i = r0; i < r1; ++i) gv[i - r0] += gc[i] * vk[j];
        }
        for (std::size_t j = 0; j < len; ++j) {
          double* gc = G.col(k + 1 + j);
          const double f = 2.0 * vk[j];
          for (std::size_t i = r0; i < r1; ++i) gc[i] -= gv[i - r0] * f;
        }
      }
    });
  }
  d.resize(n);
  e.assign(n > 1 ? n - 1 : 0, 0.0);
  for (std::size_t i = 0; i < n; ++i) d[i] = A(i, i);
  for (std::size_t i = 0; i + 1 < n; ++i) e[i] = A(i + 1, i);
}

// dispatch of band_eig.cpp:184-202 on an accumulator that is already initialised
void tridiagonalize_into(const SymBandMatrix& M, std::vector<double>& d, std::vector<double>& e,
                         DenseBlock& G) {
  const std::size_t n = M.dim(), b = M.semi_bandwidth();
  if (b <= 1 || n <= 2) {
    d.resize(n);
    e.assign(n > 1 ? n - 1 : 0, 0.0);
    for (std::size_t i = 0; i < n; ++i) d[i] = M.get(i, i);
    if (b >= 1)
      for (std::size_t i = 0; i + 1 < n; ++i) e[i] = M.get(i + 1, i);
  } else if (b >= n / 2) {
    reduce_householder(M, d, e, G);
  } else {
    reduce_band(M, d, e, G);
  }
}

DenseBlock selected_identity_rows(std::size_t dim, const std::vector<std::size_t>& rows) {
  DenseBlock G(rows.size(), dim);
  for (std::size_t t = 0; t < rows.size(); ++t) {
    if (rows[t] >= dim) throw Error("band_ritz_rows: row index out of range");
    G(t, rows[t]) = 1.0;
  }
  return G;
}

}  // namespace

void tridiagonalize(const SymBandMatrix& M, std::vector<double>& d, std::vector<double>& e,
                    DenseBlock& G) {
  G = DenseBlock::identity(M.dim());
  tridiagonalize_into(M, d, e, G);
}

void tridiag_eig(std::vector<double>& d, std::vector<double>& e, DenseBlock& G) {
  const std::size_t n = d.size();
  if (n == 0) return;
  if (G.rows() == 0 && G.cols() == 0) G = DenseBlock::identity(n);
  if (G.cols() != n) throw Error("tridiag_eig: accumulator has wrong shape");

  // off[i] couples i and i+1; off[n-1] is a zero sentinel
  std::vector<double> off(n, 0.0);
  std::copy(e.begin(), e.begin() + std::min(e.size(), n - 1), off.begin());
  const double eps = std::numeric_limits<double>::epsilon();

  // Tall accumulators (full eigenvector computations): the rotations are recorded and applied
  // to disjoint row ranges on several threads, in the recorded order — bit-identical to the
  // inline update.  Short ones (the periodic checks' few rows) are updated inline.
  struct Rot {
    std::size_t i;
    double c, s;
  };
  const bool defer = G.rows() >= 64;
  constexpr std::size_t kFlush = (std::size_t)1 << 17;
  std::vector<Rot> pending;
  auto flush = [&] {
    if (pending.empty()) return;
    parallel_rows(G.rows(), pending.size() * 4, [&](std::size_t r0, std::size_t r1) {
      for (const Rot& q : pending) {
        double* gi = G.col(q.i);
        double* gi1 = G.col(q.i + 1);
        for (std::size_t t = r0; t < r1; ++t) {
          const double hi = gi1[t];
          gi1[t] = q.s * gi[t] + q.c * hi;
          gi[t] = q.c * gi[t] - q.s * hi;
        }
      }
    });
    pending.clear();
  };
  for (std::size_t l = 0; l < n; ++l) {
    int sweeps = 0;
    while (true) {
      std::size_t m = l;  // first negligible coupling at or after l
      for (; m + 1 < n; ++m)
        if (std::abs(off[m]) <= eps * (std::abs(d[m]) + std::abs(d[m + 1]))) break;
      if (m == l) break;
      if (sweeps++ == 30)
        throw Error("tridiag_eig: eigenvalue " + std::to_string(l) +
                    " failed to converge after 30 sweeps");
      // Wilkinson-type shift from the leading 2x2, then one implicit QL sweep m -> l
      double g = (d[l + 1] - d[l]) / (2.0 * off[l]);
      double r = std::hypot(g, 1.0);
      g = d[m] - d[l] + off[l] / (g + std::copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0;
      bool deflated_early = false;
      for (std::size_t i = m; i-- > l;) {
        const double f = s * off[i];
        const double b = c * off[i];
        r = std::hypot(f, g);
        off[i + 1] = r;
        if (r == 0.0) {  // underflow: recover and restart this eigenvalue
          d[i + 1] -= p;
          off[m] = 0.0;
          deflated_early = true;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
        // columns (i, i+1) of the accumulator: [gi, gi1] <- [c gi - s gi1, s gi + c gi1]
        if (defer) {
          pending.push_back(Rot{i, c, s});
        } else {
          double* gi = G.col(i);
          double* gi1 = G.col(i + 1);
          const std::size_t rows = G.rows();
          for (std::size_t t = 0; t < rows; ++t) {
            const double hi = gi1[t];
            gi1[t] = s * gi[t] + c * hi;
            gi[t] = c * gi[t] - s * hi;
          }
        }
      }
      if (pending.size() >= kFlush) flush();
      if (deflated_early) continue;
      d[l] -= p;
      off[l] = g;
      off[m] = 0.0;
    }
  }

  flush();
  std::vector<std::size_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&d](std::size_t a, std::size_t b) { return d[a] < d[b]; });
  std::vector<double> sorted(n);
  DenseBlock Gs(G.rows(), n);
  for (std::size_t j = 0; j < n; ++j) {
    sorted[j] = d[order[j]];
    std::copy(G.col(order[j]), G.col(order[j]) + G.rows(), Gs.col(j));
  }
  d = std::move(sorted);
  G = std::move(Gs);
  e.assign(n > 1 ? n - 1 : 0, 0.0);
}

SymEig sym_band_eig(const SymBandMatrix& M) {
  std::vector<double> d, e;
  DenseBlock G;
  tridiagonalize(M, d, e, G);
  tridiag_eig(d, e, G);
  return SymEig{std::move(d), std::move(G)};
}

SymEig band_ritz_rows(const SymBandMatrix& M, const std::vector<std::size_t>& rows) {
  std::vector<double> d, e;
  DenseBlock G = selected_identity_rows(M.dim(), rows);
  if (rows.empty()) G = DenseBlock(0, M.dim());
  tridiagonalize_into(M, d, e, G);
  if (rows.empty()) {
    // tridiag_eig would replace an empty accumulator by the identity; use one dummy row
    DenseBlock dummy(1, M.dim());
    tridiag_eig(d, e, dummy);
    return SymEig{std::move(d), DenseBlock(0, M.dim())};
  }
  tridiag_eig(d, e, G);
  return SymEig{std::move(d), std::move(G)};
}

DenseBlock band_eigenvectors(const SymBandMatrix& M, const std::vector<double>& values,
                             const std::vector<std::size_t>& pick, double* max_residual,
                             double* max_ortho) {
  // Inverse iteration on the band: (M - theta I) x = b by banded LU with partial pivoting.
  // Eigenvalues closer than `cluster_tol` are treated as one cluster and their vectors are
  // Gram-Schmidt orthogonalised against each other after every solve.
  const std::size_t n = M.dim(), b = M.semi_bandwidth(), w = pick.size();
  DenseBlock W(n, w);
  const double scale = std::max(M.max_abs(), std::numeric_limits<double>::min());
  const double eps = std::numeric_limits<double>::epsilon();
  const double cluster_tol = 1e-3 * scale;
  const std::size_t kl = b, ku = b, ldab = 2 * kl + ku + 1;  // LAPACK-style band LU storage
  // clusters are independent of each other (only the vectors inside one are orthogonalised
  // against their predecessors): they are spread over host threads, each with its own
  // factorization buffers and a start-vector stream seeded by the cluster's first index, so the
  // result does not depend on the number of threads
  std::vector<std::size_t> cluster_start;
  for (std::size_t t = 0; t < w; ++t)
    if (t == 0 || std::abs(values[pick[t]] - values[pick[t - 1]]) > cluster_tol)
      cluster_start.push_back(t);
  cluster_start.push_back(w);
  auto run_clusters = [&](std::size_t c0, std::size_t c1) {
  std::vector<double> ab(ldab * n), rhs(n);
  std::vector<std::size_t> piv(n);
  auto AB = [&](std::size_t i, std::size_t j) -> double& {  // entry (i,j), |i-j| within band
    return ab[j * ldab + (kl + ku + i - j)];
  };
  for (std::size_t cl = c0; cl < c1; ++cl) {
  const std::size_t cluster_begin = cluster_start[cl];
  std::uint64_t lcg = 0x9E3779B97F4A7C15ULL * (cluster_begin + 1);
  auto next_unit = [&lcg]() {
    lcg = lcg * 6364136223846793005ULL + 1442695040888963407ULL;
    return (static_cast<double>(lcg >> 11) / 9007199254740992.0) - 0.5;
  };
  for (std::size_t t = cluster_begin; t < cluster_start[cl + 1]; ++t) {
    const double theta = values[pick[t]];
    // perturb the shift slightly inside a cluster so that the factorization differs
    const double shift = theta + (t - cluster_begin) * 10.0 * eps * scale;
    // factor M - shift*I
    std::fill(ab.begin(), ab.end(), 0.0);
    for (std::size_t j = 0; j < n; ++j)
      for (std::size_t i = j > ku ? j - ku : 0; i <= std::min(n - 1, j + kl); ++i)
        AB(i, j) = M.get(i, j) - (i == j ? shift : 0.0);
    for (std::size_t j = 0; j < n; ++j) {
      const std::size_t last = std::min(n - 1, j + kl);
      std::size_t p = j;
      for (std::size_t i = j + 1; i <= last; ++i)
        if (std::abs(AB(i, j)) > std::abs(AB(p, j))) p = i;
      piv[j] = p;
      const std::size_t cmax = std::min(n - 1, j + ku + kl);
      if (p != j)
        for (std::size_t c = j; c <= cmax; ++c) std::swap(AB(j, c), AB(p, c));
      if (AB(j, j) == 0.0) AB(j, j) = eps * scale;  // exactly singular pivot
      for (std::size_t i = j + 1; i <= last; ++i) {
        const double f = AB(i, j) / AB(j, j);
        AB(i, j) = f;
        if (f != 0.0)
          for (std::size_t c = j + 1; c <= cmax; ++c) AB(i, c) -= f * AB(j, c);
      }
    }
    double* x = W.col(t);
    for (std::size_t i = 0; i < n; ++i) x[i] = next_unit();
    for (int it = 0; it < 5; ++it) {
      // solve L U x = P b
      std::copy(x, x + n, rhs.begin());
      for (std::size_t j = 0; j < n; ++j) {
        if (piv[j] != j) std::swap(rhs[j], rhs[piv[j]]);
        const std::size_t last = std::min(n - 1, j + kl);
        for (std::size_t i = j + 1; i <= last; ++i) rhs[i] -= AB(i, j) * rhs[j];
      }
      for (std::size_t jj = n; jj-- > 0;) {
        rhs[jj] /= AB(jj, jj);
        const std::size_t first = jj > ku + kl ? jj - ku - kl : 0;
        for (std::size_t i = first; i < jj; ++i) rhs[i] -= AB(i, jj) * rhs[jj];
      }
      // orthogonalise inside the cluster, normalise
      for (int rep = 0; rep < 2; ++rep)
        for (std::size_t u = cluster_begin; u < t; ++u) {
          const double* y = W.col(u);
          double dot = 0.0;
          for (std::size_t i = 0; i < n; ++i) dot += y[i] * rhs[i];
          for (std::size_t i = 0; i < n; ++i) rhs[i] -= dot * y[i];
        }
      double nrm = 0.0;
      for (std::size_t i = 0; i < n; ++i) nrm += rhs[i] * rhs[i];
      nrm = std::sqrt(nrm);
      if (!(nrm > 0.0)) {
        for (std::size_t i = 0; i < n; ++i) rhs[i] = next_unit();
        nrm = 0.0;
        for (std::size_t i = 0; i < n; ++i) nrm += rhs[i] * rhs[i];
        nrm = std::sqrt(nrm);
      }
      for (std::size_t i = 0; i < n; ++i) x[i] = rhs[i] / nrm;
      // residual ||M x - theta x||
      double res = 0.0;
      for (std::size_t i = 0; i < n; ++i) {
        double acc = -theta * x[i];
        for (std::size_t j = i > b ? i - b : 0; j <= std::min(n - 1, i + b); ++j)
          acc += M.get(i, j) * x[j];
        res += acc * acc;
      }
      if (std::sqrt(res) <= 50.0 * eps * scale && it >= 1) break;
    }
  }
  }
  };
  {
    const std::size_t nclusters = cluster_start.size() - 1;
    unsigned threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (const char* e = std::getenv("FLZ_HOST_THREADS")) threads = (unsigned)std::max(1, std::atoi(e));
    threads = (unsigned)std::min<std::size_t>(threads, nclusters);
    if (threads <= 1 || w * n < 4096) {
      run_clusters(0, nclusters);
    } else {
      // contiguous cluster ranges of about equal vector counts
      std::vector<std::size_t> cut{0};
      for (unsigned th = 1; th < threads; ++th) {
        const std::size_t want = w * th / threads;
        std::size_t c = cut.back();
        while (c < nclusters && cluster_start[c] < want) ++c;
        cut.push_back(c);
      }
      cut.push_back(nclusters);
      std::vector<std::thread> pool;
      for (unsigned th = 0; th < threads; ++th)
        if (cut[th] < cut[th + 1])
          pool.emplace_back([&, th] { run_clusters(cut[th], cut[th + 1]); });
      for (auto& th : pool) th.join();
    }
  }
  // verification figures for the caller's fallback decision
  double worst_res = 0.0, worst_ortho = 0.0;
  for (std::size_t t = 0; t < w; ++t) {
    const double* x = W.col(t);
    const double theta = values[pick[t]];
    double res = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
      double acc = -theta * x[i];
      for (std::size_t j = i > b ? i - b : 0; j <= std::min(n - 1, i + b); ++j)
        acc += M.get(i, j) * x[j];
      res += acc * acc;
    }
    worst_res = std::max(worst_res, std::sqrt(res) / scale);
  }
  {
    std::vector<double> worst(64, 0.0);  // per chunk; a max is order independent
    const std::size_t chunks = worst.size();
    parallel_rows(chunks, w * w * n / chunks + 1, [&](std::size_t c0, std::size_t c1) {
      for (std::size_t c = c0; c < c1; ++c)
        for (std::size_t t = c; t < w; t += chunks)   // interleaved: equal work per chunk
          for (std::size_t u = 0; u <= t; ++u) {
            const double* x = W.col(t);
            const double* y = W.col(u);
            double dot = 0.0;
            for (std::size_t i = 0; i < n; ++i) dot += x[i] * y[i];
            worst[c] = std::max(worst[c], std::abs(dot - (t == u ? 1.0 : 0.0)));
          }
    });
    for (double v : worst) worst_ortho = std::max(worst_ortho, v);
  }
  if (max_residual) *max_residual = worst_res;
  if (max_ortho) *max_ortho = worst_ortho;
  return W;
}

}  // namespace flz
