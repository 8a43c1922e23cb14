// flz/projected.hpp — the small projected (banded) eigenproblem, kept on the host as
// the north star prescribes.
//
// Mirrors speig/band_eig.hpp:13-51 (SymBandMatrix, tridiagonalize, tridiag_eig,
// sym_band_eig).  Added for the GPU build: band_ritz_rows(), which
// applies the SAME rotation sequence to a few selected rows of the accumulator only —
// the periodic convergence check needs nothing else (lanczos.cpp:354-369) — turning the
// O(dim^3) check into O(dim^2 r).
#pragma once

#include <cstddef>
#include <vector>

#include "flz/matrix.hpp"

namespace flz {

// Symmetric band matrix storing the diagonal and `semi_bandwidth` sub-diagonals.
class SymBandMatrix {
 public:
  SymBandMatrix(std::size_t dim, std::size_t semi_bandwidth);
  std::size_t dim() const { return dim_; }
  std::size_t semi_bandwidth() const { return sb_; }
  double get(std::size_t i, std::size_t j) const;  // 0 outside the band
  void set(std::size_t i, std::size_t j, double v);  // requires |i-j| <= semi_bandwidth
  DenseBlock to_dense() const;
  double max_abs() const;

 private:
  std::size_t dim_, sb_;
  std::vector<double> band_;  // band_[d*dim + i] = M(i+d, i)
};

// G^T M G = tridiag(d, e), G orthogonal (dim x dim).
void tridiagonalize(const SymBandMatrix& M, std::vector<double>& d, std::vector<double>& e,
                    DenseBlock& G);
// Implicit-shift QL with accumulation into the columns of G (any row count); ascending
// eigenvalues on return.  Throws Error after 30 sweeps without convergence.
void tridiag_eig(std::vector<double>& d, std::vector<double>& e, DenseBlock& G);

struct SymEig {
  std::vector<double> values;  // ascending
  DenseBlock vectors;          // dim x dim
};
SymEig sym_band_eig(const SymBandMatrix& M);

// Eigenvalues (ascending) plus the rows `rows` of the eigenvector matrix: result.vectors is
// rows.size() x dim with vectors(t, c) = W(rows[t], c).  Identical arithmetic to
// sym_band_eig restricted to those rows.
SymEig band_ritz_rows(const SymBandMatrix& M, const std::vector<std::size_t>& rows);

// Selected eigenvectors of M by inverse iteration on the band itself (shifted banded LU
// with partial pivoting, cluster re-orthogonalisation).  `values` are eigenvalues already
// computed by band_ritz_rows/sym_band_eig, `pick` the indices wanted.  Returns dim x
// pick.size(); `max_residual` receives max ||M w - theta w|| / max|M| for verification.
DenseBlock band_eigenvectors(const SymBandMatrix& M, const std::vector<double>& values,
                             const std::vector<std::size_t>& pick, double* max_residual,
                             double* max_ortho);

}  // namespace flz
