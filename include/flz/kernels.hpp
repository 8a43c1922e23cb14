// flz/kernels.hpp — the reference's low-level kernel seam (speig/kernels.hpp:15-49) on the
// device: same names, argument meaning and backend switch, so that call sites and tests
// written against `speig::kernels` compile unchanged with `namespace speig = flz;`.
//
// The reference has two interchangeable CPU backends, a strictly sequential scalar one and an
// AVX2 one that reassociates sums.  The device library has the same pair of behaviours:
//   Backend::scalar -> EXACT mode (flz_ctx_set_exact): CSR-order, separately rounded
//                      multiply/add — bit-identical to the reference's scalar backend;
//   Backend::avx2   -> the fast production kernels (FMA, layout-order sums), which agree with
//                      the scalar results to the tolerance the reference's own cross-backend
//                      tests use (1e-13, kernels_test.cpp:60-92).
// These are HOST-pointer seams (every call moves its operands to the GPU and back): they exist
// for tests and for code that pokes the kernels directly, not for the solver, which keeps all
// blocks resident (flz/solver.hpp).  Header-only over the C ABI in flz.h.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "flz.h"
#include "flz/matrix.hpp"

namespace flz::kernels {

enum class Backend { scalar, avx2 };

namespace detail {
inline Backend& current() {
  static Backend b = Backend::avx2;   // the reference defaults to avx2 where it is available
  return b;
}
inline void check(int status) {
  if (status != FLZ_OK) throw Error(std::string("kernels: ") + flz_last_error());
}
}  // namespace detail

// The fast device path always exists (there is no CPU fallback to be unavailable).
inline bool avx2_available() { return true; }
inline Backend active_backend() { return detail::current(); }
inline void set_backend(Backend b) {
  detail::check(flz_ctx_set_exact(Device::context(), b == Backend::scalar ? 1 : 0));
  detail::current() = b;
}
inline const char* backend_name(Backend b) { return b == Backend::scalar ? "scalar" : "avx2"; }

// sum_i x[i]*y[i]
inline double dot(const double* x, const double* y, std::size_t n) {
  double out = 0.0;
  if (n) detail::check(flz_dot(Device::context(), x, y, (std::int64_t)n, &out));
  return out;
}
inline double nrm2(const double* x, std::size_t n) { return std::sqrt(dot(x, x, n)); }
// y += a*x
inline void axpy(double a, const double* x, double* y, std::size_t n) {
  if (n) detail::check(flz_axpy(Device::context(), a, x, y, (std::int64_t)n));
}
// out[i] = s1*w[i] + s2*y1[i] - y2[i] + b*x[i]; `out` may alias `y2`
inline void clenshaw_combine(std::size_t n, double s1, double s2, double b, const double* w,
                             const double* y1, const double* y2, const double* x, double* out) {
  if (n)
    detail::check(flz_clenshaw_combine(Device::context(), (std::int64_t)n, s1, s2, b, w, y1, y2, x, out));
}
// x *= a  (a*x + 0*x - 0 + 0*x on the device: the combine with zero operands)
inline void scal(double a, double* x, std::size_t n) {
  if (!n) return;
  const std::vector<double> zero(n, 0.0);
  std::vector<double> out(n);
  clenshaw_combine(n, a, 0.0, 0.0, x, zero.data(), zero.data(), zero.data(), out.data());
  for (std::size_t i = 0; i < n; ++i) x[i] = out[i];
}
// y = A*x for CSR A with n rows (uploads A for this one product: a test seam)
inline void csr_matvec(std::size_t n, const std::int64_t* row_ptr, const std::int32_t* col_idx,
                       const double* values, const double* x, double* y) {
  if (!n) return;
  flz_ctx* ctx = Device::context();
  flz_matrix* A = nullptr;
  detail::check(flz_matrix_upload(ctx, (std::int64_t)n, 0, (std::int64_t)n, row_ptr, col_idx, values, 0, &A));
  const int status = flz_spmm(ctx, A, x, 1, y, /*counted=*/0);
  flz_matrix_destroy(A);
  detail::check(status);
}

}  // namespace flz::kernels
