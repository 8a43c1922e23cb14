// A program written against the reference's public API (speig/lanczos.hpp, speig/filter.hpp,
// speig/sparse.hpp, speig/kernels.hpp), compiled unchanged against the drop-in headers with
// one alias line.  `speig_user` runs the host-only part (no GPU);
// `speig_user solve` also solves on the device and pokes the kernel seam.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "flz/kernels.hpp"
#include "flz/solver.hpp"
namespace speig = flz;

static int fail(const char* what) {
  std::printf("FAIL %s\n", what);
  return 1;
}

int main(int argc, char** argv) {
  // diag(1..5) through from_entries, as lanczos_test.cpp builds it
  std::vector<speig::Triplet> t;
  for (int i = 0; i < 5; ++i) t.push_back({i, i, double(i + 1)});
  const speig::SparseSymMatrix A = speig::SparseSymMatrix::from_entries(5, t);
  if (A.dim() != 5 || A.nnz() != 5) return fail("from_entries");
  // auto degree anchors of the reference (filter_test.cpp:96-99)
  const speig::SpectralBounds unit(-1.0, 1.0);
  if (speig::build_filter(unit, 0.1, 0.3).degree() != 48) return fail("degree 48");
  if (speig::build_filter(unit, -1.0, -0.5).degree() != 10) return fail("degree 10");
  try {
    speig::build_filter(unit, 0.5, 0.1);
    return fail("IntervalError expected");
  } catch (const speig::IntervalError&) {
  }
  speig::LanczosConfig cfg;
  if (cfg.block_size != 3 || cfg.tol != 1e-10 || cfg.check_every != 10 || cfg.seed != 20177)
    return fail("LanczosConfig defaults");
  if (argc > 1 && std::strcmp(argv[1], "solve") == 0) {
    cfg.block_size = 1;
    const speig::EigenResult r = speig::filtered_lanczos(A, 1.5, 3.5, cfg);
    if (r.eigenvalues.size() != 2 || std::abs(r.eigenvalues[0] - 2.0) > 1e-9 ||
        std::abs(r.eigenvalues[1] - 3.0) > 1e-9 || !r.stats.converged)
      return fail("filtered_lanczos on diag(1..5)");
    if (r.stats.mv_iteration != (std::uint64_t)r.stats.degree * r.stats.block_steps)
      return fail("matvec accounting");
    // kernel seam with the backend switch (kernels_test.cpp:30-58)
    namespace k = speig::kernels;
    const std::vector<double> x{1, 2, 3, 4}, y{0.5, -1, 2, 0.25};
    k::set_backend(k::Backend::scalar);
    if (k::active_backend() != k::Backend::scalar || std::strcmp(k::backend_name(k::active_backend()), "scalar"))
      return fail("backend switch");
    if (k::dot(x.data(), y.data(), 4) != 1 * 0.5 - 2 + 6 + 1) return fail("dot");
    std::vector<double> z(y);
    k::axpy(2.0, x.data(), z.data(), 4);
    if (z[0] != 2.5 || z[3] != 8.25) return fail("axpy");
    k::scal(0.5, z.data(), 4);
    if (z[0] != 1.25) return fail("scal");
    std::vector<double> out(5);
    const std::vector<double> v{1, 1, 1, 1, 1};
    k::csr_matvec(5, A.row_ptr().data(), A.col_idx().data(), A.values().data(), v.data(), out.data());
    if (out[4] != 5.0) return fail("csr_matvec");
    k::set_backend(k::Backend::avx2);
    if (std::abs(k::nrm2(x.data(), 4) - std::sqrt(30.0)) > 1e-13) return fail("nrm2");
  }
  std::printf("OK\n");
  return 0;
}
