// flz/matrix.hpp — host containers of the drop-in C++ API: errors, DenseBlock,
// SparseSymMatrix (+ Matrix Market I/O) and the device handle behind them.
//
// Mirrors the reference's speig/error.hpp:9-25, speig/dense_block.hpp:11-40 and
// speig/sparse.hpp:12-79 (same names, argument meaning and error behaviour); the
// arithmetic entry points (spmv / spmm_block / apply_uncounted) run on the GPU
// through the C ABI (include/flz.h) instead of kernels::csr_matvec.
//
// Multi-GPU: on a distributed context (flz_ctx_create_dist + Device::adopt) every n-vector
// argument of the block-level seams (spmm_block, ChebyshevFilter::apply, basis columns,
// EigenResult::eigenvectors) holds this rank's LOCAL rows only.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

struct flz_ctx;
struct flz_matrix;

namespace flz {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
struct ParseError : Error { using Error::Error; };      // malformed input file
struct IntervalError : Error { using Error::Error; };   // invalid / empty / outside interval
struct DimensionError : Error { using Error::Error; };  // shape mismatch
struct DeviceError : Error { using Error::Error; };     // CUDA / NCCL / no device

// Translates a C-ABI status into the exception the reference would throw.
void throw_status(int status);

// ------------------------------------------------------------------ device
// Process-wide default GPU context used by the C++ API (created on first use; there is
// no CPU fallback, so this throws DeviceError without an sm_100 GPU).
class Device {
 public:
  static flz_ctx* context();
  // Adopt an externally created context (e.g. a distributed one from flz_ctx_create_dist).
  static void adopt(flz_ctx* ctx);
  // tests only: the calling thread uses `ctx` (loopback ranks are threads); nullptr: undo
  static void adopt_thread(flz_ctx* ctx);
  static void set_device(int index);  // before first use
  static void shutdown();
  // Multi-GPU (one process per GPU): rank / size of the active context and the contiguous
  // block of rows this rank owns, [n*rank/size, n*(rank+1)/size).
  static int rank();
  static int nranks();
  static void row_range(std::size_t n, std::size_t& begin, std::size_t& end);
};

// -------------------------------------------------------------- DenseBlock
// Column-major rows x cols block, zero-initialised.
namespace detail {
// std::allocator whose construct() default-initialises: a vector<double, ...>(n) then leaves
// its storage untouched (no zero fill, no page faults before the first real write).
template <class T>
struct DefaultInitAllocator : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAllocator<U>;
  };
  using std::allocator<T>::allocator;
  template <class U>
  void construct(U* p) noexcept(std::is_nothrow_default_constructible_v<U>) {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};
}  // namespace detail

class DenseBlock {
 public:
  DenseBlock() = default;
  DenseBlock(std::size_t rows, std::size_t cols)
      : rows_(rows), cols_(cols), data_(rows * cols, 0.0) {}
  // storage the caller overwrites completely (device downloads): no zero fill
  static DenseBlock uninitialized(std::size_t rows, std::size_t cols) {
    DenseBlock B;
    B.rows_ = rows;
    B.cols_ = cols;
    B.data_ = Storage(rows * cols);
    return B;
  }
  // same, in page-locked host memory from the library's pool (flz_host_alloc): device
  // downloads then run at full PCIe rate and touch no fresh pageable pages.  Falls back to
  // ordinary storage when pinning fails.  Copies of such a block own ordinary storage.
  static DenseBlock pinned(std::size_t rows, std::size_t cols);
  // keeps the first `cols` columns (no reallocation, no copy); cols <= cols()
  void shrink_cols(std::size_t cols) {
    if (cols < cols_) {
      cols_ = cols;
      if (!ext_) data_.resize(rows_ * cols_);
    }
  }

  DenseBlock(const DenseBlock& o) : rows_(o.rows_), cols_(o.cols_) {
    if (o.ext_) data_.assign(o.ext_.get(), o.ext_.get() + o.size());
    else data_ = o.data_;
  }
  DenseBlock& operator=(const DenseBlock& o) {
    if (this != &o) *this = DenseBlock(o);
    return *this;
  }
  DenseBlock(DenseBlock&&) noexcept = default;
  DenseBlock& operator=(DenseBlock&&) noexcept = default;

  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  std::size_t size() const { return rows_ * cols_; }
  double* data() { return ext_ ? ext_.get() : data_.data(); }
  const double* data() const { return ext_ ? ext_.get() : data_.data(); }
  double* col(std::size_t j) { return data() + j * rows_; }
  const double* col(std::size_t j) const { return data() + j * rows_; }
  double& operator()(std::size_t i, std::size_t j) { return data()[j * rows_ + i]; }
  double operator()(std::size_t i, std::size_t j) const { return data()[j * rows_ + i]; }

  static DenseBlock identity(std::size_t n) {
    DenseBlock I(n, n);
    for (std::size_t i = 0; i < n; ++i) I(i, i) = 1.0;
    return I;
  }

 private:
  using Storage = std::vector<double, detail::DefaultInitAllocator<double>>;
  std::size_t rows_ = 0, cols_ = 0;
  Storage data_;
  std::shared_ptr<double> ext_;  // pinned pool block (data_ is empty then)
};

// ---------------------------------------------------------- SparseSymMatrix
struct Triplet {
  std::int64_t row;
  std::int64_t col;
  double value;
};

// Real symmetric CSR matrix, both triangles stored, exact symmetry enforced at
// construction, immutable afterwards.  The SELL-C-sigma device copy is created lazily on
// first arithmetic use and shared by all copies of the object.
class SparseSymMatrix {
 public:
  static SparseSymMatrix from_entries(std::size_t n, std::vector<Triplet> entries);
  // Adopts already validated CSR arrays (sorted, duplicate-free, exactly symmetric) —
  // used by generators that build CSR directly; `check` re-verifies symmetry.
  static SparseSymMatrix from_csr(std::size_t n, std::vector<std::int64_t> row_ptr,
                                  std::vector<std::int32_t> col_idx, std::vector<double> values,
                                  bool check = true);

  // Distributed construction: this rank's rows [row_begin, row_begin + row_ptr.size() - 1) of
  // an n_global x n_global matrix (global column ids).  Symmetry cannot be verified locally
  // and is the caller's responsibility; dim() is the global dimension.
  static SparseSymMatrix from_local_rows(std::size_t n_global, std::size_t row_begin,
                                         std::vector<std::int64_t> row_ptr,
                                         std::vector<std::int32_t> col_idx,
                                         std::vector<double> values);
  bool is_local_slab() const { return slab_; }
  std::size_t local_begin() const { return row_begin_; }

  std::size_t dim() const { return n_; }
  std::size_t nnz() const { return static_cast<std::size_t>(row_ptr_.back()); }
  const std::vector<std::int64_t>& row_ptr() const { return row_ptr_; }
  const std::vector<std::int32_t>& col_idx() const { return col_idx_; }
  const std::vector<double>& values() const { return values_; }
  double max_abs() const { return max_abs_; }

  void spmv(const double* x, double* y) const;                      // counted (+1)
  std::vector<double> spmv(const std::vector<double>& x) const;
  void spmm_block(const DenseBlock& X, DenseBlock& Y) const;        // counted (+X.cols())
  DenseBlock spmm_block(const DenseBlock& X) const;
  void apply_uncounted(const double* x, double* y) const;

  // Device handle on the default context (uploads on first call).
  flz_matrix* device() const;

 private:
  SparseSymMatrix() = default;
  void verify_symmetry() const;

  std::size_t n_ = 0;
  std::size_t row_begin_ = 0;  // first row held (slab mode)
  bool slab_ = false;
  std::vector<std::int64_t> row_ptr_{0};
  std::vector<std::int32_t> col_idx_;
  std::vector<double> values_;
  double max_abs_ = 0.0;
  struct DeviceCopy;
  mutable std::shared_ptr<DeviceCopy> dev_;
  // Device layout built ahead of the first use: from_csr plans a large matrix on host threads
  // beside its symmetry check (single-GPU contexts); device() uploads it and drops it.
  struct Planned;
  mutable std::shared_ptr<Planned> planned_;
};

// Matrix Market coordinate files (real / integer / pattern, general / symmetric), with the
// reference's rules and error messages (sparse.cpp:119-291).  The file is parsed by all host
// threads (csrc/host/mmio.cpp).  When the environment variable FLZ_MM_CACHE names a directory
// (or is "1": next to the file), the validated CSR arrays are kept there as a binary image
// keyed by the file's size and modification time and later loads read that instead.
SparseSymMatrix load_matrix_market(const std::string& path);
void save_matrix_market(const SparseSymMatrix& A, const std::string& path);
// Binary CSR image (extension): header + row_ptr (int64) + col_idx (int32) + values (f64).
// load_binary_csr trusts the image's symmetry (it was validated when the image was written)
// but re-checks its structure.
void save_binary_csr(const SparseSymMatrix& A, const std::string& path);
SparseSymMatrix load_binary_csr(const std::string& path);
void save_dense_matrix_market(const DenseBlock& X, const std::string& path);

std::uint64_t matvec_count();
void reset_matvec_count();

}  // namespace flz
