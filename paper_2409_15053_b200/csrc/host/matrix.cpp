// host/matrix.cpp — SparseSymMatrix, Matrix Market I/O, default device context.
//
// Behavioural contract: speig/sparse.hpp + src/sparse.cpp (from_entries :27-85, spmv /
// spmm_block / apply_uncounted :87-117, Matrix Market reader :172-291 and writers
// :293-331) and speig/error.hpp.  Products run on the GPU via include/flz.h.

#include "flz/matrix.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <atomic>
#include <mutex>
#include <thread>

#include "flz.h"

namespace flz {

// ------------------------------------------------------------ status -> throw
void throw_status(int status) {
  if (status == FLZ_OK) return;
  const std::string msg = flz_last_error();
  switch (status) {
    case FLZ_EDIM: throw DimensionError(msg);
    case FLZ_EINTERVAL: throw IntervalError(msg);
    case FLZ_EPARSE: throw ParseError(msg);
    case FLZ_ECUDA:
    case FLZ_ENODEV:
    case FLZ_ENCCL:
    case FLZ_ENOMEM: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

// ------------------------------------------------------------------ Device
namespace {
std::mutex g_dev_mutex;
flz_ctx* g_ctx = nullptr;
bool g_ctx_owned = false;
int g_dev_index = -1;
thread_local flz_ctx* t_ctx = nullptr;   // tests: per-thread override (loopback ranks)
}  // namespace

// FLZ_PLAN_AHEAD=0: the device layout is built at the first product (experiments)
static bool g_plan_ahead_off() {
  static const bool off = [] {
    const char* e = std::getenv("FLZ_PLAN_AHEAD");
    return e && e[0] == '0';
  }();
  return off;
}

void Device::adopt_thread(flz_ctx* ctx) { t_ctx = ctx; }
flz_ctx* Device::context() {
  if (t_ctx) return t_ctx;
  std::lock_guard<std::mutex> lock(g_dev_mutex);
  if (!g_ctx) {
    throw_status(flz_ctx_create(g_dev_index, &g_ctx));
    g_ctx_owned = true;
  }
  return g_ctx;
}
void Device::adopt(flz_ctx* ctx) {
  std::lock_guard<std::mutex> lock(g_dev_mutex);
  if (g_ctx && g_ctx_owned) flz_ctx_destroy(g_ctx);
  g_ctx = ctx;
  g_ctx_owned = false;
}
void Device::set_device(int index) {
  std::lock_guard<std::mutex> lock(g_dev_mutex);
  g_dev_index = index;
}
int Device::rank() { return flz_ctx_rank(context()); }
int Device::nranks() { return flz_ctx_nranks(context()); }
void Device::row_range(std::size_t n, std::size_t& begin, std::size_t& end) {
  const auto r = static_cast<std::size_t>(rank()), p = static_cast<std::size_t>(nranks());
  begin = n * r / p;
  end = n * (r + 1) / p;
}

void Device::shutdown() {
  std::lock_guard<std::mutex> lock(g_dev_mutex);
  if (g_ctx && g_ctx_owned) flz_ctx_destroy(g_ctx);
  g_ctx = nullptr;
  g_ctx_owned = false;
}

// --------------------------------------------------------- SparseSymMatrix
struct SparseSymMatrix::DeviceCopy {
  flz_matrix* handle = nullptr;
  flz_ctx* ctx = nullptr;
  ~DeviceCopy() {
    if (handle) flz_matrix_destroy(handle);
  }
};

struct SparseSymMatrix::Planned {
  flz_plan* plan = nullptr;
  ~Planned() {
    if (plan) flz_plan_destroy(plan);
  }
};

namespace {
bool coord_less(const Triplet& a, const Triplet& b) {
  return a.row < b.row || (a.row == b.row && a.col < b.col);
}
}  // namespace

SparseSymMatrix SparseSymMatrix::from_entries(std::size_t n, std::vector<Triplet> entries) {
  const auto dim = static_cast<std::int64_t>(n);
  for (const Triplet& t : entries) {
    if (t.row < 0 || t.col < 0 || t.row >= dim || t.col >= dim)
      throw Error("matrix entry index out of range");
    if (!std::isfinite(t.value)) throw Error("matrix entry is not finite");
  }
  std::sort(entries.begin(), entries.end(), coord_less);

  SparseSymMatrix A;
  A.n_ = n;
  A.row_ptr_.assign(n + 1, 0);
  A.col_idx_.reserve(entries.size());
  A.values_.reserve(entries.size());
  // merge runs of equal coordinates while emitting CSR
  for (std::size_t i = 0; i < entries.size();) {
    double sum = entries[i].value;
    std::size_t j = i + 1;
    while (j < entries.size() && entries[j].row == entries[i].row &&
           entries[j].col == entries[i].col)
      sum += entries[j++].value;
    A.row_ptr_[entries[i].row + 1] += 1;
    A.col_idx_.push_back(static_cast<std::int32_t>(entries[i].col));
    A.values_.push_back(sum);
    A.max_abs_ = std::max(A.max_abs_, std::abs(sum));
    i = j;
  }
  for (std::size_t i = 0; i < n; ++i) A.row_ptr_[i + 1] += A.row_ptr_[i];
  A.verify_symmetry();
  return A;
}

namespace {
// rows [0, n) in contiguous chunks on up to 16 threads; the first exception is rethrown
template <class F>
void parallel_rows(std::size_t n, F&& body) {
  unsigned workers = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (const char* e = std::getenv("FLZ_HOST_THREADS")) workers = std::max(1, std::atoi(e));
  workers = (unsigned)std::min<std::size_t>(workers, n / 4096 + 1);
  if (workers <= 1) {
    body(std::size_t(0), n);
    return;
  }
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  for (unsigned t = 0; t < workers; ++t)
    pool.emplace_back([&, t] {
      try {
        body(n * t / workers, n * (t + 1) / workers);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}
}  // namespace

SparseSymMatrix SparseSymMatrix::from_csr(std::size_t n, std::vector<std::int64_t> row_ptr,
                                          std::vector<std::int32_t> col_idx,
                                          std::vector<double> values, bool check) {
  if (row_ptr.size() != n + 1 || row_ptr.front() != 0 ||
      static_cast<std::size_t>(row_ptr.back()) != col_idx.size() ||
      col_idx.size() != values.size())
    throw Error("from_csr: inconsistent CSR arrays");
  SparseSymMatrix A;
  A.n_ = n;
  A.row_ptr_ = std::move(row_ptr);
  A.col_idx_ = std::move(col_idx);
  A.values_ = std::move(values);
  // First bad row (if any) is reported exactly as a sequential scan would report it.
  std::mutex mu;
  std::size_t bad_row = n;
  const char* bad_msg = nullptr;
  double max_abs = 0.0;
  parallel_rows(n, [&](std::size_t r0, std::size_t r1) {
    double local_max = 0.0;
    for (std::size_t i = r0; i < r1; ++i) {
      const char* msg = nullptr;
      if (A.row_ptr_[i] > A.row_ptr_[i + 1] || A.row_ptr_[i] < 0 ||
          static_cast<std::size_t>(A.row_ptr_[i + 1]) > A.col_idx_.size())
        msg = "from_csr: row_ptr is not monotone";
      for (std::int64_t p = A.row_ptr_[i]; !msg && p < A.row_ptr_[i + 1]; ++p) {
        const std::int32_t c = A.col_idx_[p];
        if (c < 0 || static_cast<std::size_t>(c) >= n) msg = "matrix entry index out of range";
        else if (p > A.row_ptr_[i] && A.col_idx_[p - 1] >= c)
          msg = "from_csr: columns must be strictly ascending within a row";
        else if (!std::isfinite(A.values_[p])) msg = "matrix entry is not finite";
        else local_max = std::max(local_max, std::abs(A.values_[p]));
      }
      if (msg) {
        std::lock_guard<std::mutex> lock(mu);
        if (i < bad_row) {
          bad_row = i;
          bad_msg = msg;
        }
        break;
      }
    }
    std::lock_guard<std::mutex> lock(mu);
    max_abs = std::max(max_abs, local_max);
  });
  if (bad_msg) throw Error(bad_msg);
  A.max_abs_ = max_abs;
  // Large matrices headed for a single-GPU context: the device layout (csrc/host/plan.cpp, host
  // threads only) is built now, beside the symmetry check, instead of at the first product.
  // The arrays are structurally valid at this point, which is all the planner needs; a
  // planning failure is not an error here — device() then plans again and reports it.
  const bool plan_now = A.col_idx_.size() >= (std::size_t(1) << 20) && !g_plan_ahead_off() &&
                        (g_ctx == nullptr || flz_ctx_nranks(g_ctx) == 1);
  std::shared_ptr<Planned> planned;
  std::thread planner;
  if (plan_now)
    planner = std::thread([&] {
      const std::int64_t starts[2] = {0, static_cast<std::int64_t>(n)};
      auto P = std::make_shared<Planned>();
      if (flz_plan_create(static_cast<std::int64_t>(n), 0, 1, starts, A.row_ptr_.data(),
                          A.col_idx_.data(), A.values_.data(), 0, &P->plan) == FLZ_OK)
        planned = std::move(P);
    });
  struct Join {
    std::thread& t;
    ~Join() {
      if (t.joinable()) t.join();
    }
  } join{planner};
  if (check) A.verify_symmetry();
  if (planner.joinable()) planner.join();
  A.planned_ = std::move(planned);
  return A;
}

SparseSymMatrix SparseSymMatrix::from_local_rows(std::size_t n_global, std::size_t row_begin,
                                                 std::vector<std::int64_t> row_ptr,
                                                 std::vector<std::int32_t> col_idx,
                                                 std::vector<double> values) {
  if (row_ptr.empty() || row_ptr.front() != 0 ||
      static_cast<std::size_t>(row_ptr.back()) != col_idx.size() ||
      col_idx.size() != values.size() || row_begin + row_ptr.size() - 1 > n_global)
    throw Error("from_local_rows: inconsistent CSR arrays");
  SparseSymMatrix A;
  A.n_ = n_global;
  A.row_begin_ = row_begin;
  A.slab_ = true;
  A.row_ptr_ = std::move(row_ptr);
  A.col_idx_ = std::move(col_idx);
  A.values_ = std::move(values);
  for (std::size_t p = 0; p < A.values_.size(); ++p) {
    if (A.col_idx_[p] < 0 || static_cast<std::size_t>(A.col_idx_[p]) >= n_global)
      throw Error("matrix entry index out of range");
    if (!std::isfinite(A.values_[p])) throw Error("matrix entry is not finite");
    A.max_abs_ = std::max(A.max_abs_, std::abs(A.values_[p]));
  }
  return A;
}

// exact structural + numerical symmetry (sparse.cpp:65-83): every upper entry (i,j) must
// have an equal mirror (j,i) — like the reference, lower entries are not looked up.  The
// reference's binary search per entry, threaded over rows; on a mismatch the sequential scan
// runs, so the entry the reference would report is the one reported.
void SparseSymMatrix::verify_symmetry() const {
  std::atomic<bool> ok{true};
  // Thread t owns the mirror rows j in [J0, J1).  It walks the rows i < J1 in ascending order
  // and, for every upper entry (i, j) with j in its range, advances row j's cursor to column
  // i: the mirrors of one row are asked for in ascending column order, so a cursor per row
  // replaces the reference's binary search per entry (one random access instead of ~7).
  // Lower entries without an upper partner are skipped, as the reference never looks them up.
  unsigned workers = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (const char* e = std::getenv("FLZ_HOST_THREADS")) workers = std::max(1, std::atoi(e));
  workers = (unsigned)std::min<std::size_t>(workers, n_ / 4096 + 1);
  // ranges of mirror rows with equal shares of the nonzeros
  std::vector<std::size_t> cut(workers + 1, n_);
  cut[0] = 0;
  for (unsigned t = 1; t < workers; ++t) {
    const std::int64_t want = row_ptr_[n_] / workers * t;
    cut[t] = std::lower_bound(row_ptr_.begin(), row_ptr_.end(), want) - row_ptr_.begin();
    cut[t] = std::min(std::max(cut[t], cut[t - 1]), n_);
  }
  auto body = [&](unsigned t) {
    const std::size_t J0 = cut[t], J1 = cut[t + 1];
    if (J0 >= J1) return;
    std::vector<std::int64_t> cursor(row_ptr_.begin() + J0, row_ptr_.begin() + J1);
    const std::int32_t lo = static_cast<std::int32_t>(J0), hi = static_cast<std::int32_t>(J1);
    for (std::size_t i = 0; i + 1 < J1 && ok.load(std::memory_order_relaxed); ++i) {
      const std::int32_t* first = col_idx_.data() + row_ptr_[i];
      const std::int32_t* last = col_idx_.data() + row_ptr_[i + 1];
      const std::int32_t from = std::max<std::int32_t>(lo, static_cast<std::int32_t>(i) + 1);
      for (const std::int32_t* q = std::lower_bound(first, last, from); q < last && *q < hi; ++q) {
        const std::size_t j = static_cast<std::size_t>(*q);
        std::int64_t& c = cursor[j - J0];
        const std::int64_t end = row_ptr_[j + 1];
        while (c < end && col_idx_[c] < static_cast<std::int32_t>(i)) ++c;
        if (c == end || col_idx_[c] != static_cast<std::int32_t>(i) ||
            values_[q - col_idx_.data()] != values_[c]) {
          ok.store(false, std::memory_order_relaxed);
          return;
        }
      }
    }
  };
  if (workers <= 1) {
    body(0);
  } else {
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < workers; ++t) pool.emplace_back(body, t);
    for (auto& th : pool) th.join();
  }
  if (ok) return;
  for (std::size_t i = 0; i < n_; ++i)
    for (std::int64_t p = row_ptr_[i]; p < row_ptr_[i + 1]; ++p) {
      const auto j = static_cast<std::size_t>(col_idx_[p]);
      if (j <= i) continue;
      const std::int32_t* first = col_idx_.data() + row_ptr_[j];
      const std::int32_t* last = col_idx_.data() + row_ptr_[j + 1];
      const std::int32_t* hit = std::lower_bound(first, last, static_cast<std::int32_t>(i));
      if (hit == last || *hit != static_cast<std::int32_t>(i))
        throw Error("matrix is structurally asymmetric at (" + std::to_string(i) + "," +
                    std::to_string(j) + ")");
      if (values_[p] != values_[row_ptr_[j] + (hit - first)])
        throw Error("matrix is numerically asymmetric at (" + std::to_string(i) + "," +
                    std::to_string(j) + ")");
    }
}

DenseBlock DenseBlock::pinned(std::size_t rows, std::size_t cols) {
  void* p = nullptr;
  // Larger blocks stay pageable: page-locking hundreds of MB takes ~0.25 s and stalls every
  // other CUDA call of the process meanwhile (measured on the first solves of C2), whereas
  // pre-faulted pageable memory downloads at ~19 GB/s.
  constexpr std::size_t kMaxPinned = std::size_t(64) << 20;
  const std::size_t bytes = rows * cols * sizeof(double);
  if (bytes == 0 || bytes > kMaxPinned || flz_host_alloc(bytes, &p) != FLZ_OK || !p) {
    // pageable: fault the pages in on several threads now (a device download into untouched
    // memory runs at page-fault speed, ~2 GB/s; measured 4.4 s for 8.9 GB of eigenvectors)
    DenseBlock B = uninitialized(rows, cols);
    double* base = B.data();
    const std::size_t count = rows * cols;
    parallel_rows(count / 512 + 1, [&](std::size_t p0, std::size_t p1) {
      for (std::size_t q = p0; q < p1 && q * 512 < count; ++q) base[q * 512] = 0.0;
    });
    return B;
  }
  DenseBlock B;
  B.rows_ = rows;
  B.cols_ = cols;
  B.ext_ = std::shared_ptr<double>(static_cast<double*>(p), [](double* q) { flz_host_free(q); });
  return B;
}

flz_matrix* SparseSymMatrix::device() const {
  flz_ctx* ctx = Device::context();
  if (!dev_ || dev_->ctx != ctx) {
    auto copy = std::make_shared<DeviceCopy>();
    copy->ctx = ctx;
    std::size_t b = 0, e = n_;
    Device::row_range(n_, b, e);
    const std::int64_t* rp = row_ptr_.data();
    if (slab_) {
      if (b != row_begin_ || e - b != row_ptr_.size() - 1)
        throw Error("SparseSymMatrix: the local row slab does not match this rank's row range");
    } else {
      rp += b;  // replicated global matrix: this rank's rows, absolute offsets
    }
    std::shared_ptr<Planned> planned = std::move(planned_);   // single use
    planned_.reset();
    if (planned && planned->plan && !slab_ && flz_ctx_nranks(ctx) == 1)
      throw_status(flz_matrix_upload_plan(ctx, planned->plan, &copy->handle));
    else
      throw_status(flz_matrix_upload(ctx, static_cast<std::int64_t>(n_),
                                     static_cast<std::int64_t>(b), static_cast<std::int64_t>(e),
                                     rp, col_idx_.data(), values_.data(), 0, &copy->handle));
    dev_ = std::move(copy);
  }
  return dev_->handle;
}

void SparseSymMatrix::apply_uncounted(const double* x, double* y) const {
  throw_status(flz_spmm(Device::context(), device(), x, 1, y, 0));
}
void SparseSymMatrix::spmv(const double* x, double* y) const {
  throw_status(flz_spmm(Device::context(), device(), x, 1, y, 1));
}
std::vector<double> SparseSymMatrix::spmv(const std::vector<double>& x) const {
  std::size_t b = 0, e = n_;
  Device::row_range(n_, b, e);
  if (x.size() != e - b)
    throw DimensionError("spmv: vector length " + std::to_string(x.size()) +
                         " does not match matrix dimension " + std::to_string(n_));
  std::vector<double> y(x.size());
  spmv(x.data(), y.data());
  return y;
}
void SparseSymMatrix::spmm_block(const DenseBlock& X, DenseBlock& Y) const {
  std::size_t b = 0, e = n_;
  Device::row_range(n_, b, e);
  if (X.rows() != e - b)
    throw DimensionError("spmm_block: block has " + std::to_string(X.rows()) +
                         " rows, matrix dimension is " + std::to_string(n_));
  if (Y.rows() != X.rows() || Y.cols() != X.cols()) Y = DenseBlock(X.rows(), X.cols());
  if (X.cols() == 0) return;
  throw_status(flz_spmm(Device::context(), device(), X.data(), static_cast<int>(X.cols()),
                        Y.data(), 1));
}
DenseBlock SparseSymMatrix::spmm_block(const DenseBlock& X) const {
  DenseBlock Y(X.rows(), X.cols());
  spmm_block(X, Y);
  return Y;
}

std::uint64_t matvec_count() { return flz_matvec_count(); }
void reset_matvec_count() { flz_reset_matvec_count(); }

// ------------------------------------------------------------ Matrix Market
namespace {

[[noreturn]] void parse_fail(const std::string& path, std::size_t line, const std::string& msg) {
  throw ParseError(path + ":" + std::to_string(line) + ": " + msg);
}

std::string lowered(std::string s) {
  for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

// Splits the file image into lines without copying (pointers into `text`).
struct LineCursor {
  const char* p;
  const char* end;
  std::size_t lineno = 0;
  bool next(const char*& b, const char*& e) {
    if (p >= end) return false;
    b = p;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
    e = nl ? nl : end;
    p = nl ? nl + 1 : end;
    ++lineno;
    return true;
  }
};

bool skippable(const char* b, const char* e) {
  for (; b < e; ++b) {
    if (*b == '%') return true;
    if (!std::isspace(static_cast<unsigned char>(*b))) return false;
  }
  return true;
}

enum class Field { real, integer, pattern };

}  // namespace

// The reference's loader, line by line (sparse.cpp:172-291): the fast loader in mmio.cpp
// produces the same matrix for well-formed files and hands every file it finds anything wrong
// with to this function, so that errors carry the reference's messages and line numbers.
namespace detail {
SparseSymMatrix load_matrix_market_sequential(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error("cannot open '" + path + "'");
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  text.push_back('\0');  // strto* need a terminator
  LineCursor cur{text.data(), text.data() + text.size() - 1};

  const char *b, *e;
  if (!cur.next(b, e)) throw ParseError(path + ": empty file");
  // banner: %%MatrixMarket matrix coordinate <field> <symmetry>
  std::string tok[5];
  {
    const char* q = b;
    for (int t = 0; t < 5; ++t) {
      while (q < e && std::isspace(static_cast<unsigned char>(*q))) ++q;
      const char* s = q;
      while (q < e && !std::isspace(static_cast<unsigned char>(*q))) ++q;
      tok[t].assign(s, q);
    }
  }
  if (lowered(tok[0]) != "%%matrixmarket")
    parse_fail(path, 1, "not a Matrix Market file (missing %%MatrixMarket banner)");
  if (lowered(tok[1]) != "matrix") parse_fail(path, 1, "unsupported object '" + tok[1] + "'");
  if (lowered(tok[2]) != "coordinate")
    parse_fail(path, 1, "unsupported format '" + tok[2] + "' (expected coordinate)");
  Field field = Field::real;
  const std::string f = lowered(tok[3]);
  if (f == "real") field = Field::real;
  else if (f == "integer") field = Field::integer;
  else if (f == "pattern") field = Field::pattern;
  else if (f == "complex") parse_fail(path, 1, "complex matrices are not supported");
  else parse_fail(path, 1, "unsupported field '" + tok[3] + "'");
  bool symmetric = false;
  const std::string s = lowered(tok[4]);
  if (s == "symmetric") symmetric = true;
  else if (s == "general") symmetric = false;
  else if (s == "skew-symmetric") parse_fail(path, 1, "skew-symmetric matrices are not supported");
  else if (s == "hermitian") parse_fail(path, 1, "hermitian matrices are not supported");
  else parse_fail(path, 1, "unsupported symmetry '" + tok[4] + "'");

  // size line
  std::int64_t rows = -1, cols = -1, declared = -1;
  while (cur.next(b, e)) {
    if (skippable(b, e)) continue;
    char* q = nullptr;
    const std::string line(b, e);
    const char* lp = line.c_str();
    rows = std::strtoll(lp, &q, 10);
    bool ok = q != lp;
    lp = q;
    if (ok) {
      cols = std::strtoll(lp, &q, 10);
      ok = q != lp;
      lp = q;
    }
    if (ok) {
      declared = std::strtoll(lp, &q, 10);
      ok = q != lp;
    }
    if (!ok) parse_fail(path, cur.lineno, "malformed size line (expected: rows cols nnz)");
    break;
  }
  if (rows < 0) throw ParseError(path + ": missing size line");
  if (rows != cols)
    throw ParseError(path + ": matrix is not square (" + std::to_string(rows) + "x" +
                     std::to_string(cols) + ")");
  if (declared < 0) throw ParseError(path + ": negative entry count");

  std::vector<Triplet> entries;
  entries.reserve(static_cast<std::size_t>(symmetric ? 2 * declared : declared));
  std::int64_t seen = 0;
  while (cur.next(b, e)) {
    if (skippable(b, e)) continue;
    if (seen == declared) parse_fail(path, cur.lineno, "more entries than declared in size line");
    // the line is terminated in place for strto* (restored afterwards)
    char* le = const_cast<char*>(e);
    const char saved = *le;
    *le = '\0';
    char* q = nullptr;
    const char* lp = b;
    const std::int64_t i = std::strtoll(lp, &q, 10);
    if (q == lp) parse_fail(path, cur.lineno, "malformed entry (row index)");
    lp = q;
    const std::int64_t j = std::strtoll(lp, &q, 10);
    if (q == lp) parse_fail(path, cur.lineno, "malformed entry (column index)");
    lp = q;
    double v = 1.0;
    if (field != Field::pattern) {
      v = std::strtod(lp, &q);
      if (q == lp) parse_fail(path, cur.lineno, "malformed entry (value)");
      lp = q;
    }
    while (*lp != '\0' && std::isspace(static_cast<unsigned char>(*lp))) ++lp;
    const bool trailing = *lp != '\0';
    *le = saved;
    if (trailing) parse_fail(path, cur.lineno, "trailing characters after entry");
    if (i < 1 || i > rows || j < 1 || j > cols)
      parse_fail(path, cur.lineno, "entry index out of range");
    if (symmetric && i < j) parse_fail(path, cur.lineno, "upper-triangle entry in symmetric file");
    if (!std::isfinite(v)) parse_fail(path, cur.lineno, "entry value is not finite");
    entries.push_back({i - 1, j - 1, v});
    if (symmetric && i != j) entries.push_back({j - 1, i - 1, v});
    ++seen;
  }
  if (seen != declared)
    throw ParseError(path + ": file ends after " + std::to_string(seen) + " of " +
                     std::to_string(declared) + " entries");

  if (!symmetric) {
    // general file: merge duplicates, require |a_ij - a_ji| <= 1e-12 max|A| and a
    // symmetric pattern, then replace both by their mean (sparse.cpp:236-287)
    std::sort(entries.begin(), entries.end(), coord_less);
    std::size_t out = 0;
    for (std::size_t i = 0; i < entries.size(); ++i) {
      if (out > 0 && entries[out - 1].row == entries[i].row &&
          entries[out - 1].col == entries[i].col)
        entries[out - 1].value += entries[i].value;
      else
        entries[out++] = entries[i];
    }
    entries.resize(out);
    double max_abs = 0.0;
    for (const Triplet& t : entries) max_abs = std::max(max_abs, std::abs(t.value));
    const double tol = 1e-12 * max_abs;
    auto mirror_of = [&](const Triplet& t) -> Triplet* {
      const Triplet key{t.col, t.row, 0.0};
      auto it = std::lower_bound(entries.begin(), entries.end(), key, coord_less);
      return (it != entries.end() && it->row == key.row && it->col == key.col) ? &*it : nullptr;
    };
    for (Triplet& t : entries) {
      if (t.row == t.col) continue;
      Triplet* m = mirror_of(t);
      const std::string where =
          "(" + std::to_string(t.row + 1) + "," + std::to_string(t.col + 1) + ")";
      if (t.row < t.col) {
        const double other = m ? m->value : 0.0;
        if (std::abs(t.value - other) > tol)
          throw Error(path + ": general matrix is not symmetric at " + where + ": " +
                      std::to_string(t.value) + " vs " + std::to_string(other));
        if (!m) throw Error(path + ": general matrix is structurally asymmetric at " + where);
        const double mean = 0.5 * (t.value + m->value);
        t.value = mean;
        m->value = mean;
      } else if (!m) {
        throw Error(path + ": general matrix is structurally asymmetric at " + where);
      }
    }
  }
  return SparseSymMatrix::from_entries(static_cast<std::size_t>(rows), std::move(entries));
}
}  // namespace detail

void save_matrix_market(const SparseSymMatrix& A, const std::string& path) {
  std::FILE* fp = std::fopen(path.c_str(), "w");
  if (!fp) throw Error("cannot open '" + path + "' for writing");
  const auto& rp = A.row_ptr();
  const auto& ci = A.col_idx();
  const auto& va = A.values();
  std::int64_t lower = 0;
  for (std::size_t i = 0; i < A.dim(); ++i)
    for (std::int64_t p = rp[i]; p < rp[i + 1]; ++p) lower += static_cast<std::size_t>(ci[p]) <= i;
  bool ok = std::fprintf(fp, "%%%%MatrixMarket matrix coordinate real symmetric\n%zu %zu %lld\n",
                         A.dim(), A.dim(), static_cast<long long>(lower)) > 0;
  // %.17g round-trips doubles exactly (sparse.cpp:293-315)
  for (std::size_t i = 0; i < A.dim() && ok; ++i)
    for (std::int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (static_cast<std::size_t>(ci[p]) <= i)
        ok = std::fprintf(fp, "%zu %d %.17g\n", i + 1, ci[p] + 1, va[p]) > 0 && ok;
  ok = std::fclose(fp) == 0 && ok;
  if (!ok) throw Error("write to '" + path + "' failed");
}

void save_dense_matrix_market(const DenseBlock& X, const std::string& path) {
  std::FILE* fp = std::fopen(path.c_str(), "w");
  if (!fp) throw Error("cannot open '" + path + "' for writing");
  bool ok = std::fprintf(fp, "%%%%MatrixMarket matrix array real general\n%zu %zu\n", X.rows(),
                         X.cols()) > 0;
  for (std::size_t j = 0; j < X.cols() && ok; ++j)
    for (std::size_t i = 0; i < X.rows(); ++i) ok = std::fprintf(fp, "%.17g\n", X(i, j)) > 0 && ok;
  ok = std::fclose(fp) == 0 && ok;
  if (!ok) throw Error("write to '" + path + "' failed");
}

}  // namespace flz
