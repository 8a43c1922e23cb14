// host/mmio.cpp — fast Matrix Market ingest and the binary CSR cache.
//
// Contract: load_matrix_market() returns exactly the matrix the reference's loader builds
// (sparse.cpp:172-291 -> from_entries :27-85) and fails with exactly its messages.  The fast
// path below only handles files it finds nothing wrong with: the body is cut at line ends into
// one piece per host thread, every piece is parsed with std::from_chars, rows are bucketed by
// a counting pass + scatter, every row is sorted by column and duplicates are summed in file
// order.  Anything unusual — a malformed line, an index out of range, a count that differs
// from the size line, an asymmetric "general" file — sends the file to the sequential loader
// (matrix.cpp, detail::load_matrix_market_sequential), which reports it the reference's way.
#include <sys/mman.h>
#include <sys/stat.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "flz/matrix.hpp"

namespace flz {
namespace detail {
SparseSymMatrix load_matrix_market_sequential(const std::string& path);
}

namespace {

unsigned host_threads() {
  if (const char* e = std::getenv("FLZ_HOST_THREADS")) return (unsigned)std::max(1, std::atoi(e));
  return std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
}
template <class F>
void parallel_for(unsigned pieces, F&& body) {
  if (pieces <= 1) {
    body(0u);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < pieces; ++t) pool.emplace_back([&, t] { body(t); });
  for (auto& th : pool) th.join();
}

struct MappedFile {
  const char* data = nullptr;
  size_t size = 0;
  int fd = -1;
  struct stat st {};
  explicit MappedFile(const std::string& path) {
    fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) return;
    if (::fstat(fd, &st) != 0 || !S_ISREG(st.st_mode)) {
      ::close(fd);
      fd = -1;
      return;
    }
    size = (size_t)st.st_size;
    if (size == 0) return;
    void* p = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (p == MAP_FAILED) {
      ::close(fd);
      fd = -1;
      return;
    }
    ::madvise(p, size, MADV_SEQUENTIAL | MADV_WILLNEED);
    data = static_cast<const char*>(p);
  }
  ~MappedFile() {
    if (data) ::munmap(const_cast<char*>(data), size);
    if (fd >= 0) ::close(fd);
  }
  bool ok() const { return fd >= 0; }
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }
inline const char* skip_space(const char* p, const char* e) {
  while (p < e && is_space(*p)) ++p;
  return p;
}
// blank or comment line
inline bool skippable(const char* b, const char* e) {
  b = skip_space(b, e);
  return b == e || *b == '%';
}
// strtoll-compatible decimal integer (optional sign)
inline bool parse_int(const char*& p, const char* e, std::int64_t& v) {
  p = skip_space(p, e);
  const char* q = p;
  if (q < e && *q == '+') ++q;
  const auto r = std::from_chars(q, e, v, 10);
  if (r.ec != std::errc()) return false;
  p = r.ptr;
  return true;
}
// the decimal / scientific forms from_chars and strtod agree on; anything else (hex floats,
// "infinity", locale forms) is left to the sequential loader
inline bool parse_real(const char*& p, const char* e, double& v) {
  p = skip_space(p, e);
  const char* q = p;
  if (q < e && *q == '+') ++q;
  if (q < e && !(*q == '-' || *q == '.' || (*q >= '0' && *q <= '9'))) return false;
  const auto r = std::from_chars(q, e, v, std::chars_format::general);
  if (r.ec != std::errc()) return false;
  // strtod would continue into a hex float or a longer token: only accept a clean stop
  if (r.ptr < e && !is_space(*r.ptr)) return false;
  p = r.ptr;
  return true;
}

struct Banner {
  bool pattern = false, symmetric = false;
};
std::string lowered(const char* b, const char* e) {
  std::string s(b, e);
  for (char& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

struct Entry {
  std::int32_t col;
  std::int64_t seq;   // position in the file (duplicates are summed in file order)
  double value;
};

// Fast path; false = let the sequential loader handle (and report on) this file.
bool load_fast(const MappedFile& F, std::vector<std::int64_t>& row_ptr,
               std::vector<std::int32_t>& col_idx, std::vector<double>& values, std::size_t& n_out) {
  const char* p = F.data;
  const char* end = F.data + F.size;
  auto next_line = [&](const char*& b, const char*& e) {
    if (p >= end) return false;
    b = p;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
    e = nl ? nl : end;
    p = nl ? nl + 1 : end;
    return true;
  };
  const char *b, *e;
  if (!next_line(b, e)) return false;
  Banner bn;
  {
    std::string tok[5];
    const char* q = b;
    for (auto& t : tok) {
      q = skip_space(q, e);
      const char* s = q;
      while (q < e && !is_space(*q)) ++q;
      t = lowered(s, q);
    }
    if (tok[0] != "%%matrixmarket" || tok[1] != "matrix" || tok[2] != "coordinate") return false;
    if (tok[3] == "pattern") bn.pattern = true;
    else if (tok[3] != "real" && tok[3] != "integer") return false;
    if (tok[4] == "symmetric") bn.symmetric = true;
    else if (tok[4] != "general") return false;
  }
  std::int64_t rows = -1, cols = -1, declared = -1;
  while (next_line(b, e)) {
    if (skippable(b, e)) continue;
    const char* q = b;
    if (!parse_int(q, e, rows) || !parse_int(q, e, cols) || !parse_int(q, e, declared)) return false;
    break;
  }
  if (rows < 0 || rows != cols || declared < 0 || rows >= (std::int64_t(1) << 31)) return false;
  const std::int64_t n = rows;

  // ---- cut the body into pieces at line ends and parse them
  const char* body = p;
  const size_t body_size = (size_t)(end - body);
  const unsigned pieces = (unsigned)std::max<size_t>(1, std::min<size_t>(host_threads(), body_size / (1 << 20) + 1));
  std::vector<const char*> cut(pieces + 1, end);
  cut[0] = body;
  for (unsigned t = 1; t < pieces; ++t) {
    const char* c = body + body_size * t / pieces;
    const char* nl = static_cast<const char*>(std::memchr(c, '\n', (size_t)(end - c)));
    cut[t] = nl ? nl + 1 : end;
  }
  struct Piece {
    std::vector<std::int64_t> r, c;
    std::vector<double> v;
    bool bad = false;
  };
  std::vector<Piece> piece(pieces);
  parallel_for(pieces, [&](unsigned t) {
    Piece& P = piece[t];
    const char* q = cut[t];
    const char* stop = cut[t + 1];
    const size_t guess = (size_t)(stop - q) / 24 + 16;
    P.r.reserve(guess);
    P.c.reserve(guess);
    P.v.reserve(guess);
    while (q < stop) {
      const char* nl = static_cast<const char*>(std::memchr(q, '\n', (size_t)(stop - q)));
      const char* le = nl ? nl : stop;
      const char* lb = q;
      q = nl ? nl + 1 : stop;
      if (skippable(lb, le)) continue;
      std::int64_t i, j;
      double v = 1.0;
      const char* w = lb;
      if (!parse_int(w, le, i) || !parse_int(w, le, j) || (!bn.pattern && !parse_real(w, le, v)) ||
          skip_space(w, le) != le || i < 1 || i > n || j < 1 || j > n || (bn.symmetric && i < j) ||
          !std::isfinite(v)) {
        P.bad = true;
        return;
      }
      P.r.push_back(i - 1);
      P.c.push_back(j - 1);
      P.v.push_back(v);
    }
  });
  std::int64_t seen = 0;
  std::vector<std::int64_t> first(pieces + 1, 0);
  for (unsigned t = 0; t < pieces; ++t) {
    if (piece[t].bad) return false;
    first[t] = seen;
    seen += (std::int64_t)piece[t].r.size();
  }
  if (seen != declared) return false;

  // ---- bucket by row: count, prefix, scatter (mirrors of a symmetric file included)
  std::vector<std::atomic<std::int32_t>> cnt((size_t)n);
  for (auto& c : cnt) c.store(0, std::memory_order_relaxed);
  parallel_for(pieces, [&](unsigned t) {
    const Piece& P = piece[t];
    for (size_t k = 0; k < P.r.size(); ++k) {
      cnt[(size_t)P.r[k]].fetch_add(1, std::memory_order_relaxed);
      if (bn.symmetric && P.r[k] != P.c[k]) cnt[(size_t)P.c[k]].fetch_add(1, std::memory_order_relaxed);
    }
  });
  std::vector<std::int64_t> start((size_t)n + 1, 0);
  for (std::int64_t i = 0; i < n; ++i) start[i + 1] = start[i] + cnt[(size_t)i].load(std::memory_order_relaxed);
  const std::int64_t total = start[n];
  std::vector<Entry> ent((size_t)total);
  for (auto& c : cnt) c.store(0, std::memory_order_relaxed);
  parallel_for(pieces, [&](unsigned t) {
    const Piece& P = piece[t];
    for (size_t k = 0; k < P.r.size(); ++k) {
      const std::int64_t seq = first[t] + (std::int64_t)k;
      const std::int64_t i = P.r[k], j = P.c[k];
      ent[(size_t)(start[i] + cnt[(size_t)i].fetch_add(1, std::memory_order_relaxed))] = {(std::int32_t)j, seq, P.v[k]};
      if (bn.symmetric && i != j)
        ent[(size_t)(start[j] + cnt[(size_t)j].fetch_add(1, std::memory_order_relaxed))] = {(std::int32_t)i, seq, P.v[k]};
    }
  });
  std::vector<Piece>().swap(piece);

  // ---- per row: sort by (column, file position), sum duplicates in file order
  const unsigned rpieces = (unsigned)std::max<std::int64_t>(1, std::min<std::int64_t>(host_threads(), n / 2048 + 1));
  std::vector<std::int64_t> kept((size_t)n, 0);
  parallel_for(rpieces, [&](unsigned t) {
    for (std::int64_t i = n * t / rpieces; i < n * (t + 1) / rpieces; ++i) {
      Entry* lo = ent.data() + start[i];
      Entry* hi = ent.data() + start[i + 1];
      std::sort(lo, hi, [](const Entry& a, const Entry& b) {
        return a.col < b.col || (a.col == b.col && a.seq < b.seq);
      });
      Entry* out = lo;
      for (Entry* q = lo; q < hi;) {
        Entry acc = *q++;
        while (q < hi && q->col == acc.col) acc.value += (q++)->value;
        *out++ = acc;
      }
      kept[(size_t)i] = out - lo;
    }
  });
  row_ptr.assign((size_t)n + 1, 0);
  for (std::int64_t i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + kept[(size_t)i];
  col_idx.resize((size_t)row_ptr[n]);
  values.resize((size_t)row_ptr[n]);
  parallel_for(rpieces, [&](unsigned t) {
    for (std::int64_t i = n * t / rpieces; i < n * (t + 1) / rpieces; ++i) {
      const Entry* src = ent.data() + start[i];
      for (std::int64_t k = 0; k < kept[(size_t)i]; ++k) {
        col_idx[(size_t)(row_ptr[i] + k)] = src[k].col;
        values[(size_t)(row_ptr[i] + k)] = src[k].value;
      }
    }
  });
  std::vector<Entry>().swap(ent);

  // ---- "general" files: numerically symmetric up to 1e-12 max|A|, then averaged
  // (sparse.cpp:236-287); any violation is reported by the sequential loader
  if (!bn.symmetric) {
    double max_abs = 0.0;
    for (double v : values) max_abs = std::max(max_abs, std::abs(v));
    const double tol = 1e-12 * max_abs;
    std::atomic<bool> ok{true};
    std::vector<double> mean(values.size());
    parallel_for(rpieces, [&](unsigned t) {
      for (std::int64_t i = n * t / rpieces; i < n * (t + 1) / rpieces && ok.load(std::memory_order_relaxed); ++i)
        for (std::int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
          const std::int64_t j = col_idx[(size_t)k];
          if (j == i) {
            mean[(size_t)k] = values[(size_t)k];
            continue;
          }
          const std::int32_t* fb = col_idx.data() + row_ptr[j];
          const std::int32_t* fe = col_idx.data() + row_ptr[j + 1];
          const std::int32_t* hit = std::lower_bound(fb, fe, (std::int32_t)i);
          if (hit == fe || *hit != (std::int32_t)i) {
            ok.store(false, std::memory_order_relaxed);
            return;
          }
          const double other = values[(size_t)(row_ptr[j] + (hit - fb))];
          if (std::abs(values[(size_t)k] - other) > tol) {
            ok.store(false, std::memory_order_relaxed);
            return;
          }
          // the reference forms 0.5 * (upper + lower) with the upper entry first
          mean[(size_t)k] = i < j ? 0.5 * (values[(size_t)k] + other) : 0.5 * (other + values[(size_t)k]);
        }
    });
    if (!ok) return false;
    values.swap(mean);
  }
  n_out = (std::size_t)n;
  return true;
}

// ----------------------------------------------------------------- binary CSR image
struct ImageHeader {
  char magic[8];           // "FLZCSR1\0"
  std::uint64_t n, nnz;
  std::uint64_t src_size;  // size and mtime of the text file the image was made from (0: none)
  std::int64_t src_mtime_ns;
};
constexpr char kMagic[8] = {'F', 'L', 'Z', 'C', 'S', 'R', '1', '\0'};

void write_image(const SparseSymMatrix& A, const std::string& path, std::uint64_t src_size,
                 std::int64_t src_mtime_ns) {
  const std::string tmp = path + ".tmp" + std::to_string((long)::getpid());
  std::FILE* fp = std::fopen(tmp.c_str(), "wb");
  if (!fp) throw Error("cannot open '" + path + "' for writing");
  ImageHeader h{};
  std::memcpy(h.magic, kMagic, 8);
  h.n = A.dim();
  h.nnz = A.nnz();
  h.src_size = src_size;
  h.src_mtime_ns = src_mtime_ns;
  bool ok = std::fwrite(&h, sizeof h, 1, fp) == 1;
  ok = ok && std::fwrite(A.row_ptr().data(), 8, A.dim() + 1, fp) == A.dim() + 1;
  ok = ok && (A.nnz() == 0 || std::fwrite(A.col_idx().data(), 4, A.nnz(), fp) == A.nnz());
  ok = ok && (A.nnz() == 0 || std::fwrite(A.values().data(), 8, A.nnz(), fp) == A.nnz());
  ok = std::fclose(fp) == 0 && ok;
  if (ok) ok = std::rename(tmp.c_str(), path.c_str()) == 0;   // readers never see a partial image
  if (!ok) {
    std::remove(tmp.c_str());
    throw Error("write to '" + path + "' failed");
  }
}

// false: no usable image (missing, other source, truncated)
bool read_image(const std::string& path, const struct stat* src, std::vector<std::int64_t>& rp,
                std::vector<std::int32_t>& ci, std::vector<double>& va, std::size_t& n) {
  MappedFile F(path);
  if (!F.ok() || F.size < sizeof(ImageHeader)) return false;
  ImageHeader h;
  std::memcpy(&h, F.data, sizeof h);
  if (std::memcmp(h.magic, kMagic, 8) != 0) return false;
  if (src) {
    const std::int64_t mt = (std::int64_t)src->st_mtim.tv_sec * 1000000000 + src->st_mtim.tv_nsec;
    if (h.src_size != (std::uint64_t)src->st_size || h.src_mtime_ns != mt) return false;
  }
  const size_t need = sizeof h + 8 * (h.n + 1) + 12 * h.nnz;
  if (F.size != need) return false;
  n = (std::size_t)h.n;
  rp.resize(h.n + 1);
  ci.resize(h.nnz);
  va.resize(h.nnz);
  const char* q = F.data + sizeof h;
  const unsigned pieces = (unsigned)std::max<size_t>(1, std::min<size_t>(host_threads(), h.nnz / (1 << 20) + 1));
  std::memcpy(rp.data(), q, 8 * (h.n + 1));
  const char* qc = q + 8 * (h.n + 1);
  const char* qv = qc + 4 * h.nnz;
  parallel_for(pieces, [&](unsigned t) {
    const size_t a = h.nnz * t / pieces, b = h.nnz * (t + 1) / pieces;
    std::memcpy(ci.data() + a, qc + 4 * a, 4 * (b - a));
    std::memcpy(va.data() + a, qv + 8 * a, 8 * (b - a));
  });
  return true;
}

std::string cache_path_for(const std::string& path) {
  const char* e = std::getenv("FLZ_MM_CACHE");
  if (!e || !*e || std::strcmp(e, "0") == 0) return {};
  if (std::strcmp(e, "1") == 0) return path + ".flzcsr";
  std::string base = path;
  for (char& c : base)
    if (c == '/') c = '_';
  return std::string(e) + "/" + base + ".flzcsr";
}

}  // namespace

SparseSymMatrix load_matrix_market(const std::string& path) {
  MappedFile F(path);
  if (!F.ok()) throw Error("cannot open '" + path + "'");
  std::vector<std::int64_t> rp;
  std::vector<std::int32_t> ci;
  std::vector<double> va;
  std::size_t n = 0;
  const std::string cache = cache_path_for(path);
  if (!cache.empty() && read_image(cache, &F.st, rp, ci, va, n)) {
    try {
      return SparseSymMatrix::from_csr(n, std::move(rp), std::move(ci), std::move(va), false);
    } catch (const Error&) {   // damaged image: parse the text again
      rp.clear();
      ci.clear();
      va.clear();
    }
  }
  if (F.size == 0 || !load_fast(F, rp, ci, va, n)) return detail::load_matrix_market_sequential(path);
  SparseSymMatrix A = SparseSymMatrix::from_csr(n, std::move(rp), std::move(ci), std::move(va), true);
  if (!cache.empty()) {
    try {
      write_image(A, cache, (std::uint64_t)F.st.st_size,
                  (std::int64_t)F.st.st_mtim.tv_sec * 1000000000 + F.st.st_mtim.tv_nsec);
    } catch (const Error&) {   // a cache that cannot be written is not an error of the load
    }
  }
  return A;
}

void save_binary_csr(const SparseSymMatrix& A, const std::string& path) { write_image(A, path, 0, 0); }

SparseSymMatrix load_binary_csr(const std::string& path) {
  std::vector<std::int64_t> rp;
  std::vector<std::int32_t> ci;
  std::vector<double> va;
  std::size_t n = 0;
  if (!read_image(path, nullptr, rp, ci, va, n))
    throw ParseError(path + ": not a binary CSR image (FLZCSR1) or truncated");
  return SparseSymMatrix::from_csr(n, std::move(rp), std::move(ci), std::move(va), false);
}

}  // namespace flz
