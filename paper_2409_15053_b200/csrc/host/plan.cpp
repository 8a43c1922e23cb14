// host/plan.cpp — see plan.hpp.  Pure host code, no CUDA.

#include "plan.hpp"
#include "spin_barrier.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>
#include <numeric>
#include <stdexcept>
#include <string>

namespace flz {

namespace {

#ifndef FLZ_K1_T
#define FLZ_K1_T 48  // target entries per warp before a slice is split over more warps
#endif

// Entries per warp before a slice is split over more warps.  Splitting costs (shared-memory
// reduction, barriers, more index traffic per entry), so the target is the LARGEST one that
// keeps the launch balanced: measured on B200, 3 columns — PARSEC-shaped n = 113k:
// T = 48 32.9 us, 96 30.9 us, 128 35.9 us; n = 268k: 48 65.0 us, 96 64.0 us, 192 61.6 us.
thread_local int g_task_target = FLZ_K1_T;
int warps_for(int32_t len) {
  const int T = g_task_target;
  return len <= T ? 1 : (len <= 2 * T ? 2 : (len <= 4 * T ? 4 : 8));
}
void choose_task_target(const std::vector<int32_t>& slice_len) {
  if (const char* e = std::getenv("FLZ_K1_T")) {  // experiments
    g_task_target = std::max(1, std::atoi(e));
    return;
  }
  // the longest warp must not outlast the average warp slot by much (24 resident warps on
  // each of 148 SMs): largest target whose critical path stays within 1.5x of that average
  int64_t total = 0;
  for (int32_t L : slice_len) total += L;
  const double slot_average = (double)total / (148.0 * 24.0);
  // ... and the launch must be more than one wave of CTAs (3 resident per SM): with a single
  // wave every SM keeps the two or three unequal tasks it was dealt; from ~1.5 waves on the
  // hardware scheduler evens the SMs out (PARSEC-shaped n = 113k: 468 tasks 32.3 us, 805 tasks
  // 29.1 us per step)
  auto task_count = [&] {
    int64_t tasks = 0;
    size_t i = 0;
    while (i < slice_len.size()) {
      const int W = warps_for(slice_len[i]);
      int count = 0;
      while (i < slice_len.size() && count < kPlanTaskWarps / W && warps_for(slice_len[i]) == W) {
        ++i;
        ++count;
      }
      ++tasks;
    }
    return tasks;
  };
  bool balanced = false;
  for (int T : {256, 192, 128, 96, 64, 48, 32}) {
    g_task_target = T;
    if (!balanced) {
      int32_t longest = 0;
      for (int32_t L : slice_len) longest = std::max(longest, (L + warps_for(L) - 1) / warps_for(L));
      balanced = (double)longest <= 1.5 * slot_average;
    }
    if (balanced && task_count() >= 666) return;
  }
  if (!balanced) g_task_target = 48;
}

// Groups slices (in list order) into CTA tasks: long slices get several warps each.
std::vector<PlanTask> build_tasks(const std::vector<int32_t>& ids,
                                  const std::vector<int32_t>& slice_len) {
  std::vector<PlanTask> tasks;
  size_t i = 0;
  while (i < ids.size()) {
    PlanTask t{};
    t.warps_per_slice = warps_for(slice_len[ids[i]]);
    const int cap = kPlanTaskWarps / t.warps_per_slice;
    while (i < ids.size() && t.count < cap && warps_for(slice_len[ids[i]]) == t.warps_per_slice)
      t.slice[t.count++] = ids[i++];
    tasks.push_back(t);
  }
  // longest tasks first: CTAs are dispatched in order, so the short ones fill the tail of the
  // launch (a 113k-row matrix is only ~3 waves of CTAs)
  static const bool lpt = std::getenv("FLZ_K1_NO_LPT") == nullptr;
  if (lpt)
    std::stable_sort(tasks.begin(), tasks.end(), [&](const PlanTask& a, const PlanTask& b) {
      const int32_t ca = (slice_len[a.slice[0]] + a.warps_per_slice - 1) / a.warps_per_slice;
      const int32_t cb = (slice_len[b.slice[0]] + b.warps_per_slice - 1) / b.warps_per_slice;
      return ca > cb;
    });
  return tasks;
}

// Stable sort by descending row-length CLASS inside windows of `sigma` rows.  Classes are
// geometric (ratio 1.2): rows of similar length stay in their natural order, i.e. the lanes
// of a slice are mostly neighbouring rows whose entries reference neighbouring columns — on
// the PARSEC-shaped matrix a warp-level gather then touches 12.2 instead of 15.9 128-byte lines
// (scripts/analysis/gather_lines.py) for 3 % more padding than sorting by exact length.
int32_t length_class(int32_t len) {
  if (len <= 8) return len;
  return 8 + (int32_t)std::ceil(std::log((double)len / 8.0) / std::log(1.2));
}
// `key` (optional) replaces the row length as the sorting key: the paired layout sorts PAIRS
// of adjacent rows by the length of their merged column list — both rows of a pair carry the
// same key, windows hold an even number of rows, so a stable sort keeps every pair adjacent
// and on an even position.
void sort_windows(const std::vector<int32_t>& len, int64_t sigma, std::vector<int32_t>& perm,
                  const std::vector<int32_t>* key = nullptr) {
  const int64_t nl = (int64_t)len.size();
  perm.resize(nl);
  std::iota(perm.begin(), perm.end(), 0);
  if (sigma <= 1) return;
  // classes through a table (two logarithms per row otherwise); large windows by a stable
  // counting sort over the few dozen classes, descending — the order std::stable_sort gives
  const std::vector<int32_t>& k = key ? *key : len;
  int32_t kmax = 0;
  for (int64_t i = 0; i < nl; ++i) kmax = std::max(kmax, k[i]);
  std::vector<int32_t> table((size_t)kmax + 1);
  for (int32_t v = 0; v <= kmax; ++v) table[v] = length_class(v);
  std::vector<int32_t> cls(nl);
  for (int64_t i = 0; i < nl; ++i) cls[i] = table[std::max(k[i], 0)];
  const int32_t ncls = table.empty() ? 1 : *std::max_element(table.begin(), table.end()) + 1;
  std::vector<int64_t> start;
  std::vector<int32_t> sorted;
  for (int64_t w0 = 0; w0 < nl; w0 += sigma) {
    const int64_t w1 = std::min(nl, w0 + sigma);
    if (w1 - w0 < 4096) {
      std::stable_sort(perm.begin() + w0, perm.begin() + w1,
                       [&](int32_t a, int32_t b) { return cls[a] > cls[b]; });
      continue;
    }
    start.assign((size_t)ncls + 1, 0);
    for (int64_t i = w0; i < w1; ++i) ++start[ncls - 1 - cls[perm[i]] + 1];   // descending class
    for (int32_t c = 0; c < ncls; ++c) start[c + 1] += start[c];
    sorted.resize(w1 - w0);
    for (int64_t i = w0; i < w1; ++i) sorted[start[ncls - 1 - cls[perm[i]]]++] = perm[i];
    std::copy(sorted.begin(), sorted.end(), perm.begin() + w0);
  }
}

int64_t padded_entries(const std::vector<int32_t>& len, const std::vector<int32_t>& perm) {
  int64_t total = 0;
  for (size_t s = 0; s < perm.size(); s += kPlanSliceRows) {
    int32_t mx = 0;
    for (size_t i = s; i < std::min(perm.size(), s + kPlanSliceRows); ++i)
      mx = std::max(mx, len[perm[i]]);
    total += (int64_t)mx * kPlanSliceRows;
  }
  return total;
}

// ---- host parallelism: the layout passes are independent per slice
int worker_count() {
  if (const char* e = std::getenv("FLZ_HOST_THREADS")) return std::max(1, std::atoi(e));
  return (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
}
template <class F>
void run_chunks(int nchunks, F&& body) {
  if (nchunks <= 1) {
    body(0);
    return;
  }
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  for (int t = 0; t < nchunks; ++t)
    pool.emplace_back([&, t] {
      try {
        body(t);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// Doubles the (value, mask) pairs of nuv uniform-value positions occupy in front of the
// per-lane value rows of a slice (mirrors ug_header_doubles in kernels_sell.cu)
int64_t ug_header_doubles(int nuv, int lane_rows) {
  return lane_rows > 0 ? (2 * nuv + 15) / 16 * 16 : 2 * nuv;
}

// ---- UG layout -------------------------------------------------------------------------
// A diagonal offset d = col - row that at least kUgMinLanes of a slice's 32 lanes hold is
// stored as ONE uniform position: 32 values + one int32, the lanes without it get a zero.
// Break-even against a general position (12 bytes per true entry) is 22 of 32 lanes.
constexpr int kUgMinLanes = 22;

struct OffsetCounter {  // open-addressing counter of the offsets of one slice
  std::vector<int64_t> key;
  std::vector<int32_t> cnt;
  std::vector<int32_t> used;
  size_t mask;
  explicit OffsetCounter(size_t cap_pow2) : key(cap_pow2), cnt(cap_pow2, 0), mask(cap_pow2 - 1) {}
  void add(int64_t d) {
    size_t h = (size_t)((uint64_t)d * 0x9E3779B97F4A7C15ULL >> 40) & mask;
    while (cnt[h] != 0 && key[h] != d) h = (h + 1) & mask;
    if (cnt[h] == 0) {
      key[h] = d;
      used.push_back((int32_t)h);
    }
    ++cnt[h];
  }
  void clear() {
    for (int32_t h : used) cnt[h] = 0;
    used.clear();
  }
};

// returns the number of spilled entries
int64_t build_ug(HostPlan& P, const std::vector<uint8_t>& is_boundary, bool allow_spill,
                 bool allow_uv) {
  const int64_t nslices = P.nslices, nl = P.nl;
  P.ug_slice.assign(nslices, PlanUgSlice{});
  P.ug_val.clear();
  P.ug_col.clear();
  P.ug_uoff.clear();
  P.ug_val.reserve(P.stored);
  P.ug_uniform_entries = 0;
  int32_t max_len = 0;
  for (int64_t s = 0; s < nslices; ++s) max_len = std::max(max_len, P.slice_len[s]);
  size_t cap = 64;
  while (cap < (size_t)max_len * kPlanSliceRows * 2) cap <<= 1;
  // spilled leftovers (SPLIT mode): per rest row its entries, pooled
  struct RestRow {
    int32_t row;
    int64_t begin, end;
    uint8_t boundary;
  };
  // ---- phase A (parallel over chunks of slices): uniform offsets, nu, ng, spill decision
  struct SliceInfo {
    int32_t nu = 0, ng = 0, nuv = 0;
    uint8_t spill = 0, own_first = 0;
    int64_t uni_begin = 0;  // into the chunk's offset pool (UV offsets first, each run sorted)
  };
  struct alignas(128) Chunk {   // own cache lines (vector headers change on every push_back)
    int64_t s0 = 0, s1 = 0;
    std::vector<int64_t> uni_pool;
    std::vector<double> uv_value;   // per pooled offset: the common value (UV offsets only)
    std::vector<uint32_t> uv_mask;  // per pooled offset: lanes that hold the entry
    int64_t uniform_entries = 0;
    std::vector<RestRow> rest;
    std::vector<int32_t> rest_col;
    std::vector<double> rest_val;
  };
  const int nchunks = (int)std::max<int64_t>(1, std::min<int64_t>(worker_count(), nslices / 256));
  std::vector<Chunk> chunks(nchunks);
  for (int t = 0; t < nchunks; ++t) {
    chunks[t].s0 = nslices * t / nchunks;
    chunks[t].s1 = nslices * (t + 1) / nchunks;
  }
  std::vector<SliceInfo> info(nslices);
  run_chunks(nchunks, [&](int t) {
    Chunk& C = chunks[t];
    OffsetCounter counter(cap);
    std::vector<int64_t> uni, uni_sorted;
    std::vector<double> uval;
    std::vector<uint32_t> umask;
    std::vector<uint8_t> usame;
    int32_t glen[kPlanSliceRows];
    for (int64_t s = C.s0; s < C.s1; ++s) {
      const int32_t L = P.slice_len[s];
      const int64_t base = P.slice_ptr[s];
      counter.clear();
      for (int l = 0; l < kPlanSliceRows; ++l) {
        const int64_t row = s * kPlanSliceRows + l;
        const int32_t len = row < nl ? P.row_len[row] : 0;
        for (int32_t p = 0; p < len; ++p)
          counter.add((int64_t)P.col[base + (int64_t)p * kPlanSliceRows + l] - row);
      }
      uni.clear();
      for (int32_t h : counter.used)
        if (counter.cnt[h] >= kUgMinLanes) uni.push_back(counter.key[h]);
      std::sort(uni.begin(), uni.end());
      // general part: what every lane keeps after its uniform entries are taken out
      int32_t ng = 0;
      uval.assign(uni.size(), 0.0);
      umask.assign(uni.size(), 0u);
      usame.assign(uni.size(), 1);
      if (!uni.empty()) {
        for (int l = 0; l < kPlanSliceRows; ++l) {
          const int64_t row = s * kPlanSliceRows + l;
          const int32_t len = row < nl ? P.row_len[row] : 0;
          int32_t g = 0;
          for (int32_t p = 0; p < len; ++p) {
            const int64_t e = base + (int64_t)p * kPlanSliceRows + l;
            const int64_t d = (int64_t)P.col[e] - row;
            const auto it = std::lower_bound(uni.begin(), uni.end(), d);
            if (it == uni.end() || *it != d) {
              ++g;
              continue;
            }
            const size_t i = (size_t)(it - uni.begin());  // one value for the whole position?
            if (umask[i] == 0u) uval[i] = P.val[e];
            else if (uval[i] != P.val[e]) usame[i] = 0;
            umask[i] |= 1u << l;
          }
          glen[l] = g;
          ng = std::max(ng, g);
        }
        // keep the uniform positions only when they move fewer bytes than the plain slice
        const int64_t bytes_plain = (int64_t)12 * kPlanSliceRows * L;
        const int64_t bytes_ug = (int64_t)8 * kPlanSliceRows * ((int64_t)uni.size() + ng) +
                                 4 * (int64_t)uni.size() + (int64_t)4 * kPlanSliceRows * ng;
        if (!P.split && bytes_ug >= bytes_plain) uni.clear();
      }
      if (uni.empty()) {
        ng = L;
        for (int l = 0; l < kPlanSliceRows; ++l) {
          const int64_t row = s * kPlanSliceRows + l;
          glen[l] = row < nl ? P.row_len[row] : 0;
        }
      }
      // SPLIT mode: ragged leftovers leave the slice
      bool spill = false;
      if (P.split && allow_spill && ng > 2) {
        int64_t gsum = 0;
        for (int l = 0; l < kPlanSliceRows; ++l) gsum += glen[l];
        spill = 4 * gsum < (int64_t)3 * ng * kPlanSliceRows;  // < 75 % of the padded rectangle
      }
      if (spill) ng = 0;
      SliceInfo& I = info[s];
      I.nu = (int32_t)uni.size();
      I.ng = ng;
      I.spill = spill;
      I.uni_begin = (int64_t)C.uni_pool.size();
      // uniform-value offsets first (at most 255), then the per-lane-value ones
      {
        std::vector<size_t> head, tail;
        for (size_t i = 0; i < uni.size(); ++i)
          (allow_uv && usame[i] && head.size() < 255 ? head : tail).push_back(i);
        I.nuv = (int32_t)head.size();
        I.own_first = 0;  // offsets stay ascending: the summation order of a row is its CSR order
        for (size_t i : head) {
          C.uni_pool.push_back(uni[i]);
          C.uv_value.push_back(uval[i]);
          C.uv_mask.push_back(umask[i]);
        }
        for (size_t i : tail) {
          C.uni_pool.push_back(uni[i]);
          C.uv_value.push_back(0.0);
          C.uv_mask.push_back(0u);
        }
      }
    }
  });
  // ---- phase B (serial): pointers; identical consecutive offset lists (every interior slice
  // of a stencil) share one copy
  {
    int64_t vptr = 0, cptr = 0;
    const int64_t* last_uni = nullptr;
    int32_t last_nu = -1, last_uoff_ptr = -1;
    for (int t = 0; t < nchunks; ++t)
      for (int64_t s = chunks[t].s0; s < chunks[t].s1; ++s) {
        const SliceInfo& I = info[s];
        const int64_t* uni = chunks[t].uni_pool.data() + I.uni_begin;
        PlanUgSlice& H = P.ug_slice[s];
        H.val_ptr = vptr;
        H.col_ptr = cptr;
        H.nu = I.nu;
        H.ng = I.ng;
        H.reserved = (I.spill ? 1 : 0) | (I.own_first ? 4 : 0) | (I.nuv << 16);
        if (I.nu > 0 && I.nu == last_nu && std::equal(uni, uni + I.nu, last_uni)) {
          H.uoff_ptr = last_uoff_ptr;
        } else {
          H.uoff_ptr = (int32_t)P.ug_uoff.size();
          for (int32_t i = 0; i < I.nu; ++i) P.ug_uoff.push_back((int32_t)uni[i]);
          if (I.nu > 0) {
            last_uni = uni;
            last_nu = I.nu;
            last_uoff_ptr = H.uoff_ptr;
          }
        }
        for (int i = 0; i < 8; ++i) H.inline_off[i] = i < I.nu ? (int32_t)uni[i] : 0;
        vptr += ug_header_doubles(I.nuv, I.nu + I.ng - I.nuv) +
                (int64_t)(I.nu - I.nuv + I.ng) * kPlanSliceRows;
        cptr += (int64_t)I.ng * kPlanSliceRows;
      }
    P.ug_val.assign((size_t)vptr, 0.0);
    P.ug_col.assign((size_t)cptr, 0);
  }
  // ---- phase C (parallel): values, general columns, spilled entries
  run_chunks(nchunks, [&](int t) {
    Chunk& C = chunks[t];
    for (int64_t s = C.s0; s < C.s1; ++s) {
      const SliceInfo& I = info[s];
      const PlanUgSlice& H = P.ug_slice[s];
      const int64_t* uni = C.uni_pool.data() + I.uni_begin;
      const int64_t* uv_end = uni + I.nuv;   // runs: [uni, uv_end) (diagonal first) and [uv_end, uni_end)
      const int64_t* uni_end = uni + I.nu;
      const int64_t base = P.slice_ptr[s];
      const int32_t nu = I.nu, ng = I.ng, nuv = I.nuv;
      const bool spill = I.spill;
      double* hdr = P.ug_val.data() + H.val_ptr;
      for (int32_t i = 0; i < nuv; ++i) {  // (value, lane mask) pairs
        hdr[2 * i] = C.uv_value[I.uni_begin + i];
        const uint64_t bits = C.uv_mask[I.uni_begin + i];
        std::memcpy(&hdr[2 * i + 1], &bits, sizeof(double));
      }
      // per-lane value rows: position p >= nuv lives at row p - nuv behind the header
      double* v = hdr + ug_header_doubles(nuv, nu + ng - nuv) - (int64_t)nuv * kPlanSliceRows;
      int32_t* c = P.ug_col.data() + H.col_ptr;
      for (int l = 0; l < kPlanSliceRows; ++l) {
        const int64_t row = s * kPlanSliceRows + l;
        const int32_t len = row < nl ? P.row_len[row] : 0;
        const int32_t self = (int32_t)std::min<int64_t>(row, std::max<int64_t>(nl - 1, 0));
        int32_t g = 0;
        for (int32_t p = 0; p < len; ++p) {
          const int64_t e = base + (int64_t)p * kPlanSliceRows + l;
          const int64_t d = (int64_t)P.col[e] - row;
          const int64_t* uv_sorted = uni + (I.own_first ? 1 : 0);  // the diagonal may lead the run
          const int64_t* it = std::lower_bound(uv_sorted, uv_end, d);
          bool is_uv = (I.own_first && d == 0) || (it != uv_end && *it == d);
          if (!is_uv) it = std::lower_bound(uv_end, uni_end, d);
          if (is_uv) {
            if (P.val[e] != 0.0) ++C.uniform_entries;   // value and lane bit are in the header
          } else if (it != uni_end && *it == d) {
            v[(int64_t)(it - uni) * kPlanSliceRows + l] += P.val[e];
            if (P.val[e] != 0.0) ++C.uniform_entries;
          } else if (spill) {
            if (g == 0)
              C.rest.push_back({(int32_t)row, (int64_t)C.rest_col.size(), 0, is_boundary[s]});
            C.rest_col.push_back(P.col[e]);
            C.rest_val.push_back(P.val[e]);
            C.rest.back().end = (int64_t)C.rest_col.size();
            ++g;
          } else {  // general entries keep their CSR order
            v[(int64_t)(nu + g) * kPlanSliceRows + l] = P.val[e];
            c[(int64_t)g * kPlanSliceRows + l] = P.col[e];
            ++g;
          }
        }
        if (!spill)
          for (; g < ng; ++g) c[(int64_t)g * kPlanSliceRows + l] = self;
      }
    }
  });
  // ---- phase D (serial): the chunks' spilled rows, in row order
  std::vector<RestRow> rest;
  std::vector<int32_t> rest_col;
  std::vector<double> rest_val;
  for (Chunk& C : chunks) {
    P.ug_uniform_entries += C.uniform_entries;
    const int64_t shift = (int64_t)rest_col.size();
    for (RestRow r : C.rest) {
      r.begin += shift;
      r.end += shift;
      rest.push_back(r);
    }
    rest_col.insert(rest_col.end(), C.rest_col.begin(), C.rest_col.end());
    rest_val.insert(rest_val.end(), C.rest_val.begin(), C.rest_val.end());
  }
  // ---- rest slices: interior rows first, then boundary rows.  Rows with the same column
  // extent (first, last leftover column) — e.g. the rows of one dense non-local block — are
  // kept together, 32 per slice; a column most lanes of such a slice hold becomes ONE shared
  // position (bit 1 of the flags: the position's int32 is an absolute column, every lane
  // reads the same block row — a broadcast instead of 32 scattered gathers).  Rows of small
  // groups are pooled and sorted by descending length in windows of 4096 (stable).
  P.nrest = 0;
  P.rest_rows.clear();
  P.rest_interior.clear();
  P.rest_boundary.clear();
  if (!rest.empty()) {
    constexpr int kMinGroup = 16;      // rows a column-extent group needs to get own slices
    OffsetCounter colcount(cap);
    std::vector<int32_t> order, pooled, shared;
    std::vector<int32_t> lanes;        // rest-row ids of the slice being emitted
    auto emit = [&](int pass, bool share) {
      const int h = (int)lanes.size();
      shared.clear();
      if (share) {
        colcount.clear();
        for (int32_t id : lanes)
          for (int64_t e = rest[id].begin; e < rest[id].end; ++e) colcount.add(rest_col[e]);
        const int need = std::max(2, (3 * h + 4) / 5);  // >= 60 % of the lanes
        for (int32_t hh : colcount.used)
          if (colcount.cnt[hh] >= need) shared.push_back((int32_t)colcount.key[hh]);
        std::sort(shared.begin(), shared.end());
      }
      const int32_t nu = (int32_t)shared.size();
      int32_t ng = 0;
      for (int32_t id : lanes) {
        int32_t g = 0;
        for (int64_t e = rest[id].begin; e < rest[id].end; ++e)
          if (!std::binary_search(shared.begin(), shared.end(), rest_col[e])) ++g;
        ng = std::max(ng, g);
      }
      PlanUgSlice H{};
      H.val_ptr = (int64_t)P.ug_val.size();
      H.col_ptr = (int64_t)P.ug_col.size();
      H.uoff_ptr = (int32_t)P.ug_uoff.size();
      H.nu = nu;
      H.ng = ng;
      H.reserved = nu > 0 ? 2 : 0;
      for (int i = 0; i < 8; ++i) H.inline_off[i] = i < nu ? shared[i] : 0;
      P.ug_uoff.insert(P.ug_uoff.end(), shared.begin(), shared.end());
      P.ug_val.resize(P.ug_val.size() + (size_t)(nu + ng) * kPlanSliceRows, 0.0);
      P.ug_col.resize(P.ug_col.size() + (size_t)ng * kPlanSliceRows, 0);
      double* v = P.ug_val.data() + H.val_ptr;
      int32_t* c = P.ug_col.data() + H.col_ptr;
      const int32_t fallback = rest[lanes[0]].row;
      for (int l = 0; l < kPlanSliceRows; ++l) {
        const bool on = l < h;
        const RestRow* rr = on ? &rest[lanes[l]] : nullptr;
        P.rest_rows.push_back(on ? rr->row : -1);
        int32_t g = 0;
        if (on)
          for (int64_t e = rr->begin; e < rr->end; ++e) {
            const auto it = std::lower_bound(shared.begin(), shared.end(), rest_col[e]);
            if (it != shared.end() && *it == rest_col[e]) {
              v[(int64_t)(it - shared.begin()) * kPlanSliceRows + l] = rest_val[e];
            } else {
              v[(int64_t)(nu + g) * kPlanSliceRows + l] = rest_val[e];
              c[(int64_t)g * kPlanSliceRows + l] = rest_col[e];
              ++g;
            }
          }
        for (; g < ng; ++g) c[(int64_t)g * kPlanSliceRows + l] = on ? rr->row : fallback;
      }
      const int32_t id = (int32_t)(nslices + P.nrest);
      (pass ? P.rest_boundary : P.rest_interior).push_back(id);
      P.ug_slice.push_back(H);
      ++P.nrest;
      lanes.clear();
    };
    auto key_less = [&](int32_t a, int32_t b) {
      const int32_t fa = rest_col[rest[a].begin], fb = rest_col[rest[b].begin];
      if (fa != fb) return fa < fb;
      const int32_t la = rest_col[rest[a].end - 1], lb = rest_col[rest[b].end - 1];
      if (la != lb) return la < lb;
      return rest[a].row < rest[b].row;
    };
    auto same_key = [&](int32_t a, int32_t b) {
      return rest_col[rest[a].begin] == rest_col[rest[b].begin] &&
             rest_col[rest[a].end - 1] == rest_col[rest[b].end - 1];
    };
    for (int pass = 0; pass < 2; ++pass) {
      order.clear();
      pooled.clear();
      for (size_t i = 0; i < rest.size(); ++i)
        if (rest[i].boundary == pass) order.push_back((int32_t)i);
      std::sort(order.begin(), order.end(), key_less);
      for (size_t g0 = 0; g0 < order.size();) {
        size_t g1 = g0 + 1;
        while (g1 < order.size() && same_key(order[g0], order[g1])) ++g1;
        if ((int)(g1 - g0) >= kMinGroup) {
          for (size_t i = g0; i < g1; ++i) {
            lanes.push_back(order[i]);
            if ((int)lanes.size() == kPlanSliceRows) emit(pass, true);
          }
          if (!lanes.empty()) emit(pass, true);
        } else {
          pooled.insert(pooled.end(), order.begin() + g0, order.begin() + g1);
        }
        g0 = g1;
      }
      std::sort(pooled.begin(), pooled.end(),
                [&](int32_t a, int32_t b) { return rest[a].row < rest[b].row; });
      constexpr size_t kWindow = 4096;
      for (size_t w0 = 0; w0 < pooled.size(); w0 += kWindow) {
        const size_t w1 = std::min(pooled.size(), w0 + kWindow);
        std::stable_sort(pooled.begin() + w0, pooled.begin() + w1, [&](int32_t a, int32_t b) {
          return rest[a].end - rest[a].begin > rest[b].end - rest[b].begin;
        });
      }
      for (size_t i = 0; i < pooled.size(); ++i) {
        lanes.push_back(pooled[i]);
        if ((int)lanes.size() == kPlanSliceRows) emit(pass, false);
      }
      if (!lanes.empty()) emit(pass, false);
    }
  }
  if (P.ug_val.empty()) P.ug_val.push_back(0.0);
  if (P.ug_col.empty()) P.ug_col.push_back(0);
  if (P.ug_uoff.empty()) P.ug_uoff.push_back(0);
  return (int64_t)rest_col.size();
}

struct PhaseTimer {  // FLZ_TRACE=1: phase timings of build_plan on stderr
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  bool on = std::getenv("FLZ_TRACE") != nullptr;
  void lap(const char* what) {
    if (!on) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[flz]   plan %-22s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

// ---- dense blocks (plan.hpp) ---------------------------------------------------------------
// Near-cliques among the LONG rows of the local diagonal block: rows much longer than the
// median (the members of non-local projector balls on PARSEC-like Hamiltonians).  Greedy:
// seeds in ascending row length (rows of a single ball first); candidate set K = the seed's
// still uncovered long columns; two refinement passes keep the members adjacent to >= 80 % of
// K; K is accepted when it has >= kDenseMin members and at least a quarter of K x K is new.  All
// entries (j, c), j and c in K, are then COVERED by the block.  Matrices without such blocks
// cost a bounded number of failed seeds.
struct DenseBlocks {
  std::vector<std::vector<int32_t>> members;  // local row ids, ascending
  std::vector<uint8_t> covered;               // per local CSR entry
  std::vector<int32_t> count;                 // blocks a row belongs to
  std::vector<int32_t> primary;               // the block of a row with count == 1, else -1
  int64_t covered_entries = 0;
  bool any() const { return !members.empty(); }
};
constexpr int kDenseMin = 32;

DenseBlocks extract_dense_blocks(int64_t nl, int64_t row_begin, const int64_t* row_ptr,
                                 const int32_t* col_idx, const std::vector<int32_t>& len,
                                 int64_t nnz) {
  DenseBlocks B;
  if (nl < 1024) return B;
  PhaseTimer sub;
  std::vector<int32_t> tmp(len);
  std::nth_element(tmp.begin(), tmp.begin() + nl / 2, tmp.end());
  const int32_t long_min = std::max<int32_t>(48, tmp[nl / 2] + tmp[nl / 2] / 2);
  std::vector<uint8_t> is_long(nl, 0);
  int64_t long_entries = 0;
  std::vector<int32_t> seeds;
  for (int64_t i = 0; i < nl; ++i)
    if (len[i] > long_min) {
      is_long[i] = 1;
      long_entries += len[i];
      seeds.push_back((int32_t)i);
    }
  if (5 * long_entries < nnz) return B;
  const int64_t p0 = row_ptr[0];
  auto local = [&](int64_t e) { return (int64_t)col_idx[e] - row_begin; };
  std::vector<int32_t> uncov(nl, 0);
  {
    const int64_t ns = (int64_t)seeds.size();
    const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(worker_count(), ns / 2048));
    run_chunks(chunks, [&](int t) {
      for (int64_t q = ns * t / chunks; q < ns * (t + 1) / chunks; ++q) {
        const int32_t i = seeds[q];
        int32_t u = 0;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
          const int64_t c = local(e);
          u += (c >= 0 && c < nl && is_long[c]) ? 1 : 0;
        }
        uncov[i] = u;
      }
    });
  }
  sub.lap("  blocks: long rows, uncov");
  std::stable_sort(seeds.begin(), seeds.end(), [&](int32_t a, int32_t b) { return len[a] < len[b]; });
  B.covered.assign((size_t)nnz, 0);
  sub.lap("  blocks: seed sort");
  B.count.assign(nl, 0);
  std::vector<uint8_t> mark(nl, 0);
  std::vector<int32_t> K, keep, dcount;
  // team of scanning threads (member 0 is this thread); they live for the whole search and
  // meet at a spin barrier before and after every scan — a scan is ~50 us of work
  const unsigned team = (unsigned)std::max(1, std::min(8, worker_count()));
  struct alignas(128) FreshList {   // one cache line pair per member: the list headers are
    std::vector<std::pair<int64_t, int32_t>> v;   // written on every push_back
    void clear() { v.clear(); }
    size_t size() const { return v.size(); }
    void push_back(std::pair<int64_t, int32_t> x) { v.push_back(x); }
    auto begin() const { return v.begin(); }
    auto end() const { return v.end(); }
  };
  std::vector<FreshList> fresh_at(team);
  SpinBarrier barrier(team);
  bool team_stop = false;
  int team_job = 0;   // 0: scan a share of K; 1: mark a share's new entries as covered
  auto cover_share = [&](unsigned me) {   // shares hold disjoint rows: no two members touch
    for (const auto& f : fresh_at[me]) {  // the same entry or the same uncov counter
      B.covered[f.first] = 1;
      --uncov[f.second];
    }
  };
  auto scan_share = [&](unsigned me) {
    auto& mine = fresh_at[me];
    mine.clear();   // (entry, row) of the new entries of K x K in this share
    const size_t q0 = K.size() * me / team, q1 = K.size() * (me + 1) / team;
    for (size_t q = q0; q < q1; ++q) {
      const int32_t j = K[q];
      int32_t d = 0;
      for (int64_t e = row_ptr[j]; e < row_ptr[j + 1]; ++e) {
        const int64_t c = local(e);
        const bool in = c >= 0 && c < nl && mark[c];
        d += in ? 1 : 0;
        if (in && !B.covered[e - p0]) mine.push_back({e - p0, j});
      }
      dcount[q] = d;
    }
  };
  std::vector<std::thread> scanners;
  for (unsigned m = 1; m < team; ++m)
    scanners.emplace_back([&, m] {
      while (true) {
        barrier.wait();
        if (team_stop) return;
        if (team_job == 0) scan_share(m);
        else cover_share(m);
        barrier.wait();
      }
    });
  struct StopTeam {   // also on an exception: release and join the scanners
    std::vector<std::thread>& pool;
    SpinBarrier& barrier;
    bool& stop;
    ~StopTeam() {
      if (pool.empty()) return;
      stop = true;
      barrier.wait();
      for (auto& t : pool) t.join();
    }
  } stop_team{scanners, barrier, team_stop};
  int fails = 0;
  for (int32_t seed : seeds) {
    if (uncov[seed] < kDenseMin) continue;
    K.clear();
    bool has_seed = false;
    for (int64_t e = row_ptr[seed]; e < row_ptr[seed + 1]; ++e) {
      const int64_t c = local(e);
      if (c < 0 || c >= nl || !is_long[c] || B.covered[e - p0]) continue;
      K.push_back((int32_t)c);
      has_seed = has_seed || c == seed;
    }
    if (!has_seed) K.push_back(seed);
    // (a pass that keeps every member leaves K as it was: a second pass would find the same
    // counts, and the new entries of K x K counted during that pass are the final ones)
    int64_t fresh_seen = -1;
    for (int pass = 0; pass < 2 && (int)K.size() >= kDenseMin && fresh_seen < 0; ++pass) {
      for (int32_t c : K) mark[c] = 1;
      // the rows of K are scanned by the team (member m: a contiguous share of K, its new
      // entries in its own list); counts and lists are put together in K order, so the result
      // is the sequential scan's
      dcount.resize(K.size());
      if (team > 1) {
        team_job = 0;
        barrier.wait();   // job published (K, mark)
        scan_share(0);
        barrier.wait();   // all shares done
      } else {
        scan_share(0);
      }
      keep.clear();
      int64_t fresh_pass = 0;
      for (size_t q = 0; q < K.size(); ++q)
        if (5 * (int64_t)dcount[q] >= 4 * (int64_t)K.size()) keep.push_back(K[q]);
      for (unsigned m = 0; m < team; ++m) fresh_pass += (int64_t)fresh_at[m].size();
      for (int32_t c : K) mark[c] = 0;
      if (keep.size() == K.size()) fresh_seen = fresh_pass;
      K.swap(keep);
    }
    bool ok = (int)K.size() >= kDenseMin;
    if (ok) {  // at least half of K x K must be new entries
      for (int32_t c : K) mark[c] = 1;
      int64_t fresh = 0;
      if (fresh_seen >= 0) {
        fresh = fresh_seen;
      } else {
        for (int32_t j : K)
          for (int64_t e = row_ptr[j]; e < row_ptr[j + 1]; ++e) {
            const int64_t c = local(e);
            fresh += (c >= 0 && c < nl && mark[c] && !B.covered[e - p0]) ? 1 : 0;
          }
      }
      // (a quarter is enough: a ball that overlaps an earlier block is still worth a block —
      // the hybrid layout drops the columns a task does not use, the paired layout stores zeros)
      ok = 4 * fresh >= (int64_t)K.size() * (int64_t)K.size();
      if (ok && fresh_seen >= 0) {
        // the last pass kept every member: its lists of new entries are the block's
        if (team > 1) {
          team_job = 1;
          barrier.wait();
          cover_share(0);
          barrier.wait();
        } else {
          cover_share(0);
        }
        B.covered_entries += fresh;
      } else if (ok) {
        for (int32_t j : K)
          for (int64_t e = row_ptr[j]; e < row_ptr[j + 1]; ++e) {
            const int64_t c = local(e);
            if (c >= 0 && c < nl && mark[c] && !B.covered[e - p0]) {
              B.covered[e - p0] = 1;
              --uncov[j];
            }
          }
        B.covered_entries += fresh;
      }
      for (int32_t c : K) mark[c] = 0;
    }
    if (!ok) {
      if (++fails > 64 + 4 * (int)B.members.size()) break;  // no block structure: give up
      continue;
    }
    std::sort(K.begin(), K.end());
    for (int32_t j : K) ++B.count[j];
    B.members.push_back(K);
  }
  sub.lap("  blocks: greedy search");
  if (10 * B.covered_entries < nnz) return DenseBlocks{};  // not worth a second row order
  B.primary.assign(nl, -1);
  for (size_t b = 0; b < B.members.size(); ++b)
    for (int32_t j : B.members[b])
      if (B.count[j] == 1) B.primary[j] = (int32_t)b;
  return B;
}

// ---- hybrid layout (plan.hpp) ------------------------------------------------------------
// Dense tasks from the blocks, slices from everything else; natural row order.  An entry
// (i, c) that blocks cover belongs to the FIRST block (in creation order) that holds both i
// and c — the block that covered it in extract_dense_blocks.
void require(bool ok, const char* msg);
void build_hybrid(HostPlan& P, const DenseBlocks& blocks, const int64_t* row_ptr,
                  const int32_t* col_idx, const double* values) {
  const int64_t nl = P.nl;
  const int64_t p0 = row_ptr[0];
  // gather-source index: local rows first, then the halo slots, then the zero row
  const int32_t zero_row = (int32_t)(nl + (int64_t)P.halo.size());
  PhaseTimer sub;
  auto local = [&](int64_t e) {
    const int64_t g = col_idx[e];
    if (g >= P.row_begin && g < P.row_end) return (int32_t)(g - P.row_begin);
    return (int32_t)(nl + (std::lower_bound(P.halo.begin(), P.halo.end(), g) - P.halo.begin()));
  };
  // membership lists (block, index inside the block), ascending block id
  std::vector<int32_t> mem_ptr(nl + 1, 0);
  for (const auto& K : blocks.members)
    for (int32_t j : K) ++mem_ptr[j + 1];
  for (int64_t i = 0; i < nl; ++i) mem_ptr[i + 1] += mem_ptr[i];
  std::vector<int32_t> mem_blk(mem_ptr[nl]), fill(mem_ptr.begin(), mem_ptr.end() - 1);
  for (size_t b = 0; b < blocks.members.size(); ++b)
    for (int32_t j : blocks.members[b]) mem_blk[fill[j]++] = (int32_t)b;
  auto owner = [&](int32_t i, int32_t c) -> int32_t {
    for (int32_t a = mem_ptr[i]; a < mem_ptr[i + 1]; ++a)
      for (int32_t q = mem_ptr[c]; q < mem_ptr[c + 1]; ++q)
        if (mem_blk[a] == mem_blk[q]) return mem_blk[a];
    return -1;
  };
  // ---- dense tasks: block b x 32 of its rows x the columns those rows own entries in (a task
  // whose rows sit in the overlap with an earlier block drops that block's columns)
  P.hy_dtasks.clear();
  P.hy_dcols.clear();
  std::vector<int32_t> slot_ptr(nl + 1, 0);
  for (int64_t i = 0; i < nl; ++i) slot_ptr[i + 1] = slot_ptr[i] + (mem_ptr[i + 1] - mem_ptr[i]);
  std::vector<int32_t> slots(slot_ptr[nl], 0), slot_fill(slot_ptr.begin(), slot_ptr.end() - 1);
  struct TaskSpec {
    int32_t block, g0, nrows;
  };
  std::vector<TaskSpec> spec;
  for (size_t b = 0; b < blocks.members.size(); ++b) {
    const int32_t nb = (int32_t)blocks.members[b].size();
    for (int32_t g0 = 0; g0 < nb; g0 += kPlanSliceRows)
      spec.push_back({(int32_t)b, g0, std::min<int32_t>(kPlanSliceRows, nb - g0)});
  }
  const int64_t nt = (int64_t)spec.size();
  // pass 1 (threaded): the columns every task uses
  std::vector<std::vector<int32_t>> task_cols(nt);
  const int dchunks = (int)std::max<int64_t>(1, std::min<int64_t>(worker_count(), nt / 8));
  run_chunks(dchunks, [&](int w) {
    std::vector<uint8_t> used;
    std::vector<int32_t> pos(nl, 0);   // member index of a row inside the current block
    int32_t pos_block = -1;
    for (int64_t t = nt * w / dchunks; t < nt * (w + 1) / dchunks; ++t) {
      const auto& rows = blocks.members[spec[t].block];
      if (pos_block != spec[t].block) {
        for (size_t j = 0; j < rows.size(); ++j) pos[rows[j]] = (int32_t)j;
        pos_block = spec[t].block;
      }
      used.assign(rows.size(), 0);
      for (int32_t q = 0; q < spec[t].nrows; ++q) {
        const int32_t i = rows[spec[t].g0 + q];
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
          if (!blocks.covered[e - p0]) continue;
          const int32_t c = local(e);
          if (c == i || owner(i, c) != spec[t].block) continue;
          used[pos[c]] = 1;   // c is a member: owner() found the block among c's blocks
        }
      }
      for (size_t j = 0; j < rows.size(); ++j)
        if (used[j]) task_cols[t].push_back(rows[j]);
    }
  });
  sub.lap("  hybrid: task columns");
  int64_t nslots = kPlanSliceRows, nvals = 0;
  int32_t maxcols = 1;
  for (int64_t t = 0; t < nt; ++t) {
    if (task_cols[t].empty()) continue;   // every entry of these rows belongs to earlier blocks
    const auto& rows = blocks.members[spec[t].block];
    PlanHyTask T{};
    T.val_off = nvals;
    T.col_off = (int32_t)P.hy_dcols.size();
    T.ncols = (int32_t)task_cols[t].size();
    T.slot_base = (int32_t)nslots;
    T.nrows = spec[t].nrows;
    T.pad[0] = (int32_t)t;   // spec index (host only)
    P.hy_dcols.insert(P.hy_dcols.end(), task_cols[t].begin(), task_cols[t].end());
    for (int32_t q = 0; q < T.nrows; ++q) slots[slot_fill[rows[spec[t].g0 + q]]++] = T.slot_base + q;
    nslots += kPlanSliceRows;
    nvals += T.ncols;
    maxcols = std::max(maxcols, T.ncols);
    P.hy_dtasks.push_back(T);
  }
  // rows of skipped tasks consume fewer slots than blocks they belong to: compact the lists
  std::vector<int32_t> slot_cnt(nl, 0);
  for (int64_t i = 0; i < nl; ++i) slot_cnt[i] = slot_fill[i] - slot_ptr[i];
  require(nslots < ((int64_t)1 << 31) && nvals * kPlanSliceRows < ((int64_t)1 << 40),
          "plan: hybrid layout overflow");
  P.hy_nslots = nslots;
  P.hy_maxcols = maxcols;
  P.hy_blocks = (int64_t)blocks.members.size();
  P.hy_dval.resize((size_t)std::max<int64_t>(nvals, 1) * kPlanSliceRows);   // zeroed per task below
  if (nvals == 0) std::fill(P.hy_dval.begin(), P.hy_dval.end(), 0.0);
  const int64_t ntask = (int64_t)P.hy_dtasks.size();
  std::vector<int64_t> dense_part(dchunks, 0);
  run_chunks(dchunks, [&](int w) {
    std::vector<int32_t> pos(nl, 0);   // index of a row among the current task's columns
    int64_t filled = 0;   // (a local count: the shared array would bounce between the cores)
    for (int64_t t = ntask * w / dchunks; t < ntask * (w + 1) / dchunks; ++t) {
      PlanHyTask& T = P.hy_dtasks[t];
      const TaskSpec& S = spec[T.pad[0]];
      const auto& rows = blocks.members[S.block];
      const int32_t* tc = P.hy_dcols.data() + T.col_off;
      for (int32_t j = 0; j < T.ncols; ++j) pos[tc[j]] = j;
      double* v = P.hy_dval.data() + T.val_off * kPlanSliceRows;
      std::fill(v, v + (int64_t)T.ncols * kPlanSliceRows, 0.0);
      for (int32_t q = 0; q < T.nrows; ++q) {
        const int32_t i = rows[S.g0 + q];
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
          if (!blocks.covered[e - p0]) continue;
          const int32_t c = local(e);
          if (c == i || owner(i, c) != S.block) continue;
          const int64_t j = pos[c];   // c is one of the task's columns (pass 1 marked it)
          v[j * kPlanSliceRows + q] = values[e];
          ++filled;
        }
      }
    }
    dense_part[w] = filled;
  });
  sub.lap("  hybrid: dense values");
  for (auto& T : P.hy_dtasks) T.pad[0] = 0;
  P.hy_dense_entries = 0;
  for (int64_t x : dense_part) P.hy_dense_entries += x;
  // ---- slices
  const int64_t ns = (nl + kPlanSliceRows - 1) / kPlanSliceRows;
  P.hy_slice.assign(ns, PlanHySlice{});
  P.hy_diag.assign(std::max<int64_t>(nl, 1), 0.0);
  struct alignas(128) Chunk {   // own cache lines: the vector headers change on every push_back
    std::vector<int32_t> cols;
    std::vector<double> uv, gv;
    int64_t uv_entries = 0, g_entries = 0;
  };
  const int schunks = (int)std::max<int64_t>(1, std::min<int64_t>(worker_count(), ns / 64));
  std::vector<Chunk> chunk(schunks);
  run_chunks(schunks, [&](int w) {
    Chunk& C = chunk[w];
    struct Ent {
      uint64_t bits;
      int32_t lane, col;
      double v;
    };
    std::vector<Ent> ents, sorted_ents;
    std::vector<uint64_t> gkeys;
    std::vector<size_t> gcount, goffset;
    std::vector<int> gorder;
    std::vector<int16_t> gid_of;
    std::vector<std::vector<std::pair<int32_t, double>>> gen(kPlanSliceRows);
    std::vector<std::vector<int32_t>> per(kPlanSliceRows);
    for (int64_t s = ns * w / schunks; s < ns * (w + 1) / schunks; ++s) {
      ents.clear();
      for (auto& g : gen) g.clear();
      for (int l = 0; l < kPlanSliceRows; ++l) {
        const int64_t i = s * kPlanSliceRows + l;
        if (i >= nl) break;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
          const int32_t c = local(e);
          if (c == (int32_t)i) {
            P.hy_diag[i] = values[e];
            continue;
          }
          if (blocks.covered[e - p0]) continue;
          uint64_t bits;
          std::memcpy(&bits, &values[e], 8);
          ents.push_back({bits, l, c, values[e]});
        }
      }
      // order (value bits, lane, column).  The entries arrive by lane and, inside a lane, by
      // column, so a STABLE distribution over the distinct values (a few dozen on a stencil)
      // sorted by their bits gives that order without a comparison sort of the entries
      {
        constexpr int kTab = 256;
        uint64_t tkey[kTab];
        int16_t tgid[kTab];
        std::fill(tgid, tgid + kTab, (int16_t)-1);
        gkeys.clear();
        gcount.clear();
        gid_of.resize(ents.size());
        bool small = true;
        for (size_t q = 0; q < ents.size() && small; ++q) {
          uint64_t h = ents[q].bits * 0x9E3779B97F4A7C15ULL;
          int slot = (int)(h >> 56);
          while (tgid[slot] >= 0 && tkey[slot] != ents[q].bits) slot = (slot + 1) & (kTab - 1);
          if (tgid[slot] < 0) {
            if (gkeys.size() >= 160) {   // many distinct values: no stencil, sort instead
              small = false;
              break;
            }
            tkey[slot] = ents[q].bits;
            tgid[slot] = (int16_t)gkeys.size();
            gkeys.push_back(ents[q].bits);
            gcount.push_back(0);
          }
          gid_of[q] = tgid[slot];
          ++gcount[tgid[slot]];
        }
        if (small) {
          const int ng_keys = (int)gkeys.size();
          gorder.resize(ng_keys);
          std::iota(gorder.begin(), gorder.end(), 0);
          std::sort(gorder.begin(), gorder.end(), [&](int a, int b) { return gkeys[a] < gkeys[b]; });
          goffset.assign(ng_keys, 0);
          size_t run = 0;
          for (int r = 0; r < ng_keys; ++r) {
            goffset[gorder[r]] = run;
            run += gcount[gorder[r]];
          }
          sorted_ents.resize(ents.size());
          for (size_t q = 0; q < ents.size(); ++q) sorted_ents[goffset[gid_of[q]]++] = ents[q];
          ents.swap(sorted_ents);
        } else {
          std::sort(ents.begin(), ents.end(), [](const Ent& a, const Ent& b) {
            if (a.bits != b.bits) return a.bits < b.bits;
            if (a.lane != b.lane) return a.lane < b.lane;
            return a.col < b.col;
          });
        }
      }
      PlanHySlice& H = P.hy_slice[s];
      H.col_off = (int64_t)C.cols.size() / kPlanSliceRows;   // chunk-relative for now
      H.uv_off = (int32_t)C.uv.size();
      H.g_off = (int32_t)(C.gv.size() / kPlanSliceRows);
      // uniform-value groups
      std::vector<std::vector<int32_t>> pos_cols;   // per position: 32 columns
      for (size_t a = 0; a < ents.size();) {
        size_t z = a;
        int lanes = 0, last = -1;
        while (z < ents.size() && ents[z].bits == ents[a].bits) {
          if (ents[z].lane != last) {
            ++lanes;
            last = ents[z].lane;
          }
          ++z;
        }
        if (lanes >= kHyMinLanes) {
          for (auto& v : per) v.clear();
          size_t cnt = 0;
          for (size_t q = a; q < z; ++q) {
            per[ents[q].lane].push_back(ents[q].col);
            cnt = std::max(cnt, per[ents[q].lane].size());
          }
          for (size_t q = 0; q < cnt; ++q) {
            C.uv.push_back(ents[a].v);
            pos_cols.emplace_back(kPlanSliceRows, zero_row);
            for (int l = 0; l < kPlanSliceRows; ++l)
              if (q < per[l].size()) {
                pos_cols.back()[l] = per[l][q];
                ++C.uv_entries;
              }
          }
        } else {
          for (size_t q = a; q < z; ++q) gen[ents[q].lane].push_back({ents[q].col, ents[q].v});
        }
        a = z;
      }
      while (pos_cols.size() % 4) {
        pos_cols.emplace_back(kPlanSliceRows, zero_row);
        C.uv.push_back(0.0);
      }
      H.nuv = (int32_t)pos_cols.size();
      for (size_t q = 0; q < pos_cols.size(); q += 4)
        for (int l = 0; l < kPlanSliceRows; ++l)
          for (int u = 0; u < 4; ++u) C.cols.push_back(pos_cols[q + u][l]);
      // general positions (ascending column per lane)
      size_t ng = 0;
      for (auto& g : gen) {
        std::sort(g.begin(), g.end());
        ng = std::max(ng, g.size());
      }
      for (size_t q = 0; q < ng; ++q)
        for (int l = 0; l < kPlanSliceRows; ++l) {
          const bool has = q < gen[l].size();
          C.cols.push_back(has ? gen[l][q].first : zero_row);
          C.gv.push_back(has ? gen[l][q].second : 0.0);
          C.g_entries += has;
        }
      H.ng = (int32_t)ng;
      // partial positions
      int32_t np = 0;
      for (int l = 0; l < kPlanSliceRows; ++l) {
        const int64_t i = s * kPlanSliceRows + l;
        if (i < nl) np = std::max(np, slot_cnt[i]);
      }
      for (int32_t q = 0; q < np; ++q)
        for (int l = 0; l < kPlanSliceRows; ++l) {
          const int64_t i = s * kPlanSliceRows + l;
          const bool has = i < nl && q < slot_cnt[i];
          C.cols.push_back(has ? slots[slot_ptr[i] + q] : 0);
        }
      H.np = np;
    }
  });
  sub.lap("  hybrid: slices");
  // concatenate the chunks
  int64_t ncols = 0, nuvv = 0, ngv = 0;
  for (auto& C : chunk) {
    ncols += (int64_t)C.cols.size();
    nuvv += (int64_t)C.uv.size();
    ngv += (int64_t)C.gv.size();
  }
  require(nuvv < ((int64_t)1 << 31) && ngv / kPlanSliceRows < ((int64_t)1 << 31),
          "plan: hybrid layout overflow");
  P.hy_cols.resize(std::max<int64_t>(ncols, 1));
  if (ncols == 0) P.hy_cols[0] = 0;
  P.hy_uvval.resize(std::max<int64_t>(nuvv, 1));
  P.hy_gval.resize(std::max<int64_t>(ngv, 1));
  P.hy_uv_entries = P.hy_g_entries = 0;
  std::vector<int64_t> base_c(schunks + 1, 0), base_u(schunks + 1, 0), base_g(schunks + 1, 0);
  for (int w = 0; w < schunks; ++w) {
    base_c[w + 1] = base_c[w] + (int64_t)chunk[w].cols.size();
    base_u[w + 1] = base_u[w] + (int64_t)chunk[w].uv.size();
    base_g[w + 1] = base_g[w] + (int64_t)chunk[w].gv.size();
    P.hy_uv_entries += chunk[w].uv_entries;
    P.hy_g_entries += chunk[w].g_entries;
  }
  run_chunks(schunks, [&](int w) {   // every chunk moves to its place on its own thread
    Chunk& C = chunk[w];
    const int64_t bc = base_c[w], bu = base_u[w], bg = base_g[w];
    std::copy(C.cols.begin(), C.cols.end(), P.hy_cols.begin() + bc);
    std::copy(C.uv.begin(), C.uv.end(), P.hy_uvval.begin() + bu);
    std::copy(C.gv.begin(), C.gv.end(), P.hy_gval.begin() + bg);
    for (int64_t s = ns * w / schunks; s < ns * (w + 1) / schunks; ++s) {
      P.hy_slice[s].col_off += bc / kPlanSliceRows;
      P.hy_slice[s].uv_off += (int32_t)bu;
      P.hy_slice[s].g_off += (int32_t)(bg / kPlanSliceRows);
    }
  });
  sub.lap("  hybrid: concatenate");
  P.hy = true;
}

// ---- paired layout (plan.hpp) ------------------------------------------------------------
struct P2Spec {  // rows [row0, row0 + nrows) of the permuted order, block = dense block or -1
  int32_t row0, nrows, block;
};
// `skip` (optional, parallel to P.col / P.val): entries that a dense section holds instead.
void build_p2(HostPlan& P, const std::vector<P2Spec>& specs, const std::vector<uint8_t>* skip,
              const DenseBlocks* blocks) {
  const int64_t nl = P.nl;
  const int64_t ns = P.p2_slices = (int64_t)specs.size();
  P.p2_desc.assign(ns, PlanP2Slice{});
  P.p2_ptr.assign(ns + 1, 0);
  const int nchunks = (int)std::max<int64_t>(1, std::min<int64_t>(worker_count(), ns / 64));
  // merged (column, value A, value B) list of one lane, ascending column
  struct Entry {
    int32_t col;
    double a, b;
  };
  auto merge_lane = [&](int64_t rowA, int nrows, std::vector<Entry>& out, std::vector<Entry>& tmp) {
    out.clear();
    for (int which = 0; which < std::min(2, nrows); ++which) {
      const int64_t row = rowA + which;
      const int64_t s32 = row / kPlanSliceRows, l32 = row % kPlanSliceRows;
      const int64_t base = P.slice_ptr[s32] + l32;
      tmp.clear();
      for (int32_t p = 0; p < P.row_len[row]; ++p) {
        const int64_t e = base + (int64_t)p * kPlanSliceRows;
        if (skip && (*skip)[e]) continue;
        tmp.push_back({P.col[e], which == 0 ? P.val[e] : 0.0, which == 1 ? P.val[e] : 0.0});
      }
      std::sort(tmp.begin(), tmp.end(), [](const Entry& x, const Entry& y) { return x.col < y.col; });
      if (which == 0) {
        out.swap(tmp);
      } else {  // merge into out
        std::vector<Entry> merged;
        merged.reserve(out.size() + tmp.size());
        size_t i = 0, j = 0;
        while (i < out.size() || j < tmp.size()) {
          if (j == tmp.size() || (i < out.size() && out[i].col < tmp[j].col)) merged.push_back(out[i++]);
          else if (i == out.size() || tmp[j].col < out[i].col) merged.push_back(tmp[j++]);
          else {
            merged.push_back({out[i].col, out[i].a, tmp[j].b});
            ++i;
            ++j;
          }
        }
        out.swap(merged);
      }
    }
  };
  // pass 1: general positions per slice = the longest merged lane
  std::vector<int32_t> ng(ns, 0);
  run_chunks(nchunks, [&](int t) {
    std::vector<Entry> lane, tmp;
    for (int64_t s = ns * t / nchunks; s < ns * (t + 1) / nchunks; ++s) {
      int32_t L = 0;
      for (int l = 0; 2 * l < specs[s].nrows; ++l) {
        merge_lane(specs[s].row0 + 2 * l, specs[s].nrows - 2 * l, lane, tmp);
        L = std::max<int32_t>(L, (int32_t)lane.size());
      }
      ng[s] = L;
    }
  });
  int64_t gpos = 0, dpos = 0;
  for (int64_t s = 0; s < ns; ++s) {
    PlanP2Slice& D = P.p2_desc[s];
    D.gpos = gpos;
    D.dpos = dpos;
    D.ng = ng[s];
    D.nd = specs[s].block >= 0 ? (int32_t)blocks->members[specs[s].block].size() : 0;
    D.row0 = specs[s].row0;
    D.nrows = specs[s].nrows;
    P.p2_ptr[s] = gpos;
    gpos += D.ng;
    dpos += D.nd;
  }
  P.p2_ptr[ns] = gpos;
  P.p2_entries = gpos * 32;
  P.p2_col.assign(std::max<int64_t>(gpos * 32, 1), 0);
  P.p2_val.assign(std::max<int64_t>(gpos * 64, 2), 0.0);
  P.p2_dcol.assign(std::max<int64_t>(dpos, 1), 0);
  P.p2_dval.assign(std::max<int64_t>(dpos * 64, 2), 0.0);
  // pass 2: fill.  Padding entries of a general position repeat the column of the lane below
  // (no extra line for the gather) with zero values.
  std::vector<uint8_t> boundary(ns, 0);
  std::vector<int64_t> dense_fill(nchunks, 0);
  run_chunks(nchunks, [&](int t) {
    std::vector<Entry> lanes[32], tmp;
    for (int64_t s = ns * t / nchunks; s < ns * (t + 1) / nchunks; ++s) {
      const PlanP2Slice& D = P.p2_desc[s];
      int32_t* c = P.p2_col.data() + D.gpos * 32;
      double* v = P.p2_val.data() + D.gpos * 64;
      for (int l = 0; l < 32; ++l) {
        if (2 * l < D.nrows) merge_lane(D.row0 + 2 * l, D.nrows - 2 * l, lanes[l], tmp);
        else lanes[l].clear();
      }
      for (int32_t p = 0; p < D.ng; ++p) {
        int32_t fill = (int32_t)std::min<int64_t>(D.row0, std::max<int64_t>(nl - 1, 0));
        for (int l = 0; l < 32; ++l)
          if (p < (int32_t)lanes[l].size()) {
            fill = lanes[l][p].col;
            break;
          }
        for (int l = 0; l < 32; ++l) {
          const bool on = p < (int32_t)lanes[l].size();
          if (on) fill = lanes[l][p].col;
          if (fill >= nl) boundary[s] = 1;
          c[(int64_t)p * 32 + l] = fill;
          v[((int64_t)p * 32 + l) * 2] = on ? lanes[l][p].a : 0.0;
          v[((int64_t)p * 32 + l) * 2 + 1] = on ? lanes[l][p].b : 0.0;
        }
      }
      if (D.nd > 0) {  // dense section: the block's columns once, a value pair per lane
        const int32_t b = specs[s].block;
        const std::vector<int32_t>& mem = blocks->members[b];   // old ids, ascending
        int32_t* dc = P.p2_dcol.data() + D.dpos;
        double* dv = P.p2_dval.data() + D.dpos * 64;
        for (int32_t j = 0; j < D.nd; ++j) dc[j] = P.iperm[mem[j]];
        for (int32_t r = 0; r < D.nrows; ++r) {
          const int64_t row = D.row0 + r;
          const int64_t s32 = row / kPlanSliceRows, l32 = row % kPlanSliceRows;
          const int64_t base = P.slice_ptr[s32] + l32;
          for (int32_t p = 0; p < P.row_len[row]; ++p) {
            const int64_t e = base + (int64_t)p * kPlanSliceRows;
            if (!(*skip)[e]) continue;
            const int32_t old_col = P.perm[P.col[e]];
            const int32_t j = (int32_t)(std::lower_bound(mem.begin(), mem.end(), old_col) - mem.begin());
            dv[((int64_t)j * 32 + r / 2) * 2 + (r & 1)] = P.val[e];
            ++dense_fill[t];
          }
        }
      }
    }
  });
  P.p2_dense_entries = 0;
  for (int64_t f : dense_fill) P.p2_dense_entries += f;
  P.p2_interior.clear();
  P.p2_boundary.clear();
  std::vector<int32_t> all(ns), cost(ns);
  for (int64_t s = 0; s < ns; ++s) {
    all[s] = (int32_t)s;
    (boundary[s] ? P.p2_boundary : P.p2_interior).push_back((int32_t)s);
    // a dense position costs the kernel about 0.4 general ones
    cost[s] = P.p2_desc[s].ng + (2 * P.p2_desc[s].nd + 4) / 5;
  }
  choose_task_target(cost);
  P.p2_tasks_all = build_tasks(all, cost);
  P.p2_tasks_interior = build_tasks(P.p2_interior, cost);
  P.p2_tasks_boundary = build_tasks(P.p2_boundary, cost);
}

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

}  // namespace

// ---- index-compressed layout + task lists of the UG kernels (everything between the SELL
// arrays and the paired layout).  A separate step so that matrices which are certain to run the
// paired kernel can skip it (ensure_ug builds it on demand for the plan-inspection API).
void build_ug_section(HostPlan& P, const std::vector<uint8_t>& is_boundary) {
  const int64_t nslices = P.nslices;
  std::vector<int32_t> all(nslices);
  std::iota(all.begin(), all.end(), 0);
  // a rest launch per product only pays when it carries a real share of the matrix
  // uniform-value positions are read by the stencil ("lean") kernel only: try them when the
  // slices are short, and fall back when the matrix does not qualify for that kernel after all
  int32_t longest = 0;
  for (int64_t s = 0; s < nslices; ++s) longest = std::max(longest, P.slice_len[s]);
  bool allow_uv = longest <= 16;
  bool allow_spill = true;
  if (const int64_t spilled = build_ug(P, is_boundary, allow_spill, allow_uv);
      spilled > 0 && 50 * spilled < P.nnz) {
    allow_spill = false;
    build_ug(P, is_boundary, allow_spill, allow_uv);
  }
  std::vector<int32_t> ug_len(nslices + P.nrest);  // the fast kernels walk the compressed slices
  for (int64_t s = 0; s < nslices + P.nrest; ++s) ug_len[s] = P.ug_slice[s].nu + P.ug_slice[s].ng;
  choose_task_target(ug_len);
  {
    std::vector<int32_t> rest_all(P.rest_interior);
    rest_all.insert(rest_all.end(), P.rest_boundary.begin(), P.rest_boundary.end());
    P.tasks_rest_all = build_tasks(rest_all, ug_len);
    P.tasks_rest_interior = build_tasks(P.rest_interior, ug_len);
    P.tasks_rest_boundary = build_tasks(P.rest_boundary, ug_len);
  }
  P.tasks_all = build_tasks(all, ug_len);
  P.tasks_interior = build_tasks(P.interior, ug_len);
  P.tasks_boundary = build_tasks(P.boundary, ug_len);
  P.short_rows = std::all_of(P.tasks_all.begin(), P.tasks_all.end(),
                             [](const PlanTask& t) { return t.warps_per_slice == 1; });
  auto is_lean = [&] {
    bool lean = P.short_rows;
    for (int64_t s = 0; s < nslices && lean; ++s) lean = P.ug_slice[s].nu <= 8;
    return lean;
  };
  P.lean = is_lean();
  if (!P.lean && allow_uv) {  // rare: short slices, but not a stencil — redo without pairs
    build_ug(P, is_boundary, allow_spill, false);
    std::vector<int32_t> len2(nslices + P.nrest);
    for (int64_t s = 0; s < nslices + P.nrest; ++s) len2[s] = P.ug_slice[s].nu + P.ug_slice[s].ng;
    std::vector<int32_t> rest_all(P.rest_interior);
    rest_all.insert(rest_all.end(), P.rest_boundary.begin(), P.rest_boundary.end());
    P.tasks_rest_all = build_tasks(rest_all, len2);
    P.tasks_rest_interior = build_tasks(P.rest_interior, len2);
    P.tasks_rest_boundary = build_tasks(P.rest_boundary, len2);
    P.tasks_all = build_tasks(all, len2);
    P.tasks_interior = build_tasks(P.interior, len2);
    P.tasks_boundary = build_tasks(P.boundary, len2);
    P.short_rows = std::all_of(P.tasks_all.begin(), P.tasks_all.end(),
                               [](const PlanTask& t) { return t.warps_per_slice == 1; });
    P.lean = false;
  }
}

void ensure_ug(HostPlan& P) {
  if (!P.ug_skipped) return;
  if (P.hy)   // its SELL arrays group rows through sell_rows; no kernel reads a UG copy of them
    throw std::invalid_argument("plan: a hybrid plan has no index-compressed (UG) layout");
  std::vector<uint8_t> is_boundary(P.nslices, 0);
  for (int32_t s : P.boundary) is_boundary[s] = 1;
  build_ug_section(P, is_boundary);
  P.ug_skipped = false;
}

// Tile plan of the TMA-staged stencil kernel (plan.hpp, PlanStencilTiles).  Applies when the
// matrix is a stencil ("lean") in natural row order without rest slices; the uniform-value
// positions of all slices use at most 16 distinct offsets in kPlanMaxSegs segments.  The few
// slices that also hold per-lane positions (stencil rows next to a domain boundary) are
// flagged (bit 56 of position 0's mask word): the kernel adds those positions from global
// memory.
// Row slabs (nranks > 1): the kernel stages runs of the VIRTUAL gather source
// [front halo rows | local rows | back halo rows] — front = the halo slots whose owners have
// smaller rows — so that a neighbour plane that arrives from a peer sits at the offset it has
// inside the slab (100^3 Laplacian, z slabs: the offsets stay {-P^2, -P, -1, 0, 1, P, P^2} and
// the three segments of the single-rank plan).  A position's offset d into the stored source
// [local | halo] becomes d - (nl + front) when its lanes read front halo rows and d - front
// when they read back halo rows; a position whose lanes mix classes with different shifts has
// no tile plan.  Tiles [tile_a, tile_b) stage local rows only: they run while the halo travels.
static void build_stencil_tiles(HostPlan& P) {
  P.tiles = PlanStencilTiles{};
  if (!P.lean || P.nrest > 0 || P.sigma > 1) return;
  const bool slab = P.nranks != 1 || !P.halo.empty();
  const int64_t nl = P.nl;
  const int64_t front =
      std::lower_bound(P.halo.begin(), P.halo.end(), P.row_begin) - P.halo.begin();
  const int64_t back = (int64_t)P.halo.size() - front;
  // 16-byte bulk copies: the pieces of a run start at even rows of the stored source
  if (slab && ((nl & 1) || (front & 1) || nl == 0)) return;
  if (slab) {
    static const bool off = [] {   // FLZ_ST_SLAB=0: row slabs keep the one-warp-per-slice kernel
      const char* e = std::getenv("FLZ_ST_SLAB");
      return e && e[0] == '0';
    }();
    if (off) return;
  }
  int T = 256;  // B200, 100^3 Laplacian, 3 columns: 16.4 us per step (128: 17.3, 512: 16.9)
  if (const char* e = std::getenv("FLZ_ST_TILE")) T = std::atoi(e);
  if (T <= 0) return;  // FLZ_ST_TILE=0 switches the tile kernel off
  T = std::clamp(T / kPlanSliceRows, 1, 16) * kPlanSliceRows;
  // offset of position p of slice s in the virtual source; false: lanes of mixed classes
  auto virtual_off = [&](int64_t s, int p, int32_t d, int64_t& out) {
    if (!slab) {
      out = d;
      return true;
    }
    uint64_t bits;
    std::memcpy(&bits, &P.uv_pairs[s * 16 + 2 * p + 1], 8);
    const uint32_t mask = (uint32_t)bits;
    int64_t shift = 0;
    bool have = false;
    for (int l = 0; l < kPlanSliceRows; ++l) {
      if (!((mask >> l) & 1u)) continue;
      const int64_t c = s * kPlanSliceRows + l + d;
      const int64_t sh = c < nl ? 0 : (c < nl + front ? -(nl + front) : -front);
      if (have && sh != shift) return false;
      shift = sh;
      have = true;
    }
    out = have ? d + shift : 0;
    return true;
  };
  std::vector<int32_t> offs{0};
  for (int64_t s = 0; s < P.nslices; ++s) {
    const PlanUgSlice& H = P.ug_slice[s];
    const int nuv = (H.reserved >> 16) & 0xff;
    if (nuv > 8 || H.nu > 8 || (H.reserved & 3)) return;
    for (int p = 0; p < nuv; ++p) {
      int64_t d = 0;
      if (!virtual_off(s, p, H.inline_off[p], d)) return;
      if (d < INT32_MIN / 2 || d > INT32_MAX / 2) return;
      if (std::find(offs.begin(), offs.end(), (int32_t)d) == offs.end()) {
        if (offs.size() >= 16) return;
        offs.push_back((int32_t)d);
      }
    }
  }
  std::sort(offs.begin(), offs.end());
  PlanStencilTiles G;
  G.tile_rows = T;
  auto even_down = [](int32_t v) { return v & ~1; };
  size_t i = 0;
  while (i < offs.size()) {
    size_t j = i;
    while (j + 1 < offs.size() && (int64_t)offs[j + 1] - offs[j] < T) ++j;
    if (G.nseg == kPlanMaxSegs) return;
    const int32_t base = even_down(offs[i]);
    const int32_t len = (T + (offs[j] - base) + 1) & ~1;
    G.seg_base[G.nseg] = base;
    G.seg_len[G.nseg] = len;
    G.seg_start[G.nseg] = G.y1_elems;
    G.y1_elems += len;
    ++G.nseg;
    i = j + 1;
  }
  if (G.y1_elems > 24 * T || G.y1_elems >= 65536) return;  // staging would not fit (20-bit byte offsets)
  auto staged = [&](int32_t d) {
    for (int j = G.nseg - 1; j >= 0; --j)
      if (d >= G.seg_base[j]) return G.seg_start[j] + (d - G.seg_base[j]);
    return 0;
  };
  G.own_e = staged(0);
  const int64_t per_tile = T / kPlanSliceRows;
  const int64_t ntiles = (P.nslices + per_tile - 1) / per_tile;
  // tiles whose runs stay inside the local rows (no halo row staged): [tile_a, tile_b)
  int64_t tile_a = 0, tile_b = ntiles;
  if (slab) {
    const int64_t lo = G.seg_base[0];
    const int64_t hi = (int64_t)G.seg_base[G.nseg - 1] + G.seg_len[G.nseg - 1];   // run end, tile 0
    if (front > 0 && lo < 0) tile_a = std::min(ntiles, (-lo + T - 1) / T);
    if (back > 0) tile_b = nl >= hi ? std::min(ntiles, (nl - hi) / T + 1) : 0;
    tile_b = std::max(tile_a, tile_b);
    // every slice that references a halo row (uniform or per-lane position) must lie outside
    for (int32_t s : P.boundary) {
      const int64_t t = s / per_tile;
      if (t >= tile_a && t < tile_b) return;
    }
  }
  G.front = (int32_t)front;
  G.back = (int32_t)back;
  G.tile_a = (int32_t)tile_a;
  G.tile_b = (int32_t)tile_b;
  P.uv_pairs.resize((size_t)(ntiles * per_tile) * 16, 0.0);
  for (int64_t s = 0; s < P.nslices; ++s) {
    const PlanUgSlice& H = P.ug_slice[s];
    const int nuv = (H.reserved >> 16) & 0xff;
    for (int p = 0; p < nuv; ++p) {
      int64_t d = 0;
      virtual_off(s, p, H.inline_off[p], d);
      uint64_t bits;
      std::memcpy(&bits, &P.uv_pairs[s * 16 + 2 * p + 1], 8);
      bits &= 0xffffffffull;
      bits |= (uint64_t)(uint32_t)(8 * staged((int32_t)d)) << 32;
      if (p == 0) bits |= (uint64_t)nuv << 52;
      std::memcpy(&P.uv_pairs[s * 16 + 2 * p + 1], &bits, 8);
    }
    if (H.ng != 0 || H.nu != nuv) {  // the slice also has per-lane positions (read from global)
      uint64_t bits;
      std::memcpy(&bits, &P.uv_pairs[s * 16 + 1], 8);
      bits |= 1ull << 56;
      std::memcpy(&P.uv_pairs[s * 16 + 1], &bits, 8);
    }
  }
  P.tiles = G;
}

HostPlan build_plan(int64_t n_global, int rank, int nranks, const std::vector<int64_t>& starts,
                    const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                    int sigma, bool allow_hybrid) {
  require(nranks >= 1 && rank >= 0 && rank < nranks, "plan: bad rank/nranks");
  require((int)starts.size() == nranks + 1 && starts.front() == 0 && starts.back() == n_global,
          "plan: rank row ranges must cover [0, n)");
  for (int p = 0; p < nranks; ++p)
    require(starts[p] <= starts[p + 1], "plan: rank row ranges must be ascending and contiguous");
  HostPlan P;
  P.rank = rank;
  P.nranks = nranks;
  P.n_global = n_global;
  P.starts = starts;
  P.row_begin = starts[rank];
  P.row_end = starts[rank + 1];
  const int64_t nl = P.nl = P.row_end - P.row_begin;
  require(nl < ((int64_t)1 << 31), "plan: too many local rows");
  P.nnz = nl > 0 ? row_ptr[nl] - row_ptr[0] : 0;

  std::vector<int32_t> len(nl);
  for (int64_t i = 0; i < nl; ++i) {
    const int64_t l = row_ptr[i + 1] - row_ptr[i];
    require(l >= 0 && l < ((int64_t)1 << 31), "plan: bad row_ptr");
    len[i] = (int32_t)l;
  }
  const int64_t p0 = nl > 0 ? row_ptr[0] : 0;
  {
    const int vchunks = (int)std::max<int64_t>(1, std::min<int64_t>(worker_count(), P.nnz >> 18));
    run_chunks(vchunks, [&](int t) {
      for (int64_t p = P.nnz * t / vchunks; p < P.nnz * (t + 1) / vchunks; ++p)
        require(col_idx[p0 + p] >= 0 && col_idx[p0 + p] < n_global,
                "plan: column index out of range");
    });
  }

  PhaseTimer timer;
  timer.lap("validate");
  // ---- SPLIT mode?  Count the nonzeros whose diagonal offset is shared by at least
  // kUgMinLanes rows of their natural-order slice (global indices: a good estimate of what
  // build_ug finds after the halo columns are renumbered).
  P.split = false;
  if (sigma <= 0 && nl > 0) {
    int32_t max_len = 0;
    for (int64_t i = 0; i < nl; ++i) max_len = std::max(max_len, len[i]);
    size_t cap = 64;
    while (cap < (size_t)max_len * kPlanSliceRows * 2) cap <<= 1;
    const int64_t nsl = (nl + kPlanSliceRows - 1) / kPlanSliceRows;
    const int nchunks = (int)std::max<int64_t>(1, std::min<int64_t>(worker_count(), nsl / 256));
    std::vector<int64_t> part(nchunks, 0);
    run_chunks(nchunks, [&](int t) {
      OffsetCounter counter(cap);
      for (int64_t sl = nsl * t / nchunks; sl < nsl * (t + 1) / nchunks; ++sl) {
        const int64_t i0 = sl * kPlanSliceRows;
        counter.clear();
        const int64_t i1 = std::min(nl, i0 + kPlanSliceRows);
        for (int64_t i = i0; i < i1; ++i)
          for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            counter.add((int64_t)col_idx[p] - (P.row_begin + i));
        for (int32_t h : counter.used)
          if (counter.cnt[h] >= kUgMinLanes) part[t] += counter.cnt[h];
      }
    });
    int64_t uniform = 0;
    for (int64_t v : part) uniform += v;
    P.split = 2 * uniform >= P.nnz;
    if (const char* force = std::getenv("FLZ_SPLIT")) P.split = force[0] == '1';  // experiments
  }

  timer.lap("split estimate");
  // ---- paired layout ahead?  Then rows are sorted as pairs (see sort_windows): key = size of
  // the merged column list of rows (2k, 2k+1), half of it per row so that classes stay
  // comparable with row lengths
  static const bool want_p2_sort = [] {
    const char* e = std::getenv("FLZ_P2");
    return !(e && e[0] == '0');
  }();
  // Dense blocks are searched for when the hybrid layout can use them (one rank), or when the
  // paired layout is asked to keep dense sections (FLZ_P2_DENSE=1, experiments: measured slower
  // than the plain paired layout on the PARSEC shapes, 36.3 vs 30.0 us per step at n = 113k)
  const bool p2_dense = [] {
    const char* e = std::getenv("FLZ_P2_DENSE");
    return e && e[0] == '1';
  }();
  const bool hy_wanted = allow_hybrid && [] {
    const char* e = std::getenv("FLZ_HY");
    return !(e && e[0] == '0');
  }();
  const bool want_dense = p2_dense || hy_wanted;
  int32_t longest = 0;
  for (int64_t i = 0; i < nl; ++i) longest = std::max(longest, len[i]);
  const bool p2_candidate = want_p2_sort && !P.split && longest > 24 && nl > 0;
  // size of the union of the (global, ascending) column lists of two local rows
  auto union_size = [&](int64_t i, int64_t j) {
    int64_t a = row_ptr[i], a1 = row_ptr[i + 1], b = row_ptr[j], b1 = row_ptr[j + 1];
    int32_t u = 0;
    while (a < a1 || b < b1) {
      if (b == b1 || (a < a1 && col_idx[a] < col_idx[b])) ++a;
      else if (a == a1 || col_idx[b] < col_idx[a]) ++b;
      else {
        ++a;
        ++b;
      }
      ++u;
    }
    return u;
  };
  std::vector<int32_t> pair_key;
  DenseBlocks blocks;
  std::vector<int32_t> block_order;   // new -> old when dense blocks order the rows
  std::vector<P2Spec> specs;
  if (p2_candidate && want_dense && sigma <= 0)
    blocks = extract_dense_blocks(nl, P.row_begin, row_ptr, col_idx, len, P.nnz);
  timer.lap("dense blocks");
  // HYBRID layout (plan.hpp): natural row order, dense tasks + value-grouped slices.  One rank
  // only (the slices gather local rows); FLZ_HY=0 keeps the paired layout (experiments).
  bool hybrid = hy_wanted && blocks.any();
  if (hybrid) {
    size_t widest = 0;
    for (const auto& K : blocks.members) widest = std::max(widest, K.size());
    hybrid = widest <= 1400;   // the staged block rows of a task must fit 48 KB of shared memory
  }
  if (hybrid) {
    // what the blocks leave of every row must be short (the stencil): long leftovers (balls
    // the block search missed, heavily overlapping balls) would become hundreds of general
    // positions per slice — such matrices keep the paired layout
    std::vector<int32_t> tmp(len);   // "short" = twice the 10th percentile of the row lengths
    std::nth_element(tmp.begin(), tmp.begin() + nl / 10, tmp.end());
    const int64_t limit = 2 * (int64_t)tmp[nl / 10] + 8;
    const int64_t q0 = row_ptr[0];
    const int echunks = (int)std::max<int64_t>(1, std::min<int64_t>(worker_count(), nl / 4096));
    std::vector<int64_t> part(echunks, 0);
    run_chunks(echunks, [&](int t) {
      int64_t sum = 0;
      for (int64_t i = nl * t / echunks; i < nl * (t + 1) / echunks; ++i) {
        int64_t left = 0;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) left += blocks.covered[e - q0] ? 0 : 1;
        sum += std::max<int64_t>(0, left - limit);
      }
      part[t] = sum;
    });
    int64_t excess = 0;
    for (int64_t v : part) excess += v;
    hybrid = 20 * excess <= P.nnz;
  }
  if (blocks.any() && !hybrid && !p2_dense) blocks = DenseBlocks{};   // plain paired layout
  if (blocks.any() && !hybrid) {
    // row order: rows in several blocks (all entries general, longest first), then block by
    // block the rows that belong to that block only, then the rows outside every block in
    // natural order, pairs sorted by length class inside windows.  A slice never straddles
    // two of these groups.
    block_order.reserve(nl);
    auto emit = [&](const std::vector<int32_t>& rows, int32_t block) {
      for (size_t i = 0; i < rows.size(); i += 64) {
        const int32_t cnt = (int32_t)std::min<size_t>(64, rows.size() - i);
        specs.push_back({(int32_t)block_order.size(), cnt, block});
        block_order.insert(block_order.end(), rows.begin() + i, rows.begin() + i + cnt);
      }
    };
    std::vector<int32_t> rows;
    for (int64_t i = 0; i < nl; ++i)
      if (blocks.count[i] >= 2) rows.push_back((int32_t)i);
    std::stable_sort(rows.begin(), rows.end(), [&](int32_t a, int32_t b) {
      return length_class(len[a]) > length_class(len[b]);
    });
    emit(rows, -1);
    for (size_t b = 0; b < blocks.members.size(); ++b) {
      rows.clear();
      for (int32_t j : blocks.members[b])
        if (blocks.primary[j] == (int32_t)b) rows.push_back(j);
      emit(rows, (int32_t)b);
    }
    // rows outside every block: CLUSTERS of `cluster_rows` rows that share gather targets
    // (one CTA task each), grown greedily over the matrix graph — always add the frontier row
    // with the most entries into the cluster.  On a 3D stencil a cluster is a compact brick, so
    // the block rows its lanes gather are fetched from L2 once per CTA and then hit L1: the
    // kernel is bound by L2 -> SM traffic, and in natural order a gathered row was
    // fetched again by every x-line that needs it.
    rows.clear();
    static const int cluster_rows = [] {
      const char* e = std::getenv("FLZ_P2_CLUSTER_ROWS");
      return e && *e ? std::max(64, std::atoi(e)) : 512;
    }();
    {
      // units = the pairs a lane will own: two rows with consecutive indices (x-neighbours
      // share 12 of 13 x-entries), or a single row where the neighbour is missing
      std::vector<int32_t> unit_of(nl, -1), ua, ub;
      for (int64_t i = 0; i < nl; ++i) {
        if (blocks.count[i] != 0 || unit_of[i] >= 0) continue;
        const bool pair = i + 1 < nl && blocks.count[i + 1] == 0;
        unit_of[i] = (int32_t)ua.size();
        if (pair) unit_of[i + 1] = (int32_t)ua.size();
        ua.push_back((int32_t)i);
        ub.push_back(pair ? (int32_t)(i + 1) : -1);
      }
      const int64_t nu = (int64_t)ua.size();
      const int32_t maxdeg = 2 * longest;
      std::vector<uint8_t> taken(nu, 0);
      std::vector<std::vector<int32_t>> bucket(maxdeg + 1);
      std::vector<int32_t> links(nu, 0), touched, cluster;
      int64_t next_seed = 0;
      while (true) {
        while (next_seed < nu && taken[next_seed]) ++next_seed;
        if (next_seed >= nu) break;
        cluster.clear();
        touched.clear();
        int top = 0, nrows_in = 0;
        auto add = [&](int32_t u) {
          taken[u] = 1;
          cluster.push_back(u);
          for (int32_t i : {ua[u], ub[u]}) {
            if (i < 0) continue;
            ++nrows_in;
            // STRONG connections only (|a_ij| >= 1/4 of the row's largest off-diagonal entry,
            // as in algebraic multigrid): on a high-order stencil these are the nearest
            // neighbours, so the cluster grows as a compact brick instead of along the arms
            double big = 0.0;
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
              if ((int64_t)col_idx[e] - P.row_begin != i) big = std::max(big, std::abs(values[e]));
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
              const int64_t c = (int64_t)col_idx[e] - P.row_begin;
              if (c < 0 || c >= nl || std::abs(values[e]) < 0.25 * big) continue;
              const int32_t v = unit_of[c];
              if (v < 0 || taken[v]) continue;
              if (links[v] == 0) touched.push_back(v);
              const int32_t k = std::min(++links[v], maxdeg);
              bucket[k].push_back(v);
              top = std::max(top, (int)k);
            }
          }
        };
        add((int32_t)next_seed);
        while (nrows_in < cluster_rows) {
          int32_t pick = -1;
          while (top > 0 && pick < 0) {
            auto& bk = bucket[top];
            while (!bk.empty() && pick < 0) {
              const int32_t v = bk.back();
              bk.pop_back();
              if (!taken[v] && std::min(links[v], maxdeg) == top) pick = v;  // else stale
            }
            if (pick < 0) --top;
          }
          if (pick < 0) break;  // component exhausted
          add(pick);
        }
        for (int32_t v : touched) links[v] = 0;
        for (int k = 1; k <= maxdeg; ++k) bucket[k].clear();
        // inside a cluster: ascending index, then by length class so that the lanes of a
        // slice pad little; single rows last (two of them share a lane)
        std::sort(cluster.begin(), cluster.end());
        std::vector<int32_t> cls(cluster.size());
        for (size_t q = 0; q < cluster.size(); ++q) {
          const int32_t u = cluster[q];
          cls[q] = ub[u] < 0 ? -1 : length_class((union_size(ua[u], ub[u]) + 1) / 2);
        }
        std::vector<int32_t> pid(cluster.size());
        std::iota(pid.begin(), pid.end(), 0);
        std::stable_sort(pid.begin(), pid.end(), [&](int32_t a, int32_t b) { return cls[a] > cls[b]; });
        for (int32_t q : pid) {
          rows.push_back(ua[cluster[q]]);
          if (ub[cluster[q]] >= 0) rows.push_back(ub[cluster[q]]);
        }
      }
    }
    const std::vector<int32_t>& sorted = rows;
    emit(sorted, -1);
    if (std::getenv("FLZ_TRACE"))
      std::fprintf(stderr, "[flz]   plan dense blocks: %zu blocks cover %lld of %lld entries, "
                           "%zu slices\n", blocks.members.size(), (long long)blocks.covered_entries,
                   (long long)P.nnz, specs.size());
  } else if (p2_candidate) {
    pair_key.assign(nl, 0);
    for (int64_t i = 0; i < nl; i += 2) {
      const int32_t u = i + 1 < nl ? union_size(i, i + 1) : len[i];
      pair_key[i] = (u + 1) / 2;
      if (i + 1 < nl) pair_key[i + 1] = (u + 1) / 2;
    }
  }
  const std::vector<int32_t>* sort_key = pair_key.empty() ? nullptr : &pair_key;

  // ---- halo columns: sorted unique remote global ids, grouped by owner
  if (nranks > 1) {
    for (int64_t p = 0; p < P.nnz; ++p) {
      const int64_t g = col_idx[p0 + p];
      if (g < P.row_begin || g >= P.row_end) P.halo.push_back(g);
    }
    std::sort(P.halo.begin(), P.halo.end());
    P.halo.erase(std::unique(P.halo.begin(), P.halo.end()), P.halo.end());
  }
  require(nl + (int64_t)P.halo.size() < ((int64_t)1 << 31), "plan: index overflow");
  P.need_off.assign(nranks, 0);
  P.need_cnt.assign(nranks, 0);
  {
    size_t h = 0;
    for (int p = 0; p < nranks; ++p) {
      P.need_off[p] = (int64_t)h;
      while (h < P.halo.size() && P.halo[h] < starts[p + 1]) ++h;
      P.need_cnt[p] = (int64_t)h - P.need_off[p];
    }
  }
  P.give_off.assign(nranks, 0);
  P.give_cnt.assign(nranks, 0);

  // The hybrid layout depends on the blocks only (natural row order): it is built on its own
  // thread while this one sorts the rows and fills the CSR-order SELL arrays.  build_hybrid
  // writes the hy_* members of P and nothing else.
  std::thread hybrid_thread;
  std::exception_ptr hybrid_error;
  if (hybrid)
    hybrid_thread = std::thread([&] {
      try {
        build_hybrid(P, blocks, row_ptr, col_idx, values);
      } catch (...) {
        hybrid_error = std::current_exception();
      }
    });
  struct JoinGuard {   // an exception on this thread must not leave the worker running
    std::thread& t;
    ~JoinGuard() {
      if (t.joinable()) t.join();
    }
  } hybrid_guard{hybrid_thread};

  // ---- sigma: smallest window whose padding overhead is <= 8 %
  int64_t chosen = sigma;
  if (P.split) {
    chosen = 1;  // natural order: uniform offsets only exist there
  } else if (sigma <= 0 && sort_key) {
    chosen = 16384;  // pairs: measured gathers/nnz 0.83 (1024), 0.77 (4096), 0.76 (16384), 0.75 (n)
  } else if (sigma <= 0) {
    const int64_t cands[] = {1, 256, 4096, 65536, std::max<int64_t>(nl, 1)};
    int64_t best_fill = -1;
    chosen = 1;
    for (int64_t sg : cands) {
      if (sg > 1 && sg > nl && sg != cands[4]) continue;
      sort_windows(len, sg, P.perm, sort_key);
      const int64_t f = padded_entries(len, P.perm);
      if (best_fill < 0 || f < best_fill) {
        best_fill = f;
        chosen = sg;
      }
      if ((double)f <= 1.08 * (double)std::max<int64_t>(P.nnz, 1)) {
        chosen = sg;
        break;
      }
    }
  }
  std::vector<int32_t> sell_order;   // hybrid: grouping of the exact-mode SELL arrays only
  if (hybrid) {
    chosen = 1;
    sort_windows(len, chosen, P.perm, nullptr);   // identity: the device order is the natural one
    sort_windows(len, std::max<int64_t>(nl, 2), sell_order, nullptr);
  } else if (blocks.any()) {
    P.perm = block_order;
    chosen = std::max<int64_t>(nl, 2);
  } else {
    sort_windows(len, chosen, P.perm, sort_key);
  }
  P.sigma = (int)std::min<int64_t>(chosen, 1 << 30);
  bool identity = true;
  for (int64_t i = 0; i < nl && identity; ++i) identity = P.perm[i] == i;
  if (identity) P.sigma = 1;
  P.iperm.resize(nl);
  for (int64_t i = 0; i < nl; ++i) P.iperm[P.perm[i]] = (int32_t)i;

  timer.lap("sigma / perm");
  timer.lap("halo");
  // ---- SELL-32 storage
  const int64_t nslices = P.nslices = (nl + kPlanSliceRows - 1) / kPlanSliceRows;
  P.slice_ptr.assign(nslices + 1, 0);
  P.slice_len.assign(nslices, 0);
  P.row_len.assign(nslices * kPlanSliceRows, 0);
  const std::vector<int32_t>& sell_of = hybrid ? sell_order : P.perm;   // SELL lane -> old row
  if (hybrid) {
    P.sell_rows.assign(nslices * kPlanSliceRows, -1);
    std::copy(sell_order.begin(), sell_order.end(), P.sell_rows.begin());
  }
  for (int64_t s = 0; s < nslices; ++s) {
    int32_t mx = 0;
    for (int l = 0; l < kPlanSliceRows; ++l) {
      const int64_t inew = s * kPlanSliceRows + l;
      if (inew >= nl) break;
      P.row_len[inew] = len[sell_of[inew]];
      mx = std::max(mx, P.row_len[inew]);
    }
    P.slice_len[s] = mx;
    P.slice_ptr[s + 1] = P.slice_ptr[s] + (int64_t)mx * kPlanSliceRows;
  }
  P.stored = P.slice_ptr[nslices];
  P.col.resize(std::max<int64_t>(P.stored, 1));   // uninitialised: every stored entry is written
  P.val.resize(std::max<int64_t>(P.stored, 1));   // by the fill below (real entries + padding)
  if (P.stored == 0) {
    P.col[0] = 0;
    P.val[0] = 0.0;
  }
  std::vector<uint8_t> is_boundary(nslices, 0);
  // entries the dense sections of the paired layout hold (rows that belong to one block only)
  std::vector<uint8_t> skip;
  if (blocks.any() && !hybrid) skip.assign(std::max<int64_t>(P.stored, 1), 0);
  const int fill_chunks = (int)std::max<int64_t>(1, std::min<int64_t>(worker_count(), nslices / 256));
  run_chunks(fill_chunks, [&](int t) {
  for (int64_t s = nslices * t / fill_chunks; s < nslices * (t + 1) / fill_chunks; ++s)
    for (int l = 0; l < kPlanSliceRows; ++l) {
      const int64_t inew = s * kPlanSliceRows + l;
      const int64_t base = P.slice_ptr[s] + l;
      const int32_t self = (int32_t)std::min<int64_t>(inew, std::max<int64_t>(nl - 1, 0));
      int32_t cnt = 0;
      if (inew < nl) {
        const int64_t iold = sell_of[inew];
        for (int64_t p = row_ptr[iold]; p < row_ptr[iold + 1]; ++p, ++cnt) {  // CSR order kept
          const int64_t g = col_idx[p];
          int32_t c;
          if (g >= P.row_begin && g < P.row_end) {
            c = P.iperm[g - P.row_begin];
          } else {
            const int64_t slot = std::lower_bound(P.halo.begin(), P.halo.end(), g) - P.halo.begin();
            c = (int32_t)(nl + slot);
            is_boundary[s] = 1;
          }
          P.col[base + (int64_t)cnt * kPlanSliceRows] = c;
          P.val[base + (int64_t)cnt * kPlanSliceRows] = values[p];
          if (!skip.empty() && blocks.covered[p - p0] && blocks.count[iold] == 1)
            skip[base + (int64_t)cnt * kPlanSliceRows] = 1;
        }
      }
      for (; cnt < P.slice_len[s]; ++cnt) {  // padding: zero value, harmless in-range column
        P.col[base + (int64_t)cnt * kPlanSliceRows] = self;
        P.val[base + (int64_t)cnt * kPlanSliceRows] = 0.0;
      }
    }
  });
  std::vector<int32_t> all(nslices);
  std::iota(all.begin(), all.end(), 0);
  for (int64_t s = 0; s < nslices; ++s)
    (is_boundary[s] ? P.boundary : P.interior).push_back((int32_t)s);
  timer.lap("SELL arrays");
  // Matrices that are certain to take the paired kernel never read the UG layout: a slice
  // longer than the largest entries-per-warp target cannot be a one-warp ("short rows") task,
  // so the stencil kernel is out and P.p2 below is true.  Skipping the UG build saves 55 ms of
  // a 0.2 s ingest on the PARSEC-shaped n = 113k matrix (and its upload).
  static const bool want_p2 = [] {
    const char* e = std::getenv("FLZ_P2");
    return !(e && e[0] == '0');
  }();
  {
    int32_t longest_slice = 0;
    for (int64_t s = 0; s < nslices; ++s) longest_slice = std::max(longest_slice, P.slice_len[s]);
    P.ug_skipped = want_p2 && !P.split && nl > 0 && p2_candidate && (longest_slice > 256 || blocks.any()) &&
                   std::getenv("FLZ_K1_T") == nullptr && std::getenv("FLZ_UG_ALWAYS") == nullptr;
    if (hybrid) P.ug_skipped = true;
  }
  if (P.ug_skipped) {
    P.short_rows = false;
    P.lean = false;
  } else {
    build_ug_section(P, is_boundary);
  }
  timer.lap("UG layout");
  // long ragged rows: the paired layout feeds the fast kernel (FLZ_P2=0 keeps the UG tasks)
  P.p2 = want_p2 && !P.split && !P.lean && nl > 0 && p2_candidate && !hybrid;
  if (hybrid) {
    hybrid_thread.join();
    if (hybrid_error) std::rethrow_exception(hybrid_error);
    timer.lap("hybrid layout (rest; built beside the SELL arrays)");
  }
  if (P.p2) {
    if (!blocks.any()) {
      specs.clear();
      for (int64_t r0 = 0; r0 < nl; r0 += 64)
        specs.push_back({(int32_t)r0, (int32_t)std::min<int64_t>(64, nl - r0), -1});
    }
    P.p2_blocks = (int64_t)blocks.members.size();
    build_p2(P, specs, blocks.any() ? &skip : nullptr, blocks.any() ? &blocks : nullptr);
  }
  timer.lap("paired layout");
  P.uv_pairs.clear();
  if (P.lean) {
    P.uv_pairs.assign((size_t)nslices * 16, 0.0);
    for (int64_t s = 0; s < nslices; ++s) {
      const int nuv = (P.ug_slice[s].reserved >> 16) & 0xff;
      std::copy_n(P.ug_val.data() + P.ug_slice[s].val_ptr, 2 * nuv, P.uv_pairs.data() + s * 16);
    }
    build_stencil_tiles(P);
  }
  return P;
}

void plan_set_give(HostPlan& P, int peer, int64_t count, const int64_t* global_rows) {
  require(peer >= 0 && peer < P.nranks && peer != P.rank, "plan: bad peer");
  require(P.give_cnt[peer] == 0, "plan: give list of this peer was already set");
  P.give_off[peer] = (int64_t)P.send_rows.size();
  P.give_cnt[peer] = count;
  for (int64_t i = 0; i < count; ++i) {
    require(global_rows[i] >= P.row_begin && global_rows[i] < P.row_end,
            "plan: peer requested a row this rank does not own");
    P.send_rows.push_back(P.iperm[global_rows[i] - P.row_begin]);
  }
}

}  // namespace flz
