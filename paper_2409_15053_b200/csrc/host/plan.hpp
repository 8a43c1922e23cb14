// host/plan.hpp — host-only construction of the device matrix layout and the halo plan.
//
// Everything flz_matrix_upload() decides on the host lives here so that the multi-GPU logic
// (row partition, halo lists, interior/boundary split) can be unit-tested on CPUs
// (tests/test_dist_plan.py drives it over gloo, world_size 2): SELL-32-sigma conversion of
// the local rows of a CSR matrix (reference layout: sparse.hpp:28-33), renumbering of remote
// columns to halo slots, per-peer "need" lists and, once the peers' requests are known,
// the rows to pack for them.
#pragma once

#include <cstdint>
#include <vector>
#include <memory>
#include <type_traits>
#include <utility>

namespace flz {

// std::vector whose resize() leaves trivially-constructible elements uninitialised: the big
// layout arrays (tens of MB) are then first touched by the threads that fill them instead of
// being zero-filled by one thread first (a third of the layout time on an 8M-nonzero matrix).
template <class T>
struct DefaultInitAllocator : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAllocator<U>;
  };
  using std::allocator<T>::allocator;
  template <class U>
  void construct(U* p) noexcept(std::is_nothrow_default_constructible<U>::value) {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};
template <class T>
using BigVec = std::vector<T, DefaultInitAllocator<T>>;


constexpr int kPlanSliceRows = 32;
constexpr int kPlanTaskWarps = 8;

struct PlanTask {  // mirrors SliceTask (flz_internal.hpp)
  int32_t warps_per_slice;
  int32_t count;
  int32_t slice[kPlanTaskWarps];
};

// Per-slice header of the index-compressed ("UG") layout the fast kernels read: the first
// `nu` positions of a slice are UNIFORM (every lane's column is its own row + uoff[p], one
// int32 per position instead of 32), the remaining `ng` positions are GENERAL (one int32 per
// lane).  The first `nuv` (flags bits 16-23) uniform positions also have a UNIFORM VALUE:
// every lane that holds the entry holds the same number (constant-coefficient stencils), and
// the slice stores one (value, 32-bit lane mask) pair for the position instead of 32 values.
// Value block of a slice: nuv pairs (padded to 16 doubles when rows follow), then
// [nu - nuv + ng][32] doubles; padding entries have value 0 and a harmless column.
// flags (`reserved`): bit 0 the slice adds rest partial sums, bit 1 the uniform int32 are
// absolute columns (rest slices), bit 2 position 0 is the diagonal offset 0 with a uniform
// value (its gather is the slice's own rows), bits 16-23 nuv.
struct PlanUgSlice {
  int64_t val_ptr;   // element offset into ug_val
  int64_t col_ptr;   // element offset into ug_col (general positions only)
  int32_t uoff_ptr;  // offset into ug_uoff
  int32_t nu, ng;
  int32_t reserved;
  int32_t inline_off[8];  // the first offsets again: one 64-byte load serves short slices
};

// TILE plan of a constant-coefficient stencil on one rank (every position of every slice is
// a uniform offset with a uniform value): the TMA-staged stencil kernel walks tiles of
// `tile_rows` consecutive rows and bulk-copies, per tile, the contiguous runs of the gather
// source its offsets reach.  Offsets closer than a tile are merged into one SEGMENT
// [base, base + tile_rows + extra) (base even: 16-byte aligned bulk copies); seg_start is the
// segment's first element inside the staged Y1 column (y1_elems per column).  Position p of a
// slice with offset d reads staged element seg_start[j] + (d - seg_base[j]) + (row - tile row 0);
// that number times 8 (a byte offset) sits in bits 32-51 of the position's mask word in
// uv_pairs, the slice's position count in bits 52-55 of position 0, and bit 56 of position 0
// flags a slice that also has
// per-lane positions (the kernel adds them from global memory).  nseg == 0: not applicable.
constexpr int kPlanMaxSegs = 8;
struct PlanStencilTiles {
  int32_t tile_rows = 0, nseg = 0;
  int32_t seg_base[kPlanMaxSegs] = {}, seg_len[kPlanMaxSegs] = {}, seg_start[kPlanMaxSegs] = {};
  int32_t y1_elems = 0;  // staged elements per block column (sum of the segment lengths)
  int32_t own_e = 0;     // staged element of offset 0 (the tile's own rows)
  // row slabs: the staged source is [front halo rows | local rows | back halo rows]; tiles
  // [tile_a, tile_b) stage local rows only (they run while the halo rows travel)
  int32_t front = 0, back = 0;
  int32_t tile_a = 0, tile_b = 0;
};

// Slice descriptor of the paired layout (mirrors P2Slice, flz_internal.hpp): general positions
// [gpos, gpos + ng) of p2_col / p2_val, dense positions [dpos, dpos + nd) of p2_dcol / p2_dval,
// rows [row0, row0 + nrows), nrows <= 64.
struct PlanP2Slice {
  int64_t gpos, dpos;
  int32_t ng, nd;
  int32_t row0, nrows;
};

// HYBRID layout ("HY") for matrices that are a short-row part (a stencil) plus dense blocks
// (non-local projector balls of PARSEC-like Hamiltonians), single rank.  Rows keep their
// NATURAL order (no permutation), so that the lanes of a slice — 32 consecutive rows, i.e. a
// run of grid points — gather runs of consecutive block rows.  A product is two launches:
//  (1) DENSE tasks: block b, 32 of its rows (one per lane), all its columns.  The block rows of
//      the block's columns are staged in shared memory once per task, the values stream as
//      [column][lane] (8 bytes per entry, no index).  A task leaves one partial sum per row in
//      the slot array P (slot_base + lane); slots 0..31 stay zero.
//  (2) SLICE tasks over every row: the entries no block covers, grouped by VALUE —
//      UNIFORM-VALUE positions (>= kHyMinLanes lanes of the slice hold an entry with the same
//      number, e.g. a stencil weight: one double for the position, one int32 column per lane,
//      4 bytes per entry), GENERAL positions (per-lane value and column) and PARTIAL positions
//      (per-lane slot of P, value 1).  The diagonal is an own-row operand of the epilogue.
//      Lanes without an entry at a position point at the zero row nl of the gather source.
// Columns of uniform-value positions are stored [position / 4][lane][4] (one 16-byte load per
// lane for 4 positions; nuv is padded to a multiple of 4), all others [position][lane].
constexpr int kHyMinLanes = 8;
struct PlanHySlice {   // 32 bytes
  int64_t col_off;     // first position of the slice in hy_cols (units of 32 ints)
  int32_t uv_off;      // into hy_uvval (even)
  int32_t g_off;       // into hy_gval, units of 32 doubles
  int32_t nuv, ng, np;
  int32_t pad;
};
struct PlanHyTask {    // 32 bytes
  int64_t val_off;     // into hy_dval, units of 32 doubles (one column of the task)
  int32_t col_off;     // into hy_dcols
  int32_t ncols;
  int32_t slot_base;   // the task's 32 partial slots
  int32_t nrows;
  int32_t pad[2];
};

struct HostPlan {
  // partition
  int rank = 0, nranks = 1;
  int64_t n_global = 0, row_begin = 0, row_end = 0, nl = 0, nnz = 0;
  std::vector<int64_t> starts;  // nranks + 1 row offsets
  // SELL-32-sigma of the local rows (columns: permuted local id, or nl + halo slot)
  int sigma = 1;
  int64_t nslices = 0, stored = 0;
  std::vector<int32_t> perm, iperm;      // new -> old, old -> new (local rows)
  std::vector<int64_t> slice_ptr;
  std::vector<int32_t> slice_len, row_len;
  BigVec<int32_t> col;
  BigVec<double> val;
  std::vector<int32_t> interior, boundary;  // slice ids
  std::vector<PlanTask> tasks_all, tasks_interior, tasks_boundary;
  bool short_rows = false;
  bool lean = false;   // short_rows and every main slice has <= 8 uniform positions
  // lean matrices: the (value, mask) pairs of every main slice again, at a fixed stride of 16
  // doubles per slice, so that the stencil kernel can fetch them without waiting for the
  // slice descriptor (one dependent memory round trip less per slice)
  std::vector<double> uv_pairs;
  PlanStencilTiles tiles;   // stencil tile plan (nseg == 0: none); uv_pairs is padded to whole tiles
  // index-compressed copy of the same slices (same rows, same permutation)
  std::vector<PlanUgSlice> ug_slice;
  std::vector<double> ug_val;
  std::vector<int32_t> ug_col, ug_uoff;
  int64_t ug_uniform_entries = 0;   // true nonzeros stored at uniform positions
  bool ug_skipped = false;          // paired layout certain: UG arrays not built (ensure_ug)
  // SPLIT mode (automatic sigma only; chosen when at least half of the nonzeros sit at
  // uniform offsets in natural row order — measured on B200, the PARSEC-shaped matrices with
  // 42 % uniform entries are still faster unsplit: 35 us vs 43 us per step): rows keep their natural order, main slices hold
  // the uniform part (plus small balanced leftovers), ragged leftovers ("spilled" entries,
  // e.g. dense non-local blocks) live in REST slices: general-position slices over the rows
  // that have leftovers, regrouped by length.  Rest slices are appended to ug_slice after
  // the nslices main ones; rest_rows maps their lanes to rows (-1: unused lane).  A main
  // slice whose rows have rest parts has bit 0 of `reserved` set: it adds the partial sums
  // the rest kernel left in the W workspace.
  bool split = false;
  int64_t nrest = 0;
  std::vector<int32_t> rest_rows;                    // [nrest * 32]
  std::vector<int32_t> rest_interior, rest_boundary; // slice ids (>= nslices)
  std::vector<PlanTask> tasks_rest_all, tasks_rest_interior, tasks_rest_boundary;
  // PAIRED layout ("P2") for matrices with long ragged rows (not SPLIT, not lean): slices of up
  // to 64 consecutive rows, lane l owns the ADJACENT rows row0 + 2 l and + 1, and a GENERAL
  // position holds one column and TWO values (one per row, zero where a row lacks the entry).
  // The columns of a lane are the sorted union of its two rows' columns: neighbouring rows
  // share many of them, so one 32-byte gather serves two matrix entries.
  //
  // DENSE sections.  Long rows of PARSEC-like Hamiltonians come from dense blocks (a ball of
  // grid points coupled all-to-all by a non-local projector).  extract_dense_blocks() finds
  // those near-cliques in the CSR structure; the rows that belong to exactly ONE block are
  // ordered block by block, a slice never straddles two blocks, and the slice stores the
  // block's columns ONCE (p2_dcol, shared by all lanes) with a value pair per lane and column
  // (p2_dval, zero where the entry is absent).  The kernel stages the gathered rows of 32
  // dense columns in shared memory and broadcasts them: a dense position costs the LSU ~10
  // wavefronts instead of ~30 for a general one and 8 bytes per entry instead of 10-20.
  // Rows in no block follow in (length-sorted) natural order; rows in several blocks keep all
  // their entries as general positions.  p2_desc[s] describes slice s; p2_ptr[s] repeats gpos.
  bool p2 = false;
  int64_t p2_slices = 0;
  std::vector<PlanP2Slice> p2_desc;             // [p2_slices]
  std::vector<int64_t> p2_ptr;                  // [p2_slices + 1] first general position
  std::vector<int32_t> p2_col;                  // [general positions * 32]
  std::vector<double> p2_val;                   // [general positions * 64]
  std::vector<int32_t> p2_dcol;                 // [dense positions]
  std::vector<double> p2_dval;                  // [dense positions * 64]
  std::vector<int32_t> p2_interior, p2_boundary;
  std::vector<PlanTask> p2_tasks_all, p2_tasks_interior, p2_tasks_boundary;
  int64_t p2_entries = 0;                       // general positions * 32 (gathers per product)
  int64_t p2_blocks = 0;                        // dense blocks found
  int64_t p2_dense_entries = 0;                 // true nonzeros stored in dense sections
  // HYBRID layout (see PlanHySlice); when set the device order is the natural one (perm =
  // identity) and the CSR-order SELL arrays of the exact-mode kernel group the rows by length
  // through sell_rows (SELL lane -> row, -1 = none) instead of a permutation of the vectors.
  bool hy = false;
  std::vector<PlanHySlice> hy_slice;            // [nslices]
  BigVec<int32_t> hy_cols;
  std::vector<double> hy_uvval, hy_gval, hy_diag;
  std::vector<PlanHyTask> hy_dtasks;
  std::vector<int32_t> hy_dcols;
  BigVec<double> hy_dval;
  int64_t hy_nslots = 0;                        // partial slots (multiple of 32, >= 32)
  int32_t hy_maxcols = 0;                       // widest dense block
  int64_t hy_blocks = 0, hy_dense_entries = 0, hy_uv_entries = 0, hy_g_entries = 0;
  std::vector<int32_t> sell_rows;               // [nslices * 32] when hy, else empty
  // halo: sorted unique remote global columns; slot h lives at row nl + h of a gather source
  std::vector<int64_t> halo;
  std::vector<int64_t> need_off, need_cnt;  // per owner rank: run of `halo` it must send us
  // filled by set_give(): rows (permuted local ids) to pack for each peer
  std::vector<int64_t> give_off, give_cnt;
  std::vector<int32_t> send_rows;
};

// row_ptr holds absolute offsets into col_idx/values for local rows [row_begin,row_end);
// col_idx are GLOBAL column ids.  sigma <= 0 selects the sorting window automatically.
// Throws std::invalid_argument on malformed input.
// allow_hybrid = false: no hybrid layout (a row-partitioned upload rebuilds with it when not
// every rank found dense blocks: all ranks must exchange halo rows in the same block layout).
HostPlan build_plan(int64_t n_global, int rank, int nranks, const std::vector<int64_t>& starts,
                    const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                    int sigma, bool allow_hybrid = true);

// Peer `p` asks for `count` of our rows (global ids); call once per peer, any order.
void plan_set_give(HostPlan& plan, int peer, int64_t count, const int64_t* global_rows);
// builds the UG layout of a plan that skipped it (HostPlan::ug_skipped); no-op otherwise
void ensure_ug(HostPlan& plan);

}  // namespace flz
