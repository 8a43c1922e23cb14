// flz_internal.hpp — shared declarations of the device layer behind include/flz.h.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "flz.h"
#include "host/plan.hpp"   // BigVec

namespace flz {

// ---------------------------------------------------------------- errors
struct ApiError : std::runtime_error {
  int code;
  ApiError(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

void set_last_error(const std::string& msg);

#define FLZ_CUDA(expr)                                                                  \
  do {                                                                                  \
    cudaError_t err__ = (expr);                                                         \
    if (err__ != cudaSuccess)                                                           \
      throw ::flz::ApiError(FLZ_ECUDA, std::string(#expr) + ": " +                      \
                                           cudaGetErrorString(err__));                  \
  } while (0)

#define FLZ_NCCL(expr)                                                                  \
  do {                                                                                  \
    ncclResult_t err__ = (expr);                                                        \
    if (err__ != ncclSuccess)                                                           \
      throw ::flz::ApiError(FLZ_ENCCL, std::string(#expr) + ": " +                      \
                                           ncclGetErrorString(err__));                  \
  } while (0)

#define FLZ_REQUIRE(cond, code, msg)                                                    \
  do {                                                                                  \
    if (!(cond)) throw ::flz::ApiError((code), (msg));                                  \
  } while (0)

// ------------------------------------------------------------ device buffer
// Caching allocator (pool.cu): device blocks of the current device and pinned host blocks
// are kept for reuse after they are freed; pool_trim() returns everything to the driver.
void* pool_alloc(size_t bytes);
void pool_free(void* p);
void pool_trim();
size_t pool_cached_bytes();
void* pinned_alloc(size_t bytes);
void pinned_free(void* p);

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) pool_free(p);
    p = nullptr;
    count = 0;
  }
  // grows (never shrinks); contents are NOT preserved
  void reserve(size_t n) {
    if (n <= count) return;
    release();
    p = static_cast<T*>(pool_alloc(n * sizeof(T)));
    count = n;
  }
  void reserve_zero(size_t n, cudaStream_t s) {
    reserve(n);
    FLZ_CUDA(cudaMemsetAsync(p, 0, count * sizeof(T), s));
  }
};

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

constexpr int kSliceRows = 32;   // SELL-C: C = one warp of rows per slice
constexpr int kMaxFuse = 4;      // block columns fused per Clenshaw-step launch
constexpr int kLdAlign = 32;     // leading dimensions are multiples of 32 doubles (256 B)

// Work item of the multi-warp Clenshaw-step kernel: one CTA of kTaskWarps warps processes
// `count` slices with `warps_per_slice` warps each (count * warps_per_slice <= kTaskWarps).
constexpr int kTaskWarps = 8;
constexpr int kUgInline = 8;     // uniform offsets repeated inside a slice descriptor
struct SliceTask {
  int32_t warps_per_slice;
  int32_t count;
  int32_t slice[kTaskWarps];
};

// Per-slice header of the index-compressed ("UG") layout of the fast kernels; mirrors
// PlanUgSlice (host/plan.hpp).  Positions [0, nu) are uniform (column = row + uoff[p]),
// positions [nu, nu + ng) are general (one column per lane).
// Tile plan of the TMA-staged stencil kernel (mirrors PlanStencilTiles, host/plan.hpp)
struct StencilTiles {
  int32_t tile_rows = 0, nseg = 0;
  int32_t seg_base[8] = {}, seg_len[8] = {}, seg_start[8] = {};
  int32_t y1_elems = 0, own_e = 0;
  int32_t front = 0, back = 0;     // row slabs: halo rows in front of / behind the local rows
  int32_t tile_a = 0, tile_b = 0;  // tiles [tile_a, tile_b) stage local rows only
};

// Slice descriptor of the paired layout (mirrors PlanP2Slice, host/plan.hpp)
struct P2Slice {
  int64_t gpos, dpos;
  int32_t ng, nd;
  int32_t row0, nrows;
};

// Hybrid layout (mirrors PlanHySlice / PlanHyTask, host/plan.hpp)
struct HySlice {
  int64_t col_off;
  int32_t uv_off, g_off;
  int32_t nuv, ng, np;
  int32_t pad;
};
struct HyTask {
  int64_t val_off;
  int32_t col_off, ncols;
  int32_t slot_base, nrows;
  int32_t pad[2];
};

struct UgSlice {
  int64_t val_ptr;
  int64_t col_ptr;
  int32_t uoff_ptr;
  int32_t nu, ng;
  int32_t reserved;
  int32_t inline_off[8];  // the first offsets again: one 64-byte load serves short slices
};

}  // namespace flz

// ---------------------------------------------------------------- transport (comm.cu)
namespace flz {
struct LoopHub;   // loopback transport: ranks are threads of one process on one GPU (tests)
struct CommOp {
  bool send;
  void* buf;
  size_t bytes;
  int peer;
  cudaStream_t stream;
};
}  // namespace flz

// ---------------------------------------------------------------- context
struct flz_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_halo_ready = nullptr;   // send buffer packed (compute -> comm)
  cudaEvent_t ev_halo_done = nullptr;    // halo received (comm -> compute)
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  flz::LoopHub* hub = nullptr;            // != nullptr: loopback transport instead of NCCL
  std::vector<flz::CommOp> comm_ops;      // loopback: operations of the open group
  bool comm_grouped = false;
  bool exact = false;
  int sm_count = 148;
  int refs = 1;                  // owner + every matrix/basis created on the context
  uint64_t launches = 0;
  int k1_slices_per_cta = 0, k1_tasks_per_cta = 0, k1_batch = 0;  // 0: defaults (tuning knobs)
  bool k1_packed = false;     // the last tile-kernel launch packed halo rows into send_buf
  bool k1_pdl_once = false;   // the next K1 launch carries the dependent-launch attribute (row slabs)
  cudaEvent_t t0[16] = {}, t1[16] = {};
  flz::DevBuf<double> partial;   // split-K partial sums of the tall-skinny GEMMs
  flz::DevBuf<double> small;     // small device scratch of the host-buffer test seams
  flz::DevBuf<double> stage;     // host<->device staging of blocks
  flz::DevBuf<double> stage2;
  flz::DevBuf<char> flush;       // L2 flush target
  // staged downloads into pageable host memory (capi.cu download_block): two page-locked
  // buffers filled by the copy engine and emptied by host threads
  void* dl_pinned[2] = {nullptr, nullptr};
  cudaEvent_t dl_event[2] = {nullptr, nullptr};
  flz::DevBuf<double> qr_scratch;              // block_qr_kernel: per-phase, per-CTA partial sums
  flz::DevBuf<unsigned long long> qr_barrier;  // its grid-barrier counter (monotone)
  unsigned long long qr_arrivals = 0;          // arrivals issued so far
};

// ----------------------------------------------------------------- matrix
// SELL-32-sigma, rows permuted by `perm` (new -> old local row).  The whole device
// side works in the permuted ordering; only host transfers apply perm.
struct flz_matrix {
  flz_ctx* ctx = nullptr;
  int refs = 1;           // owner + every basis built on the matrix
  int64_t n_global = 0;
  int64_t row_begin = 0, row_end = 0;
  int64_t nl = 0;         // local rows
  int64_t ld = 0;         // padded local rows (multiple of kLdAlign)
  int64_t nnz = 0;        // true local nonzeros
  bool dense_rows = false; // >= 16 nonzeros per row over the whole matrix (interleaved stride 4)
  int64_t stored = 0;     // stored entries incl. padding
  int64_t nslices = 0;
  int64_t nhalo = 0;      // halo rows appended after the nl local rows of a gather source
  int sigma = 1;
  // device arrays
  flz::DevBuf<int64_t> slice_ptr;   // [nslices+1] element offsets
  flz::DevBuf<int32_t> slice_len;   // [nslices]
  flz::DevBuf<int32_t> row_len;     // [nslices*32]
  // CSR-order SELL arrays: read only by the exact-mode kernel, uploaded on its first use
  // from the host copies below
  mutable flz::DevBuf<int32_t> col; // [stored] permuted local col or nl + halo slot
  mutable flz::DevBuf<double> val;  // [stored]
  mutable flz::BigVec<int32_t> h_col;
  mutable flz::BigVec<double> h_val;
  // index-compressed layout read by the fast kernels
  flz::DevBuf<flz::UgSlice> ug;     // [nslices]
  flz::DevBuf<double> ug_val;
  flz::DevBuf<int32_t> ug_col, ug_uoff;
  flz::DevBuf<double> uv_pairs;     // lean matrices: 16 doubles per slice (host/plan.hpp)
  flz::StencilTiles tiles;          // nseg > 0: the TMA-staged stencil kernel applies
  // paired layout (host/plan.hpp)
  bool p2 = false;
  flz::DevBuf<flz::P2Slice> p2_desc;
  flz::DevBuf<int32_t> p2_col, p2_dcol;
  flz::DevBuf<double> p2_val, p2_dval;
  int64_t p2_blocks = 0, p2_dense_entries = 0;
  // hybrid layout (host/plan.hpp): natural row order, dense tasks + value-grouped slices
  bool hy = false;
  flz::DevBuf<flz::HySlice> hy_slice;
  flz::DevBuf<flz::HyTask> hy_dtasks;
  flz::DevBuf<int32_t> hy_cols, hy_dcols;
  flz::DevBuf<double> hy_uvval, hy_gval, hy_diag, hy_dval;
  mutable flz::DevBuf<double> hy_p;      // partial sums of the dense tasks, planar [k][hy_ldp]
  mutable flz::DevBuf<double> hy_w;      // overlapped variant: slice sums, planar like y1
  int64_t hy_ndtasks = 0, hy_ldp = 0, hy_blocks = 0, hy_dense_entries = 0, hy_uv_entries = 0;
  int hy_maxcols = 0;
  int64_t hy_bytes = 0;
  flz::DevBuf<int32_t> sell_rows;        // exact-mode SELL lane -> row (hybrid only)
  // task counters of the persistent paired kernel: one per launch, zeroed kTicketSlots at a time
  mutable flz::DevBuf<unsigned> k1_tickets;
  mutable int ticket_cursor = 0;
  flz::DevBuf<flz::SliceTask> p2_tasks_all, p2_tasks_interior, p2_tasks_boundary;
  int64_t p2_nt_all = 0, p2_nt_interior = 0, p2_nt_boundary = 0;
  int64_t p2_bytes = 0;
  int64_t ug_bytes = 0;             // matrix bytes one fast step streams
  int64_t ug_uniform_entries = 0;
  // SPLIT mode (host/plan.hpp): rest slices follow the main ones in `ug`
  bool split = false;
  int64_t nrest = 0;
  flz::DevBuf<int32_t> rest_rows;   // [nrest*32] row of every rest lane, -1 = unused
  flz::DevBuf<flz::SliceTask> tasks_rest_all, tasks_rest_interior, tasks_rest_boundary;
  int64_t nt_rest_all = 0, nt_rest_interior = 0, nt_rest_boundary = 0;
  mutable flz::DevBuf<double> w;    // partial sums of the rest slices, (nl x kMaxFuse) rows
  flz::DevBuf<int32_t> perm;        // [nl] new -> old
  flz::DevBuf<int32_t> iperm;       // [nl] old -> new
  flz::DevBuf<int32_t> interior;    // slice ids without halo references
  flz::DevBuf<int32_t> boundary;    // slice ids with halo references
  int64_t n_interior = 0, n_boundary = 0;
  flz::DevBuf<flz::SliceTask> tasks_all, tasks_interior, tasks_boundary;
  int64_t nt_all = 0, nt_interior = 0, nt_boundary = 0;
  bool short_rows = false;          // every main slice fits one warp (single-warp tasks only)
  bool lean = false;                // ... with at most kUgInline uniform positions each
  std::vector<int32_t> h_perm, h_iperm;
  // halo exchange plan (distributed only)
  struct Peer {
    int rank;
    int64_t send_off, send_count;   // rows of send_rows (permuted local ids) to pack
    int64_t recv_off, recv_count;   // halo slots [recv_off, recv_off+recv_count)
  };
  std::vector<Peer> peers;
  flz::DevBuf<int32_t> send_rows;   // concatenated per-peer send lists
  int64_t n_send = 0;
  flz::DevBuf<double> send_buf;     // n_send * kMaxFuse doubles
  // tile kernel on row slabs: send slots of the rows of the halo-staging tiles (two per row,
  // -1: none; rows behind the hole [tile_a, tile_b) indexed minus the hole) — those tiles
  // write their results into send_buf as well, so the next step needs no pack launch
  flz::DevBuf<int2> send_slots;
  mutable const double* packed_from = nullptr;   // the block whose halo rows send_buf holds
  // filter workspaces (interleaved (nl+nhalo) x R), created on first use
  mutable flz::DevBuf<double> y1, y2, xs, zs;
  mutable flz::DevBuf<double> y3, y4;   // second pair of filter workspaces (multi-step launches)
  bool multistep = false;               // short-reach stencil without per-lane positions
};

// ------------------------------------------------------------------ basis
struct flz_basis {
  flz_ctx* ctx = nullptr;
  const flz_matrix* A = nullptr;
  int64_t nl = 0, ld = 0;
  int r = 0;
  int64_t max_cols = 0;
  int64_t k = 0;                       // completed blocks
  // ld x (max_cols + r) column-major; cudaMalloc is lazy about physical pages and nothing
  // is zero-filled up front (the reference zero-fills eagerly, lanczos.cpp:111); rows
  // [nl, ld) of every written column are kept zero.
  flz::DevBuf<double> Q;
  flz::DevBuf<double> Z;               // ld x r operator output / remainder
  flz::DevBuf<double> X;               // ld x r staged newest block
  flz::DevBuf<double> small;           // coefficient blocks C1/C2, S_k, scalars, op_scale
  double* pinned = nullptr;            // pinned host mirror of `small`
  size_t pinned_count = 0;
  // recovery storage
  flz::DevBuf<double> V, AV, V2, AV2;
  int w_kept = 0;
  double op_scale = 0.0;
  double mv_s = 0.0, orth_s = 0.0;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
  // Speculative operator application (one rank, fused orthogonalization): the step that has
  // just queued its small D2H copies also queues op(pending block) for the NEXT step, so the
  // device works while the host waits for and digests the step's results.  The next
  // flz_lanczos_step consumes it when its arguments match and nothing touched the basis in
  // between (basis_set / truncate / orthogonalize_column drop it and take its matvecs back).
  cudaEvent_t s0[2] = {nullptr, nullptr}, s1[2] = {nullptr, nullptr};   // around the speculative
  int spec_slot = 0;                        // application (two pairs: one read, one recorded)
  cudaEvent_t e1b = nullptr, e_done = nullptr;
  bool spec_valid = false;
  std::vector<double> spec_coeffs;          // the coefficients it was queued with (by value)
  int spec_m = 0;
  double spec_c = 0.0, spec_e = 0.0;
  uint64_t spec_matvecs = 0;
  float last_mv_ms = 0.f;
  double* col(int64_t j) const { return Q.p + j * ld; }
};

namespace flz {

// --------------------------------------------------------------- transport
// (comm.cu) NCCL, or the loopback hub when ctx->hub is set.  Sizes in bytes; a send/recv pair
// outside a group is a group of one.
LoopHub* loop_hub_create(int nranks);
void loop_hub_destroy(LoopHub* hub);
void comm_group_start(flz_ctx* ctx);
void comm_group_end(flz_ctx* ctx);
void comm_send(flz_ctx* ctx, const void* buf, size_t bytes, int peer, cudaStream_t stream);
void comm_recv(flz_ctx* ctx, void* buf, size_t bytes, int peer, cudaStream_t stream);
void comm_allreduce_sum(flz_ctx* ctx, double* buf, size_t count, cudaStream_t stream);
void comm_allgather_i64(flz_ctx* ctx, const int64_t* d_in, int64_t* d_out, cudaStream_t stream);

// --------------------------------------------------------- kernel launchers
// (kernels_sell.cu)
struct SellView {
  const SliceTask* tasks;    // task list of the fast kernel (nullptr: one warp per slice)
  int64_t ntasks;
  bool short_rows;           // every slice fits one warp: the one-warp-per-slice kernel is best
  bool lean;                 // ... and has <= kUgInline uniform positions (stencils)
  bool mostly_uniform;       // SPLIT mode: the main slices are (almost) only uniform positions
  const int64_t* slice_ptr;
  const int32_t* slice_len;
  const int32_t* row_len;
  const int32_t* col;
  const double* val;
  const int32_t* slice_ids;  // nullptr: all slices [0, nslices)
  int64_t nslices;           // number of slices this launch covers
  int64_t nl;
  // index-compressed layout (fast kernels)
  const UgSlice* ug;
  const double* ug_val;
  const int32_t* ug_col;
  const int32_t* ug_uoff;
  int64_t ncols;             // rows of a gather source: local rows + halo rows
  // SPLIT mode: rest launches map lanes to rows through rest_rows (slice ids start at
  // rest_base) and leave their sums in W; main launches add W where a slice is flagged
  const int32_t* rest_rows;
  int64_t rest_base;
  double* W;
  const double* uv_pairs;    // lean matrices: (value, mask) pairs, 16 doubles per slice
  // paired layout (host/plan.hpp): 64-row slices, two adjacent rows per lane; `tasks` then
  // lists paired slices
  bool p2;
  const P2Slice* p2_desc;
  const int32_t* p2_col;
  const double* p2_val;
  const int32_t* p2_dcol;    // dense sections: shared columns, one value pair per lane
  const double* p2_dval;
  unsigned* tickets;         // this launch's task counter (starts at 0; persistent CTAs)
  StencilTiles tiles;        // nseg > 0: tile plan of the TMA-staged stencil kernel
  const int32_t* sell_rows;  // exact-mode kernel: SELL lane -> row (nullptr: slice * 32 + lane)
  const int2* send_slots = nullptr;   // tile kernel, phase 2 of a Clenshaw step: fused halo pack
  double* send_buf = nullptr;
  int64_t n_send = 0;
  int64_t tile_slices = 0;   // the tile plan covers slices [0, tile_slices) of the matrix
  int tile_phase = 0;        // 0: all tiles, 1: tiles without halo rows, 2: the rest (row slabs)
};

// Hybrid layout (host/plan.hpp) as the kernels see it
struct HyView {
  int64_t nl, nslices;
  int ndtasks, maxcols;
  const HySlice* slice;
  const int32_t* cols;
  const double* uvval;
  const double* gval;
  const double* diag;
  const HyTask* dtasks;
  const int32_t* dcols;
  const double* dval;
  double* P;                 // partial slots, planar [k][ldp]
  int64_t ldp;
  double* W;                 // overlapped variant: the slices' sums before the finish launch
  int zero_row;              // row of the gather source that is always zero (nl + halo rows)
};

enum class StepMode { step, final, plain, rest };

// One fused Clenshaw step (or plain SpMM) for R in [1, kMaxFuse] block columns.  Layout of
// the blocks Y1/Y2: S > 0 interleaved with row stride S (S == R, or S == 4 for R == 3 on
// long-row matrices); S == 0 planar, column k at Y + k*ldy (best when the matrix is mostly
// uniform-offset positions: every gather is then a contiguous 256-byte warp load):
//   step : Y2[i,:] = s1*(A Y1)[i,:] + s2*Y1[i,:] - Y2[i,:] + b*X[i,:]   (interleaved out)
//   final: Out[:,k] column-major (ld = ldo) receives the same expression
//   plain: Out[:,k] = (A Y1)[i,k]
void launch_clenshaw_step(flz_ctx* ctx, const SellView& A, int R, int S, StepMode mode, bool exact,
                          double s1, double s2, double b, const double* Y1, double* Y2,
                          int64_t ldy, const double* X, int64_t ldx, double* Out, int64_t ldo);
// The same step on a matrix with the hybrid layout: PLANAR blocks (column k of Y1/Y2 at
// k * ldy, row nl of Y1 must be zero), two launches (dense tasks, then the slices).
// true: the overlapped variant runs (hybrid_gather + hybrid_finish), else hybrid_dense_tasks +
// hybrid_slices
bool hybrid_overlaps(const flz_ctx* ctx, int64_t nslices, int64_t ndtasks);
// phase 0: the whole step; 1: the dense tasks only (they gather LOCAL rows: a partitioned run
// launches them while the halo rows travel); 2: the slices only
void launch_hybrid_step(flz_ctx* ctx, const HyView& A, int R, StepMode mode, double s1, double s2,
                        double b, const double* Y1, double* Y2, int64_t ldy, const double* X,
                        int64_t ldx, double* Out, int64_t ldo, int phase = 0);
// Y1 = scale * X  (column-major -> interleaved with row stride S >= R, or planar for S == 0)
// several Clenshaw steps of a short-reach stencil in one launch (0: not applicable)
int launch_multistep(flz_ctx* ctx, const SellView& A, int R, int max_steps, const double* b,
                     double s1, double s2, const double* Y1, const double* Y2, int64_t ldy,
                     const double* X, int64_t ldx, double* O1, double* O2);
void launch_interleave(flz_ctx* ctx, int64_t nl, int R, int S, double scale, const double* X,
                       int64_t ldx, double* Y1, int64_t ldy);
// halo packing: buf[s*S+k] = Y1[rows[s]*S+k]; planar (S == 0): buf[k*count+s] = Y1[k*ldy+rows[s]]
void launch_pack_rows(flz_ctx* ctx, cudaStream_t stream, int64_t count, int R, int S, int64_t ldy,
                      const int32_t* rows, const double* Y1, double* buf);
// out[i] = s1*w[i] + s2*y1[i] - y2[i] + b*x[i]
void launch_combine(flz_ctx* ctx, int64_t n, bool exact, double s1, double s2, double b,
                    const double* w, const double* y1, const double* y2, const double* x,
                    double* out);

// (kernels_dense.cu)
// C[M x N] (row-major, row stride ldc) = A[:, 0..M)^T B[:, 0..N) over `rows` rows, A and B
// column-major with leading dimensions lda/ldb (multiples of 8, zero padded past `rows`).
// FP64 DMMA, deterministic split-K (partials in ctx->partial, fixed-order reduction).
void launch_gemm_tn(flz_ctx* ctx, const double* A, int64_t lda, int64_t M, const double* B,
                    int64_t ldb, int N, int64_t rows, double* C, int64_t ldc);
// Out[:, 0..N) (column-major, ldo) = alpha * A[:, 0..K) * Bs (+ Out when accumulate);
// Bs row-major [K][ldbs] with ldbs a multiple of 8 and zero padded columns.
void launch_gemm_nn(flz_ctx* ctx, const double* A, int64_t lda, int64_t K, const double* Bs,
                    int64_t ldbs, int N, int64_t rows, double alpha, bool accumulate, double* Out,
                    int64_t ldo);
// out[c] = sum_i A[i,c]*B[i,c], c < N (column-major, lda/ldb)
void launch_coldot(flz_ctx* ctx, const double* A, int64_t lda, const double* B, int64_t ldb, int N,
                   int64_t rows, double* out);
// dest[i] = src[i] * (*inv) for i < rows  (inv read from device memory)
void launch_scale_copy(flz_ctx* ctx, const double* src, const double* inv, double* dest,
                       int64_t rows);
// per column c: A[:,c] *= s[c]
void launch_scale_cols(flz_ctx* ctx, double* A, int64_t lda, int N, int64_t rows, const double* s);
// residual kernel: v = V[:,c]*inv[c]; av = AV[:,c]*inv[c] - lambda[c]*v; V[:,c] = v;
// AV[:,c] = av   (norms via coldot afterwards)
void launch_residual_prep(flz_ctx* ctx, double* V, double* AV, int64_t ld, int N, int64_t rows,
                          const double* inv, const double* lambda);
// gather/scatter rows by permutation between a host-ordered block and a device-ordered one
// dst[perm-ordered] : dst[c*ldd + inew] = src[c*lds + perm[inew]]
void launch_permute_in(flz_ctx* ctx, const double* src, int64_t lds, double* dst, int64_t ldd,
                       int N, int64_t rows, const int32_t* perm);
void launch_permute_out(flz_ctx* ctx, const double* src, int64_t lds, double* dst, int64_t ldd,
                        int N, int64_t rows, const int32_t* perm);
// block-step scalar logic (single thread kernels)
void launch_block_qr(flz_ctx* ctx, double* Z, int64_t ld, int64_t rows, int r,
                     const double* normsq0, int64_t stride, double* scale, double* Sk,
                     double* dead);
void launch_update_scale(flz_ctx* ctx, const double* gram, int r, int ldg, double* op_scale);
void launch_finish_col(flz_ctx* ctx, const double* normsq, const double* op_scale, double* Sk,
                       int r, int j, double* inv, double* dead_flag);

}  // namespace flz
