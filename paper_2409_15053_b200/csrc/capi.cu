// capi.cu — the device layer of the C ABI declared in include/flz.h.
//
// Everything here runs on the GPU; there is no CPU fallback (flz_ctx_create fails with
// FLZ_ENODEV when no sm_100 device is present).  Host code in this file only builds
// data structures (SELL-C-sigma conversion, halo plan) and sequences kernel launches.

#include <algorithm>
#include <thread>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>

#include "flz_internal.hpp"
#include "host/plan.hpp"
#include "host/spin_barrier.hpp"

using namespace flz;

namespace flz {
namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_matvecs{0};
}  // namespace
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace flz

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return FLZ_OK;
  } catch (const ApiError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return FLZ_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FLZ_EINVAL;
  }
}

// FLZ_TRACE=1: per-phase device timings on stderr (synchronises the stream; diagnostics only)
struct Trace {
  flz_ctx* ctx;
  const char* what;
  std::chrono::steady_clock::time_point t0;
  static bool on() {
    static const bool v = std::getenv("FLZ_TRACE") != nullptr;
    return v;
  }
  Trace(flz_ctx* c, const char* w) : ctx(c), what(w) {
    if (on()) {
      cudaStreamSynchronize(ctx->stream);
      t0 = std::chrono::steady_clock::now();
    }
  }
  ~Trace() {
    if (on()) {
      cudaStreamSynchronize(ctx->stream);
      const double ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      std::fprintf(stderr, "[flz]   dev %-24s %9.3f ms\n", what, ms);
    }
  }
};

void use(const flz_ctx* ctx) { FLZ_CUDA(cudaSetDevice(ctx->device)); }

struct Pinned {  // small RAII pinned host array
  double* p = nullptr;
  explicit Pinned(size_t count) { p = static_cast<double*>(pinned_alloc(count * sizeof(double))); }
  ~Pinned() { pinned_free(p); }
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
};

// FLZ_ORTH_FUSED=0: the multi-launch orthogonalization of the row-partitioned path on one
// rank too (experiments, A/B tests)
bool fused_orth_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FLZ_ORTH_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}

void allreduce(flz_ctx* ctx, double* buf, size_t count) {
  if (ctx->nranks == 1 || count == 0) return;
  comm_allreduce_sum(ctx, buf, count, ctx->stream);
}

// The CSR-order SELL arrays serve the exact-mode kernel only: they stay on the host until
// the first exact-mode product on this matrix.
void ensure_exact_arrays(const flz_matrix* A) {
  flz_ctx* ctx = A->ctx;
  if (!ctx->exact || A->col.p) return;
  A->col.reserve(std::max<size_t>(A->h_col.size(), 1));
  A->val.reserve(std::max<size_t>(A->h_val.size(), 1));
  if (!A->h_col.empty()) {
    FLZ_CUDA(cudaMemcpyAsync(A->col.p, A->h_col.data(), A->h_col.size() * sizeof(int32_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    FLZ_CUDA(cudaMemcpyAsync(A->val.p, A->h_val.data(), A->h_val.size() * sizeof(double),
                             cudaMemcpyHostToDevice, ctx->stream));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  flz::BigVec<int32_t>().swap(A->h_col);
  flz::BigVec<double>().swap(A->h_val);
}

SellView make_view(const flz_matrix* A, const SliceTask* tasks, int64_t ntasks,
                   const int32_t* slice_ids, int64_t nslices) {
  ensure_exact_arrays(A);
  return SellView{tasks,        ntasks,     A->short_rows, A->lean, A->split, A->slice_ptr.p, A->slice_len.p,
                  A->row_len.p, A->col.p,   A->val.p,      slice_ids,      nslices,
                  A->nl,        A->ug.p,    A->ug_val.p,   A->ug_col.p,    A->ug_uoff.p,
                  A->nl + A->nhalo, A->rest_rows.p, A->nslices,   A->w.p,
                  A->uv_pairs.p,    false,          A->p2_desc.p, A->p2_col.p, A->p2_val.p,
                  A->p2_dcol.p,     A->p2_dval.p,   nullptr,
                  // the tile kernel covers whole-matrix launches (and, on row slabs, its own
                  // split into tiles without and with halo rows: tiled(), below)
                  (slice_ids == nullptr && nslices == A->nslices) ? A->tiles : StencilTiles{},
                  A->hy ? A->sell_rows.p : nullptr, nullptr, nullptr, 0, A->nslices, 0};
}
// Row slabs with a tile plan: the interior / boundary launch as a phase of the tile kernel
// (the slice lists stay in place for the one-warp-per-slice kernel it falls back to).
SellView tiled(const flz_matrix* A, SellView v, int phase) {
  if (A->tiles.nseg > 0 && !A->ctx->exact) {
    v.tiles = A->tiles;
    v.tile_phase = phase;
    if (phase == 2 && A->send_slots.count > 0) {
      v.send_slots = A->send_slots.p;
      v.send_buf = A->send_buf.p;
      v.n_send = A->n_send;
    }
  }
  return v;
}
// fast mode on a matrix with the paired layout: the launch walks the paired task lists
SellView paired(const flz_matrix* A, SellView v, int which) {
  if (!A->p2 || A->ctx->exact) return v;
  v.p2 = true;
  // a fresh (zero) task counter per launch; the block of counters is cleared when it runs out
  constexpr int kTicketSlots = 4096;
  if (A->k1_tickets.count == 0 || A->ticket_cursor == kTicketSlots) {
    A->k1_tickets.reserve_zero(kTicketSlots, A->ctx->stream);
    A->ticket_cursor = 0;
  }
  v.tickets = A->k1_tickets.p + A->ticket_cursor++;
  v.tasks = which == 0 ? A->p2_tasks_all.p : (which == 1 ? A->p2_tasks_interior.p : A->p2_tasks_boundary.p);
  v.ntasks = which == 0 ? A->p2_nt_all : (which == 1 ? A->p2_nt_interior : A->p2_nt_boundary);
  return v;
}
// rest launches (SPLIT mode): task lists over the rest slices
SellView view_rest(const flz_matrix* A, int which) {
  const DevBuf<SliceTask>& t =
      which == 0 ? A->tasks_rest_all : (which == 1 ? A->tasks_rest_interior : A->tasks_rest_boundary);
  const int64_t nt =
      which == 0 ? A->nt_rest_all : (which == 1 ? A->nt_rest_interior : A->nt_rest_boundary);
  return make_view(A, t.p, nt, nullptr, A->nrest);
}
SellView paired(const flz_matrix* A, SellView v, int which);
SellView view_all(const flz_matrix* A) {
  return paired(A, make_view(A, A->tasks_all.p, A->nt_all, nullptr, A->nslices), 0);
}
SellView view_interior(const flz_matrix* A) {
  return paired(A, make_view(A, A->tasks_interior.p, A->nt_interior, A->interior.p, A->n_interior), 1);
}
SellView view_boundary(const flz_matrix* A) {
  return paired(A, make_view(A, A->tasks_boundary.p, A->nt_boundary, A->boundary.p, A->n_boundary), 2);
}

// leading dimension of the planar filter workspaces (local rows + halo rows, padded); the
// hybrid layout needs row nl as a zero row (the target of lanes without an entry)
int64_t planar_ld(const flz_matrix* A) {
  return round_up(A->nl + A->nhalo + (A->hy ? 1 : 0), kLdAlign);
}

HyView hybrid_view(const flz_matrix* A) {
  if (A->hy_p.count == 0) A->hy_p.reserve_zero((size_t)A->hy_ldp * kMaxFuse + 8, A->ctx->stream);
  if (A->hy_w.count == 0) A->hy_w.reserve_zero((size_t)planar_ld(A) * kMaxFuse + 8, A->ctx->stream);
  return HyView{A->nl,         A->nslices,    (int)A->hy_ndtasks, A->hy_maxcols, A->hy_slice.p,
                A->hy_cols.p,  A->hy_uvval.p, A->hy_gval.p,       A->hy_diag.p,  A->hy_dtasks.p,
                A->hy_dcols.p, A->hy_dval.p,  A->hy_p.p,          A->hy_ldp,     A->hy_w.p,
                (int)(A->nl + A->nhalo)};
}

void ensure_workspaces(const flz_matrix* A) {
  flz_ctx* ctx = A->ctx;
  const size_t need = (size_t)planar_ld(A) * kMaxFuse + 8;
  if (A->y1.count < need) {
    A->y1.reserve_zero(need, ctx->stream);
    A->y2.reserve_zero(need, ctx->stream);
  }
  // rows without a rest part keep W = 0 for ever; rest rows are overwritten every product
  if (A->nrest > 0 && A->w.count == 0)
    A->w.reserve_zero((size_t)A->nl * kMaxFuse + 8, ctx->stream);
}

// Halo exchange of the gather source Y1: pack the rows the peers reference, send/recv on the
// comm stream, leave ev_halo_done for the boundary launch.  The caller launches the interior
// slices in between.  Interleaved blocks (S > 0) travel as whole padded rows; planar blocks
// (S == 0) as R contiguous runs per peer, received straight into the tail of each column.
void halo_begin(const flz_matrix* A, int R, int S, double* Y1) {
  flz_ctx* ctx = A->ctx;
  const int64_t ldy = planar_ld(A);
  // (the tile kernel's last phase-2 launch may have left Y1's halo rows in send_buf already)
  if (A->packed_from != Y1)
    launch_pack_rows(ctx, ctx->stream, A->n_send, R, S, ldy, A->send_rows.p, Y1, A->send_buf.p);
  A->packed_from = nullptr;
  FLZ_CUDA(cudaEventRecord(ctx->ev_halo_ready, ctx->stream));
  FLZ_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_halo_ready, 0));
  constexpr size_t D = sizeof(double);
  // FLZ_HALO_DRY=1 (timing experiments on one GPU through the loopback transport, WRONG
  // results): pack, events and the phase split stay, the transfers are skipped — the compute
  // side of one rank of a slab run
  static const bool dry = [] {
    const char* e = std::getenv("FLZ_HALO_DRY");
    return e && e[0] == '1';
  }();
  if (dry && ctx->hub) {   // loopback contexts only: never on a production (NCCL) context
    FLZ_CUDA(cudaEventRecord(ctx->ev_halo_done, ctx->comm_stream));
    return;
  }
  comm_group_start(ctx);
  for (const auto& p : A->peers) {
    if (S > 0) {
      if (p.send_count)
        comm_send(ctx, A->send_buf.p + p.send_off * S, (size_t)p.send_count * S * D, p.rank,
                  ctx->comm_stream);
      if (p.recv_count)
        comm_recv(ctx, Y1 + (A->nl + p.recv_off) * S, (size_t)p.recv_count * S * D, p.rank,
                  ctx->comm_stream);
    } else {
      for (int k = 0; k < R; ++k) {
        if (p.send_count)
          comm_send(ctx, A->send_buf.p + (int64_t)k * A->n_send + p.send_off,
                    (size_t)p.send_count * D, p.rank, ctx->comm_stream);
        if (p.recv_count)
          comm_recv(ctx, Y1 + (int64_t)k * ldy + A->nl + p.recv_off, (size_t)p.recv_count * D,
                    p.rank, ctx->comm_stream);
      }
    }
  }
  comm_group_end(ctx);
  FLZ_CUDA(cudaEventRecord(ctx->ev_halo_done, ctx->comm_stream));
}

// One fused step over the whole local matrix, with the halo exchange overlapped with the
// interior slices when the context is distributed.
void sell_step(const flz_matrix* A, int R, int S, StepMode mode, double s1, double s2, double b,
               double* Y1, double* Y2, const double* X, int64_t ldx, double* Out, int64_t ldo) {
  flz_ctx* ctx = A->ctx;
  const int64_t ldy = planar_ld(A);
  // SPLIT mode: the rest slices leave their partial sums in W before the main slices of the
  // same rows run (the exact-mode kernel reads the unsplit CSR-order arrays instead)
  auto rest = [&](int which, int64_t ntasks) {
    if (ctx->exact || ntasks == 0) return;
    launch_clenshaw_step(ctx, view_rest(A, which), R, S, StepMode::rest, false, 0.0, 0.0, 0.0, Y1,
                         Y2, ldy, nullptr, 0, nullptr, 0);
  };
  if (A->hy && !ctx->exact) {   // hybrid layout: planar blocks, dense tasks + slices
    if (ctx->nranks == 1 || A->peers.empty()) {
      launch_hybrid_step(ctx, hybrid_view(A), R, mode, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
    } else {
      // row-partitioned: the dense blocks lie inside the local diagonal block, so their tasks
      // run while the halo rows travel; the slices (the only readers of halo rows) follow
      halo_begin(A, R, S, Y1);
      launch_hybrid_step(ctx, hybrid_view(A), R, mode, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo, 1);
      FLZ_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo_done, 0));
      launch_hybrid_step(ctx, hybrid_view(A), R, mode, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo, 2);
    }
    return;
  }
  if (ctx->nranks == 1 || A->peers.empty()) {
    rest(0, A->nt_rest_all);
    launch_clenshaw_step(ctx, view_all(A), R, S, mode, ctx->exact, s1, s2, b, Y1, Y2, ldy, X, ldx,
                         Out, ldo);
    return;
  }
  halo_begin(A, R, S, Y1);
  rest(1, A->nt_rest_interior);
  launch_clenshaw_step(ctx, tiled(A, view_interior(A), 1), R, S, mode, ctx->exact, s1, s2, b, Y1, Y2,
                       ldy, X, ldx, Out, ldo);
  FLZ_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo_done, 0));
  rest(2, A->nt_rest_boundary);
  const SellView vb = tiled(A, view_boundary(A), 2);
  launch_clenshaw_step(ctx, vb, R, S, mode, ctx->exact, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
  // a Clenshaw step through the tile kernel packed the halo rows of its result on the way
  if (mode == StepMode::step && S == 0 && vb.send_slots && vb.tiles.nseg > 0 && ctx->k1_packed) {
    A->packed_from = Y2;
  }
  ctx->k1_packed = false;
}

// Layout of the filter workspaces for R fused columns (see launch_clenshaw_step):
// interleaved rows, 3 columns padded to 4 (one aligned 32-byte sector per gathered row) when
// the matrix is gather dominated (>= 16 entries per row); planar (0) for stencil matrices
// with 3 columns.  FLZ_K1_LAYOUT=planar|interleaved|4 forces a layout (experiments).
// The exact-mode kernel always reads interleaved rows of stride R.
int row_stride(const flz_matrix* A, int R) {
  if (A->ctx->exact || A->nl == 0) return R;
  if (A->hy) return 0;   // the hybrid kernels read planar blocks
  static const char* force = std::getenv("FLZ_K1_LAYOUT");  // experiments: planar | interleaved
  // planar blocks pay for stencil matrices with 3 columns on one GPU (100^3 Laplacian: 23.0 vs
  // 25.0 us per step: a coalesced 8-byte warp load touches 2-3 lines, a 24-byte-stride one 7);
  // with 4 columns the 32-byte rows win (37.3 vs 39.4 us)
  // ... and for every column count when the TMA-staged tile kernel applies (it reads planar
  // blocks only: contiguous runs per column)
  // (row slabs: A->tiles is set only when EVERY rank has a tile plan, flz_matrix_upload)
  const bool planar = force ? force[0] == 'p'
                            : (A->lean && (A->ctx->nranks == 1 ? (R == 3 || A->tiles.nseg > 0)
                                                               : A->tiles.nseg > 0));
  if (planar) return 0;
  if (R != 3) return R;
  if (force && force[0] == '4') return 4;  // experiments: padded rows for every matrix
  return A->dense_rows ? 4 : 3;   // (nonzeros per row of the WHOLE matrix: all ranks agree)
}

// Hybrid layout: row nl of every plane of the gather source is the zero row (the target of
// lanes without an entry).  The workspaces are shared with the interleaved layouts of the
// exact-mode kernel, so the pad rows [nl, ld) are cleared whenever a block is (re)built.
void zero_pad_rows(const flz_matrix* A, int R, int S, double* Y) {
  if (!A->hy || S != 0) return;
  const int64_t ldy = planar_ld(A);
  FLZ_CUDA(cudaMemset2DAsync(Y + A->nl, (size_t)ldy * sizeof(double), 0,
                             (size_t)(ldy - A->nl) * sizeof(double), (size_t)R, A->ctx->stream));
}

// Z[:, 0..ncols) = A X[:, 0..ncols), device-resident column-major blocks (permuted rows).
void spmm_device(const flz_matrix* A, const double* X, int64_t ldx, int ncols, double* Z,
                 int64_t ldz, bool counted) {
  flz_ctx* ctx = A->ctx;
  ensure_workspaces(A);
  A->packed_from = nullptr;
  for (int c0 = 0; c0 < ncols; c0 += kMaxFuse) {
    const int R = std::min(kMaxFuse, ncols - c0);
    const int S = row_stride(A, R);
    zero_pad_rows(A, R, S, A->y1.p);
    launch_interleave(ctx, A->nl, R, S, 1.0, X + (int64_t)c0 * ldx, ldx, A->y1.p, planar_ld(A));
    sell_step(A, R, S, StepMode::plain, 1.0, 0.0, 0.0, A->y1.p, A->y2.p, nullptr, 0,
              Z + (int64_t)c0 * ldz, ldz);
  }
  if (counted) g_matvecs.fetch_add((uint64_t)ncols, std::memory_order_relaxed);
}

// Several Clenshaw steps per launch (clenshaw_multistep_stencil): constant-coefficient stencils
// on one rank with planar blocks and no per-lane positions, where a step is launch-bound
// (rows x columns below FLZ_MS_ROWS, default 2^17; FLZ_MS=0 never, FLZ_MS=1 whenever the window
// fits).  Allocates the second pair of workspaces on first use.
bool multistep_applies(const flz_matrix* A, int R, int S, bool allocate = true) {
  static const int mode = [] {
    const char* e = std::getenv("FLZ_MS");
    return e ? std::atoi(e) : -1;
  }();
  static const int64_t max_rows = [] {
    const char* e = std::getenv("FLZ_MS_ROWS");
    return e ? (int64_t)std::atoll(e) : ((int64_t)1 << 17);
  }();
  flz_ctx* ctx = A->ctx;
  if (mode == 0 || !A->multistep || ctx->exact || S != 0 || ctx->nranks != 1) return false;
  if (mode != 1 && A->nl * R > max_rows) return false;
  if (!allocate) return true;
  const size_t need = (size_t)planar_ld(A) * kMaxFuse + 8;
  if (A->y3.count < need) {
    A->y3.reserve_zero(need, ctx->stream);
    A->y4.reserve_zero(need, ctx->stream);
  }
  return true;
}

// Z = p((A - cI)/e) X by block Clenshaw (filter.cpp:122-155), device-resident blocks.
void filter_device(const flz_matrix* A, const double* coeffs, int m, double c, double e,
                   const double* X, int64_t ldx, int ncols, double* Z, int64_t ldz) {
  flz_ctx* ctx = A->ctx;
  ensure_workspaces(A);
  const double inv_e = 1.0 / e;                                  // filter.cpp:128
  const double s1 = 2.0 * inv_e, s2 = -2.0 * c * inv_e;          // filter.cpp:148
  const double f1 = inv_e, f2 = -c * inv_e;                      // filter.cpp:153
  for (int c0 = 0; c0 < ncols; c0 += kMaxFuse) {
    const int R = std::min(kMaxFuse, ncols - c0);
    const int S = row_stride(A, R);
    const double* Xc = X + (int64_t)c0 * ldx;
    double* Zc = Z + (int64_t)c0 * ldz;
    if (m == 0) {  // Y = b_0 X, no products (filter.cpp:133-136)
      for (int k = 0; k < R; ++k)
        launch_interleave(ctx, A->nl, 1, 1, coeffs[0], Xc + (int64_t)k * ldx, ldx,
                          Zc + (int64_t)k * ldz, 0);
      continue;
    }
    double* Y1 = A->y1.p;
    double* Y2 = A->y2.p;
    A->packed_from = nullptr;   // Y1 is rebuilt: nothing of it is packed yet
    zero_pad_rows(A, R, S, Y1);
    launch_interleave(ctx, A->nl, R, S, coeffs[m], Xc, ldx, Y1, planar_ld(A));   // :144
    FLZ_CUDA(cudaMemsetAsync(Y2, 0, (S > 0 ? (size_t)A->nl * S : (size_t)planar_ld(A) * R) *
                                            sizeof(double), ctx->stream));
    // short-reach stencils: several steps per launch while at least two are left (the state
    // after K steps is (y_K, y_{K-1}) in the second pair of workspaces)
    const bool multi = multistep_applies(A, R, S);
    double* O1 = multi ? A->y3.p : nullptr;
    double* O2 = multi ? A->y4.p : nullptr;
    for (int j = m - 1; j >= 1;) {                                              // :146-151
      if (multi && j >= 2) {
        double bs[8];
        const int avail = std::min(8, j);
        for (int q = 0; q < avail; ++q) bs[q] = coeffs[j - q];
        const int done = launch_multistep(ctx, view_all(A), R, avail, bs, s1, s2, Y1, Y2,
                                          planar_ld(A), Xc, ldx, O1, O2);
        if (done > 0) {
          std::swap(Y1, O1);
          std::swap(Y2, O2);
          j -= done;
          continue;
        }
      }
      sell_step(A, R, S, StepMode::step, s1, s2, coeffs[j], Y1, Y2, Xc, ldx, nullptr, 0);
      std::swap(Y1, Y2);
      --j;
    }
    sell_step(A, R, S, StepMode::final, f1, f2, coeffs[0], Y1, Y2, Xc, ldx, Zc, ldz);  // :152-154
    g_matvecs.fetch_add((uint64_t)R * (uint64_t)m, std::memory_order_relaxed);
  }
}

// host (n_local x ncols, column-major, ld = nl, original row order) -> device block in the
// matrix's permuted order (ld = A->ld, pad rows untouched)
void upload_block(const flz_matrix* A, const double* host, int ncols, double* dst) {
  flz_ctx* ctx = A->ctx;
  if (A->nl == 0 || ncols == 0) return;
  if (A->sigma <= 1) {
    FLZ_CUDA(cudaMemcpy2DAsync(dst, A->ld * sizeof(double), host, A->nl * sizeof(double),
                               A->nl * sizeof(double), ncols, cudaMemcpyHostToDevice,
                               ctx->stream));
    return;
  }
  ctx->stage.reserve((size_t)A->nl * ncols);
  FLZ_CUDA(cudaMemcpyAsync(ctx->stage.p, host, (size_t)A->nl * ncols * sizeof(double),
                           cudaMemcpyHostToDevice, ctx->stream));
  launch_permute_in(ctx, ctx->stage.p, A->nl, dst, A->ld, ncols, A->nl, A->perm.p);
}

// Large downloads into PAGEABLE host memory.  The driver stages such copies itself and reaches
// ~21 GB/s on this box; page-locked destinations reach 55 GB/s, but locking a result of
// hundreds of MB costs more than it saves (~0.25 s per GB).  So: two page-locked 16 MB buffers
// filled by cudaMemcpy2DAsync and emptied into the caller's block by a small team of host
// threads, one chunk of columns behind the copy engine.
constexpr size_t kDlChunkBytes = size_t(16) << 20;
bool staged_download(const flz_matrix* A, const double* src, int ncols, double* host) {
  flz_ctx* ctx = A->ctx;
  const size_t col_bytes = (size_t)A->nl * sizeof(double);
  const size_t total = col_bytes * (size_t)ncols;
  static const bool enabled = [] {   // FLZ_STAGED_D2H=0: the driver's pageable path
    const char* e = std::getenv("FLZ_STAGED_D2H");
    return !(e && e[0] == '0');
  }();
  if (!enabled || total < (size_t(32) << 20) || col_bytes > kDlChunkBytes) return false;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, host) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (attr.type != cudaMemoryTypeUnregistered) return false;   // already page-locked: direct copy
  for (int q = 0; q < 2; ++q) {
    if (!ctx->dl_pinned[q]) ctx->dl_pinned[q] = pinned_alloc(kDlChunkBytes);
    if (!ctx->dl_event[q])
      FLZ_CUDA(cudaEventCreateWithFlags(&ctx->dl_event[q], cudaEventDisableTiming));
  }
  const int per = (int)std::max<size_t>(1, kDlChunkBytes / col_bytes);   // columns per chunk
  const int nchunks = (ncols + per - 1) / per;
  auto issue = [&](int i) {
    const int c0 = i * per, nc = std::min(per, ncols - c0);
    FLZ_CUDA(cudaMemcpy2DAsync(ctx->dl_pinned[i & 1], col_bytes, src + (size_t)c0 * A->ld,
                               A->ld * sizeof(double), col_bytes, nc, cudaMemcpyDeviceToHost,
                               ctx->stream));
    FLZ_CUDA(cudaEventRecord(ctx->dl_event[i & 1], ctx->stream));
  };
  // team of copying threads (this thread is member 0), released chunk by chunk
  unsigned team = std::max(1u, std::min(6u, std::thread::hardware_concurrency() / 2));
  if (const char* e = std::getenv("FLZ_HOST_THREADS")) team = (unsigned)std::max(1, std::min(6, std::atoi(e)));
  SpinBarrier barrier(team);
  struct Job {
    char* dst = nullptr;
    const char* from = nullptr;
    size_t bytes = 0;
    bool stop = false;
  } job;
  auto share = [&](unsigned me) {
    const size_t b0 = job.bytes * me / team & ~size_t(63), b1 = me + 1 == team ? job.bytes : (job.bytes * (me + 1) / team & ~size_t(63));
    if (b1 > b0) std::memcpy(job.dst + b0, job.from + b0, b1 - b0);
  };
  std::vector<std::thread> pool;
  for (unsigned m = 1; m < team; ++m)
    pool.emplace_back([&, m] {
      while (true) {
        barrier.wait();
        if (job.stop) return;
        share(m);
        barrier.wait();
      }
    });
  struct Stop {
    std::vector<std::thread>& pool;
    SpinBarrier& barrier;
    Job& job;
    ~Stop() {
      if (pool.empty()) return;
      job.stop = true;
      barrier.wait();
      for (auto& t : pool) t.join();
    }
  } stop{pool, barrier, job};
  issue(0);
  for (int i = 0; i < nchunks; ++i) {
    if (i + 1 < nchunks) issue(i + 1);
    FLZ_CUDA(cudaEventSynchronize(ctx->dl_event[i & 1]));
    const int c0 = i * per, nc = std::min(per, ncols - c0);
    job.dst = reinterpret_cast<char*>(host + (size_t)c0 * A->nl);
    job.from = static_cast<const char*>(ctx->dl_pinned[i & 1]);
    job.bytes = col_bytes * (size_t)nc;
    if (team > 1) barrier.wait();
    share(0);
    if (team > 1) barrier.wait();
  }
  return true;
}

void download_block(const flz_matrix* A, const double* src, int ncols, double* host) {
  flz_ctx* ctx = A->ctx;
  if (A->nl == 0 || ncols == 0) return;
  if (A->sigma <= 1 && staged_download(A, src, ncols, host)) return;
  if (A->sigma <= 1) {
    FLZ_CUDA(cudaMemcpy2DAsync(host, A->nl * sizeof(double), src, A->ld * sizeof(double),
                               A->nl * sizeof(double), ncols, cudaMemcpyDeviceToHost,
                               ctx->stream));
  } else {
    ctx->stage2.reserve((size_t)A->nl * ncols);
    launch_permute_out(ctx, src, A->ld, ctx->stage2.p, A->nl, ncols, A->nl, A->perm.p);
    FLZ_CUDA(cudaMemcpyAsync(host, ctx->stage2.p, (size_t)A->nl * ncols * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
  }
  FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
}

void ensure_xz(const flz_matrix* A, int ncols) {
  flz_ctx* ctx = A->ctx;
  const size_t need = (size_t)A->ld * ncols;
  if (A->xs.count < need) A->xs.reserve_zero(need, ctx->stream);
  if (A->zs.count < need) A->zs.reserve_zero(need, ctx->stream);
}

// layout of ctx->small during a block step
struct SmallLayout {
  int64_t capC;     // doubles per coefficient block (cols x ldc)
  int ldc;          // row stride of C1/C2 (multiple of 8 covering r)
  int64_t C1, C2, gram, Sk, t1, t2, normsq, inv, dead, scale, total;
};
constexpr int kRMax = 16;
constexpr int kRecoverChunk = 64;  // columns of A V / rotated blocks held at a time
SmallLayout small_layout(int64_t max_cols, int r) {
  SmallLayout L;
  L.ldc = (int)round_up(r, 8);
  L.capC = (max_cols + 2 * kRMax) * L.ldc;
  L.C1 = 0;
  L.C2 = L.C1 + L.capC;
  L.gram = L.C2 + L.capC;
  L.Sk = L.gram + kRMax * kRMax;
  L.t1 = L.Sk + kRMax * kRMax;                 // [r][kRMax rows][8]
  L.t2 = L.t1 + kRMax * kRMax * 8;
  L.normsq = L.t2 + kRMax * kRMax * 8;
  L.inv = L.normsq + kRMax;
  L.dead = L.inv + kRMax;
  L.scale = L.dead + kRMax;
  L.total = L.scale + 8;
  return L;
}

}  // namespace

extern "C" {

const char* flz_last_error(void) { return g_last_error.c_str(); }
const char* flz_version(void) { return "flz 0.1 (sm_100a; SELL-32-sigma Clenshaw SpMM; DMMA GEMMs)"; }

// ---------------------------------------------------------------- context

static int ctx_create_common(int device, int rank, int nranks, const void* uid, flz_ctx** out,
                             LoopHub* hub = nullptr) {
  return guarded([&] {
    FLZ_REQUIRE(out != nullptr, FLZ_EINVAL, "ctx_create: null output");
    int count = 0;
    cudaError_t err = cudaGetDeviceCount(&count);
    if (err != cudaSuccess || count == 0)
      throw ApiError(FLZ_ENODEV,
                     std::string("no CUDA device available (") + cudaGetErrorString(err) +
                         "); libflz has no CPU fallback");
    if (device < 0) FLZ_CUDA(cudaGetDevice(&device));
    FLZ_REQUIRE(device < count, FLZ_EINVAL, "ctx_create: device index out of range");
    cudaDeviceProp prop;
    FLZ_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw ApiError(FLZ_ENODEV, std::string("device '") + prop.name +
                                     "' is not sm_100 (this library is built for sm_100a only)");
    FLZ_CUDA(cudaSetDevice(device));
    auto* ctx = new flz_ctx;
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    ctx->rank = rank;
    ctx->nranks = nranks;
    FLZ_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    FLZ_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    FLZ_CUDA(cudaEventCreateWithFlags(&ctx->ev_halo_ready, cudaEventDisableTiming));
    FLZ_CUDA(cudaEventCreateWithFlags(&ctx->ev_halo_done, cudaEventDisableTiming));
    for (int i = 0; i < 16; ++i) {
      FLZ_CUDA(cudaEventCreate(&ctx->t0[i]));
      FLZ_CUDA(cudaEventCreate(&ctx->t1[i]));
    }
    ctx->hub = hub;
    if (nranks > 1 && !hub) {
      FLZ_REQUIRE(uid != nullptr, FLZ_EINVAL, "ctx_create_dist: null NCCL unique id");
      ncclUniqueId id;
      static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
      std::memcpy(&id, uid, sizeof(id));
      FLZ_NCCL(ncclCommInitRank(&ctx->comm, nranks, id, rank));
    }
    *out = ctx;
  });
}

int flz_ctx_create(int device, flz_ctx** out) {
  return ctx_create_common(device, 0, 1, nullptr, out);
}
int flz_ctx_create_dist(int device, int rank, int nranks, const void* uid, flz_ctx** out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    set_last_error("ctx_create_dist: bad rank/nranks");
    return FLZ_EINVAL;
  }
  return ctx_create_common(device, rank, nranks, uid, out);
}
int flz_loop_hub_create(int nranks, void** out) {
  return guarded([&] {
    FLZ_REQUIRE(out && nranks >= 1 && nranks <= 8, FLZ_EINVAL, "loop_hub_create: 1..8 ranks");
    *out = loop_hub_create(nranks);
  });
}
void flz_loop_hub_destroy(void* hub) { loop_hub_destroy(static_cast<LoopHub*>(hub)); }
int flz_ctx_create_loopback(int device, int rank, int nranks, void* hub, flz_ctx** out) {
  if (!hub || nranks < 1 || rank < 0 || rank >= nranks) {
    set_last_error("ctx_create_loopback: bad hub/rank/nranks");
    return FLZ_EINVAL;
  }
  return ctx_create_common(device, rank, nranks, nullptr, out, static_cast<LoopHub*>(hub));
}
int flz_nccl_unique_id(void* out128) {
  return guarded([&] {
    ncclUniqueId id;
    FLZ_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
  });
}
// Handles are reference counted so that destroying them in any order is safe: a context
// outlives its matrices and bases, a matrix outlives the bases built on it.
static void ctx_release(flz_ctx* ctx) {
  if (!ctx || --ctx->refs > 0) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamSynchronize(ctx->comm_stream);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (int i = 0; i < 16; ++i) {
    cudaEventDestroy(ctx->t0[i]);
    cudaEventDestroy(ctx->t1[i]);
  }
  cudaEventDestroy(ctx->ev_halo_ready);
  cudaEventDestroy(ctx->ev_halo_done);
  for (int q = 0; q < 2; ++q) {
    pinned_free(ctx->dl_pinned[q]);
    if (ctx->dl_event[q]) cudaEventDestroy(ctx->dl_event[q]);
  }
  ctx->partial.release();
  ctx->small.release();
  ctx->stage.release();
  ctx->stage2.release();
  ctx->flush.release();
  pool_trim();  // cached blocks go back to the driver with the last user of the device
  cudaStreamDestroy(ctx->stream);
  cudaStreamDestroy(ctx->comm_stream);
  delete ctx;
}
void flz_ctx_destroy(flz_ctx* ctx) { ctx_release(ctx); }
int flz_ctx_sync(flz_ctx* ctx) {
  return guarded([&] {
    use(ctx);
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}
int flz_ctx_rank(const flz_ctx* ctx) { return ctx->rank; }
int flz_ctx_nranks(const flz_ctx* ctx) { return ctx->nranks; }
uint64_t flz_ctx_launch_count(const flz_ctx* ctx) { return ctx->launches; }
int flz_timer_start(flz_ctx* ctx, int slot) {
  return guarded([&] {
    FLZ_REQUIRE(slot >= 0 && slot < 16, FLZ_EINVAL, "timer slot out of range");
    use(ctx);
    FLZ_CUDA(cudaEventRecord(ctx->t0[slot], ctx->stream));
  });
}
int flz_timer_stop(flz_ctx* ctx, int slot, double* elapsed_ms) {
  return guarded([&] {
    FLZ_REQUIRE(slot >= 0 && slot < 16, FLZ_EINVAL, "timer slot out of range");
    use(ctx);
    FLZ_CUDA(cudaEventRecord(ctx->t1[slot], ctx->stream));
    FLZ_CUDA(cudaEventSynchronize(ctx->t1[slot]));
    float ms = 0.f;
    FLZ_CUDA(cudaEventElapsedTime(&ms, ctx->t0[slot], ctx->t1[slot]));
    if (elapsed_ms) *elapsed_ms = ms;
  });
}
int flz_flush_l2(flz_ctx* ctx, size_t bytes) {
  return guarded([&] {
    use(ctx);
    ctx->flush.reserve(bytes);
    FLZ_CUDA(cudaMemsetAsync(ctx->flush.p, 0, bytes, ctx->stream));
  });
}
int flz_ctx_set_exact(flz_ctx* ctx, int exact) {
  ctx->exact = exact != 0;
  return FLZ_OK;
}
int flz_ctx_make_current(const flz_ctx* ctx) {
  return guarded([&] {
    FLZ_REQUIRE(ctx, FLZ_EINVAL, "make_current: null context");
    use(ctx);
  });
}
int flz_host_alloc(size_t bytes, void** out) {
  return guarded([&] { *out = pinned_alloc(bytes); });
}
void flz_host_free(void* p) { pinned_free(p); }
int flz_mem_info(flz_ctx* ctx, size_t* free_bytes, size_t* total_bytes) {
  return guarded([&] {
    use(ctx);
    FLZ_CUDA(cudaMemGetInfo(free_bytes, total_bytes));
    *free_bytes += pool_cached_bytes();  // cached blocks are reusable (and trimmed on demand)
  });
}

uint64_t flz_matvec_count(void) { return g_matvecs.load(std::memory_order_relaxed); }
void flz_reset_matvec_count(void) { g_matvecs.store(0, std::memory_order_relaxed); }
void flz_matvec_sub(uint64_t count) { g_matvecs.fetch_sub(count, std::memory_order_relaxed); }

// ----------------------------------------------------------------- matrix

static_assert(sizeof(PlanTask) == sizeof(SliceTask), "PlanTask mirrors SliceTask");

// Device copy of a finished host plan (give lists set).
static void upload_plan(flz_ctx* ctx, HostPlan& P, flz_matrix* A) {
  A->ctx = ctx;
  A->n_global = P.n_global;
  A->row_begin = P.row_begin;
  A->row_end = P.row_end;
  A->nl = P.nl;
  A->ld = std::max<int64_t>(round_up(P.nl, kLdAlign), kLdAlign);
  A->nnz = P.nnz;
  A->dense_rows = P.nnz >= 16 * P.nl;
  A->stored = P.stored;
  A->nslices = P.nslices;
  A->nhalo = (int64_t)P.halo.size();
  A->sigma = P.sigma;
  A->short_rows = P.short_rows;
  A->lean = P.lean;
  A->n_interior = (int64_t)P.interior.size();
  A->n_boundary = (int64_t)P.boundary.size();
  A->nt_all = (int64_t)P.tasks_all.size();
  A->nt_interior = (int64_t)P.tasks_interior.size();
  A->nt_boundary = (int64_t)P.tasks_boundary.size();
  auto up = [&](auto& buf, const auto& host) {
    buf.reserve(std::max<size_t>(host.size(), 1));
    if (!host.empty())
      FLZ_CUDA(cudaMemcpyAsync(buf.p, host.data(), host.size() * sizeof(host[0]),
                               cudaMemcpyHostToDevice, ctx->stream));
  };
  up(A->slice_ptr, P.slice_ptr);
  up(A->slice_len, P.slice_len);
  up(A->row_len, P.row_len);
  A->h_col = std::move(P.col);  // exact-mode arrays: uploaded on first use
  A->h_val = std::move(P.val);
  static_assert(sizeof(PlanUgSlice) == sizeof(UgSlice), "PlanUgSlice mirrors UgSlice");
  A->ug.reserve(std::max<size_t>(P.ug_slice.size(), 1));
  if (!P.ug_slice.empty())
    FLZ_CUDA(cudaMemcpyAsync(A->ug.p, P.ug_slice.data(), P.ug_slice.size() * sizeof(UgSlice),
                             cudaMemcpyHostToDevice, ctx->stream));
  up(A->ug_val, P.ug_val);
  up(A->ug_col, P.ug_col);
  up(A->ug_uoff, P.ug_uoff);
  up(A->uv_pairs, P.uv_pairs);
  static_assert(sizeof(PlanStencilTiles) == sizeof(StencilTiles), "PlanStencilTiles mirrors StencilTiles");
  std::memcpy(static_cast<void*>(&A->tiles), &P.tiles, sizeof(StencilTiles));
  // multi-step launches: every position of every slice must be a (value, mask) pair
  A->multistep = P.tiles.nseg > 0 && P.nranks == 1 && P.halo.empty();
  for (size_t sl = 0; A->multistep && sl * 16 + 1 < P.uv_pairs.size(); ++sl) {
    uint64_t bits;
    std::memcpy(&bits, &P.uv_pairs[sl * 16 + 1], 8);
    if ((bits >> 56) & 1) A->multistep = false;
  }
  A->p2 = P.p2;
  if (P.p2) {
    static_assert(sizeof(PlanP2Slice) == sizeof(P2Slice), "PlanP2Slice mirrors P2Slice");
    A->p2_desc.reserve(std::max<size_t>(P.p2_desc.size(), 1));
    if (!P.p2_desc.empty())
      FLZ_CUDA(cudaMemcpyAsync(A->p2_desc.p, P.p2_desc.data(), P.p2_desc.size() * sizeof(P2Slice),
                               cudaMemcpyHostToDevice, ctx->stream));
    up(A->p2_col, P.p2_col);
    up(A->p2_val, P.p2_val);
    up(A->p2_dcol, P.p2_dcol);
    up(A->p2_dval, P.p2_dval);
    A->p2_blocks = P.p2_blocks;
    A->p2_dense_entries = P.p2_dense_entries;
    auto up_p2 = [&](DevBuf<SliceTask>& buf, const std::vector<PlanTask>& host, int64_t& count) {
      count = (int64_t)host.size();
      buf.reserve(std::max<size_t>(host.size(), 1));
      if (!host.empty())
        FLZ_CUDA(cudaMemcpyAsync(buf.p, host.data(), host.size() * sizeof(PlanTask),
                                 cudaMemcpyHostToDevice, ctx->stream));
    };
    up_p2(A->p2_tasks_all, P.p2_tasks_all, A->p2_nt_all);
    up_p2(A->p2_tasks_interior, P.p2_tasks_interior, A->p2_nt_interior);
    up_p2(A->p2_tasks_boundary, P.p2_tasks_boundary, A->p2_nt_boundary);
    A->p2_bytes = (int64_t)(P.p2_col.size() * 4 + P.p2_val.size() * 8 + P.p2_dcol.size() * 4 +
                            P.p2_dval.size() * 8 + P.p2_desc.size() * sizeof(P2Slice));
  }
  A->hy = P.hy;
  if (P.hy) {
    static_assert(sizeof(PlanHySlice) == sizeof(HySlice) && sizeof(PlanHyTask) == sizeof(HyTask),
                  "PlanHySlice / PlanHyTask mirror HySlice / HyTask");
    A->hy_slice.reserve(std::max<size_t>(P.hy_slice.size(), 1));
    if (!P.hy_slice.empty())
      FLZ_CUDA(cudaMemcpyAsync(A->hy_slice.p, P.hy_slice.data(), P.hy_slice.size() * sizeof(HySlice),
                               cudaMemcpyHostToDevice, ctx->stream));
    A->hy_dtasks.reserve(std::max<size_t>(P.hy_dtasks.size(), 1));
    if (!P.hy_dtasks.empty())
      FLZ_CUDA(cudaMemcpyAsync(A->hy_dtasks.p, P.hy_dtasks.data(),
                               P.hy_dtasks.size() * sizeof(HyTask), cudaMemcpyHostToDevice,
                               ctx->stream));
    up(A->hy_cols, P.hy_cols);
    up(A->hy_dcols, P.hy_dcols);
    up(A->hy_uvval, P.hy_uvval);
    up(A->hy_gval, P.hy_gval);
    up(A->hy_diag, P.hy_diag);
    up(A->hy_dval, P.hy_dval);
    up(A->sell_rows, P.sell_rows);
    A->hy_ndtasks = (int64_t)P.hy_dtasks.size();
    A->hy_ldp = round_up(P.hy_nslots, kLdAlign);
    A->hy_maxcols = P.hy_maxcols;
    A->hy_blocks = P.hy_blocks;
    A->hy_dense_entries = P.hy_dense_entries;
    A->hy_uv_entries = P.hy_uv_entries;
    A->hy_bytes = (int64_t)(P.hy_cols.size() * 4 + P.hy_dcols.size() * 4 +
                            (P.hy_uvval.size() + P.hy_gval.size() + P.hy_diag.size() +
                             P.hy_dval.size()) * 8 +
                            P.hy_slice.size() * sizeof(HySlice) + P.hy_dtasks.size() * sizeof(HyTask));
  }
  A->ug_bytes = (int64_t)(P.ug_val.size() * 8 + P.ug_col.size() * 4 + P.ug_uoff.size() * 4 +
                          P.ug_slice.size() * sizeof(UgSlice));
  A->ug_uniform_entries = P.ug_uniform_entries;
  A->split = P.split;
  A->nrest = P.nrest;
  up(A->rest_rows, P.rest_rows);
  A->ug_bytes += (int64_t)P.rest_rows.size() * 4;
  up(A->perm, P.perm);
  up(A->iperm, P.iperm);
  up(A->interior, P.interior);
  up(A->boundary, P.boundary);
  A->tasks_all.reserve(std::max<size_t>(P.tasks_all.size(), 1));
  A->tasks_interior.reserve(std::max<size_t>(P.tasks_interior.size(), 1));
  A->tasks_boundary.reserve(std::max<size_t>(P.tasks_boundary.size(), 1));
  auto up_tasks = [&](DevBuf<SliceTask>& buf, const std::vector<PlanTask>& host) {
    if (!host.empty())
      FLZ_CUDA(cudaMemcpyAsync(buf.p, host.data(), host.size() * sizeof(PlanTask),
                               cudaMemcpyHostToDevice, ctx->stream));
  };
  A->nt_rest_all = (int64_t)P.tasks_rest_all.size();
  A->nt_rest_interior = (int64_t)P.tasks_rest_interior.size();
  A->nt_rest_boundary = (int64_t)P.tasks_rest_boundary.size();
  A->tasks_rest_all.reserve(std::max<size_t>(P.tasks_rest_all.size(), 1));
  A->tasks_rest_interior.reserve(std::max<size_t>(P.tasks_rest_interior.size(), 1));
  A->tasks_rest_boundary.reserve(std::max<size_t>(P.tasks_rest_boundary.size(), 1));
  up_tasks(A->tasks_rest_all, P.tasks_rest_all);
  up_tasks(A->tasks_rest_interior, P.tasks_rest_interior);
  up_tasks(A->tasks_rest_boundary, P.tasks_rest_boundary);
  up_tasks(A->tasks_all, P.tasks_all);
  up_tasks(A->tasks_interior, P.tasks_interior);
  up_tasks(A->tasks_boundary, P.tasks_boundary);
  A->h_perm = P.perm;
  A->h_iperm = P.iperm;
  for (int p = 0; p < P.nranks; ++p) {
    if (p == P.rank || (P.need_cnt[p] == 0 && P.give_cnt[p] == 0)) continue;
    A->peers.push_back({p, P.give_off[p], P.give_cnt[p], P.need_off[p], P.need_cnt[p]});
  }
  A->n_send = (int64_t)P.send_rows.size();
  up(A->send_rows, P.send_rows);
  A->send_buf.reserve(std::max<size_t>(P.send_rows.size() * kMaxFuse, 1));
  if (P.tiles.nseg > 0 && (P.tiles.front > 0 || P.tiles.back > 0) && !P.send_rows.empty()) {
    // fused halo pack: every send row must lie in a halo-staging tile and go to <= 2 peers
    static const bool fused = [] {
      const char* e = std::getenv("FLZ_SLAB_PACK");   // 0: always the pack launch
      return !(e && e[0] == '0');
    }();
    const int64_t T = P.tiles.tile_rows;
    const int64_t hole0 = (int64_t)P.tiles.tile_a * T, hole1 = (int64_t)P.tiles.tile_b * T;
    const int64_t ntiles = (P.nslices * kPlanSliceRows + T - 1) / T;
    const int64_t rows = ntiles * T - (hole1 - hole0);
    std::vector<int2> slots((size_t)std::max<int64_t>(rows, 1), int2{-1, -1});
    bool ok = fused;
    for (size_t q = 0; ok && q < P.send_rows.size(); ++q) {
      const int64_t r = P.send_rows[q];
      if (r >= hole0 && r < hole1) { ok = false; break; }
      int2& e = slots[(size_t)(r < hole0 ? r : r - (hole1 - hole0))];
      if (e.x < 0) e.x = (int)q;
      else if (e.y < 0) e.y = (int)q;
      else ok = false;
    }
    if (ok) {
      A->send_slots.reserve(slots.size());
      FLZ_CUDA(cudaMemcpyAsync(A->send_slots.p, slots.data(), slots.size() * sizeof(int2),
                               cudaMemcpyHostToDevice, ctx->stream));
      FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  }
  FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
}

int flz_matrix_upload(flz_ctx* ctx, int64_t n_global, int64_t row_begin, int64_t row_end,
                      const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                      int sigma, flz_matrix** out) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && out && row_ptr, FLZ_EINVAL, "matrix_upload: null argument");
    FLZ_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= n_global, FLZ_EINVAL,
                "matrix_upload: bad row range");
    FLZ_REQUIRE(ctx->nranks > 1 || (row_begin == 0 && row_end == n_global), FLZ_EINVAL,
                "matrix_upload: a single-GPU context owns all rows");
    use(ctx);
    const int P = ctx->nranks;
    std::vector<int64_t> starts(P + 1, 0);
    starts[P] = n_global;
    if (P > 1) {  // every rank's first row
      DevBuf<int64_t> d;
      d.reserve(2 * (size_t)P + 2);
      FLZ_CUDA(cudaMemcpyAsync(d.p + P, &row_begin, sizeof(int64_t), cudaMemcpyHostToDevice,
                               ctx->stream));
      comm_allgather_i64(ctx, d.p + P, d.p, ctx->stream);
      FLZ_CUDA(cudaMemcpyAsync(starts.data(), d.p, P * sizeof(int64_t), cudaMemcpyDeviceToHost,
                               ctx->stream));
      FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
      FLZ_REQUIRE(starts[ctx->rank] == row_begin && (ctx->rank + 1 == P ? n_global
                                                                         : starts[ctx->rank + 1]) ==
                                                        row_end,
                  FLZ_EINVAL, "matrix_upload: rank row ranges must be ascending and contiguous");
    }
    HostPlan plan;
    try {
      plan = build_plan(n_global, ctx->rank, P, starts, row_ptr, col_idx, values, sigma);
    } catch (const std::invalid_argument& e) {
      throw ApiError(FLZ_EINVAL, std::string("matrix_upload: ") + e.what());
    }
    bool dense_rows_global = plan.nnz >= 16 * plan.nl;
    bool tiles_everywhere = true;
    if (P > 1) {
      // Halo rows travel in the block layout of the filter workspaces, so every rank must pick
      // the same one: the hybrid layout (planar blocks) only if EVERY rank found its dense
      // blocks, and the interleaved stride from the global nonzeros per row.
      DevBuf<int64_t> d;
      d.reserve(2 * (size_t)P + 2);
      std::vector<int64_t> all(P);
      auto gather = [&](int64_t mine) {
        FLZ_CUDA(cudaMemcpyAsync(d.p + P, &mine, sizeof(int64_t), cudaMemcpyHostToDevice,
                                 ctx->stream));
        comm_allgather_i64(ctx, d.p + P, d.p, ctx->stream);
        FLZ_CUDA(cudaMemcpyAsync(all.data(), d.p, P * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
      };
      gather(plan.hy ? 1 : 0);
      const bool all_hybrid = std::all_of(all.begin(), all.end(), [](int64_t v) { return v != 0; });
      // ... and the tile kernel of a stencil (planar blocks as well) only if every rank has a
      // tile plan; ranks without local rows have no say
      gather(plan.nl == 0 || plan.tiles.nseg > 0 ? 1 : 0);
      tiles_everywhere = std::all_of(all.begin(), all.end(), [](int64_t v) { return v != 0; });
      gather(plan.nnz);
      const int64_t nnz_all = std::accumulate(all.begin(), all.end(), (int64_t)0);
      dense_rows_global = nnz_all >= 16 * n_global;
      if (plan.hy && !all_hybrid) {
        try {
          plan = build_plan(n_global, ctx->rank, P, starts, row_ptr, col_idx, values, sigma, false);
        } catch (const std::invalid_argument& e) {
          throw ApiError(FLZ_EINVAL, std::string("matrix_upload: ") + e.what());
        }
      }
    }
    if (P > 1) {
      // tell every owner which of its rows we gather: counts first, then the row lists
      DevBuf<int64_t> d_cnt, d_need, d_give;
      d_cnt.reserve(2 * (size_t)P);
      FLZ_CUDA(cudaMemcpyAsync(d_cnt.p, plan.need_cnt.data(), P * sizeof(int64_t),
                               cudaMemcpyHostToDevice, ctx->stream));
      comm_group_start(ctx);
      for (int p = 0; p < P; ++p) {
        if (p == ctx->rank) continue;
        comm_send(ctx, d_cnt.p + p, sizeof(int64_t), p, ctx->stream);
        comm_recv(ctx, d_cnt.p + P + p, sizeof(int64_t), p, ctx->stream);
      }
      comm_group_end(ctx);
      std::vector<int64_t> give_cnt(P, 0), give_off(P, 0);
      FLZ_CUDA(cudaMemcpyAsync(give_cnt.data(), d_cnt.p + P, P * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, ctx->stream));
      FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
      give_cnt[ctx->rank] = 0;
      int64_t give_total = 0;
      for (int p = 0; p < P; ++p) {
        give_off[p] = give_total;
        give_total += give_cnt[p];
      }
      d_need.reserve(std::max<size_t>(plan.halo.size(), 1));
      d_give.reserve(std::max<size_t>((size_t)give_total, 1));
      if (!plan.halo.empty())
        FLZ_CUDA(cudaMemcpyAsync(d_need.p, plan.halo.data(), plan.halo.size() * sizeof(int64_t),
                                 cudaMemcpyHostToDevice, ctx->stream));
      comm_group_start(ctx);
      for (int p = 0; p < P; ++p) {
        if (p == ctx->rank) continue;
        if (plan.need_cnt[p])
          comm_send(ctx, d_need.p + plan.need_off[p], (size_t)plan.need_cnt[p] * sizeof(int64_t), p,
                    ctx->stream);
        if (give_cnt[p])
          comm_recv(ctx, d_give.p + give_off[p], (size_t)give_cnt[p] * sizeof(int64_t), p,
                    ctx->stream);
      }
      comm_group_end(ctx);
      std::vector<int64_t> give(std::max<int64_t>(give_total, 1));
      if (give_total)
        FLZ_CUDA(cudaMemcpyAsync(give.data(), d_give.p, give_total * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, ctx->stream));
      FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
      try {
        for (int p = 0; p < P; ++p)
          if (p != ctx->rank && give_cnt[p])
            plan_set_give(plan, p, give_cnt[p], give.data() + give_off[p]);
      } catch (const std::invalid_argument& e) {
        throw ApiError(FLZ_EINVAL, std::string("matrix_upload: ") + e.what());
      }
    }
    auto A = std::make_unique<flz_matrix>();
    if (!tiles_everywhere) plan.tiles = PlanStencilTiles{};
    upload_plan(ctx, plan, A.get());
    A->dense_rows = dense_rows_global;
    ctx->refs += 1;
    *out = A.release();
  });
}

// ---- host-only view of the plan (no GPU needed): used to test the multi-GPU logic on CPUs
struct flz_plan {
  HostPlan P;
  bool consumed = false;
};

int flz_plan_create(int64_t n_global, int rank, int nranks, const int64_t* starts,
                    const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                    int sigma, flz_plan** out) {
  return guarded([&] {
    FLZ_REQUIRE(starts && row_ptr && out, FLZ_EINVAL, "plan_create: null argument");
    try {
      auto plan = std::make_unique<flz_plan>();
      plan->P = build_plan(n_global, rank, nranks,
                           std::vector<int64_t>(starts, starts + nranks + 1), row_ptr, col_idx,
                           values, sigma);
      *out = plan.release();
    } catch (const std::invalid_argument& e) {
      throw ApiError(FLZ_EINVAL, e.what());
    }
  });
}
void flz_plan_destroy(flz_plan* plan) { delete plan; }
int flz_matrix_upload_plan(flz_ctx* ctx, flz_plan* plan, flz_matrix** out) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && plan && out, FLZ_EINVAL, "matrix_upload_plan: null argument");
    FLZ_REQUIRE(ctx->nranks == 1 && plan->P.nranks == 1, FLZ_EINVAL,
                "matrix_upload_plan: single-rank plans and contexts only");
    FLZ_REQUIRE(!plan->consumed, FLZ_EINVAL, "matrix_upload_plan: the plan was uploaded before");
    use(ctx);
    const Trace t(ctx, "upload of the prebuilt plan");
    auto A = std::make_unique<flz_matrix>();
    plan->consumed = true;
    upload_plan(ctx, plan->P, A.get());
    ctx->refs += 1;
    *out = A.release();
  });
}
int flz_plan_info(const flz_plan* plan, int64_t* info) {
  const HostPlan& P = plan->P;
  const int64_t v[10] = {P.nl, (int64_t)P.halo.size(), P.nslices, P.stored,
                         (int64_t)P.interior.size(), (int64_t)P.boundary.size(),
                         (int64_t)P.send_rows.size(), P.sigma, P.nnz, P.short_rows ? 1 : 0};
  std::copy(v, v + 10, info);
  return FLZ_OK;
}
int64_t flz_plan_need(const flz_plan* plan, int peer, int64_t* rows) {
  const HostPlan& P = plan->P;
  if (peer < 0 || peer >= P.nranks) return -1;
  if (rows)
    std::copy(P.halo.begin() + P.need_off[peer],
              P.halo.begin() + P.need_off[peer] + P.need_cnt[peer], rows);
  return P.need_cnt[peer];
}
int flz_plan_set_give(flz_plan* plan, int peer, int64_t count, const int64_t* rows) {
  return guarded([&] {
    try {
      plan_set_give(plan->P, peer, count, rows);
    } catch (const std::invalid_argument& e) {
      throw ApiError(FLZ_EINVAL, e.what());
    }
  });
}
int flz_plan_arrays(const flz_plan* plan, int32_t* perm, int64_t* slice_ptr, int32_t* slice_len,
                    int32_t* row_len, int32_t* col, double* val, int32_t* interior,
                    int32_t* boundary, int32_t* send_rows, int64_t* give_off, int64_t* give_cnt,
                    int64_t* need_off) {
  const HostPlan& P = plan->P;
  auto cp = [](const auto& v, auto* dst) {
    if (dst) std::copy(v.begin(), v.end(), dst);
  };
  cp(P.perm, perm);
  cp(P.slice_ptr, slice_ptr);
  cp(P.slice_len, slice_len);
  cp(P.row_len, row_len);
  if (col) std::copy(P.col.begin(), P.col.begin() + P.stored, col);
  if (val) std::copy(P.val.begin(), P.val.begin() + P.stored, val);
  cp(P.interior, interior);
  cp(P.boundary, boundary);
  cp(P.send_rows, send_rows);
  cp(P.give_off, give_off);
  cp(P.give_cnt, give_cnt);
  cp(P.need_off, need_off);
  return FLZ_OK;
}

int flz_plan_ug(const flz_plan* plan, int64_t* sizes, int32_t* descriptors, double* ug_val,
                int32_t* ug_col, int32_t* ug_uoff, int32_t* rest_rows) {
  if (!plan) return FLZ_EINVAL;
  try {
    flz::ensure_ug(const_cast<flz_plan*>(plan)->P);  // skipped when the paired layout was certain
  } catch (...) {
    return FLZ_EINVAL;
  }
  const HostPlan& P = plan->P;
  if (sizes) {
    sizes[0] = (int64_t)P.ug_slice.size();
    sizes[1] = (int64_t)P.ug_val.size();
    sizes[2] = (int64_t)P.ug_col.size();
    sizes[3] = (int64_t)P.ug_uoff.size();
    sizes[4] = P.ug_uniform_entries;
    sizes[5] = P.nrest;
    sizes[6] = P.split ? 1 : 0;
    sizes[7] = (int64_t)P.rest_interior.size();
  }
  if (rest_rows) std::copy(P.rest_rows.begin(), P.rest_rows.end(), rest_rows);
  if (descriptors && !P.ug_slice.empty())
    std::memcpy(descriptors, P.ug_slice.data(), P.ug_slice.size() * sizeof(PlanUgSlice));
  if (ug_val) std::copy(P.ug_val.begin(), P.ug_val.end(), ug_val);
  if (ug_col) std::copy(P.ug_col.begin(), P.ug_col.end(), ug_col);
  if (ug_uoff) std::copy(P.ug_uoff.begin(), P.ug_uoff.end(), ug_uoff);
  return FLZ_OK;
}

int flz_plan_p2(const flz_plan* plan, int64_t* sizes, int64_t* ptr, int32_t* col, double* val,
                int64_t* desc, int32_t* dcol, double* dval) {
  if (!plan) return FLZ_EINVAL;
  const HostPlan& P = plan->P;
  const int64_t dense_positions =
      P.p2 && !P.p2_desc.empty() ? P.p2_desc.back().dpos + P.p2_desc.back().nd : 0;
  if (sizes) {
    std::fill(sizes, sizes + 8, (int64_t)0);
    sizes[0] = P.p2 ? 1 : 0;
    sizes[1] = P.p2_slices;
    sizes[2] = P.p2 ? P.p2_ptr.back() : 0;   // general positions
    sizes[3] = (int64_t)P.p2_interior.size();
    sizes[4] = dense_positions;
    sizes[5] = P.p2_blocks;
    sizes[6] = P.p2_dense_entries;
  }
  if (!P.p2) return FLZ_OK;
  if (ptr) std::copy(P.p2_ptr.begin(), P.p2_ptr.end(), ptr);
  if (col) std::copy(P.p2_col.begin(), P.p2_col.end(), col);
  if (val) std::copy(P.p2_val.begin(), P.p2_val.end(), val);
  if (desc)
    for (size_t s = 0; s < P.p2_desc.size(); ++s) {
      const PlanP2Slice& D = P.p2_desc[s];
      const int64_t row[6] = {D.gpos, D.dpos, D.ng, D.nd, D.row0, D.nrows};
      std::copy(row, row + 6, desc + 6 * s);
    }
  if (dcol) std::copy_n(P.p2_dcol.begin(), dense_positions, dcol);
  if (dval) std::copy_n(P.p2_dval.begin(), dense_positions * 64, dval);
  return FLZ_OK;
}

int flz_plan_hy(const flz_plan* plan, int64_t* sizes, int64_t* slices, int32_t* cols,
                double* uvval, double* gval, double* diag, int64_t* tasks, int32_t* dcols,
                double* dval, int32_t* sell_rows) {
  if (!plan) return FLZ_EINVAL;
  const HostPlan& P = plan->P;
  if (sizes) {
    std::fill(sizes, sizes + 12, (int64_t)0);
    if (P.hy) {
      const int64_t v[12] = {1, (int64_t)P.hy_slice.size(), (int64_t)P.hy_dtasks.size(),
                             (int64_t)P.hy_cols.size(), (int64_t)P.hy_uvval.size(),
                             (int64_t)P.hy_gval.size(), (int64_t)P.hy_dcols.size(),
                             (int64_t)P.hy_dval.size(), P.hy_nslots, P.hy_blocks,
                             P.hy_dense_entries, P.hy_uv_entries};
      std::copy(v, v + 12, sizes);
    }
  }
  if (!P.hy) return FLZ_OK;
  if (slices)
    for (size_t s = 0; s < P.hy_slice.size(); ++s) {
      const PlanHySlice& H = P.hy_slice[s];
      const int64_t row[6] = {H.col_off, H.uv_off, H.g_off, H.nuv, H.ng, H.np};
      std::copy(row, row + 6, slices + 6 * s);
    }
  if (tasks)
    for (size_t t = 0; t < P.hy_dtasks.size(); ++t) {
      const PlanHyTask& T = P.hy_dtasks[t];
      const int64_t row[5] = {T.val_off, T.col_off, T.ncols, T.slot_base, T.nrows};
      std::copy(row, row + 5, tasks + 5 * t);
    }
  if (cols) std::copy(P.hy_cols.begin(), P.hy_cols.end(), cols);
  if (uvval) std::copy(P.hy_uvval.begin(), P.hy_uvval.end(), uvval);
  if (gval) std::copy(P.hy_gval.begin(), P.hy_gval.end(), gval);
  if (diag) std::copy_n(P.hy_diag.begin(), P.nl, diag);
  if (dcols) std::copy(P.hy_dcols.begin(), P.hy_dcols.end(), dcols);
  if (dval) std::copy(P.hy_dval.begin(), P.hy_dval.end(), dval);
  if (sell_rows) std::copy(P.sell_rows.begin(), P.sell_rows.end(), sell_rows);
  return FLZ_OK;
}

int flz_plan_tiles(const flz_plan* plan, int64_t* info, double* pairs) {
  if (!plan || !info) return FLZ_EINVAL;
  const HostPlan& P = plan->P;
  const PlanStencilTiles& G = P.tiles;
  std::fill(info, info + 30, (int64_t)0);
  info[0] = G.tile_rows;
  info[1] = G.nseg;
  for (int j = 0; j < kPlanMaxSegs; ++j) {
    info[2 + j] = G.seg_base[j];
    info[10 + j] = G.seg_len[j];
    info[18 + j] = G.seg_start[j];
  }
  info[26] = G.y1_elems;
  info[27] = G.own_e;
  info[28] = G.nseg ? (int64_t)P.uv_pairs.size() : 0;
  if (G.nseg && pairs) std::copy(P.uv_pairs.begin(), P.uv_pairs.end(), pairs);
  return FLZ_OK;
}
int flz_plan_tile_slab(const flz_plan* plan, int64_t* info) {
  if (!plan || !info) return FLZ_EINVAL;
  const PlanStencilTiles& G = plan->P.tiles;
  info[0] = G.front;
  info[1] = G.back;
  info[2] = G.tile_a;
  info[3] = G.tile_b;
  return FLZ_OK;
}

static void matrix_release(flz_matrix* A) {
  if (!A || --A->refs > 0) return;
  flz_ctx* ctx = A->ctx;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete A;
  ctx_release(ctx);
}
void flz_matrix_destroy(flz_matrix* A) { matrix_release(A); }
int64_t flz_matrix_rows_local(const flz_matrix* A) { return A->nl; }
int64_t flz_matrix_nnz_local(const flz_matrix* A) { return A->nnz; }
int flz_matrix_stats(const flz_matrix* A, int64_t* stored_entries, int64_t* slices,
                     int64_t* halo_rows, int64_t* boundary_slices) {
  if (stored_entries) *stored_entries = A->stored;
  if (slices) *slices = A->nslices;
  if (halo_rows) *halo_rows = A->nhalo;
  if (boundary_slices) *boundary_slices = A->n_boundary;
  return A->sigma;
}

int flz_matrix_layout(const flz_matrix* A, int64_t* matrix_bytes, int64_t* uniform_entries) {
  if (!A) return FLZ_EINVAL;
  // stencils with a tile plan: the TMA-staged kernel streams the (value, mask) pairs only
  if (matrix_bytes)
    *matrix_bytes = A->hy ? A->hy_bytes
                          : (A->p2 ? A->p2_bytes
                                   : (A->tiles.nseg > 0 ? (int64_t)A->uv_pairs.count * 8 : A->ug_bytes));
  if (uniform_entries) *uniform_entries = A->ug_uniform_entries;
  return FLZ_OK;
}
int flz_matrix_k1_info(const flz_matrix* A, int r, int64_t* info, char* kernel, int cap) {
  if (!A || r < 1 || r > kMaxFuse) return FLZ_EINVAL;
  const int S = row_stride(A, r);
  const char* name;
  int64_t matrix_bytes;
  if (A->ctx->exact) {
    name = "clenshaw_step_sell<EXACT>";
    matrix_bytes = A->stored * 12;
  } else if (A->hy) {
    const bool overlap = hybrid_overlaps(A->ctx, A->nslices, A->hy_ndtasks);
    name = overlap ? "hybrid_gather + hybrid_finish (dense tasks and slices overlapped)"
                   : "hybrid_dense_tasks + hybrid_slices (dense blocks + value-grouped slices)";
    // dense partials: written once and read once per row and block; the overlapped variant
    // also writes and reads the slices' sums once
    matrix_bytes = A->hy_bytes + 16 * A->hy_ndtasks * 32 * r + (overlap ? 16 * A->nl * r : 0);
  } else if (A->p2) {
    name = A->p2_blocks > 0 ? "clenshaw_step_p2_tasks (paired + dense sections)"
                            : "clenshaw_step_p2_tasks (paired)";
    matrix_bytes = A->p2_bytes;
  } else if (A->short_rows && A->lean) {
    const bool tile = A->tiles.nseg > 0 && (S == 0 || (S == 1 && r == 1));
    name = tile ? (multistep_applies(A, r, S, false)
                       ? "clenshaw_multistep_stencil (several Clenshaw steps per launch) + "
                         "clenshaw_step_stencil_tma"
                       : "clenshaw_step_stencil_tma")
                : "clenshaw_step_ug_warp";
    matrix_bytes = tile ? (int64_t)A->uv_pairs.count * 8 : A->ug_bytes;
  } else {
    name = "clenshaw_step_ug_tasks";
    matrix_bytes = A->ug_bytes;
  }
  const int64_t stride = S > 0 ? S : r;
  if (info) {
    info[0] = matrix_bytes + 8 * A->nl * (3 * stride + r);
    info[1] = A->hy ? A->hy_blocks : A->p2_blocks;
    info[2] = A->hy ? A->hy_dense_entries : A->p2_dense_entries;
    info[3] = S;
  }
  if (kernel && cap > 0) {
    std::strncpy(kernel, name, (size_t)cap - 1);
    kernel[cap - 1] = 0;
  }
  return FLZ_OK;
}
int flz_ctx_set_tuning(flz_ctx* ctx, int slices_per_cta, int tasks_per_cta, int batch) {
  if (!ctx || slices_per_cta < 0 || tasks_per_cta < 0 || batch < 0) return FLZ_EINVAL;
  ctx->k1_slices_per_cta = slices_per_cta;
  ctx->k1_tasks_per_cta = tasks_per_cta;
  ctx->k1_batch = batch;
  return FLZ_OK;
}

// ------------------------------------------------- block products & filter

int flz_spmm(flz_ctx* ctx, const flz_matrix* A, const double* X, int r, double* Y, int counted) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && A && X && Y && r >= 1, FLZ_EINVAL, "spmm: bad argument");
    use(ctx);
    ensure_xz(A, r);
    upload_block(A, X, r, A->xs.p);
    spmm_device(A, A->xs.p, A->ld, r, A->zs.p, A->ld, counted != 0);
    download_block(A, A->zs.p, r, Y);
  });
}

int flz_filter_apply(flz_ctx* ctx, const flz_matrix* A, const double* coeffs, int m, double c,
                     double e, const double* X, int r, double* Y) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && A && X && Y && coeffs && r >= 1, FLZ_EINVAL, "filter_apply: bad argument");
    FLZ_REQUIRE(m >= 0, FLZ_EINVAL, "filter needs at least one coefficient");
    FLZ_REQUIRE(e > 0.0, FLZ_EINTERVAL, "spectral bounds require lambda_min < lambda_max");
    use(ctx);
    ensure_xz(A, r);
    upload_block(A, X, r, A->xs.p);
    filter_device(A, coeffs, m, c, e, A->xs.p, A->ld, r, A->zs.p, A->ld);
    download_block(A, A->zs.p, r, Y);
  });
}

int flz_filter_bench(flz_ctx* ctx, const flz_matrix* A, const double* coeffs, int m, double c,
                     double e, const double* X, int r, int reps, int flush_l2, double* ms_total,
                     double* Y_last) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && A && X && coeffs && r >= 1 && m >= 1 && reps >= 1, FLZ_EINVAL,
                "filter_bench: bad argument");
    use(ctx);
    ensure_xz(A, r);
    upload_block(A, X, r, A->xs.p);
    if (flush_l2) {
      ctx->flush.reserve((size_t)256 << 20);
      FLZ_CUDA(cudaMemsetAsync(ctx->flush.p, 0, (size_t)256 << 20, ctx->stream));
    }
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
    FLZ_CUDA(cudaEventRecord(ctx->t0[15], ctx->stream));
    for (int rep = 0; rep < reps; ++rep)
      filter_device(A, coeffs, m, c, e, A->xs.p, A->ld, r, A->zs.p, A->ld);
    FLZ_CUDA(cudaEventRecord(ctx->t1[15], ctx->stream));
    FLZ_CUDA(cudaEventSynchronize(ctx->t1[15]));
    float ms = 0.f;
    FLZ_CUDA(cudaEventElapsedTime(&ms, ctx->t0[15], ctx->t1[15]));
    if (ms_total) *ms_total = ms;
    if (Y_last) download_block(A, A->zs.p, r, Y_last);
  });
}

int flz_dot(flz_ctx* ctx, const double* x, const double* y, int64_t n, double* out) {
  return guarded([&] {
    use(ctx);
    const int64_t ld = std::max<int64_t>(round_up(n, kLdAlign), kLdAlign);
    ctx->stage.reserve_zero((size_t)ld * 2, ctx->stream);
    ctx->small.reserve(64);
    FLZ_CUDA(cudaMemcpyAsync(ctx->stage.p, x, n * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    FLZ_CUDA(cudaMemcpyAsync(ctx->stage.p + ld, y, n * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    launch_gemm_tn(ctx, ctx->stage.p, ld, 1, ctx->stage.p + ld, ld, 1, n, ctx->small.p, 8);
    FLZ_CUDA(cudaMemcpyAsync(out, ctx->small.p, sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int flz_axpy(flz_ctx* ctx, double a, const double* x, double* y, int64_t n) {
  return guarded([&] {
    use(ctx);
    const int64_t ld = std::max<int64_t>(round_up(n, kLdAlign), kLdAlign);
    ctx->stage.reserve_zero((size_t)ld * 2, ctx->stream);
    ctx->small.reserve(64);
    FLZ_CUDA(cudaMemcpyAsync(ctx->stage.p, x, n * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    FLZ_CUDA(cudaMemcpyAsync(ctx->stage.p + ld, y, n * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    double bs[8] = {a, 0, 0, 0, 0, 0, 0, 0};
    FLZ_CUDA(cudaMemcpyAsync(ctx->small.p, bs, sizeof(bs), cudaMemcpyHostToDevice, ctx->stream));
    launch_gemm_nn(ctx, ctx->stage.p, ld, 1, ctx->small.p, 8, 1, n, 1.0, true, ctx->stage.p + ld,
                   ld);
    FLZ_CUDA(cudaMemcpyAsync(y, ctx->stage.p + ld, n * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int flz_clenshaw_combine(flz_ctx* ctx, int64_t n, double s1, double s2, double b,
                         const double* w, const double* y1, const double* y2, const double* x,
                         double* out) {
  return guarded([&] {
    use(ctx);
    ctx->stage.reserve((size_t)n * 5 + 8);
    double* d = ctx->stage.p;
    const double* src[4] = {w, y1, y2, x};
    for (int i = 0; i < 4; ++i)
      FLZ_CUDA(cudaMemcpyAsync(d + (size_t)i * n, src[i], n * sizeof(double),
                               cudaMemcpyHostToDevice, ctx->stream));
    launch_combine(ctx, n, ctx->exact, s1, s2, b, d, d + n, d + 2 * n, d + 3 * n, d + 4 * n);
    FLZ_CUDA(cudaMemcpyAsync(out, d + 4 * n, n * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ------------------------------------------------- Lanczos factorization

// A queued speculative application that will not be consumed (flz_basis, flz_internal.hpp);
// its products enter the matvec counter only when a step consumes it
static void drop_speculation(flz_basis* B) { B->spec_valid = false; }
// FLZ_SPECULATE=0: no speculative applications (experiments, A/B tests)
static bool speculation_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FLZ_SPECULATE");
    return !(e && e[0] == '0');
  }();
  return on;
}

int flz_basis_create(flz_ctx* ctx, const flz_matrix* A, int64_t max_cols, int r,
                     const double* start, flz_basis** out) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && A && start && out, FLZ_EINVAL, "basis_create: null argument");
    FLZ_REQUIRE(r >= 1 && r <= kRMax, FLZ_EINVAL,
                "basis_create: block_size must lie in [1, 16] on the device path");
    FLZ_REQUIRE(max_cols >= 2 * r, FLZ_EINVAL, "LanczosFactorization: column budget too small");
    use(ctx);
    auto B = std::make_unique<flz_basis>();
    B->ctx = ctx;
    B->A = A;
    B->nl = A->nl;
    B->ld = A->ld;
    B->r = r;
    B->max_cols = max_cols;
    const size_t total = (size_t)B->ld * (size_t)(max_cols + r);
    size_t free_b = 0, total_b = 0;
    FLZ_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (total * sizeof(double) > free_b)
      throw ApiError(FLZ_ENOMEM, "basis_create: basis of " +
                                     std::to_string(total * sizeof(double) >> 20) +
                                     " MiB does not fit in free device memory (" +
                                     std::to_string(free_b >> 20) + " MiB); lower max_dim");
    B->Q.reserve(total);
    if (B->ld > B->nl)  // keep the pad rows of every column zero
      FLZ_CUDA(cudaMemset2DAsync(B->Q.p + B->nl, B->ld * sizeof(double), 0,
                                 (B->ld - B->nl) * sizeof(double), max_cols + r, ctx->stream));
    B->Z.reserve_zero((size_t)B->ld * r, ctx->stream);
    B->X.reserve_zero((size_t)B->ld * r, ctx->stream);
    upload_block(A, start, r, B->Q.p);
    const SmallLayout L = small_layout(max_cols, r);
    B->small.reserve_zero((size_t)L.total, ctx->stream);
    B->pinned = static_cast<double*>(pinned_alloc((size_t)L.total * sizeof(double)));
    B->pinned_count = (size_t)L.total;
    FLZ_CUDA(cudaEventCreate(&B->e0));
    FLZ_CUDA(cudaEventCreate(&B->e1));
    FLZ_CUDA(cudaEventCreate(&B->e2));
    for (int q = 0; q < 2; ++q) {
      FLZ_CUDA(cudaEventCreate(&B->s0[q]));
      FLZ_CUDA(cudaEventCreate(&B->s1[q]));
    }
    FLZ_CUDA(cudaEventCreate(&B->e1b));
    FLZ_CUDA(cudaEventCreateWithFlags(&B->e_done, cudaEventDisableTiming));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->refs += 1;
    const_cast<flz_matrix*>(A)->refs += 1;
    *out = B.release();
  });
}

void flz_basis_destroy(flz_basis* B) {
  if (!B) return;
  cudaSetDevice(B->ctx->device);
  cudaStreamSynchronize(B->ctx->stream);
  if (B->e0) cudaEventDestroy(B->e0);
  if (B->e1) cudaEventDestroy(B->e1);
  if (B->e2) cudaEventDestroy(B->e2);
  for (int q = 0; q < 2; ++q) {
    if (B->s0[q]) cudaEventDestroy(B->s0[q]);
    if (B->s1[q]) cudaEventDestroy(B->s1[q]);
  }
  if (B->e1b) cudaEventDestroy(B->e1b);
  if (B->e_done) cudaEventDestroy(B->e_done);
  pinned_free(B->pinned);
  flz_ctx* ctx = B->ctx;
  flz_matrix* A = const_cast<flz_matrix*>(B->A);
  delete B;
  matrix_release(A);
  ctx_release(ctx);
}
int64_t flz_basis_blocks(const flz_basis* B) { return B->k; }

int flz_basis_get(flz_ctx* ctx, const flz_basis* B, int64_t j0, int64_t count, double* out) {
  return guarded([&] {
    FLZ_REQUIRE(j0 >= 0 && count >= 0 && j0 + count <= B->max_cols + B->r, FLZ_EDIM,
                "basis_get: column range out of bounds");
    use(ctx);
    for (int64_t c = 0; c < count; c += 64) {
      const int nc = (int)std::min<int64_t>(64, count - c);
      download_block(B->A, B->col(j0 + c), nc, out + (size_t)c * B->nl);
    }
  });
}

int flz_basis_set(flz_ctx* ctx, flz_basis* B, int64_t j, const double* col) {
  return guarded([&] {
    FLZ_REQUIRE(j >= 0 && j < B->max_cols + B->r, FLZ_EDIM, "basis_set: column out of bounds");
    use(ctx);
    drop_speculation(B);
    upload_block(B->A, col, 1, B->col(j));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int flz_basis_truncate(flz_ctx* ctx, flz_basis* B, int64_t k, double op_scale) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && B, FLZ_EINVAL, "basis_truncate: null argument");
    FLZ_REQUIRE(k >= 0 && k <= B->k, FLZ_EDIM, "basis_truncate: k exceeds the completed blocks");
    use(ctx);
    const SmallLayout L = small_layout(B->max_cols, B->r);
    drop_speculation(B);
    B->k = k;
    B->op_scale = op_scale;
    B->pinned[L.scale] = op_scale;
    FLZ_CUDA(cudaMemcpyAsync(B->small.p + L.scale, B->pinned + L.scale, sizeof(double),
                             cudaMemcpyHostToDevice, ctx->stream));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int flz_lanczos_step(flz_ctx* ctx, const flz_matrix* A, flz_basis* B, const double* coeffs,
                     int m, double c, double e, double* Dk, double* Sk, double* op_scale,
                     uint8_t* dead) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && A && B && Dk && Sk && dead, FLZ_EINVAL, "lanczos_step: null argument");
    FLZ_REQUIRE(B->A == A, FLZ_EINVAL, "lanczos_step: basis belongs to another matrix");
    const int r = B->r;
    FLZ_REQUIRE((B->k + 1) * r <= B->max_cols, FLZ_EDIM, "lanczos_step: column budget exhausted");
    FLZ_REQUIRE(m < 0 || (coeffs && e > 0.0), FLZ_EINVAL, "lanczos_step: bad filter");
    use(ctx);
    const int64_t nl = B->nl, ld = B->ld;
    const SmallLayout L = small_layout(B->max_cols, r);
    double* sm = B->small.p;

    // promote the pending block (lanczos.cpp:153); undone if anything below throws, so the
    // device basis never runs ahead of the host's LanczosFactorization
    struct Promote {
      flz_basis* B;
      bool committed = false;
      ~Promote() {
        if (!committed) B->k -= 1;
      }
    } promote{B};
    B->k += 1;
    const int64_t cols = B->k * r, newest = cols - r;

    const bool fused = ctx->nranks == 1 && fused_orth_enabled();
    // Z = op(newest block); the block is staged first, as the reference copies it
    // (lanczos.cpp:161-164) — it keeps the filter's X operand at a fixed address.  One rank:
    // Z goes straight into the pending block's storage.
    auto apply_op = [&](int64_t from_col, double* out) {
      FLZ_CUDA(cudaMemcpyAsync(B->X.p, B->col(from_col), (size_t)ld * r * sizeof(double),
                               cudaMemcpyDeviceToDevice, ctx->stream));
      if (m >= 0)
        filter_device(A, coeffs, m, c, e, B->X.p, ld, r, out, ld);
      else
        spmm_device(A, B->X.p, ld, r, out, ld, true);
    };
    const bool consumed =
        fused && B->spec_valid && B->spec_m == m && B->spec_c == c && B->spec_e == e &&
        (m < 0 || std::equal(coeffs, coeffs + m + 1, B->spec_coeffs.begin(), B->spec_coeffs.end()));
    const int read_slot = B->spec_slot;   // events around a consumed application
    if (consumed) {
      B->spec_valid = false;   // op(newest) is already in the pending block
      g_matvecs.fetch_add(B->spec_matvecs, std::memory_order_relaxed);
    } else {
      drop_speculation(B);
      FLZ_CUDA(cudaEventRecord(B->e0, ctx->stream));
      apply_op(newest, fused ? B->col(cols) : B->Z.p);
      FLZ_CUDA(cudaEventRecord(B->e1, ctx->stream));
    }
    FLZ_CUDA(cudaEventRecord(B->e1b, ctx->stream));

    if (fused) {
      // One rank: Z already sits in the pending block's storage, so [Q_k Z]^T Z gives the
      // projection coefficients AND Z^T Z (op_scale) in one sweep; the intra-block QR is one
      // cooperative launch that normalises the pending block in place.
      double* P = B->col(cols);
      launch_gemm_tn(ctx, B->Q.p, ld, cols + r, P, ld, r, nl, sm + L.C1, L.ldc);
      launch_gemm_nn(ctx, B->Q.p, ld, cols, sm + L.C1, L.ldc, r, nl, -1.0, true, P, ld);
      launch_gemm_tn(ctx, B->Q.p, ld, cols, P, ld, r, nl, sm + L.C2, L.ldc);
      launch_gemm_nn(ctx, B->Q.p, ld, cols, sm + L.C2, L.ldc, r, nl, -1.0, true, P, ld);
      launch_block_qr(ctx, P, ld, nl, r, sm + L.C1 + cols * L.ldc, L.ldc + 1, sm + L.scale,
                      sm + L.Sk, sm + L.dead);
    } else {
      // op_scale = max(op_scale, ||Z_j||) (lanczos.cpp:169-170)
      launch_coldot(ctx, B->Z.p, ld, B->Z.p, ld, r, nl, sm + L.normsq);
      allreduce(ctx, sm + L.normsq, r);
      launch_update_scale(ctx, sm + L.normsq, r, 0, sm + L.scale);

      // two full Gram-Schmidt sweeps in GEMM form (lanczos.cpp:177-182)
      launch_gemm_tn(ctx, B->Q.p, ld, cols, B->Z.p, ld, r, nl, sm + L.C1, L.ldc);
      allreduce(ctx, sm + L.C1, (size_t)cols * L.ldc);
      launch_gemm_nn(ctx, B->Q.p, ld, cols, sm + L.C1, L.ldc, r, nl, -1.0, true, B->Z.p, ld);
      launch_gemm_tn(ctx, B->Q.p, ld, cols, B->Z.p, ld, r, nl, sm + L.C2, L.ldc);
      allreduce(ctx, sm + L.C2, (size_t)cols * L.ldc);
      launch_gemm_nn(ctx, B->Q.p, ld, cols, sm + L.C2, L.ldc, r, nl, -1.0, true, B->Z.p, ld);

      // intra-block QR, two sweeps against the finished pending columns (lanczos.cpp:205-230)
      FLZ_CUDA(cudaMemsetAsync(sm + L.Sk, 0, (size_t)(L.normsq - L.Sk) * sizeof(double),
                               ctx->stream));
      double* P = B->col(cols);
      for (int j = 0; j < r; ++j) {
        double* zj = B->Z.p + (int64_t)j * ld;
        if (j > 0) {
          for (int pass = 0; pass < 2; ++pass) {
            double* t = sm + (pass == 0 ? L.t1 : L.t2) + (int64_t)j * kRMax * 8;
            launch_gemm_tn(ctx, P, ld, j, zj, ld, 1, nl, t, 8);
            allreduce(ctx, t, (size_t)j * 8);
            launch_gemm_nn(ctx, P, ld, j, t, 8, 1, nl, -1.0, true, zj, ld);
          }
        }
        launch_coldot(ctx, zj, ld, zj, ld, 1, nl, sm + L.normsq + j);
        allreduce(ctx, sm + L.normsq + j, 1);
        launch_finish_col(ctx, sm + L.normsq + j, sm + L.scale, sm + L.Sk, r, j, sm + L.inv + j,
                          sm + L.dead + j);
        launch_scale_copy(ctx, zj, sm + L.inv + j, P + (int64_t)j * ld, nl);
      }
    }
    FLZ_CUDA(cudaEventRecord(B->e2, ctx->stream));

    // small results back: D_k rows of C1, Sk + t1 + t2 + norms + flags + scale
    double* h = B->pinned;
    FLZ_CUDA(cudaMemcpyAsync(h, sm + L.C1 + newest * L.ldc, (size_t)r * L.ldc * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
    FLZ_CUDA(cudaMemcpyAsync(h + L.Sk, sm + L.Sk, (size_t)(L.total - L.Sk) * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
    FLZ_CUDA(cudaEventRecord(B->e_done, ctx->stream));
    // Speculation: op(pending block) for the next step, queued behind this step's copies.
    // Only short applications (< 2 ms measured on the previous step): a long one hides nothing
    // worth hiding and is the work thrown away when the solve stops here.
    const float prev_mv_ms = B->last_mv_ms;
    bool speculated = false;
    if (fused && speculation_enabled() && prev_mv_ms > 0.f && prev_mv_ms < 2.f &&
        (B->k + 1) * r <= B->max_cols) {
      const uint64_t before = g_matvecs.load(std::memory_order_relaxed);
      B->spec_slot = read_slot ^ 1;
      FLZ_CUDA(cudaEventRecord(B->s0[B->spec_slot], ctx->stream));
      apply_op(cols, B->col(cols + r));
      FLZ_CUDA(cudaEventRecord(B->s1[B->spec_slot], ctx->stream));
      B->spec_matvecs = g_matvecs.load(std::memory_order_relaxed) - before;
      g_matvecs.fetch_sub(B->spec_matvecs, std::memory_order_relaxed);   // counted when consumed
      if (m >= 0) B->spec_coeffs.assign(coeffs, coeffs + m + 1);
      B->spec_m = m;
      B->spec_c = c;
      B->spec_e = e;
      speculated = true;
    }
    FLZ_CUDA(cudaEventSynchronize(B->e_done));
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < r; ++j) Dk[i * r + j] = h[i * L.ldc + j];  // coeff[newest+i] of col j
    for (int i = 0; i < r * r; ++i) Sk[i] = 0.0;
    for (int j = 0; j < r; ++j) {
      for (int i = 0; i < j; ++i)
        Sk[i * r + j] = fused ? h[L.Sk + i * r + j]
                              : h[L.t1 + (int64_t)j * kRMax * 8 + i * 8] +
                                    h[L.t2 + (int64_t)j * kRMax * 8 + i * 8];
      Sk[j * r + j] = h[L.Sk + j * r + j];
      dead[j] = h[L.dead + j] != 0.0 ? 1 : 0;
    }
    B->op_scale = h[L.scale];
    if (op_scale) *op_scale = B->op_scale;
    float ms_mv = 0.f, ms_orth = 0.f;
    FLZ_CUDA(cudaEventElapsedTime(&ms_mv, consumed ? B->s0[read_slot] : B->e0,
                                  consumed ? B->s1[read_slot] : B->e1));
    FLZ_CUDA(cudaEventElapsedTime(&ms_orth, B->e1b, B->e2));
    B->mv_s += 1e-3 * ms_mv;
    B->orth_s += 1e-3 * ms_orth;
    B->last_mv_ms = ms_mv;
    B->spec_valid = speculated;
    promote.committed = true;
  });
}

int flz_orthogonalize_column(flz_ctx* ctx, const flz_basis* B, int64_t cols, int pending,
                             double* v, double* norm) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && B && v && norm, FLZ_EINVAL, "orthogonalize_column: null argument");
    FLZ_REQUIRE(cols + pending <= B->max_cols + B->r, FLZ_EDIM,
                "orthogonalize_column: too many columns");
    use(ctx);
    const int64_t nl = B->nl, ld = B->ld, M = cols + pending;
    const SmallLayout L = small_layout(B->max_cols, B->r);
    double* sm = B->small.p;
    double* z = B->Z.p;  // scratch: the step that owns Z has finished
    FLZ_CUDA(cudaMemsetAsync(z, 0, (size_t)ld * sizeof(double), ctx->stream));
    upload_block(B->A, v, 1, z);
    for (int pass = 0; pass < 2; ++pass) {
      launch_gemm_tn(ctx, B->Q.p, ld, M, z, ld, 1, nl, sm + L.C1, L.ldc);
      allreduce(ctx, sm + L.C1, (size_t)M * L.ldc);
      launch_gemm_nn(ctx, B->Q.p, ld, M, sm + L.C1, L.ldc, 1, nl, -1.0, true, z, ld);
    }
    launch_coldot(ctx, z, ld, z, ld, 1, nl, sm + L.normsq);
    allreduce(ctx, sm + L.normsq, 1);
    FLZ_CUDA(cudaMemcpyAsync(B->pinned, sm + L.normsq, sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    download_block(B->A, z, 1, v);
    *norm = std::sqrt(std::max(B->pinned[0], 0.0));
  });
}

int flz_basis_ortho_error(flz_ctx* ctx, const flz_basis* B, const uint8_t* dead, double* out) {
  return guarded([&] {
    use(ctx);
    const int64_t cols = B->k * B->r;
    double worst = 0.0;
    const int panel = 128;
    DevBuf<double> G;
    G.reserve((size_t)cols * panel + 8);
    std::vector<double> h((size_t)cols * panel);
    for (int64_t j0 = 0; j0 < cols; j0 += panel) {
      const int nb = (int)std::min<int64_t>(panel, cols - j0);
      launch_gemm_tn(ctx, B->Q.p, B->ld, cols, B->col(j0), B->ld, nb, B->nl, G.p, panel);
      allreduce(ctx, G.p, (size_t)cols * panel);
      FLZ_CUDA(cudaMemcpyAsync(h.data(), G.p, (size_t)cols * panel * sizeof(double),
                               cudaMemcpyDeviceToHost, ctx->stream));
      FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int64_t i = 0; i < cols; ++i) {
        if (dead && dead[i]) continue;
        for (int jj = 0; jj < nb; ++jj) {
          const int64_t j = j0 + jj;
          if (j < i || (dead && dead[j])) continue;
          worst = std::max(worst, std::abs(h[i * panel + jj] - (i == j ? 1.0 : 0.0)));
        }
      }
    }
    *out = worst;
  });
}

int flz_basis_times(const flz_basis* B, double* mv_s, double* orth_s) {
  if (mv_s) *mv_s = B->mv_s;
  if (orth_s) *orth_s = B->orth_s;
  return FLZ_OK;
}

// ------------------------------------------------------- Ritz recovery

int flz_ritz_lift(flz_ctx* ctx, const flz_matrix* A, const flz_basis* Bc, int64_t dim,
                  const double* W, int w, double* vnorm, uint8_t* keep, int* w_kept, double* Bm) {
  return guarded([&] {
    flz_basis* B = const_cast<flz_basis*>(Bc);
    FLZ_REQUIRE(ctx && A && B && W && vnorm && keep && w_kept && Bm, FLZ_EINVAL,
                "ritz_lift: null argument");
    FLZ_REQUIRE(dim == B->k * B->r, FLZ_EDIM, "ritz_lift: dim does not match the basis");
    use(ctx);
    *w_kept = 0;
    B->w_kept = 0;
    if (w == 0) return;
    const int64_t nl = B->nl, ld = B->ld;
    const int64_t ldw = round_up(w, 64);
    // V is the only n x w block of the recovery; A V and the rotated blocks are produced in
    // chunks of kRecoverChunk columns (memory: the 27M-row Laplacian with 345 wanted pairs
    // needs 37 GB per n x w block on each of 2 GPUs, next to a 97 GB basis)
    { Trace tr(ctx, "lift: reserve V, AV chunk");
    B->V.reserve_zero((size_t)ld * w, ctx->stream);
    B->AV.reserve_zero((size_t)ld * std::min(w, kRecoverChunk), ctx->stream); }
    // W (dim x w column-major) -> row-major [dim][ldw]
    std::vector<double> Wt((size_t)dim * ldw, 0.0);
    DevBuf<double> dW;
    { Trace tr(ctx, "lift: W transpose + H2D");
    for (int c = 0; c < w; ++c)
      for (int64_t j = 0; j < dim; ++j) Wt[(size_t)j * ldw + c] = W[(size_t)c * dim + j];
    dW.reserve(Wt.size() + 8);
    FLZ_CUDA(cudaMemcpyAsync(dW.p, Wt.data(), Wt.size() * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream)); }
    { Trace tr(ctx, "lift: V = Q W (gemm_nn)");
    launch_gemm_nn(ctx, B->Q.p, ld, dim, dW.p, ldw, w, nl, 1.0, false, B->V.p, ld); }
    DevBuf<double> dn;
    dn.reserve((size_t)2 * w + 8);
    launch_coldot(ctx, B->V.p, ld, B->V.p, ld, w, nl, dn.p);
    allreduce(ctx, dn.p, w);
    std::vector<double> hn(w), hs(w);
    FLZ_CUDA(cudaMemcpyAsync(hn.data(), dn.p, w * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
    int wk = 0;
    for (int c = 0; c < w; ++c) {
      vnorm[c] = std::sqrt(std::max(hn[c], 0.0));
      keep[c] = vnorm[c] >= 0.5 ? 1 : 0;  // lanczos.cpp:430-431
      if (!keep[c]) continue;
      if (wk != c)
        FLZ_CUDA(cudaMemcpyAsync(B->V.p + (size_t)wk * ld, B->V.p + (size_t)c * ld,
                                 ld * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
      hs[wk] = 1.0 / vnorm[c];
      ++wk;
    }
    *w_kept = wk;
    B->w_kept = wk;
    if (wk == 0) return;
    FLZ_CUDA(cudaMemcpyAsync(dn.p + w, hs.data(), wk * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    launch_scale_cols(ctx, B->V.p, ld, wk, nl, dn.p + w);
    const int64_t ldb = round_up(wk, 8);
    DevBuf<double> dB;
    dB.reserve((size_t)wk * ldb + 8);
    { Trace tr(ctx, "lift: A V, V'AV by chunks");
    for (int c0 = 0; c0 < wk; c0 += kRecoverChunk) {
      const int nc = std::min(kRecoverChunk, wk - c0);
      // uncounted products (lanczos.cpp:448-449); columns c0.. of V^T (A V) (:451-457)
      spmm_device(A, B->V.p + (size_t)c0 * ld, ld, nc, B->AV.p, ld, false);
      launch_gemm_tn(ctx, B->V.p, ld, wk, B->AV.p, ld, nc, nl, dB.p + c0, ldb);
    } }
    allreduce(ctx, dB.p, (size_t)wk * ldb);
    std::vector<double> hB((size_t)wk * ldb);
    FLZ_CUDA(cudaMemcpyAsync(hB.data(), dB.p, hB.size() * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < wk; ++i)  // 0.5*(v_i.Av_j + v_j.Av_i) (lanczos.cpp:451-457)
      for (int j = 0; j < wk; ++j)
        Bm[(size_t)j * wk + i] = 0.5 * (hB[(size_t)i * ldb + j] + hB[(size_t)j * ldb + i]);
  });
}

static void residuals_and_vectors(flz_ctx* ctx, const flz_basis* B, double* V, double* AV,
                                  const double* lambda, int w2, double scale, bool normalize,
                                  double* residuals, double* eigvecs) {
  const int64_t nl = B->nl, ld = B->ld;
  DevBuf<double> d;
  d.reserve((size_t)3 * w2 + 8);
  std::vector<double> h(w2), inv(w2, 1.0);
  if (normalize) {
    launch_coldot(ctx, V, ld, V, ld, w2, nl, d.p);
    allreduce(ctx, d.p, w2);
    FLZ_CUDA(cudaMemcpyAsync(h.data(), d.p, w2 * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int c = 0; c < w2; ++c) inv[c] = 1.0 / std::sqrt(h[c]);  // lanczos.cpp:473-475
  }
  FLZ_CUDA(cudaMemcpyAsync(d.p + w2, inv.data(), w2 * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
  FLZ_CUDA(cudaMemcpyAsync(d.p + 2 * w2, lambda, w2 * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
  launch_residual_prep(ctx, V, AV, ld, w2, nl, d.p + w2, d.p + 2 * w2);  // :476
  launch_coldot(ctx, AV, ld, AV, ld, w2, nl, d.p);
  allreduce(ctx, d.p, w2);
  FLZ_CUDA(cudaMemcpyAsync(h.data(), d.p, w2 * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int c = 0; c < w2; ++c) residuals[c] = std::sqrt(std::max(h[c], 0.0)) / scale;  // :477
  Trace tr(ctx, "eigenvectors D2H");
  if (eigvecs)
    for (int c = 0; c < w2; c += 64) {
      const int nc = std::min(64, w2 - c);
      download_block(B->A, V + (size_t)c * ld, nc, eigvecs + (size_t)c * nl);
    }
}

int flz_ritz_rotate(flz_ctx* ctx, const flz_basis* Bc, const double* U, const double* lambda,
                    int w2, double scale, double* residuals, double* eigvecs) {
  return guarded([&] {
    flz_basis* B = const_cast<flz_basis*>(Bc);
    FLZ_REQUIRE(ctx && B && (w2 == 0 || (U && lambda && residuals)), FLZ_EINVAL,
                "ritz_rotate: null argument");
    use(ctx);
    if (w2 == 0) return;
    const int wk = B->w_kept;
    FLZ_REQUIRE(wk > 0, FLZ_EINVAL, "ritz_rotate: call ritz_lift first");
    const int64_t nl = B->nl, ld = B->ld;
    const int64_t ldu = round_up(w2, 64);
    std::vector<double> Ut((size_t)wk * ldu, 0.0);
    for (int c = 0; c < w2; ++c)
      for (int j = 0; j < wk; ++j) Ut[(size_t)j * ldu + c] = U[(size_t)c * wk + j];
    DevBuf<double> dU;
    dU.reserve(Ut.size() + 8);
    FLZ_CUDA(cudaMemcpyAsync(dU.p, Ut.data(), Ut.size() * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    const int cmax = std::min(w2, kRecoverChunk);
    B->V2.reserve_zero((size_t)ld * cmax, ctx->stream);
    B->AV2.reserve_zero((size_t)ld * cmax, ctx->stream);
    Trace tr(ctx, "rotate: V U, A (V U), residuals, D2H by chunks");
    for (int c0 = 0; c0 < w2; c0 += kRecoverChunk) {
      const int nc = std::min(kRecoverChunk, w2 - c0);
      // v = V u (:467-470); A v is formed from v (the reference rotates A V: the same vector
      // up to rounding) so that no second n x w block has to be kept
      launch_gemm_nn(ctx, B->V.p, ld, wk, dU.p + c0, ldu, nc, nl, 1.0, false, B->V2.p, ld);
      spmm_device(B->A, B->V2.p, ld, nc, B->AV2.p, ld, false);
      residuals_and_vectors(ctx, B, B->V2.p, B->AV2.p, lambda + c0, nc, scale, true,
                            residuals + c0, eigvecs ? eigvecs + (size_t)c0 * nl : nullptr);
    }
  });
}

int flz_ritz_plain(flz_ctx* ctx, const flz_matrix* A, const flz_basis* Bc, const double* lambda,
                   int w_kept, double scale, double* residuals, double* eigvecs) {
  return guarded([&] {
    flz_basis* B = const_cast<flz_basis*>(Bc);
    FLZ_REQUIRE(ctx && A && B, FLZ_EINVAL, "ritz_plain: null argument");
    FLZ_REQUIRE(w_kept == B->w_kept, FLZ_EDIM, "ritz_plain: w_kept mismatch");
    use(ctx);
    if (w_kept == 0) return;
    // V holds the normalised lifted vectors; A V by chunks (lanczos.cpp:480-495)
    B->AV.reserve_zero((size_t)B->ld * std::min(w_kept, kRecoverChunk), ctx->stream);
    for (int c0 = 0; c0 < w_kept; c0 += kRecoverChunk) {
      const int nc = std::min(kRecoverChunk, w_kept - c0);
      double* Vc = B->V.p + (size_t)c0 * B->ld;
      spmm_device(A, Vc, B->ld, nc, B->AV.p, B->ld, false);
      residuals_and_vectors(ctx, B, Vc, B->AV.p, lambda + c0, nc, scale, false, residuals + c0,
                            eigvecs ? eigvecs + (size_t)c0 * B->nl : nullptr);
    }
  });
}

// ------------------------------------------------------- spectral bounds

int flz_bounds_lanczos(flz_ctx* ctx, const flz_matrix* A, int steps, const double* q0, double* d,
                       double* e, double* beta_last, int* done) {
  return guarded([&] {
    FLZ_REQUIRE(ctx && A && q0 && d && e && beta_last && done, FLZ_EINVAL,
                "bounds_lanczos: null argument");
    FLZ_REQUIRE(steps >= 1, FLZ_EINVAL, "bounds_lanczos: steps must be >= 1");
    use(ctx);
    const int64_t nl = A->nl, ld = A->ld;
    DevBuf<double> Q, w, sm;
    Q.reserve_zero((size_t)ld * steps, ctx->stream);
    w.reserve_zero((size_t)ld, ctx->stream);
    sm.reserve_zero((size_t)(steps + 4) * 8 * 2 + 64, ctx->stream);
    double* C = sm.p;                                   // [steps+..][8]
    double* sc = sm.p + (size_t)(steps + 4) * 8;        // scalars: nw2, a, beta2, inv, dead, ...
    double* one = sc + 16;                              // op_scale stand-in (=huge so never dead)
    Pinned pin(64);
    upload_block(A, q0, 1, Q.p);
    double scale = 0.0;
    *beta_last = 0.0;
    *done = 0;
    for (int s = 0; s < steps; ++s) {
      double* qs = Q.p + (size_t)s * ld;
      spmm_device(A, qs, ld, 1, w.p, ld, true);                          // lanczos.cpp:533
      launch_coldot(ctx, w.p, ld, w.p, ld, 1, nl, sc + 0);               // :534
      launch_coldot(ctx, qs, ld, w.p, ld, 1, nl, sc + 1);                // :535
      allreduce(ctx, sc, 2);
      for (int pass = 0; pass < 2; ++pass) {                             // :537-538
        launch_gemm_tn(ctx, Q.p, ld, s + 1, w.p, ld, 1, nl, C, 8);
        allreduce(ctx, C, (size_t)(s + 1) * 8);
        launch_gemm_nn(ctx, Q.p, ld, s + 1, C, 8, 1, nl, -1.0, true, w.p, ld);
      }
      launch_coldot(ctx, w.p, ld, w.p, ld, 1, nl, sc + 2);               // :539
      allreduce(ctx, sc + 2, 1);
      // inv = 1/beta via the finish kernel (op_scale slot = 0 => dead_tol = 1e-310)
      launch_finish_col(ctx, sc + 2, one, sc + 8, 1, 0, sc + 3, sc + 4);
      if (s + 1 < steps) launch_scale_copy(ctx, w.p, sc + 3, Q.p + (size_t)(s + 1) * ld, nl);
      FLZ_CUDA(cudaMemcpyAsync(pin.p, sc, 8 * sizeof(double), cudaMemcpyDeviceToHost,
                               ctx->stream));
      FLZ_CUDA(cudaStreamSynchronize(ctx->stream));
      const double nw = std::sqrt(std::max(pin.p[0], 0.0));
      scale = std::max(scale, nw);
      d[s] = pin.p[1];
      const double beta = std::sqrt(std::max(pin.p[2], 0.0));
      *beta_last = beta;
      *done = s + 1;
      if (beta <= 1e-14 * std::max(scale, 1e-300)) {                     // :541-544
        *beta_last = 0.0;
        break;
      }
      if (s + 1 < steps) e[s] = beta;                                    // :545-549
    }
  });
}

}  // extern "C"
