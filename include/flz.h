/* flz.h — C ABI of libflz.so: the B200-native filter-and-Lanczos hot path.
 *
 * This is the drop-in boundary for the reference CPU library `speig`
 * (/root/reference/proj): every entry point below names the reference
 * interface (file:line) it replaces.  Plain pointers and sizes only; no C++
 * or torch types; functions return 0 on success and a negative FLZ_E* code on
 * failure (message via flz_last_error()), and never throw across the ABI.
 *
 * Conventions
 *   - dense blocks passed from / to the host are COLUMN-MAJOR n x r with leading
 *     dimension n, exactly like speig::DenseBlock (dense_block.hpp:11-40);
 *   - CSR is int64 row_ptr / int32 col_idx / f64 values, exactly like
 *     speig::SparseSymMatrix (sparse.hpp:28-33);
 *   - r x r blocks (D_k, S_k) are row-major like LanczosFactorization::diag_blocks()
 *     (lanczos.hpp:86-88);
 *   - all arithmetic is IEEE FP64 on the device.  There is NO CPU fallback: every
 *     compute entry point fails with FLZ_ENODEV when no sm_100 device is usable.
 *
 * Multi-GPU: one process per GPU.  A context created with flz_ctx_create_dist()
 * owns rows [row_begin,row_end) of every n-vector and of the matrix; SpMV halos
 * travel by NCCL send/recv overlapped with interior rows, dot-product blocks by
 * NCCL all-reduce.  Host arrays passed to such a context are the LOCAL rows.
 */
#ifndef FLZ_H
#define FLZ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FLZ_OK 0
#define FLZ_EINVAL -1   /* bad argument            -> speig::Error            */
#define FLZ_EDIM -2     /* shape mismatch          -> speig::DimensionError   */
#define FLZ_EINTERVAL -3/* bad interval            -> speig::IntervalError    */
#define FLZ_ECUDA -4    /* CUDA runtime failure                               */
#define FLZ_ENODEV -5   /* no usable sm_100 device (no CPU fallback exists)   */
#define FLZ_ENCCL -6    /* NCCL failure                                       */
#define FLZ_ENOMEM -7
#define FLZ_EPARSE -8   /* Matrix Market parse error -> speig::ParseError     */
#define FLZ_ENUMERIC -9 /* e.g. QL failed to converge (band_eig.cpp:224-226)  */

typedef struct flz_ctx flz_ctx;       /* one GPU + stream + workspaces (+ NCCL comm) */
typedef struct flz_matrix flz_matrix; /* device-resident SELL-C-sigma matrix         */
typedef struct flz_basis flz_basis;   /* device-resident Lanczos factorization       */

const char* flz_last_error(void);
const char* flz_version(void);

/* ---------------------------------------------------------------- context */
/* device < 0 selects the current device. */
int flz_ctx_create(int device, flz_ctx** out);
/* nccl_unique_id: the 128-byte ncclUniqueId created on rank 0 (flz_nccl_unique_id)
 * and distributed by the caller (torch.distributed / MPI / file). */
int flz_ctx_create_dist(int device, int rank, int nranks, const void* nccl_unique_id,
                        flz_ctx** out);
/* LOOPBACK transport — TESTS ONLY.  NCCL refuses two ranks on one device; with a hub the ranks
 * of a "distributed" run are host threads of this process that share one GPU, and halo
 * send/recv, all-reduce and all-gather go through device-to-device copies ordered by CUDA
 * events (csrc/comm.cu).  Every rank calls the library from its own thread with its own
 * context; the row-partitioned device code that runs is exactly the NCCL build's. */
int flz_loop_hub_create(int nranks, void** hub);
void flz_loop_hub_destroy(void* hub);
int flz_ctx_create_loopback(int device, int rank, int nranks, void* hub, flz_ctx** out);
int flz_nccl_unique_id(void* out128);
void flz_ctx_destroy(flz_ctx* ctx);
int flz_ctx_sync(flz_ctx* ctx);
/* binds the calling host thread to the context's device (worker threads that allocate
 * page-locked memory or issue calls of their own) */
int flz_ctx_make_current(const flz_ctx* ctx);
int flz_ctx_rank(const flz_ctx* ctx);
int flz_ctx_nranks(const flz_ctx* ctx);
/* Launch counters: kernels of THIS library launched on the context since creation. */
uint64_t flz_ctx_launch_count(const flz_ctx* ctx);
/* Device timer on the context's stream (CUDA events). slot in [0,16). */
int flz_timer_start(flz_ctx* ctx, int slot);
int flz_timer_stop(flz_ctx* ctx, int slot, double* elapsed_ms); /* syncs the stop event */
/* Writes `bytes` of zeros to a scratch buffer: L2 flush between timed iterations. */
int flz_flush_l2(flz_ctx* ctx, size_t bytes);
/* 0: fast (FMA contraction) — default.  1: exact — the filter recurrence performs the
 * reference scalar backend's operations in the reference's order (kernels.cpp:25-41)
 * with separately rounded mul/add, making flz_filter_apply bit-identical to it. */
int flz_ctx_set_exact(flz_ctx* ctx, int exact);
/* Pinned host memory for the e2e path. */
int flz_host_alloc(size_t bytes, void** out);
void flz_host_free(void* p);
/* Device memory info (bytes). */
int flz_mem_info(flz_ctx* ctx, size_t* free_bytes, size_t* total_bytes);

/* ----------------------------------------------------------------- matrix */
/* Replaces the CSR arrays of speig::SparseSymMatrix as consumed by
 * kernels::csr_matvec (kernels.hpp:40-43, kernels.cpp:25-34).
 * Single-GPU: rows [0,n).  Distributed: pass the LOCAL rows [row_begin,row_end)
 * (row_ptr has row_end-row_begin+1 entries starting at 0, col_idx holds GLOBAL
 * column ids); every rank must call it collectively.
 * sigma: SELL-C-sigma sorting window in rows (0 = library default, 1 = no sorting). */
int flz_matrix_upload(flz_ctx* ctx, int64_t n_global, int64_t row_begin, int64_t row_end,
                      const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                      int sigma, flz_matrix** out);
void flz_matrix_destroy(flz_matrix* A);
int64_t flz_matrix_rows_local(const flz_matrix* A);
int64_t flz_matrix_nnz_local(const flz_matrix* A);
/* storage statistics: stored (padded) entries, slices, halo rows received per SpMV */
int flz_matrix_stats(const flz_matrix* A, int64_t* stored_entries, int64_t* slices,
                     int64_t* halo_rows, int64_t* boundary_slices);
/* index-compressed layout the fast kernels stream: matrix bytes read per product (paired
 * layout for long ragged rows; the (value, mask) pairs alone for stencils with a tile plan)
 * and the number of true nonzeros held at uniform-offset positions */
int flz_matrix_layout(const flz_matrix* A, int64_t* matrix_bytes, int64_t* uniform_entries);
/* what one fused Clenshaw step of `r` block columns (1..4) runs and moves in fast mode on
 * this matrix: name of the kernel (copied into kernel[cap]) and the bytes its layout has to
 * stream per launch (compressed matrix + the block streams: gather source once, Y2 in,
 * X in, result out), for the roofline record of bench.py.
 * info[4] = {streamed bytes, dense blocks, nonzeros held in dense sections, block row stride
 * (0 = planar)} */
int flz_matrix_k1_info(const flz_matrix* A, int r, int64_t* info, char* kernel, int cap);
/* launch-shape knobs of the fused Clenshaw-step kernels (0 = built-in default): slices per
 * CTA of the one-warp-per-slice kernel, tasks per CTA of the multi-warp kernel, positions
 * per pipeline stage of the one-warp-per-slice kernel (4 or 8) */
int flz_ctx_set_tuning(flz_ctx* ctx, int slices_per_cta, int tasks_per_cta, int batch);

/* Host-only half of flz_matrix_upload (no GPU, no NCCL): the SELL-32-sigma layout of this
 * rank's rows and its halo plan.  Exists so that the multi-GPU logic can be exercised on
 * CPUs; flz_matrix_upload runs exactly this code and then exchanges the need lists by NCCL.
 *   starts[nranks+1]: first row of every rank (+ n_global).
 *   info[10] = {rows_local, halo_rows, slices, stored_entries, interior_slices,
 *               boundary_slices, send_rows, sigma, nnz_local, short_rows}
 *   need(peer): global rows of `peer` this rank gathers (sorted); returns the count.
 *   set_give(peer): the rows `peer` needs from this rank (its need list), once per peer.
 *   arrays: any pointer may be NULL; sizes follow info[] (give/need offsets: nranks each). */
typedef struct flz_plan flz_plan;
int flz_plan_create(int64_t n_global, int rank, int nranks, const int64_t* starts,
                    const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                    int sigma, flz_plan** out);
void flz_plan_destroy(flz_plan* plan);
/* Device copy of a finished single-rank plan (nranks == 1 on both sides): what
 * flz_matrix_upload does after building the plan itself.  Lets a caller build the layout on
 * host threads ahead of time (SparseSymMatrix::from_csr builds it beside its symmetry check).
 * The plan is consumed: its arrays move into the matrix, a second upload is refused. */
int flz_matrix_upload_plan(flz_ctx* ctx, flz_plan* plan, flz_matrix** out);
int flz_plan_info(const flz_plan* plan, int64_t* info);
int64_t flz_plan_need(const flz_plan* plan, int peer, int64_t* rows);
int flz_plan_set_give(flz_plan* plan, int peer, int64_t count, const int64_t* rows);
int flz_plan_arrays(const flz_plan* plan, int32_t* perm, int64_t* slice_ptr, int32_t* slice_len,
                    int32_t* row_len, int32_t* col, double* val, int32_t* interior,
                    int32_t* boundary, int32_t* send_rows, int64_t* give_off, int64_t* give_cnt,
                    int64_t* need_off);
/* index-compressed layout of the plan (what the fast kernels stream), for host-side checks:
 * sizes[8] = {slices (main + rest), values, general columns, uniform offsets, uniform true
 * entries, rest slices, split mode, interior rest slices};
 * descriptors: 16 int32 per slice {val_ptr lo/hi, col_ptr lo/hi, uoff_ptr, nu, ng, flags,
 * first 8 offsets}; rest_rows: 32 int32 per rest slice (row of each lane, -1 = unused).
 * Any pointer may be NULL. */
int flz_plan_ug(const flz_plan* plan, int64_t* sizes, int32_t* descriptors, double* ug_val,
                int32_t* ug_col, int32_t* ug_uoff, int32_t* rest_rows);
/* paired layout of the plan (long ragged rows; host/plan.hpp), for host-side checks:
 * sizes[8] = {used, slices, general positions, interior slices, dense positions, dense
 * blocks, nonzeros in dense sections, 0}; ptr[slices + 1] first general position of every
 * slice; col[positions * 32]; val[positions * 64] (two values per lane and position);
 * desc[slices * 6] = {gpos, dpos, ng, nd, row0, nrows} per slice; dcol[dense positions]
 * shared columns; dval[dense positions * 64].  Any pointer may be NULL. */
int flz_plan_p2(const flz_plan* plan, int64_t* sizes, int64_t* ptr, int32_t* col, double* val,
                int64_t* desc, int32_t* dcol, double* dval);
/* hybrid layout of the plan (stencil + dense blocks, natural row order; host/plan.hpp), for
 * host-side checks: sizes[12] = {used, slices, dense tasks, ints in cols, doubles in uvval,
 * doubles in gval, ints in dcols, doubles in dval, partial slots, dense blocks, nonzeros in
 * dense tasks, nonzeros at uniform-value positions}; slices[slices * 6] = {col_off, uv_off,
 * g_off, nuv, ng, np}; tasks[dense tasks * 5] = {val_off, col_off, ncols, slot_base, nrows};
 * diag[rows]; sell_rows[SELL slices * 32] row of every lane of the exact-mode arrays.  Any
 * pointer may be NULL. */
int flz_plan_hy(const flz_plan* plan, int64_t* sizes, int64_t* slices, int32_t* cols,
                double* uvval, double* gval, double* diag, int64_t* tasks, int32_t* dcols,
                double* dval, int32_t* sell_rows);
/* tile plan of the TMA-staged stencil kernel (constant-coefficient stencils, one rank or row slabs;
 * host/plan.hpp), for host-side checks: info[30] = {tile_rows, segments, seg_base[8],
 * seg_len[8], seg_start[8], staged elements per column, staged element of offset 0,
 * doubles in pairs, 0}; info[1] == 0: the matrix has no tile plan.  pairs: 16 doubles per
 * slice, padded to whole tiles — (value, mask word) per position, mask word = lane mask |
 * 8 * staged element << 32 | (position 0 only) position count << 52 | (position 0 only,
 * slice also has per-lane positions) 1 << 56.  pairs may be NULL. */
int flz_plan_tiles(const flz_plan* plan, int64_t* info, double* pairs);
/* ... on a row slab (nranks > 1): info[4] = {front, back, tile_a, tile_b} — the kernel stages
 * runs of the virtual source [front halo rows | local rows | back halo rows] (front = halo
 * slots owned by lower ranks; stored source: [local | front halo | back halo]), and tiles
 * [tile_a, tile_b) stage local rows only: they run while the halo rows travel. */
int flz_plan_tile_slab(const flz_plan* plan, int64_t* info);

/* Global matvec counter: speig::matvec_count()/reset (sparse.hpp:74-79).  One count per
 * vector-column product, so a fused r-column block product adds r. */
uint64_t flz_matvec_count(void);
void flz_reset_matvec_count(void);
/* takes back the counts of block steps that were rolled back (flz_basis_truncate) */
void flz_matvec_sub(uint64_t count);

/* ------------------------------------------------- block products & filter */
/* Y = A X, r columns, host buffers.  Replaces SparseSymMatrix::spmm_block
 * (sparse.cpp:105-111) / spmv (:91-94); counted!=0 bumps the matvec counter by r
 * (apply_uncounted, :87-89, otherwise). */
int flz_spmm(flz_ctx* ctx, const flz_matrix* A, const double* X, int r, double* Y, int counted);

/* Y = p_m((A - cI)/e) X by the block Clenshaw recurrence with coefficients b[0..m].
 * Replaces ChebyshevFilter::apply (filter.cpp:122-155): exactly m fused block
 * products (r*m counted matvecs); m == 0 gives Y = b_0 X with no product. */
int flz_filter_apply(flz_ctx* ctx, const flz_matrix* A, const double* coeffs, int m, double c,
                     double e, const double* X, int r, double* Y);

/* Same, device-resident, for benchmarking the recurrence alone: runs `reps` filter
 * applications on an internal n x r block (filled from X once), returns the device time
 * of the timed region in ms (CUDA events on the context's stream). */
int flz_filter_bench(flz_ctx* ctx, const flz_matrix* A, const double* coeffs, int m, double c,
                     double e, const double* X, int r, int reps, int flush_l2, double* ms_total,
                     double* Y_last);

/* L0 kernels on host buffers — test seams for kernels.hpp:29-49. */
int flz_dot(flz_ctx* ctx, const double* x, const double* y, int64_t n, double* out);
int flz_axpy(flz_ctx* ctx, double a, const double* x, double* y, int64_t n);
int flz_clenshaw_combine(flz_ctx* ctx, int64_t n, double s1, double s2, double b,
                         const double* w, const double* y1, const double* y2, const double* x,
                         double* out);

/* ------------------------------------------------- Lanczos factorization  */
/* Replaces LanczosFactorization's ctor (lanczos.cpp:105-118): device basis with room for
 * max_cols + r columns (allocated lazily in chunks, not eagerly), first block = start. */
int flz_basis_create(flz_ctx* ctx, const flz_matrix* A, int64_t max_cols, int r,
                     const double* start, flz_basis** out);
void flz_basis_destroy(flz_basis* B);
int64_t flz_basis_blocks(const flz_basis* B); /* k */
/* Rolls the factorization back to its first k completed blocks (k <= current): block k
 * becomes the pending block again — it still holds what it held when it was pending — and
 * the running operator-output scale is reset to `op_scale`, its value at that point.  Used by
 * the solver when block steps ran speculatively beside a host-side convergence check. */
int flz_basis_truncate(flz_ctx* ctx, flz_basis* B, int64_t k, double op_scale);
/* Copies basis columns [j0, j0+count) (local rows) to the host, column-major. */
int flz_basis_get(flz_ctx* ctx, const flz_basis* B, int64_t j0, int64_t count, double* out);
/* Overwrites one column (breakdown replacement path, lanczos.cpp:232-262). */
int flz_basis_set(flz_ctx* ctx, flz_basis* B, int64_t j, const double* col);

/* One block step of expand() (lanczos.cpp:134-271) without the breakdown replacement:
 *   Z = op(newest block)            [m >= 0: Clenshaw filter; m < 0: plain A]
 *   op_scale = max(op_scale, ||Z_j||)
 *   two full Gram-Schmidt sweeps against all k*r basis columns (FP64 DMMA GEMMs)
 *   D_k = first-sweep coefficients against the newest block (NOT symmetrized here)
 *   intra-block QR (two sweeps) -> S_k upper triangular, diag = norms, next pending block
 * Outputs (host): Dk, Sk row-major r x r; colnorm[j] = ||z_j|| before normalisation;
 * dead[j] = 1 where ||z_j|| <= dead_tol = 1e-10*max(op_scale,1e-300) — such a column is
 * left ZERO in the pending block and the caller (host driver) runs the replacement
 * policy with flz_orthogonalize_column()/flz_basis_set(). */
int flz_lanczos_step(flz_ctx* ctx, const flz_matrix* A, flz_basis* B, const double* coeffs,
                     int m, double c, double e, double* Dk, double* Sk, double* op_scale,
                     uint8_t* dead);
/* Replacement helper: orthogonalizes host vector v (local rows) against the first `cols`
 * basis columns and the first `pending` pending columns twice (lanczos.cpp:237-247),
 * returns its norm; v is overwritten with the orthogonalized (unnormalised) vector. */
int flz_orthogonalize_column(flz_ctx* ctx, const flz_basis* B, int64_t cols, int pending,
                             double* v, double* norm);
/* ortho_error() (lanczos.cpp:120-132): max |Q^T Q - I| over live columns. */
int flz_basis_ortho_error(flz_ctx* ctx, const flz_basis* B, const uint8_t* dead, double* out);
/* Device seconds spent in the filter (MV) and orthogonalization (ORTH) buckets, the
 * reference's ExpandTimes (lanczos.hpp:58-61), measured with CUDA events. */
int flz_basis_times(const flz_basis* B, double* mv_s, double* orth_s);

/* ------------------------------------------------------- Ritz recovery    */
/* recover_eigenpairs (lanczos.cpp:407-510), device part 1:
 *   V = Q_k W (dim x w column-major W from the host), vnorm[c] = ||V_c||, V_c /= vnorm[c]
 *   for columns with vnorm >= 0.5 (others are dropped, keep[c] = 0);
 *   AV = A V (uncounted); Bm = sym(V^T A V) over kept columns (w_kept x w_kept, col-major).
 * Returns w_kept through *w_kept. */
int flz_ritz_lift(flz_ctx* ctx, const flz_matrix* A, const flz_basis* B, int64_t dim,
                  const double* W, int w, double* vnorm, uint8_t* keep, int* w_kept,
                  double* Bm);
/* part 2: for the `w2` selected eigenpairs (U: w_kept x w2 column-major, lambda[w2]):
 *   v = V u / ||V u||, residual = ||A v - lambda v|| / scale; eigvecs (n_local x w2,
 *   column-major) may be NULL. */
int flz_ritz_rotate(flz_ctx* ctx, const flz_basis* B, const double* U, const double* lambda,
                    int w2, double scale, double* residuals, double* eigvecs);
/* plain-mode variant (lanczos.cpp:480-495): residuals of the lifted vectors themselves */
int flz_ritz_plain(flz_ctx* ctx, const flz_matrix* A, const flz_basis* B, const double* lambda,
                   int w_kept, double scale, double* residuals, double* eigvecs);

/* estimate_spectral_bounds' Lanczos loop (lanczos.cpp:529-551) on the device: q0 (unit
 * start vector, local rows) -> d[steps], e[steps-1], beta_last, *done steps. Counted. */
int flz_bounds_lanczos(flz_ctx* ctx, const flz_matrix* A, int steps, const double* q0, double* d,
                       double* e, double* beta_last, int* done);

#ifdef __cplusplus
}
#endif
#endif /* FLZ_H */
