// kernels_sell.cu — K1: the fused Clenshaw-step SpMM on a SELL-32-sigma matrix.
//
// Replaces, per Clenshaw step, the reference's r separate csr_matvec sweeps
// (sparse.cpp:105-111 -> kernels.cpp:25-34) plus one clenshaw_combine pass
// (kernels.cpp:36-41) as driven by ChebyshevFilter::apply (filter.cpp:146-154):
// the matrix is streamed ONCE for all R block columns and the combine is applied
// in the epilogue, so a step moves 12*nnz + 4*n(row lengths) + 32*n*R bytes.
//
// Layout: slices of 32 consecutive (permuted) rows, one lane per row; the slice's
// (val, col) pairs are stored column-major so that step p of all 32 rows is one
// coalesced 256 B + 128 B load.  Block vectors are row-interleaved with a row stride of
// S >= R doubles, so a nonzero costs one gather of a whole row of the block; for
// stencil-like matrices neighbouring lanes gather neighbouring rows, i.e. the gathers are
// coalesced too.  S = 4 for R = 3 on long-row (PARSEC-like) matrices: a 32-byte aligned
// row is exactly one sector and two 16-byte loads, which halves the L1 traffic of the
// gathers (ncu: l1tex at 76 % with S = 3); short-row stencils keep S = R because there the
// block vectors are half of the HBM traffic.
//
// Two kernels:
//  * clenshaw_step_tasks<R,S,MODE>  — fast path.  CTAs of 8 warps work through a host-built
//    task list; long slices are split over 2/4/8 warps whose partial sums meet in shared
//    memory in a fixed order (deterministic).  The (val, col) stream is software pipelined
//    one batch ahead of the dependent gathers.
//  * clenshaw_step_sell<R,MODE,EXACT> — one warp per slice, strictly sequential per row.
//    EXACT = true reproduces the reference scalar backend bit for bit: products are
//    accumulated left to right in CSR order with separately rounded multiply and add (the
//    reference's scalar TU is built without FMA), the combine is ((s1*w + s2*y1) - y2) + b*x.

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "flz_internal.hpp"

namespace flz {

namespace {

constexpr int kWarpsPerBlock = 4;
#ifndef FLZ_K1_BATCH
#define FLZ_K1_BATCH 4
#endif
constexpr int kBatch = FLZ_K1_BATCH;  // matrix entries per row requested per pipeline stage

// Programmatic dependent launch: consecutive Clenshaw steps depend on each other through Y1/Y2
// only, so step j+1 may be scheduled while step j drains and read its (immutable) matrix
// stream; pdl_wait() orders everything after it behind the complete previous grid.  Both are
// no-ops for a launch without the attribute.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// integer environment switch (experiments: FLZ_ST_STAGES, FLZ_ST_CTAS, FLZ_HY_OVERLAP, ...)
inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

// FLZ_K1_PDL=0 restores plain stream-ordered launches (experiments)
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FLZ_K1_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class... KArgs, class... Args>
void launch_k1_smem(flz_ctx* ctx, void (*kernel)(KArgs...), unsigned grid, unsigned block,
                    size_t smem, Args&&... args);
template <class... KArgs, class... Args>
void launch_k1(flz_ctx* ctx, void (*kernel)(KArgs...), unsigned grid, unsigned block,
               Args&&... args) {
  launch_k1_smem(ctx, kernel, grid, block, 0, std::forward<Args>(args)...);
}
template <class... KArgs, class... Args>
void launch_k1_smem(flz_ctx* ctx, void (*kernel)(KArgs...), unsigned grid, unsigned block,
                    size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  const bool pdl = pdl_enabled() && (ctx->nranks == 1 || ctx->k1_pdl_once);
  ctx->k1_pdl_once = false;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  FLZ_CUDA(cudaLaunchKernelEx(&cfg, kernel, KArgs(std::forward<Args>(args))...));
}

template <bool EXACT>
__device__ __forceinline__ double mul_add(double a, double b, double c) {
  if constexpr (EXACT)
    return __dadd_rn(__dmul_rn(a, b), c);
  else
    return fma(a, b, c);
}

template <bool EXACT>
__device__ __forceinline__ double combine(double s1, double w, double s2, double y1, double y2,
                                          double b, double x) {
  if constexpr (EXACT) {
    // s1*w + s2*y1 - y2 + b*x, evaluated left to right as the C expression is
    const double t = __dadd_rn(__dmul_rn(s1, w), __dmul_rn(s2, y1));
    return __dadd_rn(__dsub_rn(t, y2), __dmul_rn(b, x));
  } else {
    return fma(b, x, fma(s1, w, fma(s2, y1, -y2)));
  }
}

__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream_s32(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// One row of an interleaved block (R useful doubles, row stride S) with the widest load the
// alignment allows: S = 2 -> one 16-byte load, S = 4 -> one 32-byte load (LDG.E.256, new on
// sm_100: a whole padded row = one sector = ONE L1 tag lookup per lane instead of three),
// otherwise scalar 8-byte loads.
template <int R, int S, bool READONLY>
__device__ __forceinline__ void load_row(const double* Y, int64_t ldy, int64_t row,
                                         double (&out)[R]) {
  if constexpr (S == 0) {  // planar: column k of the block is Y + k*ldy
#pragma unroll
    for (int k = 0; k < R; ++k) out[k] = READONLY ? __ldg(Y + k * ldy + row) : Y[k * ldy + row];
    return;
  }
  const double* p = Y + row * S;
  if constexpr (S == 4) {
    double a, b, c, d;
    if constexpr (READONLY)
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
    else
      asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p) : "memory");
    out[0] = a;
    if constexpr (R > 1) out[1] = b;
    if constexpr (R > 2) out[2] = c;
    if constexpr (R > 3) out[3] = d;
  } else if constexpr (S == 2 && R == 2) {
    const double2* q = reinterpret_cast<const double2*>(p);
    const double2 a = READONLY ? __ldg(q) : *q;
    out[0] = a.x;
    out[1] = a.y;
  } else {
#pragma unroll
    for (int k = 0; k < R; ++k) out[k] = READONLY ? __ldg(p + k) : p[k];
  }
}

// Predicated gather of one block row: zeros when !on (no branch, so the loads of a batch
// stay independent and in flight together).
template <int R, int S>
__device__ __forceinline__ void gather_row(const double* __restrict__ Y, int64_t ldy, int64_t row,
                                           bool on, double (&out)[R]) {
  if constexpr (S == 0) {
#pragma unroll
    for (int k = 0; k < R; ++k) out[k] = on ? __ldg(Y + k * ldy + row) : 0.0;
    return;
  }
  const double* p = Y + row * S;
  if constexpr (S == 4) {
    double a, b, c, d;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %5, 0;\n\t"
        "mov.f64 %0, 0d0000000000000000;\n\tmov.f64 %1, 0d0000000000000000;\n\t"
        "mov.f64 %2, 0d0000000000000000;\n\tmov.f64 %3, 0d0000000000000000;\n\t"
        "@q ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n\t}"
        : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
        : "l"(p), "r"((int)on));
    out[0] = a;
    if constexpr (R > 1) out[1] = b;
    if constexpr (R > 2) out[2] = c;
    if constexpr (R > 3) out[3] = d;
  } else if constexpr (S == 2 && R == 2) {
    const double2 a = on ? __ldg(reinterpret_cast<const double2*>(p)) : make_double2(0.0, 0.0);
    out[0] = a.x;
    out[1] = a.y;
  } else {
#pragma unroll
    for (int k = 0; k < R; ++k) out[k] = on ? __ldg(p + k) : 0.0;
  }
}

template <int R, int S>
__device__ __forceinline__ void store_row(double* Y, int64_t ldy, int64_t row,
                                          const double (&v)[R]) {
  if constexpr (S == 0) {
#pragma unroll
    for (int k = 0; k < R; ++k) Y[k * ldy + row] = v[k];
    return;
  }
  double* p = Y + row * S;
  if constexpr (S == 4) {
    double w[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < R; ++k) w[k] = v[k];
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(w[0]), "d"(w[1]),
                 "d"(w[2]), "d"(w[3]) : "memory");
  } else if constexpr (S == 2 && R == 2) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  } else {
#pragma unroll
    for (int k = 0; k < R; ++k) p[k] = v[k];
  }
}

// Doubles the (value, mask) pairs of nuv uniform-value positions occupy in front of the
// per-lane value rows of a slice: padded to a 128-byte line when per-lane rows follow.
__host__ __device__ __forceinline__ int ug_header_doubles(int nuv, int lane_rows) {
  return lane_rows > 0 ? (2 * nuv + 15) / 16 * 16 : 2 * nuv;
}

// acc[k] += sum over positions [p0, p1) of one compressed slice for one lane (= one row).
// Position classes, in this order (see host/plan.hpp):
//   [0, nu)    uniform offset, per-lane values
//   [nu, L)    general: per-lane value and column (padding: zero value, own row as column)
// Uniform columns are row + uoff[p] (or the absolute column uoff[p] when flag bit 1 is set),
// clamped into the block because lanes that do not hold the offset carry a zero there; the
// offsets are fetched 32 at a time, one per lane, and broadcast by shuffle.
// The gathers depend only on the index stream, never on the values.  The per-lane loops are
// software pipelined: the values (and columns) of batch b+1 are requested before the gathers
// of batch b are consumed; all loads of a batch are independent.
template <int R, int S, int U>
__device__ __forceinline__ void ug_accumulate(const SellView& A, const UgSlice& H, int lane,
                                              int64_t row, int p0, int p1,
                                              const double* __restrict__ Y1, int64_t ldy,
                                              double (&acc)[R]) {
  // (slices with uniform-value pairs only occur in matrices the stencil kernel handles)
  const double* __restrict__ val = A.ug_val + H.val_ptr + lane;
  constexpr int nuv = 0;
  const int32_t* __restrict__ uoff = A.ug_uoff + H.uoff_ptr + lane;
  const int cmax = (int)A.ncols - 1;
  const int crow = (H.reserved & 2) ? 0 : (int)row;  // flag bit 1: absolute shared columns
  double v[U], vn[U];
  // ---- uniform positions with per-lane values [pu0, pu1)
  const int pu0 = max(p0, nuv), pu1 = min(p1, H.nu);
  if (pu0 < pu1) {
    int myoff = pu0 + lane < pu1 ? __ldg(uoff + pu0) : 0;
    const double* vp = val + (int64_t)pu0 * kSliceRows;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = pu0 + u < pu1 ? ld_stream_f64(vp + u * kSliceRows) : 0.0;
    for (int p = pu0; p < pu1; p += U) {
      vp += U * kSliceRows;
#pragma unroll
      for (int u = 0; u < U; ++u)
        vn[u] = p + U + u < pu1 ? ld_stream_f64(vp + u * kSliceRows) : 0.0;
      const int q = (p - pu0) & 31;
      if (q == 0 && p > pu0) myoff = p + lane < pu1 ? __ldg(uoff + p) : 0;
      double g[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = min(max(crow + __shfl_sync(0xffffffffu, myoff, q + u), 0), cmax);
        gather_row<R, S>(Y1, ldy, c, p + u < pu1, g[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = fma(v[u], g[u][k], acc[k]);
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = vn[u];
    }
  }
  // ---- general positions [q0, p1)
  const int q0 = max(p0, H.nu);
  if (q0 < p1) {
    const double* vp = val + (int64_t)q0 * kSliceRows;
    const int32_t* cp = A.ug_col + H.col_ptr + lane + (int64_t)(q0 - H.nu) * kSliceRows;
    int c[U], cn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = q0 + u < p1;
      v[u] = ok ? ld_stream_f64(vp + u * kSliceRows) : 0.0;
      c[u] = ok ? ld_stream_s32(cp + u * kSliceRows) : 0;
    }
    for (int p = q0; p < p1; p += U) {
      vp += U * kSliceRows;
      cp += U * kSliceRows;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = p + U + u < p1;
        vn[u] = ok ? ld_stream_f64(vp + u * kSliceRows) : 0.0;
        cn[u] = ok ? ld_stream_s32(cp + u * kSliceRows) : 0;
      }
      double g[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u) gather_row<R, S>(Y1, ldy, c[u], p + u < p1, g[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = fma(v[u], g[u][k], acc[k]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = vn[u];
        c[u] = cn[u];
      }
    }
  }
}

__device__ __forceinline__ UgSlice load_ug_header(const UgSlice* __restrict__ h) {
  const int4 a = __ldg(reinterpret_cast<const int4*>(h));
  const int4 b = __ldg(reinterpret_cast<const int4*>(h) + 1);
  UgSlice H{};
  H.val_ptr = (int64_t)(((uint64_t)(uint32_t)a.y << 32) | (uint32_t)a.x);
  H.col_ptr = (int64_t)(((uint64_t)(uint32_t)a.w << 32) | (uint32_t)a.z);
  H.uoff_ptr = b.x;
  H.nu = b.y;
  H.ng = b.z;
  H.reserved = b.w;
  return H;
}

// ---------------------------------------------------------------- exact / simple kernel
template <int R, int MODE, bool EXACT>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    clenshaw_step_sell(SellView A, double s1, double s2, double b,
                       const double* __restrict__ Y1, double* __restrict__ Y2,
                       const double* __restrict__ X, int64_t ldx, double* __restrict__ Out,
                       int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t widx = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (widx >= A.nslices) return;
  const int64_t slice = A.slice_ids ? (int64_t)A.slice_ids[widx] : widx;
  const int64_t sell_lane = slice * kSliceRows + lane;
  // hybrid matrices group the rows of a SELL slice by length without permuting the vectors
  const int64_t row = A.sell_rows ? (int64_t)A.sell_rows[sell_lane] : sell_lane;
  const int len = A.row_len[sell_lane];
  const int L = A.slice_len[slice];
  const int64_t base = A.slice_ptr[slice] + lane;
  const double* __restrict__ val = A.val + base;
  const int* __restrict__ col = A.col + base;

  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  int p = 0;
  for (; p < L; ++p) {
    const double v = ld_stream_f64(val + (int64_t)p * kSliceRows);
    const int c = ld_stream_s32(col + (int64_t)p * kSliceRows);
    if (p < len) {
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] = mul_add<EXACT>(v, Y1[(int64_t)c * R + k], acc[k]);
    }
  }
  if (row < 0 || row >= A.nl) return;
  if constexpr (MODE == 2) {  // plain: Out = A*Y1
#pragma unroll
    for (int k = 0; k < R; ++k) Out[(int64_t)k * ldo + row] = acc[k];
  } else {
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const double y1 = Y1[row * R + k];
      const double y2 = Y2[row * R + k];
      const double x = X[(int64_t)k * ldx + row];
      const double o = combine<EXACT>(s1, acc[k], s2, y1, y2, b, x);
      if constexpr (MODE == 0)
        Y2[row * R + k] = o;
      else
        Out[(int64_t)k * ldo + row] = o;
    }
  }
}

// ----------------------------------------------------------------------- fast kernels
// Epilogue shared by the fast kernels: own-row operands were requested before the matrix
// stream so that they are in flight together with it.
template <int R, int S, int MODE>
__device__ __forceinline__ void load_own(const SellView& A, int64_t row, const double* Y1,
                                         const double* Y2, int64_t ldy,
                                         const double* __restrict__ X,
                                         int64_t ldx, double (&y1o)[R], double (&y2o)[R],
                                         double (&xo)[R]) {
#pragma unroll
  for (int k = 0; k < R; ++k) y1o[k] = y2o[k] = xo[k] = 0.0;
  if constexpr (MODE != 2 && MODE != 3) {
    if (row < A.nl) {
      load_row<R, S, true>(Y1, ldy, row, y1o);
      load_row<R, S, false>(Y2, ldy, row, y2o);
#pragma unroll
      for (int k = 0; k < R; ++k) xo[k] = __ldg(X + (int64_t)k * ldx + row);
    }
  }
}

template <int R, int S, int MODE>
__device__ __forceinline__ void finish_row(int64_t row, double s1, double s2, double b,
                                           const double (&acc)[R], const double (&y1o)[R],
                                           const double (&y2o)[R], const double (&xo)[R],
                                           double* Y2, int64_t ldy, double* __restrict__ Out,
                                           int64_t ldo) {
  if constexpr (MODE == 2) {
#pragma unroll
    for (int k = 0; k < R; ++k) Out[(int64_t)k * ldo + row] = acc[k];
  } else {
    double o[R];
#pragma unroll
    for (int k = 0; k < R; ++k) o[k] = combine<false>(s1, acc[k], s2, y1o[k], y2o[k], b, xo[k]);
    if constexpr (MODE == 0) {
      store_row<R, S>(Y2, ldy, row, o);
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) Out[(int64_t)k * ldo + row] = o[k];
    }
  }
}

// L2 prefetch of the own-row operands of the epilogue (streamed once: Y2 row, X entries);
// the loads themselves are issued after the accumulation so that they hold no registers
// while the gathers are in flight.
template <int R, int S, int MODE>
__device__ __forceinline__ void prefetch_own(const SellView& A, int64_t row, const double* Y2,
                                             int64_t ldy, const double* X, int64_t ldx) {
  if constexpr (MODE != 2 && MODE != 3) {
    if (row < A.nl) {
      if constexpr (S == 0) {
#pragma unroll
        for (int k = 0; k < R; ++k)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(Y2 + k * ldy + row));
      } else {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(Y2 + row * S));
        if constexpr (S == 3) asm volatile("prefetch.global.L2 [%0];" ::"l"(Y2 + row * S + 2));
      }
#pragma unroll
      for (int k = 0; k < R; ++k)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(X + (int64_t)k * ldx + row));
    }
  }
}

// SPLIT mode: partial sums the rest launch left for this row (kMaxFuse doubles per row)
template <int R>
__device__ __forceinline__ void add_rest(const SellView& A, int64_t row, double (&acc)[R]) {
  if (row < A.nl) {
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] += A.W[row * kMaxFuse + k];
  }
}

// Short slices (stencils): one warp per slice; a CTA walks a contiguous range of slices so
// that the block rows gathered by one slice are still in L1 for its neighbours.  The slice
// descriptor (header + the first kUgInline uniform offsets) is one coalesced 64-byte load;
// values and gathers of a batch are then all independent, so a slice costs two dependent
// memory round trips (descriptor, then everything else).
//   Every slice has at most kUgInline uniform positions and a few general ones (stencils);
//   the code then needs no offset lists and no software pipeline, which keeps the
//   register count at 64 (eight CTAs per SM) — occupancy is what hides the latency of
//   seven-position slices (measured, 100^3 Laplacian, 3 columns: 24 warps/SM 37 us, 28 warps
//   29 us, 32 warps 27.7 us per step).
#ifndef FLZ_K1_LEAN_CTAS
#define FLZ_K1_LEAN_CTAS 8
#endif
#ifndef FLZ_K1_EARLY_OWN
#define FLZ_K1_LATE_OWN 1  // own-row operands: L2 prefetch up front, loads after the gathers
#endif
template <int R, int S, int MODE, int U>
__global__ void __launch_bounds__(kWarpsPerBlock * 32,
                                  R == 1 ? 12 : (R <= 3 ? FLZ_K1_LEAN_CTAS : 1))  // R = 1 fits 40 registers
    clenshaw_step_ug_warp(SellView A, int slices_per_cta, double s1, double s2, double b,
                          const double* __restrict__ Y1, double* __restrict__ Y2, int64_t ldy,
                          const double* __restrict__ X, int64_t ldx, double* __restrict__ Out,
                          int64_t ldo) {
  static_assert(sizeof(UgSlice) == 64, "descriptor is 16 words");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t first = (int64_t)blockIdx.x * slices_per_cta;
  const int64_t last = min(A.nslices, first + slices_per_cta);
  const int cmax = (int)A.ncols - 1;
  pdl_launch_dependents();
  for (int64_t w = first + warp; w < last; w += kWarpsPerBlock) {
    const int64_t slice = A.slice_ids ? (int64_t)A.slice_ids[w] : w;
    const int word = __ldg(reinterpret_cast<const int*>(A.ug + slice) + (lane & 15));
    // (value, mask) pairs of the uniform-value positions: fixed stride, no descriptor needed
    const double pair = ld_stream_f64(A.uv_pairs + slice * 16 + (lane & 15));
    const int64_t row = slice * kSliceRows + lane;
    double acc[R], y1o[R], y2o[R], xo[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    if (w == first + warp) pdl_wait();  // matrix words above are requested before the wait
#ifdef FLZ_K1_LATE_OWN
    prefetch_own<R, S, MODE>(A, row, Y2, ldy, X, ldx);
#else
    load_own<R, S, MODE>(A, row, Y1, Y2, ldy, X, ldx, y1o, y2o, xo);
#endif
    const int64_t val_ptr = (int64_t)(((uint64_t)(uint32_t)__shfl_sync(0xffffffffu, word, 1) << 32) |
                                      (uint32_t)__shfl_sync(0xffffffffu, word, 0));
    const int nu = __shfl_sync(0xffffffffu, word, 5);
    const int ng = __shfl_sync(0xffffffffu, word, 6);
    const int nuv = (__shfl_sync(0xffffffffu, word, 7) >> 16) & 0xff;
    const double* __restrict__ vbase = A.ug_val + val_ptr;
    // ---- uniform-value positions: batches of 4, 2, 1 — no predicated loads, no zero fills
    {
      const int maskword = __double2loint(pair);  // lanes 2i+1 hold the lane mask of position i
      auto uv_batch = [&](auto count, int p) {
        constexpr int N = decltype(count)::value;
        double g[N][R];
#pragma unroll
        for (int u = 0; u < N; ++u) {  // the gathers need the descriptor only
          const int d = __shfl_sync(0xffffffffu, word, 8 + p + u);
          gather_row<R, S>(Y1, ldy, min(max((int)row + d, 0), cmax), true, g[u]);
        }

#pragma unroll
        for (int u = 0; u < N; ++u) {
          const double value = __shfl_sync(0xffffffffu, pair, 2 * (p + u));
          const int mask = __shfl_sync(0xffffffffu, maskword, 2 * (p + u) + 1);
          const double v = ((mask >> lane) & 1) ? value : 0.0;
#pragma unroll
          for (int k = 0; k < R; ++k) acc[k] = fma(v, g[u][k], acc[k]);
        }
      };
      int p = 0;
      if (p + 4 <= nuv) { uv_batch(std::integral_constant<int, 4>{}, p); p += 4; }
      if (p + 4 <= nuv) { uv_batch(std::integral_constant<int, 4>{}, p); p += 4; }
      if (p + 2 <= nuv) { uv_batch(std::integral_constant<int, 2>{}, p); p += 2; }
      if (p < nuv) uv_batch(std::integral_constant<int, 1>{}, p);
    }
    // ---- uniform positions with per-lane values
    const double* __restrict__ val = vbase + ug_header_doubles(nuv, nu + ng - nuv) + lane;
    for (int p = nuv; p < nu; p += U) {
      double v[U], g[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = p + u < nu;
        v[u] = ok ? ld_stream_f64(val + (int64_t)(p + u - nuv) * kSliceRows) : 0.0;
        const int d = __shfl_sync(0xffffffffu, word, 8 + ((p + u) & (kUgInline - 1)));
        gather_row<R, S>(Y1, ldy, min(max((int)row + d, 0), cmax), ok, g[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = fma(v[u], g[u][k], acc[k]);
    }
    // ---- the few general positions of a stencil slice
    if (ng > 0) {
      const int64_t col_ptr =
          (int64_t)(((uint64_t)(uint32_t)__shfl_sync(0xffffffffu, word, 3) << 32) |
                    (uint32_t)__shfl_sync(0xffffffffu, word, 2));
      const int32_t* __restrict__ col = A.ug_col + col_ptr + lane;
      for (int q = 0; q < ng; q += 4) {
        double v[4], g[4][R];
        int c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = q + u < ng;
          v[u] = ok ? ld_stream_f64(val + (int64_t)(nu - nuv + q + u) * kSliceRows) : 0.0;
          c[u] = ok ? ld_stream_s32(col + (int64_t)(q + u) * kSliceRows) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) gather_row<R, S>(Y1, ldy, c[u], q + u < ng, g[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < R; ++k) acc[k] = fma(v[u], g[u][k], acc[k]);
      }
    }
    if (__shfl_sync(0xffffffffu, word, 7) & 1) add_rest<R>(A, row, acc);
#ifdef FLZ_K1_LATE_OWN
    load_own<R, S, MODE>(A, row, Y1, Y2, ldy, X, ldx, y1o, y2o, xo);
#endif
    if (row < A.nl) finish_row<R, S, MODE>(row, s1, s2, b, acc, y1o, y2o, xo, Y2, ldy, Out, ldo);
  }
}

// Long slices: CTAs of 8 warps walk a contiguous range of a host-built task list; a task
// gives each of its slices 1, 2, 4 or 8 warps, whose partial sums meet in shared memory in
// a fixed order (deterministic).
template <int R, int S, int MODE>
#ifndef FLZ_K1_TASK_CTAS
#define FLZ_K1_TASK_CTAS 3
#endif
__global__ void __launch_bounds__(kTaskWarps * 32, FLZ_K1_TASK_CTAS)
    clenshaw_step_ug_tasks(SellView A, int tasks_per_cta, double s1, double s2, double b,
                           const double* __restrict__ Y1, double* __restrict__ Y2, int64_t ldy,
                           const double* __restrict__ X, int64_t ldx, double* __restrict__ Out,
                           int64_t ldo) {
  __shared__ double part[kTaskWarps][R][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * tasks_per_cta;
  const int64_t t1 = min(A.ntasks, t0 + tasks_per_cta);
  pdl_launch_dependents();
  pdl_wait();
  for (int64_t t = t0; t < t1; ++t) {
    const SliceTask task = A.tasks[t];
    const int W = task.warps_per_slice;
    const int sub = warp / W, piece = warp - sub * W;
    const bool active = sub < task.count;
    double acc[R], y1o[R], y2o[R], xo[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = y1o[k] = y2o[k] = xo[k] = 0.0;
    int64_t row = 0;
    bool has_rest = false;
    if (active) {
      const int64_t slice = task.slice[sub];
      const UgSlice H = load_ug_header(A.ug + slice);
      if constexpr (MODE == 3) {  // rest slice: lanes map to rows through rest_rows
        const int r = A.rest_rows[(slice - A.rest_base) * kSliceRows + lane];
        row = r < 0 ? A.nl : r;
      } else {
        row = slice * kSliceRows + lane;
        has_rest = H.reserved & 1;
      }
      if (piece == 0) load_own<R, S, MODE>(A, row, Y1, Y2, ldy, X, ldx, y1o, y2o, xo);
      const int L = H.nu + H.ng;
      const int chunk = (((L + W - 1) / W) + kBatch - 1) / kBatch * kBatch;
      const int p0 = piece * chunk, p1 = min(L, p0 + chunk);
      if (p0 < p1) ug_accumulate<R, S, kBatch>(A, H, lane, row, p0, p1, Y1, ldy, acc);
    }
    if (W > 1) {  // uniform across the CTA
      if (active && piece > 0) {
#pragma unroll
        for (int k = 0; k < R; ++k) part[warp][k][lane] = acc[k];
      }
      __syncthreads();
      if (active && piece == 0) {
        for (int q = 1; q < W; ++q)
#pragma unroll
          for (int k = 0; k < R; ++k) acc[k] += part[warp + q][k][lane];
      }
      if (t + 1 < t1) __syncthreads();  // `part` is reused by the next task
    }
    if (active && piece == 0 && row < A.nl) {
      if constexpr (MODE == 3) {
#pragma unroll
        for (int k = 0; k < R; ++k) A.W[row * kMaxFuse + k] = acc[k];
      } else {
        if (has_rest) add_rest<R>(A, row, acc);
        finish_row<R, S, MODE>(row, s1, s2, b, acc, y1o, y2o, xo, Y2, ldy, Out, ldo);
      }
    }
  }
}

// Paired layout (host/plan.hpp): slices of up to 64 rows, lane l owns the adjacent rows
// row0 + 2l and + 1.  GENERAL positions: one column per lane and two values; one gathered block
// row feeds two rows of the product.  DENSE positions (rows of one dense block, host/plan.hpp):
// the column is shared by the whole slice, so a warp gathers the block rows of 32 dense
// columns at once (one 32-byte gather per LANE instead of per lane and position), parks them
// in its own shared-memory strip and every position then costs a broadcast shared load plus
// the coalesced 512-byte value stream — about a third of the LSU wavefronts of a general
// position.  Task list and multi-warp split as in clenshaw_step_ug_tasks: the W warps of a
// slice share its general AND its dense positions evenly.
template <int R, int S, int MODE>
__global__ void __launch_bounds__(kTaskWarps * 32, FLZ_K1_TASK_CTAS)
    clenshaw_step_p2_tasks(SellView A, double s1, double s2, double b,
                           const double* __restrict__ Y1, double* __restrict__ Y2, int64_t ldy,
                           const double* __restrict__ X, int64_t ldx, double* __restrict__ Out,
                           int64_t ldo) {
  // Persistent CTAs take tasks from a ticket counter (tasks are sorted longest first): an SM
  // that was dealt long tasks simply takes fewer of them.  With one CTA per task the SMs were
  // active 41k-83k cycles of a 90k-cycle launch (ncu, PARSEC-shaped n = 113k).
  // One 1.5 KB strip per warp: the gathered rows of 32 dense columns ([32][4]) while the dense
  // section runs, then the warp's partial sums ([2R][32]).  Shared memory is kept small on
  // purpose: what the CTAs do not claim stays L1 for the gathered block rows.
  __shared__ __align__(16) double scratch[kTaskWarps][2 * kMaxFuse * 32];
  __shared__ int next_task;
  auto part = [&](int w, int k) -> double* { return scratch[w] + k * 32; };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_launch_dependents();
  if (threadIdx.x == 0) next_task = (int)atomicAdd(A.tickets, 1u);
  __syncthreads();
  int t = next_task;
  if (t >= A.ntasks) return;
  pdl_wait();
  for (;;) {
    const int2 head = __ldg(reinterpret_cast<const int2*>(A.tasks + t));
    const int W = head.x;   // warps per slice; head.y slices in this task
    const int sub = warp / W, piece = warp - sub * W;
    const bool active = sub < head.y;
    double acc[2][R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[0][k] = acc[1][k] = 0.0;
    int64_t row = 0;
    int row_end = 0;
    if (active) {
      const int4* hp = reinterpret_cast<const int4*>(A.p2_desc + __ldg(&A.tasks[t].slice[sub]));
      const int4 h0 = __ldg(hp), h1 = __ldg(hp + 1);
      const int64_t gpos = ((int64_t)(uint32_t)h0.y << 32) | (uint32_t)h0.x;
      const int64_t dpos = ((int64_t)(uint32_t)h0.w << 32) | (uint32_t)h0.z;
      const int ng = h1.x, nd = h1.y;
      row = (int64_t)h1.z + 2 * lane;
      row_end = h1.z + h1.w;
      const int chunk = (((ng + W - 1) / W) + kBatch - 1) / kBatch * kBatch;
      const int p0 = piece * chunk, p1 = min(ng, p0 + chunk);
      const int dchunk = (((nd + W - 1) / W) + 31) / 32 * 32;
      const int d0 = min(nd, piece * dchunk), d1 = min(nd, d0 + dchunk);
      const int32_t* __restrict__ col = A.p2_col + (gpos + p0) * 32 + lane;
      const double* __restrict__ val = A.p2_val + ((gpos + p0) * 32 + lane) * 2;
      const int32_t* __restrict__ dcol = A.p2_dcol + dpos;
      const double* __restrict__ dval = A.p2_dval + (dpos * 32 + lane) * 2;
      // general positions, kBatch per round.  The columns of round i+1 are requested before
      // the gathers of round i are consumed, so a round exposes ONE memory round trip (the
      // gathers, with the values beside them), not two (columns, then gathers).
      int c[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) c[u] = p0 + u < p1 ? ld_stream_s32(col + u * 32) : 0;
      // first dense round: its column and gather do not depend on the general part
      int dc = (d0 < d1 && lane < d1 - d0) ? ld_stream_s32(dcol + d0 + lane) : -1;
      for (int p = p0; p < p1; p += kBatch) {
        double va[kBatch], vb[kBatch], g[kBatch][R];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) gather_row<R, S>(Y1, ldy, c[u], p + u < p1, g[u]);
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          va[u] = vb[u] = 0.0;
          if (p + u < p1)
            asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                         : "=d"(va[u]), "=d"(vb[u]) : "l"(val + u * 64));
        }
        col += kBatch * 32;
        val += kBatch * 64;
#pragma unroll
        for (int u = 0; u < kBatch; ++u)
          c[u] = p + kBatch + u < p1 ? ld_stream_s32(col + u * 32) : 0;
#pragma unroll
        for (int u = 0; u < kBatch; ++u)
#pragma unroll
          for (int k = 0; k < R; ++k) {
            acc[0][k] = fma(va[u], g[u][k], acc[0][k]);
            acc[1][k] = fma(vb[u], g[u][k], acc[1][k]);
          }
      }
      // dense section: 32 columns per round; the next round's column and gathered row are
      // requested before this round's positions are consumed
      double (*mine)[4] = reinterpret_cast<double (*)[4]>(scratch[warp]);
      double g[R];
      gather_row<R, S>(Y1, ldy, max(dc, 0), dc >= 0, g);
      for (int q = d0; q < d1; q += 32) {
        const int cnt = min(32, d1 - q);
        const double* __restrict__ v = dval + (int64_t)q * 64;
        double va[4], vb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          va[u] = vb[u] = 0.0;
          if (u < cnt)
            asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                         : "=d"(va[u]), "=d"(vb[u]) : "l"(v + u * 64));
        }
        __syncwarp();                      // the previous round's reads of the strip are done
#pragma unroll
        for (int k = 0; k < R; ++k) mine[lane][k] = g[k];
        __syncwarp();
        dc = (q + 32 < d1 && lane < d1 - q - 32) ? ld_stream_s32(dcol + q + 32 + lane) : -1;
        bool gathered = false;
        for (int j = 0; j < cnt; j += 4) {
          double na[4], nb[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {    // next batch in flight while this one is consumed
            na[u] = nb[u] = 0.0;
            if (j + 4 + u < cnt)
              asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                           : "=d"(na[u]), "=d"(nb[u]) : "l"(v + (j + 4 + u) * 64));
          }
          if (!gathered && j >= 4) {       // the next round's column has had a batch to arrive
            gather_row<R, S>(Y1, ldy, max(dc, 0), dc >= 0, g);
            gathered = true;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int jj = min(j + u, 31);  // past cnt: zero values times a staged (finite) row
#pragma unroll
            for (int k = 0; k < R; ++k) {
              const double y = mine[jj][k];
              acc[0][k] = fma(va[u], y, acc[0][k]);
              acc[1][k] = fma(vb[u], y, acc[1][k]);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            va[u] = na[u];
            vb[u] = nb[u];
          }
        }
        if (!gathered) gather_row<R, S>(Y1, ldy, max(dc, 0), dc >= 0, g);
      }
    }
    if (W > 1) {  // uniform across the CTA
      if (active && piece > 0) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
          part(warp, k)[lane] = acc[0][k];
          part(warp, R + k)[lane] = acc[1][k];
        }
      }
    }
    if (threadIdx.x == 0) next_task = (int)atomicAdd(A.tickets, 1u);
    __syncthreads();
    t = next_task;
    if (active && piece == 0) {
      for (int q = 1; q < W; ++q)
#pragma unroll
        for (int k = 0; k < R; ++k) {
          acc[0][k] += part(warp + q, k)[lane];
          acc[1][k] += part(warp + q, R + k)[lane];
        }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = row + h;
        if (r >= row_end) break;
        double y1o[R], y2o[R], xo[R];
        load_own<R, S, MODE>(A, r, Y1, Y2, ldy, X, ldx, y1o, y2o, xo);
        finish_row<R, S, MODE>(r, s1, s2, b, acc[h], y1o, y2o, xo, Y2, ldy, Out, ldo);
      }
    }
    if (t >= A.ntasks) break;
    __syncthreads();   // `part` and next_task are reused by the next task
  }
}

// ---- mbarrier / bulk-copy (TMA) primitives
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// the same with an L2 eviction-priority policy (createpolicy) for the lines the copy touches
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes,
                                              uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(policy) : "memory");
}

// ------------------------------------------------------------ TMA-staged stencil kernel
// Constant-coefficient stencils on one GPU, planar blocks (host/plan.hpp, PlanStencilTiles).
// A persistent CTA walks tiles of T = tile_rows consecutive rows (tile t, t + grid, ...).
// Everything a tile touches is CONTIGUOUS in global memory — per block column the runs of Y1
// its offsets reach (offsets closer than a tile share one run), its own rows of Y2 and X,
// and its slices' (value, mask) pairs — so the tile is requested with a handful of
// cp.async.bulk copies into a ring of shared-memory stages (full/empty mbarriers,
// complete_tx), `nstages` tiles ahead of the consumers.
//   * T consumer threads (one row each, T/32 warps = the tile's slices) need no global load at
//     all: a position costs one broadcast 16-byte shared load (value, lane mask, staged byte
//     offset) and R conflict-free 8-byte shared loads — no shuffles, no address clamps, no
//     dependent global round trips; only the results go back to global memory.
//   * nprod producer warps: lane l of producer warp w owns copy l*nprod + w of every tile.
//     A warp issues its bulk copies one after the other (UBLKCP takes uniform operands, the
//     compiler loops over the lanes; ~150 cycles per copy on B200), so ONE producer warp
//     cannot feed the ring (measured: 34 us per step with one, 16.4 us with four).
// Memory-level parallelism comes from the ring (stages x CTAs per SM x ~36 KB in flight), not
// from occupancy and registers as in clenshaw_step_ug_warp.  Runs that leave [0, rows) are
// clipped and the producers zero-fill the clipped part (the lanes that would read it carry a
// zero mask bit, but 0 * stale bits must stay finite).  Positions are added in the order of
// clenshaw_step_ug_warp: results are bit-identical (tests/test_gpu_variants.py).
// The positions of a stencil slice that are not uniform-value pairs (rows next to a domain
// boundary: per-lane values at uniform offsets, then general positions), gathered from global
// memory in the order clenshaw_step_ug_warp adds them.  Rare: a few slices per matrix.
template <int R>
struct SliceAcc {
  double v[R];
};
template <int R>
__device__ __noinline__ SliceAcc<R> stencil_slice_rest(const SellView& A, int64_t slice, int lane,
                                                       int64_t row, const double* __restrict__ Y1,
                                                       int64_t ldy, SliceAcc<R> acc) {
  const UgSlice H = load_ug_header(A.ug + slice);
  const int* __restrict__ desc = reinterpret_cast<const int*>(A.ug + slice);
  const int nuv = (H.reserved >> 16) & 0xff;
  const int cmax = (int)A.ncols - 1;
  const double* __restrict__ val =
      A.ug_val + H.val_ptr + ug_header_doubles(nuv, H.nu + H.ng - nuv) + lane;
  for (int p = nuv; p < H.nu; ++p) {
    const double v = ld_stream_f64(val + (int64_t)(p - nuv) * kSliceRows);
    const int c = min(max((int)row + __ldg(desc + 8 + p), 0), cmax);
#pragma unroll
    for (int k = 0; k < R; ++k) acc.v[k] = fma(v, __ldg(Y1 + (int64_t)k * ldy + c), acc.v[k]);
  }
  const int32_t* __restrict__ col = A.ug_col + H.col_ptr + lane;
  for (int q = 0; q < H.ng; ++q) {
    const double v = ld_stream_f64(val + (int64_t)(H.nu - nuv + q) * kSliceRows);
    const int c = ld_stream_s32(col + (int64_t)q * kSliceRows);
#pragma unroll
    for (int k = 0; k < R; ++k) acc.v[k] = fma(v, __ldg(Y1 + (int64_t)k * ldy + c), acc.v[k]);
  }
  return acc;
}

// SLAB (row slabs, the tiles that stage halo rows): a run covers rows [-front, y_rows - front)
// of the VIRTUAL source column [front halo | local | back halo]; rows [-front, 0) are stored at
// base + nl + (g + front), rows [0, nl) at base + g, rows [nl, ...) at base + front + g — up
// to three bulk copies per run — and the launch walks the tiles outside [hole_lo, hole_lo +
// hole_len).  !SLAB: tiles [tile_lo, tile_lo + ntiles), one copy per run (the single-rank
// kernel; on row slabs the tiles whose runs stay inside the local rows).
template <int R, int MODE, bool SLAB>
__global__ void __launch_bounds__(768)
    clenshaw_step_stencil_tma(const __grid_constant__ SellView A,
                              const __grid_constant__ StencilTiles G,
                              const double* __restrict__ pairs, int64_t nl,
                              int64_t ntiles, int64_t tile_lo, int64_t hole_lo, int64_t hole_len,
                              int nstages, int nprod, int l2hint, int64_t y_rows,
                              int64_t x_rows,
                              double s1, double s2, double b, const double* __restrict__ Y1,
                              double* __restrict__ Y2, int64_t ldy, const double* __restrict__ X,
                              int64_t ldx, double* __restrict__ Out, int64_t ldo) {
  extern __shared__ __align__(128) unsigned char st_smem[];
  constexpr bool kOwn = MODE != 2;
  // consumer threads = rows of a tile; the last nprod warps produce (a warp issues its bulk
  // copies one after the other, ~150 cycles each on B200: one producer warp cannot keep up)
  const int T = (int)blockDim.x - 32 * nprod;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int spt = T >> 5;
  const int pair_d = spt * 16;
  const int y1e = G.y1_elems;
  const int y1_d = R * y1e;
  const int stage_d = pair_d + y1_d + (kOwn ? 2 * R * T : 0);  // doubles per stage
  double* const ring = reinterpret_cast<double*>(st_smem);
  const uint32_t ring_s = smem_addr(ring);
  const uint32_t full_bars = ring_s + (uint32_t)nstages * stage_d * 8;  // tile has landed
  const uint32_t empty_bars = full_bars + (uint32_t)nstages * 8;        // all warps consumed it
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    for (int st = 0; st < nstages; ++st) {
      mbar_init(full_bars + st * 8, nprod);
      mbar_init(empty_bars + st * 8, spt);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // Y1/Y2 belong to the previous step until here

  if (warp >= spt) {
    // ---------------------------------------------------------------- producer warps
    // Lane l of producer warp pw owns copy c = l*nprod + pw of EVERY tile (the launcher makes
    // 32*nprod >= copies per tile): what does not depend on the tile is set up once.
    const int pw = warp - spt;
    const int c = lane * nprod + pw;
    const int ncopy = 1 + G.nseg * R + (kOwn ? 2 * R : 0);
    int dst = 0, full = 0, off = 0;   // staged element, run length, first row relative to the tile
    int64_t lim = 0;                  // readable rows of the source column
    const double* base = nullptr;
    bool y1run = false;               // SLAB: a run of the gather source (halo pieces)
    const int64_t front = SLAB ? G.front : 0;
    // L2 policy: X and the matrix pairs are read again by every later step of the filter and
    // never written (evict_last); the Y blocks take the default priority
    bool keep = false;
    uint64_t pol_keep = 0;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    if (c == 0) {
      keep = true;
      full = pair_d;
    } else if (c < 1 + G.nseg * R) {
      const int q = c - 1, j = q / R, k = q - j * R;
      dst = pair_d + k * y1e + G.seg_start[j];
      full = G.seg_len[j];
      off = G.seg_base[j];
      lim = y_rows;
      base = Y1 + (int64_t)k * ldy;
      y1run = true;
    } else if (c < ncopy) {
      const int q = c - 1 - G.nseg * R, which = q / R, k = q - which * R;
      dst = pair_d + y1_d + q * T;
      full = T;
      lim = which ? x_rows : y_rows;
      base = which ? X + (int64_t)k * ldx : Y2 + (int64_t)k * ldy;
      keep = which != 0;
    }
    keep = keep && l2hint;
    int st = 0;
    uint32_t parity = 1;  // first pass over the ring: the stages are empty (wait falls through)
    for (int64_t u = blockIdx.x; u < ntiles; u += gridDim.x) {
      int64_t t = tile_lo + u;
      if constexpr (SLAB) {
        if (t >= hole_lo) t += hole_len;
      }
      mbar_wait(empty_bars + st * 8, parity);
      double* sb = ring + (int64_t)st * stage_d;
      const uint32_t bar = full_bars + st * 8;
      int lead = 0, count = full;
      const double* src = pairs + t * pair_d;
      int64_t g0 = 0;
      if (base) {
        g0 = t * T + off;
        const int64_t lo = (SLAB && y1run) ? -front : 0, hi = (SLAB && y1run) ? lim - front : lim;
        const int64_t a0 = max(g0, lo), a1 = min(g0 + full, hi);
        lead = (int)min(a0 - g0, (int64_t)full);
        count = (int)max(a1 - a0, (int64_t)0);
        src = base + a0;
      }
      // clipped runs (first and last tiles): all lanes zero the part no copy fills
      unsigned clipped = __ballot_sync(0xffffffffu, count < full);
      while (clipped) {
        const int l = __ffs(clipped) - 1;
        clipped &= clipped - 1;
        const int zd = __shfl_sync(0xffffffffu, dst, l), zf = __shfl_sync(0xffffffffu, full, l);
        const int zl = __shfl_sync(0xffffffffu, lead, l), zc = __shfl_sync(0xffffffffu, count, l);
        for (int i = lane; i < zl; i += 32) sb[zd + i] = 0.0;
        for (int i = zl + zc + lane; i < zf; i += 32) sb[zd + i] = 0.0;
      }
      const uint32_t bytes = (uint32_t)count * 8u;
      const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
      __syncwarp();  // orders every lane's zero fills before lane 0's release below
      // release: the zero fills above are visible to whoever sees the phase flip
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(total) : "memory");
      __syncwarp();
      if (SLAB && y1run && front > 0) {
        // the stored pieces of the run: local rows, halo rows in front, halo rows behind
        const uint32_t to = ring_s + (uint32_t)(st * stage_d + dst) * 8u;
        const int64_t g1 = g0 + full;
        const int64_t b0 = max(g0, (int64_t)0), b1 = min(g1, nl);
        if (b1 > b0) bulk_g2s(to + (uint32_t)(b0 - g0) * 8u, base + b0, (uint32_t)(b1 - b0) * 8u, bar);
        const int64_t f0 = max(g0, -front), f1 = min(g1, (int64_t)0);
        if (f1 > f0)
          bulk_g2s(to + (uint32_t)(f0 - g0) * 8u, base + nl + front + f0, (uint32_t)(f1 - f0) * 8u, bar);
        const int64_t c0 = max(g0, nl), c1 = min(g1, lim - front);
        if (c1 > c0)
          bulk_g2s(to + (uint32_t)(c0 - g0) * 8u, base + front + c0, (uint32_t)(c1 - c0) * 8u, bar);
      } else if (count > 0) {
        const uint32_t to = ring_s + (uint32_t)(st * stage_d + dst + lead) * 8u;
        if (keep) bulk_g2s_hint(to, src, bytes, bar, pol_keep);
        else bulk_g2s(to, src, bytes, bar);
      }
      if (++st == nstages) { st = 0; parity ^= 1u; }
    }
    return;
  }

  // ------------------------------------------------------------------ consumer warps
  int st = 0;
  uint32_t parity = 0;
  const uint32_t y1e8 = (uint32_t)y1e * 8u;
  const uint32_t lanebit = 1u << lane;
  const uint32_t own8 = (uint32_t)G.own_e * 8u;
  int64_t row = (((int64_t)blockIdx.x + tile_lo) * spt + warp) * 32 + lane;
  const int64_t row_step = (int64_t)gridDim.x * T;
  double* dst = (MODE == 0 ? Y2 : Out) + row;
  const int64_t ldd = MODE == 0 ? ldy : ldo;
  for (int64_t u = blockIdx.x; u < ntiles; u += gridDim.x, row += row_step, dst += row_step) {
    int64_t t = tile_lo + u;
    if constexpr (SLAB) {   // the tiles behind the hole
      if (t >= hole_lo) {
        t += hole_len;
        row = (t * spt + warp) * 32 + lane;
        dst = (MODE == 0 ? Y2 : Out) + row;
      }
    }
    mbar_wait(full_bars + st * 8, parity);
    const double* sb = ring + (int64_t)st * stage_d;
    const double2* sP = reinterpret_cast<const double2*>(sb + warp * 16);
    const unsigned char* sY1 = reinterpret_cast<const unsigned char*>(sb + pair_d + threadIdx.x);
    double acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    double2 pr[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) pr[p] = sP[p];  // unused positions: value 0, mask 0, element 0
    const uint32_t word0 = (uint32_t)__double2hiint(pr[0].y);
    const int nuv = (word0 >> 20) & 0xf;
    auto position = [&](int p) {
      const uint32_t e8 = (uint32_t)__double2hiint(pr[p].y) & 0xfffffu;  // staged BYTE offset
      const double v = ((uint32_t)__double2loint(pr[p].y) & lanebit) ? pr[p].x : 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k)
        acc[k] = fma(v, *reinterpret_cast<const double*>(sY1 + k * y1e8 + e8), acc[k]);
    };
    position(0); position(1); position(2); position(3);
    if (nuv > 4) { position(4); position(5); }
    if (nuv > 6) { position(6); position(7); }
    if ((word0 >> 24) & 1) {  // rare: the slice also has per-lane positions
      SliceAcc<R> tmp;
#pragma unroll
      for (int k = 0; k < R; ++k) tmp.v[k] = acc[k];
      tmp = stencil_slice_rest<R>(A, t * spt + warp, lane, row, Y1, ldy, tmp);
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] = tmp.v[k];
    }
    double o[R];
    if constexpr (MODE == 2) {
#pragma unroll
      for (int k = 0; k < R; ++k) o[k] = acc[k];
    } else {
      const double* sY2 = sb + pair_d + y1_d + threadIdx.x;
      const double* sX = sY2 + R * T;
#pragma unroll
      for (int k = 0; k < R; ++k)
        o[k] = combine<false>(s1, acc[k], s2,
                              *reinterpret_cast<const double*>(sY1 + k * y1e8 + own8), sY2[k * T],
                              b, sX[k * T]);
    }
    __syncwarp();
    if (lane == 0)  // this warp is done with the stage
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(empty_bars + st * 8)
                   : "memory");
    if (row < nl) {
#pragma unroll
      for (int k = 0; k < R; ++k) dst[(int64_t)k * ldd] = o[k];
      if constexpr (SLAB && MODE == 0) {
        // fused halo pack: the rows the peers gather from go to the send buffer as well
        if (A.send_slots) {
          const int2 sl = __ldg(A.send_slots + (row < hole_lo * T ? row : row - hole_len * T));
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if (sl.x >= 0) A.send_buf[(int64_t)k * A.n_send + sl.x] = o[k];
            if (sl.y >= 0) A.send_buf[(int64_t)k * A.n_send + sl.y] = o[k];
          }
        }
      }
    }
    if (++st == nstages) { st = 0; parity ^= 1u; }
  }
}


// ------------------------------------------------ several Clenshaw steps per launch (stencils)
// Temporal blocking for stencils with a short reach (2-D grids: reach = one grid line).  A CTA
// owns `core` consecutive rows and loads the window [r0 - K*reach, r0 + core + K*reach) of Y1,
// Y2 and X into shared memory; step s of the launch updates the rows that are still s*reach
// inside the window (their neighbours were updated by step s-1 in this CTA), so after K steps
// the core rows hold the state a sequence of K one-step launches would have produced — the halo
// rows are recomputed by the neighbouring CTAs.  The recurrence state after K steps is two
// blocks (y_K, y_{K-1}); they go to O1 / O2 (not in place: other CTAs still read the old
// state of these rows as their halo).  Positions are added in the order of
// clenshaw_step_stencil_tma (same masked values, same fma chain, same combine): bit-identical
// to K launches of it.  One launch replaces K dependent launches where a step is launch-bound
// (200 x 200 grid: 2.9 us per launch) and divides the DRAM traffic of a step by ~K where it
// is bandwidth-bound.
struct StepCoeffs {
  double b[8];
};
__device__ __forceinline__ void ms_cp_async8(double* dst_smem, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  const int bytes = valid ? 8 : 0;   // 0: the destination is zero filled
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
template <int R>
__global__ void __launch_bounds__(1024)
    clenshaw_multistep_stencil(const __grid_constant__ StencilTiles G,
                               const double* __restrict__ pairs, int64_t nl, int64_t npair_slices,
                               int core, int reach, int K, const __grid_constant__ StepCoeffs cf,
                               double s1, double s2, const double* __restrict__ Y1,
                               const double* __restrict__ Y2, int64_t ldy,
                               const double* __restrict__ X, int64_t ldx, double* __restrict__ O1,
                               double* __restrict__ O2) {
  extern __shared__ __align__(16) unsigned char ms_smem[];
  const int W = core + 2 * K * reach;            // window rows (multiple of 32)
  const int nq = W >> 5;                         // slices of the window
  double* ybuf = reinterpret_cast<double*>(ms_smem);          // [3][R][W]
  double* xs = ybuf + 3 * R * W;                              // [R][W]
  // per slice and position: (value, lane mask | row offset << 32) — one 16-byte broadcast load
  double2* prs = reinterpret_cast<double2*>(xs + R * W);      // [nq][8]
  int* pnuv = reinterpret_cast<int*>(prs + nq * 8);           // [nq]
  const int64_t w0 = (int64_t)blockIdx.x * core - (int64_t)K * reach;   // first row of the window
  pdl_launch_dependents();
  // the slices' (value, mask, offset) triples: immutable, read before the dependency wait
  for (int e = threadIdx.x; e < nq * 8; e += blockDim.x) {
    const int q = e >> 3, p = e & 7;
    const int64_t sl = (w0 >> 5) + q;
    double v = 0.0;
    unsigned mask = 0;
    int off = 0, nuv = 0;
    if (sl >= 0 && sl < npair_slices) {
      const double2 pr = __ldg(reinterpret_cast<const double2*>(pairs + sl * 16) + p);
      const unsigned hi = (unsigned)__double2hiint(pr.y);
      const int elem = (int)((hi & 0xfffffu) >> 3);          // staged element of the tile kernel
      v = pr.x;
      mask = (unsigned)__double2loint(pr.y);
      nuv = (int)((hi >> 20) & 0xf);
      off = G.seg_base[0] + elem;                            // ... back to a row offset
      for (int j = 1; j < G.nseg; ++j)
        if (elem >= G.seg_start[j]) off = G.seg_base[j] + (elem - G.seg_start[j]);
    }
    prs[e] = make_double2(v, __hiloint2double(off, (int)mask));
    if (p == 0) pnuv[q] = nuv;
  }
  pdl_wait();
  // the window: 8-byte cp.async (zero fill outside the matrix) — every element of the window
  // is in flight at once, no registers staged
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    const int64_t row = w0 + i;
    const bool in = row >= 0 && row < nl;
    const int64_t at = in ? row : 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      ms_cp_async8(ybuf + (0 * R + k) * W + i, Y2 + (int64_t)k * ldy + at, in);   // y_{j+1}
      ms_cp_async8(ybuf + (1 * R + k) * W + i, Y1 + (int64_t)k * ldy + at, in);   // y_j
      ms_cp_async8(xs + k * W + i, X + (int64_t)k * ldx + at, in);
      ybuf[(2 * R + k) * W + i] = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  int prev = 0, cur = 1, next = 2;
  for (int s = 1; s <= K; ++s) {
    const double b = cf.b[s - 1];
    const double* yc = ybuf + cur * R * W;
    const double* yp = ybuf + prev * R * W;
    double* yn = ybuf + next * R * W;
    for (int i = s * reach + threadIdx.x; i < W - s * reach; i += blockDim.x) {
      const int64_t row = w0 + i;
      if (row < 0 || row >= nl) {
#pragma unroll
        for (int k = 0; k < R; ++k) yn[k * W + i] = 0.0;
        continue;
      }
      const int q = i >> 5;
      const unsigned lanebit = 1u << (i & 31);
      const int nuv = pnuv[q];
      double acc[R];
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] = 0.0;
      auto position = [&](int p) {
        const double2 pr = prs[q * 8 + p];
        const double v = ((unsigned)__double2loint(pr.y) & lanebit) ? pr.x : 0.0;
        const int at = i + __double2hiint(pr.y);
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = fma(v, yc[k * W + at], acc[k]);
      };
      position(0); position(1); position(2); position(3);
      if (nuv > 4) { position(4); position(5); }
      if (nuv > 6) { position(6); position(7); }
#pragma unroll
      for (int k = 0; k < R; ++k)
        yn[k * W + i] = combine<false>(s1, acc[k], s2, yc[k * W + i], yp[k * W + i], b, xs[k * W + i]);
    }
    __syncthreads();
    const int t = prev;
    prev = cur;
    cur = next;
    next = t;
  }
  for (int i = K * reach + threadIdx.x; i < K * reach + core; i += blockDim.x) {
    const int64_t row = w0 + i;
    if (row >= nl) break;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      O1[(int64_t)k * ldy + row] = ybuf[(cur * R + k) * W + i];
      O2[(int64_t)k * ldy + row] = ybuf[(prev * R + k) * W + i];
    }
  }
}

template <int R, int S>
__global__ void interleave_kernel(int64_t nl, double scale, const double* __restrict__ X,
                                  int64_t ldx, double* __restrict__ Y1, int64_t ldy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nl) return;
  double v[R];
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = __dmul_rn(scale, X[(int64_t)k * ldx + i]);
  store_row<R, S>(Y1, ldy, i, v);
}

template <int S>
__global__ void pack_rows_kernel(int64_t count, const int32_t* __restrict__ rows,
                                 const double* __restrict__ Y1, double* __restrict__ buf) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  const int64_t r = rows[s];
#pragma unroll
  for (int k = 0; k < S; ++k) buf[s * S + k] = Y1[r * S + k];
}

// planar blocks: buf[k*count + s] = Y1[k*ldy + rows[s]]
__global__ void pack_rows_planar_kernel(int64_t count, int R, const int32_t* __restrict__ rows,
                                        const double* __restrict__ Y1, int64_t ldy,
                                        double* __restrict__ buf) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  const int64_t r = rows[s];
  for (int k = 0; k < R; ++k) buf[(int64_t)k * count + s] = Y1[(int64_t)k * ldy + r];
}

template <bool EXACT>
__global__ void combine_kernel(int64_t n, double s1, double s2, double b,
                               const double* __restrict__ w, const double* __restrict__ y1,
                               const double* y2, const double* __restrict__ x, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = combine<EXACT>(s1, w[i], s2, y1[i], y2[i], b, x[i]);
}

// --------------------------------------------------------------------- hybrid layout
// (host/plan.hpp) Matrices that are a stencil plus dense blocks, natural row order, PLANAR
// blocks.  Two launches per product, chained by programmatic dependent launch; everything a
// CTA reads before its grid-dependency wait is immutable matrix data (the value stream of a
// dense task, the first column words of a slice), so it overlaps the previous launch's tail.
__device__ __forceinline__ int4 ld_stream_s32x4(const int* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

constexpr int kHyDenseWarps = 4;
#ifndef FLZ_HY_DU
#define FLZ_HY_DU 4
#endif
#ifndef FLZ_HY_SLICE_CTAS
#define FLZ_HY_SLICE_CTAS 8
#endif
#ifndef FLZ_HY_OVERLAP_DEFAULT
#define FLZ_HY_OVERLAP_DEFAULT -1
#endif

// Dense task: 4 warps share the columns of the block; the block rows of ALL its columns are
// staged in shared memory once (ys[ncols][4]), a lane owns one row of the task and streams its
// values ([column][lane], 256 coalesced bytes per column).  Partial sums meet in shared memory
// in a fixed order; warp 0 stores the task's 32 partials.
template <int R>
__global__ void __launch_bounds__(kHyDenseWarps * 32)
    hybrid_dense_tasks(HyView A, const double* __restrict__ Y1, int64_t ldy) {
  extern __shared__ __align__(16) double hy_smem[];
  double (*ys)[4] = reinterpret_cast<double (*)[4]>(hy_smem);
  double (*part)[R][32] = reinterpret_cast<double (*)[R][32]>(hy_smem + 4 * A.maxcols);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_launch_dependents();
  const int4* tp = reinterpret_cast<const int4*>(A.dtasks + blockIdx.x);
  const int4 t0 = __ldg(tp), t1 = __ldg(tp + 1);
  const int64_t val_off = ((int64_t)(uint32_t)t0.y << 32) | (uint32_t)t0.x;
  const int col_off = t0.z, ncols = t0.w, slot_base = t1.x;
  const int chunk = (ncols + kHyDenseWarps - 1) / kHyDenseWarps;
  const int j0 = min(ncols, warp * chunk), j1 = min(ncols, j0 + chunk);
  const double* __restrict__ v = A.dval + val_off * 32 + lane;
  constexpr int U = FLZ_HY_DU;
  double a[U], nx[U];
  auto fetch = [&](double (&dst)[U], int j) {
#pragma unroll
    for (int u = 0; u < U; ++u) dst[u] = j + u < j1 ? ld_stream_f64(v + (int64_t)(j + u) * 32) : 0.0;
  };
  fetch(a, j0);
  fetch(nx, j0 + U);
  {  // the rest of this warp's value chunk: into L2 while the previous launch drains
    const char* base = reinterpret_cast<const char*>(v - lane + (int64_t)(j0 + 2 * U) * 32);
    const int lines = max(0, j1 - j0 - 2 * U) * 2;
    for (int l = lane; l < lines; l += 32) prefetch_l2(base + (size_t)l * 128);
  }
  pdl_wait();
  for (int j = threadIdx.x; j < ncols; j += kHyDenseWarps * 32) {
    const int c = __ldg(A.dcols + col_off + j);
#pragma unroll
    for (int k = 0; k < R; ++k) ys[j][k] = __ldg(Y1 + (int64_t)k * ldy + c);
  }
  __syncthreads();
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  for (int j = j0; j < j1; j += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int jj = min(j + u, ncols - 1);   // past j1: zero value times a staged (finite) row
      if constexpr (R >= 2) {
        const double2 y01 = *reinterpret_cast<const double2*>(&ys[jj][0]);
        acc[0] = fma(a[u], y01.x, acc[0]);
        acc[1] = fma(a[u], y01.y, acc[1]);
        if constexpr (R >= 3) {
          const double2 y23 = *reinterpret_cast<const double2*>(&ys[jj][2]);
          acc[2] = fma(a[u], y23.x, acc[2]);
          if constexpr (R == 4) acc[3] = fma(a[u], y23.y, acc[3]);
        }
      } else {
        acc[0] = fma(a[u], ys[jj][0], acc[0]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = nx[u];
    fetch(nx, j + 2 * U);
  }
  if (warp > 0) {
#pragma unroll
    for (int k = 0; k < R; ++k) part[warp - 1][k][lane] = acc[k];
  }
  __syncthreads();
  if (warp == 0) {
    for (int q = 0; q < kHyDenseWarps - 1; ++q)
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] += part[q][k][lane];
#pragma unroll
    for (int k = 0; k < R; ++k) A.P[(int64_t)k * A.ldp + slot_base + lane] = acc[k];
  }
}

// Slices: one warp per 32 consecutive rows.  MODE 0 step (planar Y2 in place), 1 final (Out,
// column-major ldo), 2 plain (Out = A Y1).
// CTAS = resident CTAs per SM the register budget is cut for: 8 (64 registers) or 6 (80).
template <int R, int MODE, int CTAS>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, CTAS)
    hybrid_slices(HyView A, double s1, double s2, double b, const double* __restrict__ Y1,
                  double* __restrict__ Y2, int64_t ldy, const double* __restrict__ X, int64_t ldx,
                  double* __restrict__ Out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t slice = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  pdl_launch_dependents();
  if (slice >= A.nslices) {
    pdl_wait();
    return;
  }
  const int4* hp = reinterpret_cast<const int4*>(A.slice + slice);
  const int4 h0 = __ldg(hp), h1 = __ldg(hp + 1);
  const int64_t col_off = ((int64_t)(uint32_t)h0.y << 32) | (uint32_t)h0.x;
  const int uv_off = h0.z, g_off = h0.w, nuv = h1.x, ng = h1.y, np = h1.z;
  const int zero_row = A.zero_row;
  const int64_t row = slice * kSliceRows + lane;
  const int* __restrict__ col = A.cols + col_off * 32 + lane * 4;
  const double2* __restrict__ uv = reinterpret_cast<const double2*>(A.uvval + uv_off);
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  int4 c = nuv > 0 ? ld_stream_s32x4(col) : make_int4(zero_row, zero_row, zero_row, zero_row);
  {  // this slice's remaining column words and position values: into L2 ahead of their use
    const char* base = reinterpret_cast<const char*>(A.cols + col_off * 32);
    const int lines = nuv + ng + np;   // 128 bytes per position
    for (int l = lane + 4; l < lines; l += 32) prefetch_l2(base + (size_t)l * 128);
    if (lane * 16 < nuv) prefetch_l2(reinterpret_cast<const char*>(uv) + lane * 128);
  }
  pdl_wait();
  // uniform-value positions, 4 per round; the columns of round i+1 are requested before the
  // gathers of round i are consumed
  for (int p = 0; p < nuv; p += 4) {
    double g[4][R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      g[0][k] = __ldg(Y1 + (int64_t)k * ldy + c.x);
      g[1][k] = __ldg(Y1 + (int64_t)k * ldy + c.y);
      g[2][k] = __ldg(Y1 + (int64_t)k * ldy + c.z);
      g[3][k] = __ldg(Y1 + (int64_t)k * ldy + c.w);
    }
    const double2 v01 = __ldg(uv + (p >> 1)), v23 = __ldg(uv + (p >> 1) + 1);
    col += 128;
    if (p + 4 < nuv) c = ld_stream_s32x4(col);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      acc[k] = fma(v01.x, g[0][k], acc[k]);
      acc[k] = fma(v01.y, g[1][k], acc[k]);
      acc[k] = fma(v23.x, g[2][k], acc[k]);
      acc[k] = fma(v23.y, g[3][k], acc[k]);
    }
  }
  const int* __restrict__ gcol = A.cols + (col_off + nuv) * 32 + lane;
  // general positions: per-lane value and column
  if (ng > 0) {
    const double* __restrict__ gv = A.gval + (int64_t)g_off * 32 + lane;
    for (int p = 0; p < ng; p += 4) {
      int cc[4];
      double v[4], g[4][R];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cc[u] = p + u < ng ? ld_stream_s32(gcol + (p + u) * 32) : zero_row;
        v[u] = p + u < ng ? ld_stream_f64(gv + (int64_t)(p + u) * 32) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) g[u][k] = __ldg(Y1 + (int64_t)k * ldy + cc[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = fma(v[u], g[u][k], acc[k]);
    }
    gcol += ng * 32;
  }
  // partial positions: what the dense tasks of this product left for the row
  for (int p = 0; p < np; ++p) {
    const int sl = ld_stream_s32(gcol + p * 32);
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] += A.P[(int64_t)k * A.ldp + sl];
  }
  if (row >= A.nl) return;
  const double d = ld_stream_f64(A.diag + row);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const double y1 = __ldg(Y1 + (int64_t)k * ldy + row);
    const double w = fma(d, y1, acc[k]);
    if constexpr (MODE == 2) {
      Out[(int64_t)k * ldo + row] = w;
    } else {
      const double y2 = Y2[(int64_t)k * ldy + row];
      const double x = ld_stream_f64(X + (int64_t)k * ldx + row);
      const double o = combine<false>(s1, w, s2, y1, y2, b, x);
      if constexpr (MODE == 0)
        Y2[(int64_t)k * ldy + row] = o;
      else
        Out[(int64_t)k * ldo + row] = o;
    }
  }
}

// ---- overlapped variant: ONE launch holds the dense tasks and the slices' gather work, CTA
// roles interleaved by blockIdx (Bresenham: of every nd + ns consecutive CTAs, nd are dense
// tasks), so that every SM runs DRAM-bound dense CTAs next to LSU-bound slice CTAs.  No CTA
// waits for another: the slices leave their sums in W, and a second, small launch adds the
// partial sums of the dense tasks and applies the Clenshaw combine (same order of additions as
// hybrid_slices: bit-identical results).
template <int R, int CTAS>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, CTAS)
    hybrid_gather(HyView A, const double* __restrict__ Y1, int64_t ldy) {
  extern __shared__ __align__(16) double hy_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t total = gridDim.x, nd = A.ndtasks, bid = blockIdx.x;
  const int64_t d0 = bid * nd / total, d1 = (bid + 1) * nd / total;
  pdl_launch_dependents();
  if (d1 > d0) {   // ---- dense task d0 (as hybrid_dense_tasks)
    double (*ys)[4] = reinterpret_cast<double (*)[4]>(hy_smem);
    double (*part)[R][32] = reinterpret_cast<double (*)[R][32]>(hy_smem + 4 * A.maxcols);
    const int4* tp = reinterpret_cast<const int4*>(A.dtasks + d0);
    const int4 t0 = __ldg(tp), t1 = __ldg(tp + 1);
    const int64_t val_off = ((int64_t)(uint32_t)t0.y << 32) | (uint32_t)t0.x;
    const int col_off = t0.z, ncols = t0.w, slot_base = t1.x;
    const int chunk = (ncols + kHyDenseWarps - 1) / kHyDenseWarps;
    const int j0 = min(ncols, warp * chunk), j1 = min(ncols, j0 + chunk);
    const double* __restrict__ v = A.dval + val_off * 32 + lane;
    constexpr int U = FLZ_HY_DU;
    double a[U], nx[U];
    auto fetch = [&](double (&dst)[U], int j) {
#pragma unroll
      for (int u = 0; u < U; ++u) dst[u] = j + u < j1 ? ld_stream_f64(v + (int64_t)(j + u) * 32) : 0.0;
    };
    fetch(a, j0);
    fetch(nx, j0 + U);
    {
      const char* base = reinterpret_cast<const char*>(v - lane + (int64_t)(j0 + 2 * U) * 32);
      const int lines = max(0, j1 - j0 - 2 * U) * 2;
      for (int l = lane; l < lines; l += 32) prefetch_l2(base + (size_t)l * 128);
    }
    pdl_wait();
    for (int j = threadIdx.x; j < ncols; j += kHyDenseWarps * 32) {
      const int c = __ldg(A.dcols + col_off + j);
#pragma unroll
      for (int k = 0; k < R; ++k) ys[j][k] = __ldg(Y1 + (int64_t)k * ldy + c);
    }
    __syncthreads();
    double acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    for (int j = j0; j < j1; j += U) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int jj = min(j + u, ncols - 1);
        if constexpr (R >= 2) {
          const double2 y01 = *reinterpret_cast<const double2*>(&ys[jj][0]);
          acc[0] = fma(a[u], y01.x, acc[0]);
          acc[1] = fma(a[u], y01.y, acc[1]);
          if constexpr (R >= 3) {
            const double2 y23 = *reinterpret_cast<const double2*>(&ys[jj][2]);
            acc[2] = fma(a[u], y23.x, acc[2]);
            if constexpr (R == 4) acc[3] = fma(a[u], y23.y, acc[3]);
          }
        } else {
          acc[0] = fma(a[u], ys[jj][0], acc[0]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) a[u] = nx[u];
      fetch(nx, j + 2 * U);
    }
    if (warp > 0) {
#pragma unroll
      for (int k = 0; k < R; ++k) part[warp - 1][k][lane] = acc[k];
    }
    __syncthreads();
    if (warp == 0) {
      for (int q = 0; q < kHyDenseWarps - 1; ++q)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] += part[q][k][lane];
#pragma unroll
      for (int k = 0; k < R; ++k) A.P[(int64_t)k * A.ldp + slot_base + lane] = acc[k];
    }
    return;
  }
  // ---- slice CTA (bid - d0): uniform-value and general positions into W
  const int64_t slice = (bid - d0) * kWarpsPerBlock + warp;
  if (slice >= A.nslices) {
    pdl_wait();
    return;
  }
  const int4* hp = reinterpret_cast<const int4*>(A.slice + slice);
  const int4 h0 = __ldg(hp), h1 = __ldg(hp + 1);
  const int64_t col_off = ((int64_t)(uint32_t)h0.y << 32) | (uint32_t)h0.x;
  const int uv_off = h0.z, g_off = h0.w, nuv = h1.x, ng = h1.y;
  const int zero_row = A.zero_row;
  const int64_t row = slice * kSliceRows + lane;
  const int* __restrict__ col = A.cols + col_off * 32 + lane * 4;
  const double2* __restrict__ uv = reinterpret_cast<const double2*>(A.uvval + uv_off);
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  int4 c = nuv > 0 ? ld_stream_s32x4(col) : make_int4(zero_row, zero_row, zero_row, zero_row);
  {
    const char* base = reinterpret_cast<const char*>(A.cols + col_off * 32);
    const int lines = nuv + ng;
    for (int l = lane + 4; l < lines; l += 32) prefetch_l2(base + (size_t)l * 128);
    if (lane * 16 < nuv) prefetch_l2(reinterpret_cast<const char*>(uv) + lane * 128);
  }
  pdl_wait();
  for (int p = 0; p < nuv; p += 4) {
    double g[4][R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      g[0][k] = __ldg(Y1 + (int64_t)k * ldy + c.x);
      g[1][k] = __ldg(Y1 + (int64_t)k * ldy + c.y);
      g[2][k] = __ldg(Y1 + (int64_t)k * ldy + c.z);
      g[3][k] = __ldg(Y1 + (int64_t)k * ldy + c.w);
    }
    const double2 v01 = __ldg(uv + (p >> 1)), v23 = __ldg(uv + (p >> 1) + 1);
    col += 128;
    if (p + 4 < nuv) c = ld_stream_s32x4(col);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      acc[k] = fma(v01.x, g[0][k], acc[k]);
      acc[k] = fma(v01.y, g[1][k], acc[k]);
      acc[k] = fma(v23.x, g[2][k], acc[k]);
      acc[k] = fma(v23.y, g[3][k], acc[k]);
    }
  }
  if (ng > 0) {
    const int* __restrict__ gcol = A.cols + (col_off + nuv) * 32 + lane;
    const double* __restrict__ gv = A.gval + (int64_t)g_off * 32 + lane;
    for (int p = 0; p < ng; p += 4) {
      int cc[4];
      double v[4], g[4][R];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cc[u] = p + u < ng ? ld_stream_s32(gcol + (p + u) * 32) : zero_row;
        v[u] = p + u < ng ? ld_stream_f64(gv + (int64_t)(p + u) * 32) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) g[u][k] = __ldg(Y1 + (int64_t)k * ldy + cc[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = fma(v[u], g[u][k], acc[k]);
    }
  }
  if (row < A.nl) {
#pragma unroll
    for (int k = 0; k < R; ++k) A.W[(int64_t)k * ldy + row] = acc[k];
  }
}

// Second launch of the overlapped variant: W + partial sums + diagonal, then the combine.
template <int R, int MODE>
__global__ void __launch_bounds__(256)
    hybrid_finish(HyView A, double s1, double s2, double b, const double* __restrict__ Y1,
                  double* __restrict__ Y2, int64_t ldy, const double* __restrict__ X, int64_t ldx,
                  double* __restrict__ Out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t slice = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  pdl_launch_dependents();
  if (slice >= A.nslices) {
    pdl_wait();
    return;
  }
  const int4* hp = reinterpret_cast<const int4*>(A.slice + slice);
  const int4 h0 = __ldg(hp), h1 = __ldg(hp + 1);
  const int64_t col_off = ((int64_t)(uint32_t)h0.y << 32) | (uint32_t)h0.x;
  const int nuv = h1.x, ng = h1.y, np = h1.z;
  const int64_t row = slice * kSliceRows + lane;
  const int* __restrict__ pcol = A.cols + (col_off + nuv + ng) * 32 + lane;
  const bool live = row < A.nl;
  const double d = live ? ld_stream_f64(A.diag + row) : 0.0;
  double x[R];
  int sl[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) sl[p] = p < np ? ld_stream_s32(pcol + p * 32) : 0;
  if constexpr (MODE != 2) {
#pragma unroll
    for (int k = 0; k < R; ++k) x[k] = live ? ld_stream_f64(X + (int64_t)k * ldx + row) : 0.0;
  }
  pdl_wait();
  if (!live) return;
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = A.W[(int64_t)k * ldy + row];
  for (int p = 0; p < np; ++p) {
    const int s = p < 4 ? sl[p] : ld_stream_s32(pcol + p * 32);
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] += A.P[(int64_t)k * A.ldp + s];
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const double y1 = __ldg(Y1 + (int64_t)k * ldy + row);
    const double w = fma(d, y1, acc[k]);
    if constexpr (MODE == 2) {
      Out[(int64_t)k * ldo + row] = w;
    } else {
      const double y2 = Y2[(int64_t)k * ldy + row];
      const double o = combine<false>(s1, w, s2, y1, y2, b, x[k]);
      if constexpr (MODE == 0)
        Y2[(int64_t)k * ldy + row] = o;
      else
        Out[(int64_t)k * ldo + row] = o;
    }
  }
}

template <int R>
void launch_hybrid_r(flz_ctx* ctx, const HyView& A, StepMode mode, double s1, double s2, double b,
                     const double* Y1, double* Y2, int64_t ldy, const double* X, int64_t ldx,
                     double* Out, int64_t ldo, int phase) {
  if (A.nslices == 0) return;
  const size_t smem = (size_t)A.maxcols * 32 + (size_t)(kHyDenseWarps - 1) * R * 32 * 8;
  const unsigned grid = (unsigned)((A.nslices + kWarpsPerBlock - 1) / kWarpsPerBlock);
  if (phase == 0 && hybrid_overlaps(ctx, A.nslices, A.ndtasks)) {
    const unsigned total = grid + (unsigned)A.ndtasks;
    launch_k1_smem(ctx, hybrid_gather<R, 6>, total, kWarpsPerBlock * 32, smem, A, Y1, ldy);
    const unsigned fgrid = (unsigned)((A.nslices + 7) / 8);
    switch (mode) {
      case StepMode::step:
        launch_k1(ctx, hybrid_finish<R, 0>, fgrid, 256, A, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
        break;
      case StepMode::final:
        launch_k1(ctx, hybrid_finish<R, 1>, fgrid, 256, A, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
        break;
      case StepMode::plain:
        launch_k1(ctx, hybrid_finish<R, 2>, fgrid, 256, A, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
        break;
      default:
        throw ApiError(FLZ_EINVAL, "hybrid step: unsupported mode");
    }
    ctx->launches += 2;
    return;
  }
  if (A.ndtasks > 0 && phase != 2) {
    launch_k1_smem(ctx, hybrid_dense_tasks<R>, (unsigned)A.ndtasks, kHyDenseWarps * 32, smem, A, Y1, ldy);
    ctx->launches++;
  }
  if (phase == 1) return;
  // Registers against waves: 6 CTAs per SM (80 registers, no spills) when that needs no more
  // waves of CTAs than 8 per SM would (measured on B200: n = 113k, one wave either way, 24.2 ->
  // 21.4 us per step; n = 268k, 2 waves against 3, 40.2 against 42.9 us)
  const int64_t per8 = (int64_t)ctx->sm_count * 8, per6 = (int64_t)ctx->sm_count * 6;
  const bool roomy = FLZ_HY_SLICE_CTAS != 8 ? FLZ_HY_SLICE_CTAS == 6
                                            : (grid + per6 - 1) / per6 <= (grid + per8 - 1) / per8;
#define FLZ_HY_LAUNCH(MODEV)                                                                       \
  if (roomy)                                                                                       \
    launch_k1(ctx, hybrid_slices<R, MODEV, 6>, grid, kWarpsPerBlock * 32, A, s1, s2, b, Y1, Y2, ldy, \
              X, ldx, Out, ldo);                                                                   \
  else                                                                                             \
    launch_k1(ctx, hybrid_slices<R, MODEV, 8>, grid, kWarpsPerBlock * 32, A, s1, s2, b, Y1, Y2, ldy, \
              X, ldx, Out, ldo)
  switch (mode) {
    case StepMode::step: FLZ_HY_LAUNCH(0); break;
    case StepMode::final: FLZ_HY_LAUNCH(1); break;
    case StepMode::plain: FLZ_HY_LAUNCH(2); break;
    default:
      throw ApiError(FLZ_EINVAL, "hybrid step: unsupported mode");
  }
#undef FLZ_HY_LAUNCH
  ctx->launches++;
}

template <int R, int MODE>
void launch_simple(flz_ctx* ctx, const SellView& A, double s1, double s2, double b,
                   const double* Y1, double* Y2, const double* X, int64_t ldx, double* Out,
                   int64_t ldo) {
  const unsigned grid = (unsigned)((A.nslices + kWarpsPerBlock - 1) / kWarpsPerBlock);
  if (grid == 0) return;
  clenshaw_step_sell<R, MODE, true><<<grid, kWarpsPerBlock * 32, 0, ctx->stream>>>(
      A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
  ctx->launches++;
}

#ifndef FLZ_K1_UB
#define FLZ_K1_UB 4
#endif
#ifndef FLZ_K1_SLICES_PER_CTA
#define FLZ_K1_SLICES_PER_CTA 4
#endif
#ifndef FLZ_K1_TASKS_PER_CTA
#define FLZ_K1_TASKS_PER_CTA 1
#endif



// Launches the TMA-staged stencil kernel when the matrix has a tile plan and the operands
// allow 16-byte bulk copies; false: the caller falls back to the one-warp-per-slice kernel.
template <int R, int MODE>
bool launch_stencil_tma(flz_ctx* ctx, const SellView& A, double s1, double s2, double b,
                        const double* Y1, double* Y2, int64_t ldy, const double* X, int64_t ldx,
                        double* Out, int64_t ldo) {
  const StencilTiles& G = A.tiles;
  if (G.nseg == 0 || A.tile_slices == 0) return false;
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!aligned(Y1) || (ldy & 1) || ldy < A.nl) return false;
  if (MODE != 2 && (!aligned(Y2) || !aligned(X) || (ldx & 1) || ldx < A.nl)) return false;
  const int T = G.tile_rows;
  const int64_t y_rows = ldy, x_rows = ldx;   // readable rows of a block column
  const size_t stage_bytes =
      8 * ((size_t)(T / 32) * 16 + (size_t)R * G.y1_elems + (MODE != 2 ? 2 * (size_t)R * T : 0));
  static const int want_stages = std::clamp(env_int("FLZ_ST_STAGES", 3), 1, 8);
  static const int want_ctas = std::clamp(env_int("FLZ_ST_CTAS", 2), 1, 8);
  static const int want_prod = std::clamp(env_int("FLZ_ST_PRODUCERS", 4), 1, 8);
  const int ncopy = 1 + G.nseg * R + (MODE != 2 ? 2 * R : 0);
  const int nprod = std::max(want_prod, (ncopy + 31) / 32);
  static const int l2hint = env_int("FLZ_ST_L2HINT", 0);  // measured: no change (16.4 us either way)
  static const int sms = [] {
    int dev = 0, n = 0;
    FLZ_CUDA(cudaGetDevice(&dev));
    FLZ_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
  }();
  constexpr size_t kSmemPerSm = 227 * 1024, kMaxCta = 227 * 1024;
  int ctas = want_ctas, stages = want_stages;
  while (stages > 2 && (stages * (stage_bytes + 16) + 1024) * ctas > kSmemPerSm) --stages;
  while (ctas > 1 && (stages * (stage_bytes + 16) + 1024) * ctas > kSmemPerSm) --ctas;
  const size_t smem = stages * (stage_bytes + 16);
  if (smem > kMaxCta) return false;
  static const bool configured = [] {
    FLZ_CUDA(cudaFuncSetAttribute(clenshaw_step_stencil_tma<R, MODE, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxCta));
    FLZ_CUDA(cudaFuncSetAttribute(clenshaw_step_stencil_tma<R, MODE, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxCta));
    return true;
  }();
  (void)configured;
  // tile_phase 0: every tile; 1: the tiles that stage local rows only; 2: the others (row
  // slabs: the halo rows have arrived)
  const int64_t all = (A.tile_slices + T / 32 - 1) / (T / 32);
  int64_t ntiles = all, tile_lo = 0, hole_lo = all, hole_len = 0;
  if (A.tile_phase == 1) {
    tile_lo = G.tile_a;
    ntiles = G.tile_b - G.tile_a;
  } else if (A.tile_phase == 2) {
    hole_lo = G.tile_a;
    hole_len = G.tile_b - G.tile_a;
    ntiles = all - hole_len;
  }
  if (ntiles <= 0) return true;
  // row slabs: the two phases of a step are chained by programmatic dependent launch as the
  // steps of a single-rank run are (the pack kernel in between has no early trigger, the
  // event waits of the stream serialise as usual)
  static const int slab_pdl = env_int("FLZ_SLAB_PDL", 1);
  ctx->k1_pdl_once = A.tile_phase != 0 && slab_pdl != 0;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * ctas);
  // the halo-aware instantiation only where a tile can stage halo rows
  const bool slab = (G.front > 0 || G.back > 0) && A.tile_phase != 1;
  ctx->k1_packed = slab && MODE == 0 && A.send_slots != nullptr;
  if (slab)
    launch_k1_smem(ctx, clenshaw_step_stencil_tma<R, MODE, true>, grid, (unsigned)(T + 32 * nprod), smem,
                   A, G, A.uv_pairs, A.nl, ntiles, tile_lo, hole_lo, hole_len, stages, nprod, l2hint,
                   y_rows, x_rows, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
  else
    launch_k1_smem(ctx, clenshaw_step_stencil_tma<R, MODE, false>, grid, (unsigned)(T + 32 * nprod), smem,
                   A, G, A.uv_pairs, A.nl, ntiles, tile_lo, hole_lo, hole_len, stages, nprod, l2hint,
                   y_rows, x_rows, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
  return true;
}


template <int R, int S, int MODE>
void launch_ug(flz_ctx* ctx, const SellView& A, double s1, double s2, double b, const double* Y1,
               double* Y2, int64_t ldy, const double* X, int64_t ldx, double* Out, int64_t ldo) {
  // kernel choice: stencils (every slice <= 8 uniform positions) -> lean one-warp-per-slice
  // kernel; everything else -> multi-warp task kernel.  (A "sub-slice" kernel — rows x position
  // groups inside a warp, shuffle reduction, no shared memory — was measured and dropped: on
  // the PARSEC-shaped matrix it took 40.8-49.6 us per step against 34.9 us, because lanes that
  // mix positions touch more L1 lines on general positions.)
  if constexpr (MODE != 3) {
    if (A.p2) {
      if (A.ntasks == 0) return;
      const unsigned grid =
          (unsigned)std::min<int64_t>(A.ntasks, (int64_t)ctx->sm_count * FLZ_K1_TASK_CTAS);
      static const bool configured = [] {   // smallest shared-memory carve-out that fits: rest is L1
        const int pct = env_int("FLZ_K1_CARVEOUT", 25);
        FLZ_CUDA(cudaFuncSetAttribute(clenshaw_step_p2_tasks<R, S, MODE>,
                                      cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        return true;
      }();
      (void)configured;
      launch_k1(ctx, clenshaw_step_p2_tasks<R, S, MODE>, grid, kTaskWarps * 32, A, s1, s2, b, Y1,
                Y2, ldy, X, ldx, Out, ldo);
      ctx->launches++;
      return;
    }
  }
  bool lean = false;
  if constexpr (MODE != 3) lean = A.short_rows && A.lean;
  if (lean) {
    if constexpr (MODE != 3) {
      if (A.nslices == 0) return;
      if constexpr (S == 0 || (S == 1 && R == 1)) {
        if (launch_stencil_tma<R, MODE>(ctx, A, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo)) {
          ctx->launches++;
          return;
        }
      }
      const int spc = ctx->k1_slices_per_cta > 0 ? ctx->k1_slices_per_cta : FLZ_K1_SLICES_PER_CTA;
      const unsigned grid = (unsigned)((A.nslices + spc - 1) / spc);
      if ((ctx->k1_batch > 0 ? ctx->k1_batch : FLZ_K1_UB) >= 8)
        launch_k1(ctx, clenshaw_step_ug_warp<R, S, MODE, 8>, grid, kWarpsPerBlock * 32, A, spc, s1,
                  s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
      else
        launch_k1(ctx, clenshaw_step_ug_warp<R, S, MODE, 4>, grid, kWarpsPerBlock * 32, A, spc, s1,
                  s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
    }
  } else {
    if (A.ntasks == 0) return;
    const int tpc = ctx->k1_tasks_per_cta > 0 ? ctx->k1_tasks_per_cta : FLZ_K1_TASKS_PER_CTA;
    const unsigned grid = (unsigned)((A.ntasks + tpc - 1) / tpc);
    launch_k1(ctx, clenshaw_step_ug_tasks<R, S, MODE>, grid, kTaskWarps * 32, A, tpc, s1, s2, b,
              Y1, Y2, ldy, X, ldx, Out, ldo);
  }
  ctx->launches++;
}

template <int R, int S>
void launch_rs(flz_ctx* ctx, const SellView& A, StepMode mode, bool exact, double s1, double s2,
               double b, const double* Y1, double* Y2, int64_t ldy, const double* X, int64_t ldx,
               double* Out, int64_t ldo) {
  if constexpr (S != R) {
    if (exact)
      throw ApiError(FLZ_EINVAL, "clenshaw step: exact mode needs interleaved blocks, stride R");
  }
  switch (mode) {
    case StepMode::step:
      if (!exact) launch_ug<R, S, 0>(ctx, A, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
      else if constexpr (S == R) launch_simple<R, 0>(ctx, A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      break;
    case StepMode::final:
      if (!exact) launch_ug<R, S, 1>(ctx, A, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
      else if constexpr (S == R) launch_simple<R, 1>(ctx, A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      break;
    case StepMode::rest:
      if (!exact) launch_ug<R, S, 3>(ctx, A, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
      break;
    case StepMode::plain:
      if (!exact) launch_ug<R, S, 2>(ctx, A, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);
      else if constexpr (S == R) launch_simple<R, 2>(ctx, A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      break;
  }
}

}  // namespace

void launch_clenshaw_step(flz_ctx* ctx, const SellView& A, int R, int S, StepMode mode, bool exact,
                          double s1, double s2, double b, const double* Y1, double* Y2,
                          int64_t ldy, const double* X, int64_t ldx, double* Out, int64_t ldo) {
#define FLZ_K1_CASE(RR, SS)                                                                  \
  case RR * 10 + SS:                                                                         \
    launch_rs<RR, SS>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo);        \
    break;
  switch (R * 10 + S) {
    FLZ_K1_CASE(1, 1) FLZ_K1_CASE(2, 2) FLZ_K1_CASE(3, 3) FLZ_K1_CASE(3, 4) FLZ_K1_CASE(4, 4)
    FLZ_K1_CASE(1, 0) FLZ_K1_CASE(2, 0) FLZ_K1_CASE(3, 0) FLZ_K1_CASE(4, 0)
    default: throw ApiError(FLZ_EINVAL, "clenshaw step: unsupported (columns, stride) pair");
  }
#undef FLZ_K1_CASE
  FLZ_CUDA(cudaGetLastError());
}

// Overlapping pays for its second launch once a product is several waves of CTAs (measured on
// B200: n = 268k, 3.7 waves, 40.2 -> 37.3 us per step; n = 113k, 2.3 waves, 21.4 -> 22.0).
// FLZ_HY_OVERLAP=0|1 forces a variant.
bool hybrid_overlaps(const flz_ctx* ctx, int64_t nslices, int64_t ndtasks) {
  static const int forced = env_int("FLZ_HY_OVERLAP", FLZ_HY_OVERLAP_DEFAULT);
  if (ndtasks <= 0 || ctx->nranks > 1) return false;   // partitioned: the dense launch hides the halo exchange
  if (forced >= 0) return forced != 0;
  const int64_t ctas = (nslices + kWarpsPerBlock - 1) / kWarpsPerBlock + ndtasks;
  return ctas >= 3 * (int64_t)ctx->sm_count * 6;
}

void launch_hybrid_step(flz_ctx* ctx, const HyView& A, int R, StepMode mode, double s1, double s2,
                        double b, const double* Y1, double* Y2, int64_t ldy, const double* X,
                        int64_t ldx, double* Out, int64_t ldo, int phase) {
  switch (R) {
    case 1: launch_hybrid_r<1>(ctx, A, mode, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo, phase); break;
    case 2: launch_hybrid_r<2>(ctx, A, mode, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo, phase); break;
    case 3: launch_hybrid_r<3>(ctx, A, mode, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo, phase); break;
    case 4: launch_hybrid_r<4>(ctx, A, mode, s1, s2, b, Y1, Y2, ldy, X, ldx, Out, ldo, phase); break;
    default: throw ApiError(FLZ_EINVAL, "hybrid step: unsupported column count");
  }
  FLZ_CUDA(cudaGetLastError());
}

// K Clenshaw steps (StepMode::step, coefficients b[0..K)) of a short-reach stencil in one
// launch; planar blocks.  0: not applicable (the caller runs single steps); else the number
// of steps done.  Geometry: reach = the largest |offset| rounded up to 32 rows, K steps, core
// rows per CTA such that the window fits the shared memory and the grid is about one CTA per
// SM (FLZ_MS_K, FLZ_MS_CORE override).  Measured on B200, 200 x 200 grid, us per step of a
// degree-50 filter application (one launch per step: 4.07 with one column, 4.0 with three):
// K = 3, core = K * reach: 2.08 (K = 2: 2.22-2.42, K = 4: 2.14, K = 6: 3.6; core = 2 K reach:
// 2.5; K = 6 / 8 with small cores: 1.98-2.3 — the fixed cost of an application, ~1.2 us per
// step at degree 50, is in all of these); three columns: K = 3, core = 2 * reach 2.84
// (K = 2: 3.04, core = 3 * reach: 3.29).
template <int R>
int launch_multistep_r(flz_ctx* ctx, const SellView& A, int max_steps, const double* b, double s1,
                       double s2, const double* Y1, const double* Y2, int64_t ldy, const double* X,
                       int64_t ldx, double* O1, double* O2) {
  const StencilTiles& G = A.tiles;
  static const int forced_k = std::clamp(env_int("FLZ_MS_K", 0), 0, 8);
  const int want_k = forced_k > 0 ? forced_k : 3;
  static const int want_core = env_int("FLZ_MS_CORE", 0);
  if (G.nseg == 0 || want_k < 2 || max_steps < 2) return 0;
  const int lo = -G.seg_base[0];
  const int hi = G.seg_base[G.nseg - 1] + G.seg_len[G.nseg - 1] - G.tile_rows;
  const int reach = (std::max(lo, hi) + 31) / 32 * 32;
  if (reach <= 0) return 0;
  const int K = std::min(want_k, max_steps);
  constexpr size_t kMaxCta = 227 * 1024;
  auto smem_for = [&](int core) {
    const size_t W = (size_t)core + 2 * (size_t)K * reach, nq = W / 32;
    return 8 * (4 * (size_t)R * W) + 16 * (nq * 8) + 4 * nq + 64;
  };
  // as many core rows as halo rows on one side (the window is 3x the core), more when the
  // matrix has more rows than that per SM
  int core = want_core > 0 ? (want_core + 31) / 32 * 32
                           : (int)std::max<int64_t>((int64_t)(R == 1 ? K : 2) * reach,
                                                    ((A.nl + ctx->sm_count - 1) / ctx->sm_count + 31) / 32 * 32);
  while (core > 32 && smem_for(core) > kMaxCta) core -= 32;
  if (smem_for(core) > kMaxCta || (want_core <= 0 && core < 2 * reach)) return 0;   // halo would dominate
  static const bool configured = [] {
    FLZ_CUDA(cudaFuncSetAttribute(clenshaw_multistep_stencil<R>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxCta));
    return true;
  }();
  (void)configured;
  StepCoeffs cf{};
  for (int s = 0; s < K; ++s) cf.b[s] = b[s];
  const unsigned grid = (unsigned)((A.nl + core - 1) / core);
  const int64_t npair_slices = (A.tile_slices + G.tile_rows / 32 - 1) / (G.tile_rows / 32) * (G.tile_rows / 32);
  launch_k1_smem(ctx, clenshaw_multistep_stencil<R>, grid, 1024u, smem_for(core), G, A.uv_pairs, A.nl,
                 npair_slices, core, reach, K, cf, s1, s2, Y1, Y2, ldy, X, ldx, O1, O2);
  ctx->launches++;
  return K;
}

int launch_multistep(flz_ctx* ctx, const SellView& A, int R, int max_steps, const double* b,
                     double s1, double s2, const double* Y1, const double* Y2, int64_t ldy,
                     const double* X, int64_t ldx, double* O1, double* O2) {
  int done = 0;
  switch (R) {
    case 1: done = launch_multistep_r<1>(ctx, A, max_steps, b, s1, s2, Y1, Y2, ldy, X, ldx, O1, O2); break;
    case 2: done = launch_multistep_r<2>(ctx, A, max_steps, b, s1, s2, Y1, Y2, ldy, X, ldx, O1, O2); break;
    case 3: done = launch_multistep_r<3>(ctx, A, max_steps, b, s1, s2, Y1, Y2, ldy, X, ldx, O1, O2); break;
    case 4: done = launch_multistep_r<4>(ctx, A, max_steps, b, s1, s2, Y1, Y2, ldy, X, ldx, O1, O2); break;
    default: break;
  }
  if (done) FLZ_CUDA(cudaGetLastError());
  return done;
}

void launch_interleave(flz_ctx* ctx, int64_t nl, int R, int S, double scale, const double* X,
                       int64_t ldx, double* Y1, int64_t ldy) {
  if (nl == 0) return;
  const unsigned grid = (unsigned)((nl + 255) / 256);
#define FLZ_IL_CASE(RR, SS)                                                                  \
  case RR * 10 + SS:                                                                         \
    interleave_kernel<RR, SS><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1, ldy);    \
    break;
  switch (R * 10 + S) {
    FLZ_IL_CASE(1, 1) FLZ_IL_CASE(2, 2) FLZ_IL_CASE(3, 3) FLZ_IL_CASE(3, 4) FLZ_IL_CASE(4, 4)
    FLZ_IL_CASE(1, 0) FLZ_IL_CASE(2, 0) FLZ_IL_CASE(3, 0) FLZ_IL_CASE(4, 0)
    default: throw ApiError(FLZ_EINVAL, "interleave: unsupported (columns, stride) pair");
  }
#undef FLZ_IL_CASE
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_pack_rows(flz_ctx* ctx, cudaStream_t stream, int64_t count, int R, int S, int64_t ldy,
                      const int32_t* rows, const double* Y1, double* buf) {
  if (count == 0) return;
  const unsigned grid = (unsigned)((count + 255) / 256);
  switch (S) {
    case 0: {
      // planar halo rows belong to the tile kernel's steps: same shared-memory carve-out, so
      // that the SMs are not reconfigured twice per step
      static const bool configured = [] {
        if (env_int("FLZ_PACK_CARVEOUT", 1))
          FLZ_CUDA(cudaFuncSetAttribute(pack_rows_planar_kernel,
                                        cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        return true;
      }();
      (void)configured;
      pack_rows_planar_kernel<<<grid, 256, 0, stream>>>(count, R, rows, Y1, ldy, buf);
      break;
    }
    case 1: pack_rows_kernel<1><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    case 2: pack_rows_kernel<2><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    case 3: pack_rows_kernel<3><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    case 4: pack_rows_kernel<4><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    default: throw ApiError(FLZ_EINVAL, "pack: row stride must be 0..4");
  }
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_combine(flz_ctx* ctx, int64_t n, bool exact, double s1, double s2, double b,
                    const double* w, const double* y1, const double* y2, const double* x,
                    double* out) {
  if (n == 0) return;
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (exact)
    combine_kernel<true><<<grid, 256, 0, ctx->stream>>>(n, s1, s2, b, w, y1, y2, x, out);
  else
    combine_kernel<false><<<grid, 256, 0, ctx->stream>>>(n, s1, s2, b, w, y1, y2, x, out);
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

}  // namespace flz
