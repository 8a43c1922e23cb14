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

#include "flz_internal.hpp"

namespace flz {

namespace {

constexpr int kWarpsPerBlock = 4;
#ifndef FLZ_K1_BATCH
#define FLZ_K1_BATCH 4
#endif
constexpr int kBatch = FLZ_K1_BATCH;  // matrix entries per row requested per pipeline stage

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
__device__ __forceinline__ void load_row(const double* Y, int64_t row, double (&out)[R]) {
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
__device__ __forceinline__ void gather_row(const double* __restrict__ Y, int64_t row, bool on,
                                           double (&out)[R]) {
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
__device__ __forceinline__ void store_row(double* Y, int64_t row, const double (&v)[R]) {
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

// acc[k] += sum_{p in [p0,p1), p < len} val[p] * Y1[col[p]*S + k] for one lane (= one row).
// Software pipelined: the (val, col) pairs of batch b+1 are requested before the gathers of
// batch b are consumed, so a row of L entries costs about 1 + ceil(L/U) memory latencies
// instead of 2*ceil(L/U); all loads of a batch are independent.
template <int R, int S, int U>
__device__ __forceinline__ void accumulate_range(const double* __restrict__ val,
                                                 const int* __restrict__ col, int len, int p0,
                                                 int p1, const double* __restrict__ Y1,
                                                 double (&acc)[R]) {
  double v[U], vn[U];
  int c[U], cn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool ok = p0 + u < p1;
    v[u] = ok ? ld_stream_f64(val + (int64_t)(p0 + u) * kSliceRows) : 0.0;
    c[u] = ok ? ld_stream_s32(col + (int64_t)(p0 + u) * kSliceRows) : 0;
  }
  for (int p = p0; p < p1; p += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {  // next batch of the matrix stream
      const bool ok = p + U + u < p1;
      vn[u] = ok ? ld_stream_f64(val + (int64_t)(p + U + u) * kSliceRows) : 0.0;
      cn[u] = ok ? ld_stream_s32(col + (int64_t)(p + U + u) * kSliceRows) : 0;
    }
    double g[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) gather_row<R, S>(Y1, c[u], p + u < len && p + u < p1, g[u]);
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
  const int64_t row = slice * kSliceRows + lane;
  const int len = A.row_len[row];
  const int L = A.slice_len[slice];
  const int64_t base = A.slice_ptr[slice] + lane;
  const double* __restrict__ val = A.val + base;
  const int* __restrict__ col = A.col + base;

  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  int p = 0;
  if constexpr (!EXACT) {
    // short-row fast path (stencils, <= 24 entries per row): four entries of every row in
    // flight before the dependent gathers; measured best for 5..7-point stencils
    for (; p + 4 <= L; p += 4) {
      double v[4];
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = ld_stream_f64(val + (int64_t)(p + u) * kSliceRows);
        c[u] = ld_stream_s32(col + (int64_t)(p + u) * kSliceRows);
      }
      double g[4][R];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) g[u][k] = (p + u < len) ? Y1[(int64_t)c[u] * R + k] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (p + u < len) {
#pragma unroll
          for (int k = 0; k < R; ++k) acc[k] = fma(v[u], g[u][k], acc[k]);
        }
    }
  }
  for (; p < L; ++p) {
    const double v = ld_stream_f64(val + (int64_t)p * kSliceRows);
    const int c = ld_stream_s32(col + (int64_t)p * kSliceRows);
    if (p < len) {
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] = mul_add<EXACT>(v, Y1[(int64_t)c * R + k], acc[k]);
    }
  }
  if (row >= A.nl) return;
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

// ------------------------------------------------------------------------ fast kernel
template <int R, int S, int MODE>
__global__ void __launch_bounds__(kTaskWarps * 32, 4)
    clenshaw_step_tasks(SellView A, double s1, double s2, double b,
                        const double* __restrict__ Y1, double* __restrict__ Y2,
                        const double* __restrict__ X, int64_t ldx, double* __restrict__ Out,
                        int64_t ldo) {
  __shared__ double part[kTaskWarps][R][32];
  const SliceTask task = A.tasks[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = task.warps_per_slice;
  const int sub = warp / W, piece = warp - sub * W;
  const bool active = sub < task.count;

  double acc[R], y1o[R], y2o[R], xo[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = y1o[k] = y2o[k] = xo[k] = 0.0;
  int64_t row = 0;
  if (active) {
    const int64_t slice = task.slice[sub];
    row = slice * kSliceRows + lane;
    if constexpr (MODE != 2) {  // own-row operands of the epilogue: requested up front
      if (piece == 0 && row < A.nl) {
        load_row<R, S, true>(Y1, row, y1o);
        load_row<R, S, false>(Y2, row, y2o);
#pragma unroll
        for (int k = 0; k < R; ++k) xo[k] = __ldg(X + (int64_t)k * ldx + row);
      }
    }
    const int len = A.row_len[row];
    const int L = A.slice_len[slice];
    const int chunk = (L + W - 1) / W;
    const int p0 = piece * chunk, p1 = min(L, p0 + chunk);
    const int64_t base = A.slice_ptr[slice] + lane;
    accumulate_range<R, S, kBatch>(A.val + base, A.col + base, len, p0, p1, Y1, acc);
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
  }
  if (!active || piece != 0 || row >= A.nl) return;
  if constexpr (MODE == 2) {
#pragma unroll
    for (int k = 0; k < R; ++k) Out[(int64_t)k * ldo + row] = acc[k];
  } else {
    double o[R];
#pragma unroll
    for (int k = 0; k < R; ++k) o[k] = combine<false>(s1, acc[k], s2, y1o[k], y2o[k], b, xo[k]);
    if constexpr (MODE == 0) {
      store_row<R, S>(Y2, row, o);
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) Out[(int64_t)k * ldo + row] = o[k];
    }
  }
}

// Y1[i*S+k] = scale * X[k*ldx+i], k < R; pad entries (R <= k < S) are zeroed
template <int R, int S>
__global__ void interleave_kernel(int64_t nl, double scale, const double* __restrict__ X,
                                  int64_t ldx, double* __restrict__ Y1) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nl) return;
  double v[R];
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = __dmul_rn(scale, X[(int64_t)k * ldx + i]);
  store_row<R, S>(Y1, i, v);
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

template <bool EXACT>
__global__ void combine_kernel(int64_t n, double s1, double s2, double b,
                               const double* __restrict__ w, const double* __restrict__ y1,
                               const double* y2, const double* __restrict__ x, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = combine<EXACT>(s1, w[i], s2, y1[i], y2[i], b, x[i]);
}

template <int R, int MODE>
void launch_simple(flz_ctx* ctx, const SellView& A, bool exact, double s1, double s2, double b,
                   const double* Y1, double* Y2, const double* X, int64_t ldx, double* Out,
                   int64_t ldo) {
  const unsigned grid = (unsigned)((A.nslices + kWarpsPerBlock - 1) / kWarpsPerBlock);
  if (grid == 0) return;
  if (exact)
    clenshaw_step_sell<R, MODE, true><<<grid, kWarpsPerBlock * 32, 0, ctx->stream>>>(
        A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
  else
    clenshaw_step_sell<R, MODE, false><<<grid, kWarpsPerBlock * 32, 0, ctx->stream>>>(
        A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
  ctx->launches++;
}

template <int R, int S, int MODE>
void launch_tasks(flz_ctx* ctx, const SellView& A, double s1, double s2, double b,
                  const double* Y1, double* Y2, const double* X, int64_t ldx, double* Out,
                  int64_t ldo) {
  if (A.ntasks == 0) return;
  clenshaw_step_tasks<R, S, MODE><<<(unsigned)A.ntasks, kTaskWarps * 32, 0, ctx->stream>>>(
      A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
  ctx->launches++;
}

template <int R, int S>
void launch_rs(flz_ctx* ctx, const SellView& A, StepMode mode, bool exact, double s1, double s2,
               double b, const double* Y1, double* Y2, const double* X, int64_t ldx, double* Out,
               int64_t ldo) {
  const bool fast = !exact && A.tasks != nullptr && !(A.short_rows && S == R);
  if (!fast && S != R)
    throw ApiError(FLZ_EINVAL, "clenshaw step: a padded row stride needs the fast path");
  switch (mode) {
    case StepMode::step:
      if (fast) launch_tasks<R, S, 0>(ctx, A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      else launch_simple<R, 0>(ctx, A, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      break;
    case StepMode::final:
      if (fast) launch_tasks<R, S, 1>(ctx, A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      else launch_simple<R, 1>(ctx, A, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      break;
    case StepMode::plain:
      if (fast) launch_tasks<R, S, 2>(ctx, A, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      else launch_simple<R, 2>(ctx, A, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      break;
  }
}

}  // namespace

void launch_clenshaw_step(flz_ctx* ctx, const SellView& A, int R, int S, StepMode mode, bool exact,
                          double s1, double s2, double b, const double* Y1, double* Y2,
                          const double* X, int64_t ldx, double* Out, int64_t ldo) {
  switch (R * 10 + S) {
    case 11: launch_rs<1, 1>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo); break;
    case 22: launch_rs<2, 2>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo); break;
    case 33: launch_rs<3, 3>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo); break;
    case 34: launch_rs<3, 4>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo); break;
    case 44: launch_rs<4, 4>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo); break;
    default: throw ApiError(FLZ_EINVAL, "clenshaw step: unsupported (columns, stride) pair");
  }
  FLZ_CUDA(cudaGetLastError());
}

void launch_interleave(flz_ctx* ctx, int64_t nl, int R, int S, double scale, const double* X,
                       int64_t ldx, double* Y1) {
  if (nl == 0) return;
  const unsigned grid = (unsigned)((nl + 255) / 256);
  switch (R * 10 + S) {
    case 11: interleave_kernel<1, 1><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1); break;
    case 22: interleave_kernel<2, 2><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1); break;
    case 33: interleave_kernel<3, 3><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1); break;
    case 34: interleave_kernel<3, 4><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1); break;
    case 44: interleave_kernel<4, 4><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1); break;
    default: throw ApiError(FLZ_EINVAL, "interleave: unsupported (columns, stride) pair");
  }
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_pack_rows(flz_ctx* ctx, cudaStream_t stream, int64_t count, int S,
                      const int32_t* rows, const double* Y1, double* buf) {
  if (count == 0) return;
  const unsigned grid = (unsigned)((count + 255) / 256);
  switch (S) {
    case 1: pack_rows_kernel<1><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    case 2: pack_rows_kernel<2><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    case 3: pack_rows_kernel<3><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    case 4: pack_rows_kernel<4><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    default: throw ApiError(FLZ_EINVAL, "pack: row stride must be 1..4");
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
