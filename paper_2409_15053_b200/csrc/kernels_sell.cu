// kernels_sell.cu — K1: the fused Clenshaw-step SpMM on a SELL-32-sigma matrix.
//
// Replaces, per Clenshaw step, the reference's r separate csr_matvec sweeps
// (sparse.cpp:105-111 -> kernels.cpp:25-34) plus one clenshaw_combine pass
// (kernels.cpp:36-41) as driven by ChebyshevFilter::apply (filter.cpp:146-154):
// the matrix is streamed ONCE for all R block columns and the combine is applied
// in the epilogue, so a step moves 12*nnz + 4*n(row lengths) + 32*n*R bytes.
//
// Layout: slices of 32 consecutive (permuted) rows, one warp per slice, one lane per
// row; the slice's (val, col) pairs are stored column-major so that step p of all 32
// rows is one coalesced 256 B + 128 B load.  Block vectors are row-interleaved
// (R doubles per row) so a nonzero costs one R-wide gather; for stencil-like matrices
// neighbouring lanes gather neighbouring rows, i.e. the gathers are coalesced too.
//
// exact = true reproduces the reference scalar backend bit for bit: per row the
// products are accumulated left to right in CSR order with separately rounded
// multiply and add (the scalar TU is built without FMA), and the combine is
// ((s1*w + s2*y1) - y2) + b*x.

#include "flz_internal.hpp"

namespace flz {

namespace {

constexpr int kWarpsPerBlock = 4;

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
  // main loop: four entries of every row in flight before the dependent gathers
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
        for (int k = 0; k < R; ++k) acc[k] = mul_add<EXACT>(v[u], g[u][k], acc[k]);
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

template <int R>
__global__ void interleave_kernel(int64_t nl, double scale, const double* __restrict__ X,
                                  int64_t ldx, double* __restrict__ Y1) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nl) return;
#pragma unroll
  for (int k = 0; k < R; ++k) Y1[i * R + k] = __dmul_rn(scale, X[(int64_t)k * ldx + i]);
}

template <int R>
__global__ void pack_rows_kernel(int64_t count, const int32_t* __restrict__ rows,
                                 const double* __restrict__ Y1, double* __restrict__ buf) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  const int64_t r = rows[s];
#pragma unroll
  for (int k = 0; k < R; ++k) buf[s * R + k] = Y1[r * R + k];
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
void launch_step_rm(flz_ctx* ctx, const SellView& A, bool exact, double s1, double s2, double b,
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

template <int R>
void launch_step_r(flz_ctx* ctx, const SellView& A, StepMode mode, bool exact, double s1,
                   double s2, double b, const double* Y1, double* Y2, const double* X,
                   int64_t ldx, double* Out, int64_t ldo) {
  switch (mode) {
    case StepMode::step:
      launch_step_rm<R, 0>(ctx, A, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      break;
    case StepMode::final:
      launch_step_rm<R, 1>(ctx, A, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      break;
    case StepMode::plain:
      launch_step_rm<R, 2>(ctx, A, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo);
      break;
  }
}

}  // namespace

void launch_clenshaw_step(flz_ctx* ctx, const SellView& A, int R, StepMode mode, bool exact,
                          double s1, double s2, double b, const double* Y1, double* Y2,
                          const double* X, int64_t ldx, double* Out, int64_t ldo) {
  switch (R) {
    case 1: launch_step_r<1>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo); break;
    case 2: launch_step_r<2>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo); break;
    case 3: launch_step_r<3>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo); break;
    case 4: launch_step_r<4>(ctx, A, mode, exact, s1, s2, b, Y1, Y2, X, ldx, Out, ldo); break;
    default: throw ApiError(FLZ_EINVAL, "clenshaw step: fused column count must be 1..4");
  }
  FLZ_CUDA(cudaGetLastError());
}

void launch_interleave(flz_ctx* ctx, int64_t nl, int R, double scale, const double* X,
                       int64_t ldx, double* Y1) {
  if (nl == 0) return;
  const unsigned grid = (unsigned)((nl + 255) / 256);
  switch (R) {
    case 1: interleave_kernel<1><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1); break;
    case 2: interleave_kernel<2><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1); break;
    case 3: interleave_kernel<3><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1); break;
    case 4: interleave_kernel<4><<<grid, 256, 0, ctx->stream>>>(nl, scale, X, ldx, Y1); break;
    default: throw ApiError(FLZ_EINVAL, "interleave: fused column count must be 1..4");
  }
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_pack_rows(flz_ctx* ctx, cudaStream_t stream, int64_t count, int R,
                      const int32_t* rows, const double* Y1, double* buf) {
  if (count == 0) return;
  const unsigned grid = (unsigned)((count + 255) / 256);
  switch (R) {
    case 1: pack_rows_kernel<1><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    case 2: pack_rows_kernel<2><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    case 3: pack_rows_kernel<3><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    case 4: pack_rows_kernel<4><<<grid, 256, 0, stream>>>(count, rows, Y1, buf); break;
    default: throw ApiError(FLZ_EINVAL, "pack: fused column count must be 1..4");
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
