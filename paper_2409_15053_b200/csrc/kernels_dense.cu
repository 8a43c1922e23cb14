// kernels_dense.cu — K3..K9: the dense contractions of the Lanczos engine as FP64
// tensor-core (DMMA, mma.sync.m8n8k4.f64) GEMMs, plus the small vector helpers.
//
// Reference call sites replaced:
//   gemm_tn  C = A^T B  (reduction over the long dimension n):
//            cgs_pass projections  (lanczos.cpp:35-42, :177-182)      M = k*r, N = r
//            intra-block QR dots   (lanczos.cpp:205-230)              M < r,   N = 1
//            B = V^T A V           (lanczos.cpp:451-457)              M = N = w
//   gemm_nn  Out (+)= alpha A Bs  (long dimension n is the M side):
//            cgs_pass updates      (lanczos.cpp:35-42)                K = k*r, N = r
//            Ritz lift V = Q_k W   (lanczos.cpp:422-433)              K = dim, N = w
//            rotation V U, AV U    (lanczos.cpp:461-472)              K = N = w
//
// tcgen05.mma has no f64 kind, so FP64 tensor work on sm_100a is the warp-level
// mma.sync path (SASS: DMMA.8x8x4).  Both GEMMs are HBM-bound for N = r <= 4 (0.75
// flop/B); the tensor pipe just takes the multiply-add issue pressure off the FP64 ALUs.
//
// Determinism: every reduction has a fixed order (split-K partials are combined by a
// second kernel in chunk order), so repeated solves are bitwise identical, like the
// reference (kernels.hpp:9-11).

#include "flz_internal.hpp"

namespace flz {

namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// 16-byte streaming load, volatile so that the loads of a group are all issued before the
// (volatile) DMMAs that consume them — left to itself the compiler interleaves load and DMMA
// pairs to save registers, which leaves one load in flight per warp
__device__ __forceinline__ double2 ld_stream_f64x2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_cached_f64x2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// ---------------------------------------------------------------- gemm_tn
// Work item = (8-column tile of A, k-chunk): one CTA of 8 warps each.  The warps of a CTA
// interleave over the chunk's rows in groups of 64 (eight 8-row MMA steps, all loads of a
// group in flight together), so that at any moment a CTA reads 4 KB of CONTIGUOUS memory from
// each of its 8 columns: DRAM pages are
// used whole.  (The first version gave every warp its own column tile and a private row
// range: ~38k concurrent 64-byte streams, 2.2 TB/s on a 3.4M x 600 basis.)  The eight partial
// fragments meet in shared memory in warp order; chunk partials are combined by
// reduce_partials_kernel in chunk order: deterministic.
// The k-chunking adapts to M: a 3-column projection (first Lanczos steps, intra-block QR) is
// split into hundreds of chunks, a 3000-column one into a few.
// Lane (g = lane>>2, t = lane&3) loads the double2 at rows k+2t, k+2t+1 of column g: the
// .x halves of a warp form one 8x4 k-slab, the .y halves the next (the k order inside an
// MMA is free as long as A and B agree), so every load is a full 16 B per lane.
template <int NT>
__global__ void __launch_bounds__(256)
    gemm_tn_kernel(const double* __restrict__ A, int64_t lda, int64_t M,
                   const double* __restrict__ B, int64_t ldb, int N, int64_t rows8,
                   int64_t rows_per_chunk, int64_t mtiles, int64_t nitems,
                   double* __restrict__ part, int64_t Mpad, int Npad) {
  __shared__ double frag[8][NT][2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t item = blockIdx.x;
  if (item >= nitems) return;
  const int64_t chunk = item / mtiles;
  const int64_t m0 = (item - chunk * mtiles) * 8;
  const int n0 = blockIdx.y * 8 * NT;
  const int64_t k0 = chunk * rows_per_chunk;
  const int64_t k1 = min(k0 + rows_per_chunk, rows8);

  const bool a_ok = (m0 + g) < M;
  const double* ap = A + (a_ok ? (m0 + g) : 0) * lda + 2 * t;
  const double* bp[NT];
  bool b_ok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    b_ok[nt] = (n0 + 8 * nt + g) < N;
    bp[nt] = B + (int64_t)(b_ok[nt] ? (n0 + 8 * nt + g) : 0) * ldb + 2 * t;
  }
  double c[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) c[nt][0] = c[nt][1] = 0.0;

  constexpr int U = NT >= 4 ? 4 : 8;  // 8-row MMA steps per group: 16 B x 2U loads in flight
  for (int64_t kb = k0 + warp * (8 * U); kb < k1; kb += 8 * (8 * U)) {
    double2 a2[U], b2[U][NT];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // all loads of the group first
      const int64_t k = kb + 8 * u;
      const bool in = k < k1;
      a2[u] = (a_ok && in) ? ld_stream_f64x2(ap + k) : make_double2(0.0, 0.0);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        b2[u][nt] = (b_ok[nt] && in) ? ld_cached_f64x2(bp[nt] + k) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        dmma(c[nt][0], c[nt][1], a2[u].x, b2[u][nt].x);
        dmma(c[nt][0], c[nt][1], a2[u].y, b2[u][nt].y);
      }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    frag[warp][nt][0][lane] = c[nt][0];
    frag[warp][nt][1][lane] = c[nt][1];
  }
  __syncthreads();
  if (warp != 0) return;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
    for (int w = 1; w < 8; ++w) {
      c[nt][0] += frag[w][nt][0][lane];
      c[nt][1] += frag[w][nt][1][lane];
    }
  // C fragment: row g, columns 2t, 2t+1 of each 8x8 tile
  double* out = part + (chunk * Mpad + m0 + g) * Npad + n0 + 2 * t;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    out[8 * nt] = c[nt][0];
    out[8 * nt + 1] = c[nt][1];
  }
}

// C[m][n] = sum over chunks of part[chunk][m][n]: one warp per output element, lanes stride
// over the chunks, fixed shuffle tree -> the summation order never changes between runs.
__global__ void __launch_bounds__(256)
    reduce_partials_kernel(const double* __restrict__ part, int64_t nchunks, int64_t M, int N,
                           int64_t Mpad, int Npad, double* __restrict__ C, int64_t ldc) {
  const int lane = threadIdx.x & 31;
  const int64_t idx = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (idx >= M * N) return;
  const int64_t m = idx / N;
  const int n = (int)(idx - m * N);
  double s = 0.0;
  for (int64_t ch = lane; ch < nchunks; ch += 32) s += part[(ch * Mpad + m) * Npad + n];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) C[m * ldc + n] = s;
}

// ---------------------------------------------------------------- gemm_nn
// grid (ceil(rows/128), ceil(N/(8*NT))), 256 threads; warp w owns rows i0 = blockIdx.x*128
// + 16w .. +16 as two interleaved 8-row tiles (even rows / odd rows, again so that each
// lane loads a double2), and 8*NT output columns.  Bs (row-major [K][ldbs]) stays in L1/L2.
template <int NT, bool ACCUM>
__global__ void __launch_bounds__(256)
    gemm_nn_kernel(const double* __restrict__ A, int64_t lda, int64_t K,
                   const double* __restrict__ Bs, int64_t ldbs, int N, int64_t rows, double alpha,
                   double* __restrict__ Out, int64_t ldo) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t i0 = (int64_t)blockIdx.x * 128 + warp * 16;
  if (i0 >= rows) return;
  const int n0 = blockIdx.y * 8 * NT;

  double ce[NT][2], co[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) ce[nt][0] = ce[nt][1] = co[nt][0] = co[nt][1] = 0.0;

  const double* ap = A + i0 + 2 * g;     // + (j0+t)*lda
  const double* bp = Bs + n0 + g;        // + (j0+t)*ldbs + 8*nt
  const int64_t K4 = K & ~(int64_t)3;
#pragma unroll 4
  for (int64_t j0 = 0; j0 < K4; j0 += 4) {
    const double2 a2 = *reinterpret_cast<const double2*>(ap + (j0 + t) * lda);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const double b = bp[(j0 + t) * ldbs + 8 * nt];
      dmma(ce[nt][0], ce[nt][1], a2.x, b);
      dmma(co[nt][0], co[nt][1], a2.y, b);
    }
  }
  if (K4 < K) {
    const bool ok = (K4 + t) < K;
    const double2 a2 = ok ? *reinterpret_cast<const double2*>(ap + (K4 + t) * lda)
                          : make_double2(0.0, 0.0);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const double b = ok ? bp[(K4 + t) * ldbs + 8 * nt] : 0.0;
      dmma(ce[nt][0], ce[nt][1], a2.x, b);
      dmma(co[nt][0], co[nt][1], a2.y, b);
    }
  }
  // fragment (row g of the even/odd tile, columns 2t, 2t+1) -> rows i0+2g, i0+2g+1
  const int64_t i = i0 + 2 * g;
  if (i >= rows) return;
  const bool second = (i + 1) < rows;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = n0 + 8 * nt + 2 * t + e;
      if (n >= N) continue;
      double* o = Out + (int64_t)n * ldo + i;
      double v0 = alpha * ce[nt][e], v1 = alpha * co[nt][e];
      if constexpr (ACCUM) {
        const double2 old = *reinterpret_cast<const double2*>(o);
        v0 += old.x;
        v1 += old.y;
      }
      if (second)
        *reinterpret_cast<double2*>(o) = make_double2(v0, v1);
      else
        o[0] = v0;
    }
}

// ---------------------------------------------------------------- ts_update (K4, N <= 8)
// Out[i, 0..N) += alpha * sum_j A[i, j] * Bs[j][0..N): the Gram-Schmidt update of a block of
// N <= 8 columns against K basis columns, gemm_nn_kernel<1, true>'s fragment mapping (a warp
// owns 16 rows as two interleaved 8-row tiles, one k-step = 4 columns) with two changes the
// small-n shapes need:
//  * U = 8 k-steps are requested together (volatile loads, 8 x 512 B per warp in flight; the
//    compiler had interleaved loads and DMMAs of the unrolled loop);
//  * the 8 warps of a CTA are RW = 8 / KW row groups x KW column sets, so that a 40k-row basis
//    still gives several waves of CTAs (gemm_nn: 313 CTAs = 0.42 waves, 3.5 TB/s at
//    40k x 1700; 864 CTAs = 1.17 waves, 4.2 TB/s at 110k x 630 with a quarter of the time in
//    the tail).  The KW partial fragments of a row group meet in shared memory in warp order:
//    deterministic.
template <int KW>
__global__ void __launch_bounds__(256)
    ts_update_kernel(const double* __restrict__ A, int64_t lda, int64_t K,
                     const double* __restrict__ Bs, int64_t ldbs, int N, int64_t rows,
                     double alpha, double* __restrict__ Out, int64_t ldo) {
  constexpr int RW = 8 / KW, U = 8;
  __shared__ double part[KW > 1 ? KW - 1 : 1][RW][4][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int rg = warp / KW, kw = warp % KW;
  const int64_t i0 = ((int64_t)blockIdx.x * RW + rg) * 16;
  const bool live = i0 < rows;
  double ce0 = 0.0, ce1 = 0.0, co0 = 0.0, co1 = 0.0;
  const double* ap = A + (live ? i0 : 0) + 2 * g;
  const double* bp = Bs + g;
  const int64_t ngroups = (K + 3) / 4, full = K / 4;   // groups with all four columns < K
  const int64_t step_a = 4 * (int64_t)KW * lda, step_b = 4 * (int64_t)KW * ldbs;
  const double* pa = ap + (4 * (int64_t)kw + t) * lda;
  const double* pb = bp + (4 * (int64_t)kw + t) * ldbs;
  int64_t q0 = kw;
  if (live) {
    for (; q0 + (int64_t)(U - 1) * KW < full; q0 += (int64_t)KW * U) {   // whole batches: no checks
      double2 a2[U];
      double b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a2[u] = ld_stream_f64x2(pa + u * step_a);
        b[u] = __ldg(pb + u * step_b);
      }
      pa += U * step_a;
      pb += U * step_b;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        dmma(ce0, ce1, a2[u].x, b[u]);
        dmma(co0, co1, a2[u].y, b[u]);
      }
    }
  }
  for (; q0 < ngroups; q0 += KW) {   // the last, partial batch
    const int64_t j = 4 * q0 + t;
    const bool ok = live && j < K;
    const double2 a2 = ok ? ld_stream_f64x2(ap + j * lda) : make_double2(0.0, 0.0);
    const double b = ok ? __ldg(bp + j * ldbs) : 0.0;
    dmma(ce0, ce1, a2.x, b);
    dmma(co0, co1, a2.y, b);
  }
  if constexpr (KW > 1) {
    if (kw > 0) {
      part[kw - 1][rg][0][lane] = ce0;
      part[kw - 1][rg][1][lane] = ce1;
      part[kw - 1][rg][2][lane] = co0;
      part[kw - 1][rg][3][lane] = co1;
    }
    __syncthreads();
    if (kw > 0) return;
#pragma unroll
    for (int w = 0; w < KW - 1; ++w) {
      ce0 += part[w][rg][0][lane];
      ce1 += part[w][rg][1][lane];
      co0 += part[w][rg][2][lane];
      co1 += part[w][rg][3][lane];
    }
  }
  // fragment (row g of the even/odd tile, columns 2t, 2t+1) -> rows i0+2g, i0+2g+1
  const int64_t i = i0 + 2 * g;
  if (!live || i >= rows) return;
  const bool second = (i + 1) < rows;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int n = 2 * t + e;
    if (n >= N) continue;
    double* o = Out + (int64_t)n * ldo + i;
    const double2 old = *reinterpret_cast<const double2*>(o);
    const double v0 = fma(alpha, e == 0 ? ce0 : ce1, old.x);
    const double v1 = fma(alpha, e == 0 ? co0 : co1, old.y);
    if (second)
      *reinterpret_cast<double2*>(o) = make_double2(v0, v1);
    else
      o[0] = v0;
  }
}

// ---------------------------------------------------------------- block QR (one rank)
// Intra-block QR of the r twice-projected columns (lanczos.cpp:205-230) in ONE cooperative
// launch: CTA c owns a fixed range of rows; a reduction is per-CTA partials (fixed tree) ->
// scratch slot -> grid barrier -> every CTA adds the slots in the same order.  Column j:
//   [scale column j-1 +] dots against P_0..P_{j-1}   | reduce
//   first update + second-pass dots                    | reduce
//   second update + sum of squares                     | reduce
//   norm -> S_k(j,j), dead flag; the scaling is folded into the next column's first phase.
// 1 + 3 (r - 1) reductions instead of ~6 launches per column.  Columns are normalised in
// place (Z is the pending block's storage in the basis).
struct QrArgs {
  double* Z;            // r columns, leading dimension ld, normalised in place
  int64_t ld, rows;
  int r;
  const double* normsq0;  // z_j . z_j BEFORE the Gram-Schmidt sweeps at normsq0[j * stride] (op_scale)
  int64_t stride;
  double* scale;        // op_scale, in/out
  double* Sk;           // r x r row-major, written whole
  double* dead;         // r flags (0.0 / 1.0)
  double* scratch;      // [phases][gridDim.x][RQ] partial sums
  unsigned long long* barrier;
  unsigned long long base;   // arrivals before this launch
};

__device__ __forceinline__ void grid_barrier(unsigned long long* ctr, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1ULL);
    unsigned long long seen;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(ctr) : "memory");
    } while (seen < target);
  }
  __syncthreads();
}

template <int RQ>
__global__ void __launch_bounds__(256) block_qr_kernel(QrArgs a) {
  __shared__ double red[8][RQ];
  __shared__ double tot[RQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x, r = a.r;
  const int64_t per = ((a.rows + G - 1) / G + 1) & ~(int64_t)1;
  const int64_t r0 = min(a.rows, (int64_t)blockIdx.x * per), r1 = min(a.rows, r0 + per);
  int phase = 0;
  unsigned long long arrived = a.base;
  // sum `v[0..count)` over the grid; every thread of every CTA receives the totals in tot[]
  auto reduce = [&](double (&v)[RQ], int count) {
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      if (q < count) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], off);
        if (lane == 0) red[warp][q] = v[q];
      }
    }
    __syncthreads();
    double* slot = a.scratch + ((int64_t)phase * G + blockIdx.x) * RQ;
    if (threadIdx.x < count) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
      slot[threadIdx.x] = s;
    }
    arrived += (unsigned long long)G;
    grid_barrier(a.barrier, arrived);
    if (warp < count && warp < 8) {   // warp q adds slot q of every CTA: lanes stride, fixed tree
      double s = 0.0;
      for (int c = lane; c < G; c += 32) s += __ldcg(a.scratch + ((int64_t)phase * G + c) * RQ + warp);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
      if (lane == 0) tot[warp] = s;
    }
    if constexpr (RQ > 8) {
      if (warp == 0)
        for (int q = 8; q < count; ++q) {
          double s = 0.0;
          for (int c = lane; c < G; c += 32) s += __ldcg(a.scratch + ((int64_t)phase * G + c) * RQ + q);
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
          if (lane == 0) tot[q] = s;
        }
    }
    __syncthreads();
    ++phase;
  };
  // op_scale = max(op_scale, ||z_j||) over the block, before the sweeps (lanczos.cpp:169-170)
  double scale = *a.scale;
  for (int j = 0; j < r; ++j) scale = fmax(scale, sqrt(fmax(a.normsq0[j * a.stride], 0.0)));
  const double dead_tol = 1e-10 * fmax(scale, 1e-300);
  double inv_prev = 1.0;   // scaling still owed to column j - 1
  for (int j = 0; j < r; ++j) {
    double* zj = a.Z + (int64_t)j * a.ld;
    double coeff[RQ], d[RQ];
#pragma unroll
    for (int q = 0; q < RQ; ++q) coeff[q] = d[q] = 0.0;
    if (j > 0) {
      // phase A: scale column j-1 (owed), first-pass dots
      double* zp = a.Z + (int64_t)(j - 1) * a.ld;
      for (int64_t i = r0 + threadIdx.x; i < r1; i += 256) {
        const double p = zp[i] * inv_prev;
        zp[i] = p;
        const double z = zj[i];
#pragma unroll
        for (int q = 0; q < RQ; ++q)
          if (q < j) d[q] = fma(q == j - 1 ? p : a.Z[(int64_t)q * a.ld + i], z, d[q]);
      }
      reduce(d, j);
#pragma unroll
      for (int q = 0; q < RQ; ++q)
        if (q < j) coeff[q] = tot[q];
      // phase B: first update, second-pass dots
      double c1[RQ];
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        c1[q] = q < j ? tot[q] : 0.0;
        d[q] = 0.0;
      }
      for (int64_t i = r0 + threadIdx.x; i < r1; i += 256) {
        double z = zj[i];
        double pq[RQ];
#pragma unroll
        for (int q = 0; q < RQ; ++q)
          if (q < j) {
            pq[q] = a.Z[(int64_t)q * a.ld + i];
            z = fma(-c1[q], pq[q], z);
          }
        zj[i] = z;
#pragma unroll
        for (int q = 0; q < RQ; ++q)
          if (q < j) d[q] = fma(pq[q], z, d[q]);
      }
      reduce(d, j);
#pragma unroll
      for (int q = 0; q < RQ; ++q)
        if (q < j) {
          c1[q] = tot[q];
          coeff[q] += tot[q];
        }
      // phase C: second update, sum of squares
      double ss[RQ];
#pragma unroll
      for (int q = 0; q < RQ; ++q) ss[q] = 0.0;
      for (int64_t i = r0 + threadIdx.x; i < r1; i += 256) {
        double z = zj[i];
#pragma unroll
        for (int q = 0; q < RQ; ++q)
          if (q < j) z = fma(-c1[q], a.Z[(int64_t)q * a.ld + i], z);
        zj[i] = z;
        ss[0] = fma(z, z, ss[0]);
      }
      reduce(ss, 1);
    } else {
      double ss[RQ];
#pragma unroll
      for (int q = 0; q < RQ; ++q) ss[q] = 0.0;
      for (int64_t i = r0 + threadIdx.x; i < r1; i += 256) ss[0] = fma(zj[i], zj[i], ss[0]);
      reduce(ss, 1);
    }
    const double norm = sqrt(fmax(tot[0], 0.0));
    const bool alive = norm > dead_tol;
    inv_prev = alive ? 1.0 / norm : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      for (int q = 0; q < r; ++q) a.Sk[q * r + j] = q < j ? coeff[q] : 0.0;
      a.Sk[j * r + j] = alive ? norm : 0.0;
      a.dead[j] = alive ? 0.0 : 1.0;
    }
    __syncthreads();   // tot[] is rewritten by the next reduction
  }
  // the last column's scaling
  double* zl = a.Z + (int64_t)(r - 1) * a.ld;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += 256) zl[i] *= inv_prev;
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.scale = scale;
}

// ---------------------------------------------------------------- helpers
// out[c] = sum_i A[i,c]*B[i,c]: one block row-chunk per (chunk, c), fixed-order tree
__global__ void __launch_bounds__(256)
    coldot_partial_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                          int64_t ldb, int64_t rows, int64_t rows_per_chunk,
                          double* __restrict__ part, int N) {
  __shared__ double sm[256];
  const int c = blockIdx.y;
  const int64_t k0 = (int64_t)blockIdx.x * rows_per_chunk;
  const int64_t k1 = min(k0 + rows_per_chunk, rows);
  const double* a = A + (int64_t)c * lda;
  const double* b = B + (int64_t)c * ldb;
  double s = 0.0;
  for (int64_t i = k0 + threadIdx.x; i < k1; i += 256) s = fma(a[i], b[i], s);
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)blockIdx.x * N + c] = sm[0];
}

__global__ void coldot_reduce_kernel(const double* __restrict__ part, int64_t nchunks, int N,
                                     double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  double s = 0.0;
  for (int64_t ch = 0; ch < nchunks; ++ch) s += part[ch * N + c];
  out[c] = s;
}

__global__ void scale_copy_kernel(const double* __restrict__ src, const double* __restrict__ inv,
                                  double* __restrict__ dest, int64_t rows) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  dest[i] = src[i] * (*inv);
}

__global__ void scale_cols_kernel(double* __restrict__ A, int64_t lda, int64_t rows,
                                  const double* __restrict__ s) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int c = blockIdx.y;
  A[(int64_t)c * lda + i] *= s[c];
}

__global__ void residual_prep_kernel(double* __restrict__ V, double* __restrict__ AV, int64_t ld,
                                     int64_t rows, const double* __restrict__ inv,
                                     const double* __restrict__ lambda) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int c = blockIdx.y;
  const double s = inv[c];
  const double v = V[(int64_t)c * ld + i] * s;
  const double av = AV[(int64_t)c * ld + i] * s;
  V[(int64_t)c * ld + i] = v;
  AV[(int64_t)c * ld + i] = fma(-lambda[c], v, av);
}

__global__ void permute_in_kernel(const double* __restrict__ src, int64_t lds,
                                  double* __restrict__ dst, int64_t ldd, int64_t rows,
                                  const int32_t* __restrict__ perm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int c = blockIdx.y;
  dst[(int64_t)c * ldd + i] = src[(int64_t)c * lds + perm[i]];
}

__global__ void permute_out_kernel(const double* __restrict__ src, int64_t lds,
                                   double* __restrict__ dst, int64_t ldd, int64_t rows,
                                   const int32_t* __restrict__ perm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int c = blockIdx.y;
  dst[(int64_t)c * ldd + perm[i]] = src[(int64_t)c * lds + i];
}

// op_scale = max(op_scale, sqrt(gram[j][j])) (lanczos.cpp:169-170)
__global__ void update_scale_kernel(const double* gram, int r, int ldg, double* op_scale) {
  double s = *op_scale;
  for (int j = 0; j < r; ++j) s = fmax(s, sqrt(fmax(gram[j * ldg + j], 0.0)));
  *op_scale = s;
}

// norm = sqrt(normsq); live iff norm > 1e-10*max(op_scale,1e-300) (lanczos.cpp:201, :224-230)
__global__ void finish_col_kernel(const double* normsq, const double* op_scale, double* Sk, int r,
                                  int j, double* inv, double* dead_flag) {
  const double norm = sqrt(fmax(*normsq, 0.0));
  const double dead_tol = 1e-10 * fmax(*op_scale, 1e-300);
  if (norm > dead_tol) {
    Sk[j * r + j] = norm;
    *inv = 1.0 / norm;
    *dead_flag = 0.0;
  } else {
    Sk[j * r + j] = 0.0;
    *inv = 0.0;
    *dead_flag = 1.0;
  }
}

}  // namespace

// --------------------------------------------------------------- launchers

// FLZ_TS_UPDATE=0: the DMMA gemm_nn for the Gram-Schmidt updates too (experiments)
static bool ts_update_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FLZ_TS_UPDATE");
    return !(e && e[0] == '0');
  }();
  return on;
}

void launch_gemm_tn(flz_ctx* ctx, const double* A, int64_t lda, int64_t M, const double* B,
                    int64_t ldb, int N, int64_t rows, double* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return;
  const int64_t rows8 = round_up(rows, 8);
  FLZ_REQUIRE(rows8 <= lda && rows8 <= ldb, FLZ_EDIM, "gemm_tn: leading dimension too small");
  const int NT = N > 16 ? 4 : (N > 8 ? 2 : 1);
  const int64_t mtiles = (M + 7) / 8;
  const int nblocks = (N + 8 * NT - 1) / (8 * NT);
  // ~4 CTAs (32 warps) per SM over the whole grid, chunks of at least 2048 rows
  // (3 to 16 work items per SM measured the same on B200 for 40k x 1740, 110k x 630, 1M x 210)
  const int64_t want_ctas = (int64_t)ctx->sm_count * 6;
  int64_t nchunks = (want_ctas + mtiles * nblocks - 1) / (mtiles * nblocks);
  const int64_t max_chunks = (rows8 + 2047) / 2048;
  if (nchunks > max_chunks) nchunks = max_chunks;
  if (nchunks < 1) nchunks = 1;
  const int64_t rpc = round_up((rows8 + nchunks - 1) / nchunks, 512);
  nchunks = (rows8 + rpc - 1) / rpc;
  const int64_t Mpad = mtiles * 8;
  const int Npad = nblocks * 8 * NT;
  const int64_t nitems = mtiles * nchunks;
  ctx->partial.reserve((size_t)(nchunks * Mpad * Npad));
  dim3 grid((unsigned)nitems, (unsigned)nblocks);
  switch (NT) {
    case 1:
      gemm_tn_kernel<1><<<grid, 256, 0, ctx->stream>>>(A, lda, M, B, ldb, N, rows8, rpc, mtiles,
                                                       nitems, ctx->partial.p, Mpad, Npad);
      break;
    case 2:
      gemm_tn_kernel<2><<<grid, 256, 0, ctx->stream>>>(A, lda, M, B, ldb, N, rows8, rpc, mtiles,
                                                       nitems, ctx->partial.p, Mpad, Npad);
      break;
    default:
      gemm_tn_kernel<4><<<grid, 256, 0, ctx->stream>>>(A, lda, M, B, ldb, N, rows8, rpc, mtiles,
                                                       nitems, ctx->partial.p, Mpad, Npad);
      break;
  }
  const int64_t total = M * N;
  reduce_partials_kernel<<<(unsigned)((total + 7) / 8), 256, 0, ctx->stream>>>(
      ctx->partial.p, nchunks, M, N, Mpad, Npad, C, ldc);
  ctx->launches += 2;
  FLZ_CUDA(cudaGetLastError());
}

void launch_gemm_nn(flz_ctx* ctx, const double* A, int64_t lda, int64_t K, const double* Bs,
                    int64_t ldbs, int N, int64_t rows, double alpha, bool accumulate, double* Out,
                    int64_t ldo) {
  if (rows <= 0 || N <= 0) return;
  FLZ_REQUIRE(round_up(rows, 2) <= lda && round_up(rows, 2) <= ldo, FLZ_EDIM,
              "gemm_nn: leading dimension too small");
  if (accumulate && N <= 8 && K > 0 && ldbs >= 8 && ts_update_enabled()) {
    // tall-skinny update: as many column sets per CTA as it takes to have ~2 waves of CTAs
    // (4 resident CTAs per SM).  Measured on B200 (orthogonalization time of a whole
    // factorization, row groups per CTA 8 / 4 / 2 / 1): 110k rows 56.8 / 53.6 / 57.2 / 62.9 ms,
    // 40k rows 434 / 438 / 421 / 420 ms, 1M rows 52.9 / 58.3 ms, 262k rows 85.6 / 85.6 ms.
    const int64_t want = (int64_t)ctx->sm_count * 8;
    int rw = 8;
    while (rw > 1 && (rows + 16 * rw - 1) / (16 * rw) < want) rw >>= 1;
    static const int forced_rw = [] {   // experiments: FLZ_TSU_RW = 8 | 4 | 2 | 1 row groups per CTA
      const char* e = std::getenv("FLZ_TSU_RW");
      return e && *e ? std::atoi(e) : 0;
    }();
    if (forced_rw == 8 || forced_rw == 4 || forced_rw == 2 || forced_rw == 1) rw = forced_rw;
    const unsigned grid = (unsigned)((rows + 16 * rw - 1) / (16 * rw));
#define FLZ_TSU(KWV)                                                                          \
  ts_update_kernel<KWV><<<grid, 256, 0, ctx->stream>>>(A, lda, K, Bs, ldbs, N, rows, alpha, Out, ldo)
    switch (rw) {
      case 8: FLZ_TSU(1); break;
      case 4: FLZ_TSU(2); break;
      case 2: FLZ_TSU(4); break;
      default: FLZ_TSU(8); break;
    }
#undef FLZ_TSU
    ctx->launches++;
    FLZ_CUDA(cudaGetLastError());
    return;
  }
  const int NT = N > 32 ? 8 : (N > 16 ? 4 : (N > 8 ? 2 : 1));
  FLZ_REQUIRE(ldbs >= round_up(N, 8 * NT), FLZ_EDIM, "gemm_nn: Bs row stride too small");
  dim3 grid((unsigned)((rows + 127) / 128), (unsigned)((N + 8 * NT - 1) / (8 * NT)));
#define FLZ_NN(NTV)                                                                              \
  if (accumulate)                                                                                \
    gemm_nn_kernel<NTV, true><<<grid, 256, 0, ctx->stream>>>(A, lda, K, Bs, ldbs, N, rows, alpha, \
                                                             Out, ldo);                          \
  else                                                                                           \
    gemm_nn_kernel<NTV, false><<<grid, 256, 0, ctx->stream>>>(A, lda, K, Bs, ldbs, N, rows,      \
                                                              alpha, Out, ldo)
  switch (NT) {
    case 1: FLZ_NN(1); break;
    case 2: FLZ_NN(2); break;
    case 4: FLZ_NN(4); break;
    default: FLZ_NN(8); break;
  }
#undef FLZ_NN
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

// Intra-block QR in one cooperative launch (one rank).  normsq0: z_j . z_j before the sweeps at
// stride `stride`.  Sk (r x r row-major), dead (r flags) and *scale are device pointers.
void launch_block_qr(flz_ctx* ctx, double* Z, int64_t ld, int64_t rows, int r,
                     const double* normsq0, int64_t stride, double* scale, double* Sk,
                     double* dead) {
  FLZ_REQUIRE(r >= 1 && r <= 16, FLZ_EINVAL, "block_qr: block size out of range");
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->sm_count, (rows + 511) / 512));
  const int RQ = r <= 4 ? 4 : 16;
  const int phases = 1 + 3 * (r - 1);
  if (ctx->qr_scratch.count == 0) {
    ctx->qr_scratch.reserve((size_t)(1 + 3 * 15) * ctx->sm_count * 16);
    ctx->qr_barrier.reserve_zero(1, ctx->stream);
    ctx->qr_arrivals = 0;
  }
  QrArgs a{Z, ld, rows, r, normsq0, stride, scale, Sk, dead, ctx->qr_scratch.p,
           reinterpret_cast<unsigned long long*>(ctx->qr_barrier.p), ctx->qr_arrivals};
  void* args[] = {&a};
  if (RQ == 4)
    FLZ_CUDA(cudaLaunchCooperativeKernel((const void*)block_qr_kernel<4>, dim3(G), dim3(256), args,
                                         0, ctx->stream));
  else
    FLZ_CUDA(cudaLaunchCooperativeKernel((const void*)block_qr_kernel<16>, dim3(G), dim3(256),
                                         args, 0, ctx->stream));
  ctx->qr_arrivals += (unsigned long long)phases * G;
  ctx->launches++;
}

void launch_coldot(flz_ctx* ctx, const double* A, int64_t lda, const double* B, int64_t ldb, int N,
                   int64_t rows, double* out) {
  if (N <= 0) return;
  int64_t nchunks = ((int64_t)ctx->sm_count * 8 + N - 1) / N;
  const int64_t max_chunks = (rows + 2047) / 2048;
  if (nchunks > max_chunks) nchunks = max_chunks;
  if (nchunks < 1) nchunks = 1;
  const int64_t rpc = (rows + nchunks - 1) / nchunks;
  nchunks = rpc > 0 ? (rows + rpc - 1) / rpc : 1;
  if (nchunks < 1) nchunks = 1;
  ctx->partial.reserve((size_t)(nchunks * N));
  dim3 grid((unsigned)nchunks, (unsigned)N);
  coldot_partial_kernel<<<grid, 256, 0, ctx->stream>>>(A, lda, B, ldb, rows, rpc, ctx->partial.p,
                                                       N);
  coldot_reduce_kernel<<<(N + 127) / 128, 128, 0, ctx->stream>>>(ctx->partial.p, nchunks, N, out);
  ctx->launches += 2;
  FLZ_CUDA(cudaGetLastError());
}

void launch_scale_copy(flz_ctx* ctx, const double* src, const double* inv, double* dest,
                       int64_t rows) {
  if (rows <= 0) return;
  scale_copy_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, ctx->stream>>>(src, inv, dest, rows);
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_scale_cols(flz_ctx* ctx, double* A, int64_t lda, int N, int64_t rows,
                       const double* s) {
  if (rows <= 0 || N <= 0) return;
  dim3 grid((unsigned)((rows + 255) / 256), (unsigned)N);
  scale_cols_kernel<<<grid, 256, 0, ctx->stream>>>(A, lda, rows, s);
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_residual_prep(flz_ctx* ctx, double* V, double* AV, int64_t ld, int N, int64_t rows,
                          const double* inv, const double* lambda) {
  if (rows <= 0 || N <= 0) return;
  dim3 grid((unsigned)((rows + 255) / 256), (unsigned)N);
  residual_prep_kernel<<<grid, 256, 0, ctx->stream>>>(V, AV, ld, rows, inv, lambda);
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_permute_in(flz_ctx* ctx, const double* src, int64_t lds, double* dst, int64_t ldd,
                       int N, int64_t rows, const int32_t* perm) {
  if (rows <= 0 || N <= 0) return;
  dim3 grid((unsigned)((rows + 255) / 256), (unsigned)N);
  permute_in_kernel<<<grid, 256, 0, ctx->stream>>>(src, lds, dst, ldd, rows, perm);
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_permute_out(flz_ctx* ctx, const double* src, int64_t lds, double* dst, int64_t ldd,
                        int N, int64_t rows, const int32_t* perm) {
  if (rows <= 0 || N <= 0) return;
  dim3 grid((unsigned)((rows + 255) / 256), (unsigned)N);
  permute_out_kernel<<<grid, 256, 0, ctx->stream>>>(src, lds, dst, ldd, rows, perm);
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_update_scale(flz_ctx* ctx, const double* gram, int r, int ldg, double* op_scale) {
  update_scale_kernel<<<1, 1, 0, ctx->stream>>>(gram, r, ldg, op_scale);
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

void launch_finish_col(flz_ctx* ctx, const double* normsq, const double* op_scale, double* Sk,
                       int r, int j, double* inv, double* dead_flag) {
  finish_col_kernel<<<1, 1, 0, ctx->stream>>>(normsq, op_scale, Sk, r, j, inv, dead_flag);
  ctx->launches++;
  FLZ_CUDA(cudaGetLastError());
}

}  // namespace flz
