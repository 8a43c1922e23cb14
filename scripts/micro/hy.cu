// hy.cu — stand-alone prototype of the HYBRID layout for PARSEC-shaped matrices (stencil +
// dense non-local blocks).  Not part of the library: a bench bed for the kernel design.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o hy hy.cu
//   ./hy [radius=30] [atoms=199] [ball=3.384] [steps=200]
//
// Phase A (dense tasks): one CTA per (block, group of 64 rows); the block rows of the block's
//   columns are staged in shared memory once, the values stream as [col][lane] pairs; result =
//   one partial per (block, row), stored in a slot array P.
// Phase B (slice tasks): natural row order, one warp per 32-row slice, planar block vectors.
//   Positions are UNIFORM-VALUE (one double for the position, per-lane columns), GENERAL
//   (per-lane value and column) or PARTIAL (per-lane slot of P, value 1).  Diagonal in the
//   epilogue together with the Clenshaw combine.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

constexpr int R = 3;
#ifndef BATCH
#define BATCH 1   // groups of 4 uniform-value positions per round
#endif
#ifndef SLICE_CTAS
#define SLICE_CTAS 6
#endif
#ifndef DH
#define DH 1   // rows per lane in a dense task (group = 32 * DH rows)
#endif
constexpr int GR = 32 * DH;
#ifndef NGRP
#define NGRP 10   // groups of 4 uniform-value positions kept in registers
#endif
#ifndef DMAXC
#define DMAXC 48
#endif
#ifndef PREF
#define PREF 1
#endif
#ifndef EXP
#define EXP 0
#endif
#ifndef DU
#define DU 4
#endif
#ifndef UV_MIN_LANES
#define UV_MIN_LANES 8
#endif

struct Csr {
  int n = 0;
  std::vector<int64_t> rp;
  std::vector<int> ci;
  std::vector<double> va;
};

struct Gen {
  Csr A;
  std::vector<std::vector<int>> balls;  // rows of every dense block (ascending)
};

static Gen generate(double radius, int n_atoms, double ball_radius, double h = 0.567) {
  const double fd[7] = {-5369.0 / 1800, 12.0 / 7, -15.0 / 56, 10.0 / 189, -1.0 / 112, 2.0 / 1925,
                        -1.0 / 16632};
  const int Rg = (int)std::ceil(radius), L = 2 * Rg + 1;
  std::vector<int> ident((size_t)L * L * L, -1);
  std::vector<int> px, py, pz;
  for (int z = -Rg; z <= Rg; ++z)
    for (int y = -Rg; y <= Rg; ++y)
      for (int x = -Rg; x <= Rg; ++x)
        if (x * x + y * y + z * z < radius * radius) {
          ident[((size_t)(z + Rg) * L + (y + Rg)) * L + (x + Rg)] = (int)px.size();
          px.push_back(x);
          py.push_back(y);
          pz.push_back(z);
        }
  const int n = (int)px.size();
  std::vector<std::map<int, double>> rows(n);
  const double kin = -0.5 / (h * h);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> pot(-1.2, 0.3), uni(0.0, 1.0);
  for (int i = 0; i < n; ++i) {
    rows[i][i] = 3 * kin * fd[0] + pot(rng);
    const int d[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    for (auto& a : d)
      for (int k = -6; k <= 6; ++k) {
        if (!k) continue;
        const int x = px[i] + k * a[0] + Rg, y = py[i] + k * a[1] + Rg, z = pz[i] + k * a[2] + Rg;
        if (x < 0 || y < 0 || z < 0 || x >= L || y >= L || z >= L) continue;
        const int j = ident[((size_t)z * L + y) * L + x];
        if (j >= 0) rows[i][j] += kin * fd[std::abs(k)];
      }
  }
  Gen G;
  std::uniform_real_distribution<double> pos(-radius, radius);
  while ((int)G.balls.size() < n_atoms) {
    const double a[3] = {pos(rng), pos(rng), pos(rng)};
    if (a[0] * a[0] + a[1] * a[1] + a[2] * a[2] >= (radius - ball_radius) * (radius - ball_radius))
      continue;
    std::vector<int> ball;
    std::vector<double> p;
    double nrm = 0;
    for (int i = 0; i < n; ++i) {
      const double d2 = (px[i] - a[0]) * (px[i] - a[0]) + (py[i] - a[1]) * (py[i] - a[1]) +
                        (pz[i] - a[2]) * (pz[i] - a[2]);
      if (d2 < ball_radius * ball_radius) {
        ball.push_back(i);
        p.push_back(std::exp(-d2 / (0.5 * ball_radius * ball_radius)));
        nrm += p.back() * p.back();
      }
    }
    if (ball.size() < 2) continue;
    const double w = 0.35 * (0.5 + uni(rng)) * (uni(rng) < 0.7 ? 1 : -1) / nrm;
    for (size_t s = 0; s < ball.size(); ++s)
      for (size_t t = 0; t < ball.size(); ++t) rows[ball[s]][ball[t]] += w * p[s] * p[t];
    G.balls.push_back(ball);
  }
  G.A.n = n;
  G.A.rp.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    G.A.rp[i + 1] = G.A.rp[i] + (int64_t)rows[i].size();
    for (auto& kv : rows[i]) {
      G.A.ci.push_back(kv.first);
      G.A.va.push_back(kv.second);
    }
  }
  return G;
}

// ------------------------------------------------------------------------------ layout
struct SliceHdr {      // 32 bytes
  int64_t col_off;     // into cols, in units of 32 ints (positions)
  int uv_off;          // into uvval
  int g_off;           // into gval, in units of 32 doubles
  int nuv, ng, np;
  int pad;
};
struct DenseTask {     // 32 bytes
  int64_t val_off;     // into dval, units of 64 doubles (one column: 32 lanes x 2 rows)
  int col_off;         // into dcols
  int ncols;
  int slot_base;       // 64 slots: [h][lane]
  int nrows;
  int pad[2];
};
struct Layout {
  int n, ld, nslices, nslots, ldp;
  std::vector<SliceHdr> hdr;
  std::vector<int> cols;
  std::vector<double> uvval, gval, diag;
  std::vector<DenseTask> dtasks;
  std::vector<int> dcols;
  std::vector<double> dval;
  int64_t dense_entries = 0, uv_entries = 0, g_entries = 0, p_entries = 0, uv_pos = 0, g_pos = 0,
          p_pos = 0;
};

static Layout build(const Gen& G) {
  const Csr& A = G.A;
  const int n = A.n;
  Layout Ly;
  Ly.n = n;
  Ly.ld = (n + 1 + 31) / 32 * 32;  // row n = zero row
  Ly.nslices = (n + 31) / 32;
  Ly.diag.assign(n, 0.0);
  // block membership: for every row, the blocks that contain it and its index inside them
  std::vector<std::vector<std::pair<int, int>>> member(n);
  for (size_t b = 0; b < G.balls.size(); ++b)
    for (size_t s = 0; s < G.balls[b].size(); ++s) member[G.balls[b][s]].push_back({(int)b, (int)s});
  // dense tasks: block b, groups of 64 rows; entry (i,j) is owned by the FIRST block holding both
  std::vector<std::vector<int>> slot_of(n);  // partial slots a row consumes
  int nslots = 64;                           // slots 0..63 unused: slot 0 = zero slot
  auto owner = [&](int i, int j) {
    for (auto& mi : member[i])
      for (auto& mj : member[j])
        if (mi.first == mj.first) return mi.first;
    return -1;
  };
  for (size_t b = 0; b < G.balls.size(); ++b) {
    const auto& rows = G.balls[b];
    const int nb = (int)rows.size();
    const int col_off = (int)Ly.dcols.size();
    Ly.dcols.insert(Ly.dcols.end(), rows.begin(), rows.end());
    for (int g0 = 0; g0 < nb; g0 += GR) {
      DenseTask T{};
      T.val_off = (int64_t)Ly.dval.size() / GR;
      T.col_off = col_off;
      T.ncols = nb;
      T.slot_base = nslots;
      T.nrows = std::min(GR, nb - g0);
      nslots += GR;
      Ly.dval.resize(Ly.dval.size() + (size_t)nb * GR, 0.0);
      double* v = Ly.dval.data() + T.val_off * GR;
      for (int q = 0; q < T.nrows; ++q) {
        const int i = rows[g0 + q], lane = q & 31, hh = q >> 5;
        slot_of[i].push_back(T.slot_base + hh * 32 + lane);
        for (int64_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
          const int j = A.ci[e];
          if (j == i) continue;
          auto it = std::lower_bound(rows.begin(), rows.end(), j);
          if (it == rows.end() || *it != j) continue;
          if (owner(i, j) != (int)b) continue;
          v[(size_t)(it - rows.begin()) * GR + lane * DH + hh] = A.va[e];
          ++Ly.dense_entries;
        }
      }
      Ly.dtasks.push_back(T);
    }
  }
  Ly.nslots = nslots;
  Ly.ldp = (nslots + 31) / 32 * 32;
  // slices
  for (int s = 0; s < Ly.nslices; ++s) {
    std::map<double, std::vector<std::vector<int>>> byval;  // value -> per lane cols
    std::vector<std::vector<std::pair<int, double>>> gen(32);
    std::map<double, int> lanes_with;
    std::vector<std::vector<std::pair<int, double>>> rest(32);
    for (int l = 0; l < 32; ++l) {
      const int i = s * 32 + l;
      if (i >= n) continue;
      std::map<double, int> seen;
      for (int64_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
        const int j = A.ci[e];
        if (j == i) {
          Ly.diag[i] = A.va[e];
          continue;
        }
        if (owner(i, j) >= 0) continue;
        rest[l].push_back({j, A.va[e]});
        if (!seen[A.va[e]]++) ++lanes_with[A.va[e]];
      }
    }
    for (int l = 0; l < 32; ++l)
      for (auto& cv : rest[l]) {
        if (lanes_with[cv.second] >= UV_MIN_LANES) {
          auto& per = byval[cv.second];
          per.resize(32);
          per[l].push_back(cv.first);
        } else {
          gen[l].push_back(cv);
        }
      }
    SliceHdr H{};
    H.col_off = (int64_t)Ly.cols.size() / 32;
    H.uv_off = (int)Ly.uvval.size();
    H.g_off = (int)(Ly.gval.size() / 32);
    {
      std::vector<std::vector<int>> pc;  // per position: 32 columns
      for (auto& kv : byval) {
        size_t cnt = 0;
        for (auto& per : kv.second) cnt = std::max(cnt, per.size());
        for (size_t q = 0; q < cnt; ++q) {
          Ly.uvval.push_back(kv.first);
          pc.emplace_back(32, n);
          for (int l = 0; l < 32; ++l)
            if (q < kv.second[l].size()) {
              pc.back()[l] = kv.second[l][q];
              ++Ly.uv_entries;
            }
        }
      }
      while (pc.size() % 4) {
        pc.emplace_back(32, n);
        Ly.uvval.push_back(0.0);
      }
      H.nuv = (int)pc.size();
      for (size_t q = 0; q < pc.size(); q += 4)
        for (int l = 0; l < 32; ++l)
          for (int u = 0; u < 4; ++u) Ly.cols.push_back(pc[q + u][l]);
    }
    size_t ng = 0;
    for (auto& g : gen) ng = std::max(ng, g.size());
    for (size_t q = 0; q < ng; ++q) {
      for (int l = 0; l < 32; ++l) {
        const bool has = q < gen[l].size();
        Ly.cols.push_back(has ? gen[l][q].first : n);
        Ly.gval.push_back(has ? gen[l][q].second : 0.0);
        Ly.g_entries += has;
      }
      ++H.ng;
    }
    size_t np = 0;
    for (int l = 0; l < 32; ++l)
      if (s * 32 + l < n) np = std::max(np, slot_of[s * 32 + l].size());
    for (size_t q = 0; q < np; ++q) {
      for (int l = 0; l < 32; ++l) {
        const int i = s * 32 + l;
        const bool has = i < n && q < slot_of[i].size();
        Ly.cols.push_back(has ? slot_of[i][q] : 0);
        Ly.p_entries += has;
      }
      ++H.np;
    }
    Ly.uv_pos += H.nuv;
    Ly.g_pos += H.ng;
    Ly.p_pos += H.np;
    Ly.hdr.push_back(H);
  }
  return Ly;
}

// ------------------------------------------------------------------------------ kernels
struct View {
  int n, ld, nslices, ldp, ndtasks;
  const SliceHdr* hdr;
  const int* cols;
  const double* uvval;
  const double* gval;
  const double* diag;
  const DenseTask* dtasks;
  const int* dcols;
  const double* dval;
  double2* P;         // [k][slot] {partial sum, tag}: tag == epoch of the launch that wrote it
  unsigned* tickets;  // this launch's ticket counter
  double epoch;
  int nbtasks;        // slice tasks (4 slices each)
  int maxcols;
  unsigned long long* trace;  // optional: per task {start, end, smid} in ns
};

__device__ __forceinline__ double ldnc(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldnc_s32(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int4 ldnc_s32x4(const int* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldcg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ---- one slice by one warp.  G = groups of 4 uniform-value positions per round.
template <int G, bool WAIT, bool PDL = false>
__device__ __forceinline__ void slice_body(const View& V, int slice, int lane, double s1, double s2,
                                           double b, const double* __restrict__ Y1,
                                           double* __restrict__ Y2, const double* __restrict__ X) {
  unsigned long long ts[8];
  int nts = 0;
  const bool tr = V.trace != nullptr && slice % 500 == 0 && lane == 0;
  auto stamp = [&]() {
    if (tr && nts < 8) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[nts]));
    ++nts;
  };
  stamp();
  const int4* hp = reinterpret_cast<const int4*>(V.hdr + slice);
  const int4 h0 = __ldg(hp), h1 = __ldg(hp + 1);
  const int64_t col_off = ((int64_t)(uint32_t)h0.y << 32) | (uint32_t)h0.x;
  const int uv_off = h0.z, g_off = h0.w, nuv = h1.x, ng = h1.y, np = h1.z;
  const int ld = V.ld;
  const int row = slice * 32 + lane;
  double acc[R] = {0.0, 0.0, 0.0};
  // uniform-value positions.  Everything immutable is requested BEFORE the grid-dependency
  // wait: all column words of up to 4*NGR positions (registers) and the position values (lane l
  // keeps the values of positions l and 32 + l; a shuffle broadcasts them).  After the wait only
  // the gathers remain, 4G positions per round.
  {
    constexpr int NGR = NGRP;
    const int* __restrict__ col = V.cols + col_off * 32 + lane * 4;
    const double* __restrict__ uv = V.uvval + uv_off;
    int4 c[NGR];
#pragma unroll
    for (int u = 0; u < NGR; ++u)
      c[u] = 4 * u < nuv ? ldnc_s32x4(col + u * 128) : make_int4(V.n, V.n, V.n, V.n);
    const double uvA = lane < nuv ? ldnc(uv + lane) : 0.0;
    const double uvB = 32 + lane < nuv ? ldnc(uv + 32 + lane) : 0.0;
    if (tr) { volatile int x = c[0].x; (void)x; }
    stamp();   // 1: header and first columns have arrived
    if (PDL) pdl_wait();
    stamp();   // 2: previous kernel complete
#pragma unroll
    for (int r0 = 0; r0 < NGR; r0 += G) {
      if (4 * r0 < nuv) {
        double g[G][4][R];
#pragma unroll
        for (int u = 0; u < G; ++u)
          if (r0 + u < NGR) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
              g[u][0][k] = __ldg(Y1 + (int64_t)k * ld + c[r0 + u].x);
              g[u][1][k] = __ldg(Y1 + (int64_t)k * ld + c[r0 + u].y);
              g[u][2][k] = __ldg(Y1 + (int64_t)k * ld + c[r0 + u].z);
              g[u][3][k] = __ldg(Y1 + (int64_t)k * ld + c[r0 + u].w);
            }
          }
#pragma unroll
        for (int u = 0; u < G; ++u)
          if (r0 + u < NGR) {
            const int p = 4 * (r0 + u);
            const double src = p < 32 ? uvA : uvB;
            const double v0 = __shfl_sync(0xffffffffu, src, (p + 0) & 31);
            const double v1 = __shfl_sync(0xffffffffu, src, (p + 1) & 31);
            const double v2 = __shfl_sync(0xffffffffu, src, (p + 2) & 31);
            const double v3 = __shfl_sync(0xffffffffu, src, (p + 3) & 31);
#pragma unroll
            for (int k = 0; k < R; ++k) {
              acc[k] = fma(v0, g[u][0][k], acc[k]);
              acc[k] = fma(v1, g[u][1][k], acc[k]);
              acc[k] = fma(v2, g[u][2][k], acc[k]);
              acc[k] = fma(v3, g[u][3][k], acc[k]);
            }
          }
      }
    }
    // slices with more than 4*NGR uniform-value positions: plain loop (rare)
    for (int p = 4 * NGR; p < nuv; p += 4) {
      const int4 cc = ldnc_s32x4(col + (p >> 2) * 128);
      const int cs[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double v = __ldg(uv + p + u);
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = fma(v, __ldg(Y1 + (int64_t)k * ld + cs[u]), acc[k]);
      }
    }
  }
  if (tr) { volatile double x = acc[0]; (void)x; }
  stamp();     // 3: uniform-value positions done
  const int* __restrict__ col = V.cols + (col_off + nuv) * 32 + lane;
  // general positions
  {
    const double* __restrict__ gv = V.gval + (int64_t)g_off * 32 + lane;
    for (int p = 0; p < ng; p += 4) {
      int c[4];
      double v[4], g[4][R];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = p + u < ng ? ldnc_s32(col + (p + u) * 32) : V.n;
        v[u] = p + u < ng ? ldnc(gv + (p + u) * 32) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) g[u][k] = __ldg(Y1 + (int64_t)k * ld + c[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = fma(v[u], g[u][k], acc[k]);
    }
    col += ng * 32;
  }
  // own-row operands (requested before the partials are waited for)
  double y1o[R], y2o[R], xo[R], d = 0.0;
  if (row < V.n) {
    d = ldnc(V.diag + row);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int64_t o = (int64_t)k * ld + row;
      y1o[k] = __ldg(Y1 + o);
      y2o[k] = Y2[o];
      xo[k] = ldnc(X + o);
    }
  }
  // partial positions: results of dense tasks of THIS launch.  Slot s belongs to dense task
  // s / 64 - 1, whose flag carries the epoch of the launch that completed it.
  if (tr) { volatile double x = y2o[0] + xo[0] + y1o[0]; (void)x; }
  stamp();     // 4: own-row operands have arrived
  // Each partial carries the epoch of the launch that wrote it in the same 16-byte word, so no
  // flag, no fence and no L1 invalidation is needed: poll the word (L2) until the tag matches.
  for (int p = 0; p < np; ++p) {
    const int sl = ldnc_s32(col + p * 32);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const double2* q = V.P + (int64_t)k * V.ldp + sl;
      double2 w;
      for (;;) {
        asm volatile("ld.relaxed.gpu.global.v2.f64 {%0,%1}, [%2];" : "=d"(w.x), "=d"(w.y) : "l"(q) : "memory");
        if (!WAIT || sl < 64 || w.y == V.epoch) break;
        __nanosleep(32);
      }
      acc[k] += w.x;
    }
  }
  if (row < V.n) {
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const double w = fma(d, y1o[k], acc[k]);
      Y2[(int64_t)k * ld + row] = fma(s1, w, fma(s2, y1o[k], fma(b, xo[k], -y2o[k])));
    }
  }
  stamp();     // 5: stored
  if (tr)
    for (int i = 0; i < 6; ++i) V.trace[(slice / 500) * 8 + i] = ts[i];
}

// ---- one dense task by 4 warps (warp index wd, named barrier `bar`).
// smem: ys[maxcols][4] then part[3][DH * R][32]
__device__ __forceinline__ void bar4(int id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }

__device__ __forceinline__ void dense_body(const View& V, int t, double* smem,
                                           const double* __restrict__ Y1, int wd, int bar, int tid,
                                           bool pdl = false) {
  double (*ys)[4] = reinterpret_cast<double (*)[4]>(smem);
  double (*part)[DH * R][32] = reinterpret_cast<double (*)[DH * R][32]>(smem + 4 * V.maxcols);
  const int lane = threadIdx.x & 31;
  const int4* tp = reinterpret_cast<const int4*>(V.dtasks + t);
  const int4 t0 = __ldg(tp), t1 = __ldg(tp + 1);
  const int64_t val_off = ((int64_t)(uint32_t)t0.y << 32) | (uint32_t)t0.x;
  const int col_off = t0.z, ncols = t0.w, slot_base = t1.x;
  const int chunk = (ncols + 3) / 4;
  const int j0 = wd * chunk, j1 = min(ncols, j0 + chunk);
  const double* __restrict__ v = V.dval + val_off * GR + lane * DH;
  // ALL values of this warp's column chunk are requested before the grid-dependency wait
  // (they are immutable): up to DMAX columns live in registers, longer chunks loop.
  constexpr int DMAX = DMAXC;
  double a[DMAX][DH];
  auto fetch = [&](int j) {
#pragma unroll
    for (int u = 0; u < DMAX; ++u) {
#pragma unroll
      for (int h = 0; h < DH; ++h) a[u][h] = 0.0;
      if (j + u < j1) {
        if (DH == 2)
          asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                       : "=d"(a[u][0]), "=d"(a[u][DH - 1]) : "l"(v + (int64_t)(j + u) * GR));
        else
          asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];"
                       : "=d"(a[u][0]) : "l"(v + (int64_t)(j + u) * GR));
      }
    }
  };
  fetch(j0);
  if (pdl) pdl_wait();
  for (int j = tid; j < ncols; j += 128) {
    const int c = __ldg(V.dcols + col_off + j);
#pragma unroll
    for (int k = 0; k < R; ++k) ys[j][k] = __ldg(Y1 + (int64_t)k * V.ld + c);
  }
  bar4(bar);
  double acc[DH][R];
#pragma unroll
  for (int h = 0; h < DH; ++h)
#pragma unroll
    for (int k = 0; k < R; ++k) acc[h][k] = 0.0;
  for (int j = j0; j < j1; j += DMAX) {
    if (j > j0) fetch(j);
#pragma unroll
    for (int u = 0; u < DMAX; ++u) {
      const int jj = min(j + u, ncols - 1);
      const double2 y01 = *reinterpret_cast<const double2*>(&ys[jj][0]);
      const double y2 = ys[jj][2];
#pragma unroll
      for (int h = 0; h < DH; ++h) {
        acc[h][0] = fma(a[u][h], y01.x, acc[h][0]);
        acc[h][1] = fma(a[u][h], y01.y, acc[h][1]);
        acc[h][2] = fma(a[u][h], y2, acc[h][2]);
      }
    }
  }
  if (wd > 0) {
#pragma unroll
    for (int h = 0; h < DH; ++h)
#pragma unroll
      for (int k = 0; k < R; ++k) part[wd - 1][h * R + k][lane] = acc[h][k];
  }
  bar4(bar);
  if (wd == 0) {
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int h = 0; h < DH; ++h)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[h][k] += part[q][h * R + k][lane];
#pragma unroll
    for (int h = 0; h < DH; ++h)
#pragma unroll
      for (int k = 0; k < R; ++k)
        V.P[(int64_t)k * V.ldp + slot_base + h * 32 + lane] = make_double2(acc[h][k], V.epoch);
  }
}

// Separate launches (upper bound of the design): dense, then slices
__global__ void __launch_bounds__(128) dense_kernel(View V, const double* __restrict__ Y1) {
  extern __shared__ __align__(16) double smem[];
  pdl_launch();
  dense_body(V, blockIdx.x, smem, Y1, threadIdx.x >> 5, 1, threadIdx.x, true);
}
__global__ void __launch_bounds__(128) dense_kernel_pdl(View V, const double* __restrict__ Y1) {
  extern __shared__ __align__(16) double smem[];
  pdl_launch();
  dense_body(V, blockIdx.x, smem, Y1, threadIdx.x >> 5, 1, threadIdx.x, true);
}
template <int G>
__global__ void __launch_bounds__(128, SLICE_CTAS)
    slice_kernel_pdl(View V, double s1, double s2, double b, const double* __restrict__ Y1,
                     double* __restrict__ Y2, const double* __restrict__ X) {
  pdl_launch();
  const int slice = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (slice < V.nslices) slice_body<G, false, true>(V, slice, threadIdx.x & 31, s1, s2, b, Y1, Y2, X);
  else pdl_wait();
}

template <int G>
__global__ void __launch_bounds__(128, SLICE_CTAS)
    slice_kernel(View V, double s1, double s2, double b, const double* __restrict__ Y1,
                 double* __restrict__ Y2, const double* __restrict__ X) {
  pdl_launch();
  const int slice = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (slice < V.nslices) slice_body<G, false, true>(V, slice, threadIdx.x & 31, s1, s2, b, Y1, Y2, X);
  else pdl_wait();
}

// One launch: persistent CTAs take tickets; dense tasks first, then the slices in natural order.
// A slice waits (per lane, per partial slot) for the flag of the dense task that produces the
// slot — dense tasks never wait and all hold earlier tickets, so this cannot deadlock.
template <int G>
__global__ void __launch_bounds__(128, SLICE_CTAS)
    fused_kernel(View V, double s1, double s2, double b, const double* __restrict__ Y1,
                 double* __restrict__ Y2, const double* __restrict__ X) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int next;
  const int total = V.ndtasks + V.nbtasks;
  pdl_launch();
  pdl_wait();
  for (;;) {
    if (threadIdx.x == 0) next = (int)atomicAdd(V.tickets, 1u);
    __syncthreads();
    const int t = next;
    if (t >= total) break;
    unsigned long long t_begin = 0;
    if (V.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
    if (t < V.ndtasks) {
      dense_body(V, t, smem, Y1, threadIdx.x >> 5, 1, threadIdx.x);
    } else {
      const int slice = (t - V.ndtasks) * 4 + (threadIdx.x >> 5);
      if (slice < V.nslices) slice_body<G, true>(V, slice, threadIdx.x & 31, s1, s2, b, Y1, Y2, X);
    }
    __syncthreads();  // `next` and smem are reused
    if (V.trace && threadIdx.x == 0) {
      unsigned long long t_end;
      unsigned sm;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      V.trace[3 * t] = t_begin;
      V.trace[3 * t + 1] = t_end;
      V.trace[3 * t + 2] = sm;
    }
  }
}

// One launch, static schedule, warp-specialised CTAs of 8 warps: warps 0-3 run slices (each its
// own contiguous share), warps 4-7 run dense tasks t = blockIdx.x, + gridDim.x, ...  All CTAs
// are co-resident (grid = SMs x 3), a slice polls the tagged partials it needs at its very end.
#ifndef F2_CTAS
#define F2_CTAS 3
#endif
template <int G>
__global__ void __launch_bounds__(256, F2_CTAS)
    fused2_kernel(View V, double s1, double s2, double b, const double* __restrict__ Y1,
                  double* __restrict__ Y2, const double* __restrict__ X, int spw) {
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5;
  pdl_launch();
  pdl_wait();
  if (warp < 4) {
    const int s0 = (blockIdx.x * 4 + warp) * spw;
    for (int i = 0; i < spw; ++i)
      if (s0 + i < V.nslices) slice_body<G, true>(V, s0 + i, threadIdx.x & 31, s1, s2, b, Y1, Y2, X);
  } else {
    for (int t = blockIdx.x; t < V.ndtasks; t += gridDim.x)
      dense_body(V, t, smem, Y1, warp - 4, 1, threadIdx.x - 128);
  }
}

// ------------------------------------------------------------------------------ host
template <class T>
static T* upload(const std::vector<T>& v) {
  T* d = nullptr;
  CK(cudaMalloc(&d, std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

int main(int argc, char** argv) {
  const double radius = argc > 1 ? std::atof(argv[1]) : 30.0;
  const int atoms = argc > 2 ? std::atoi(argv[2]) : 199;
  const double ball = argc > 3 ? std::atof(argv[3]) : 3.384;
  const int steps = argc > 4 ? std::atoi(argv[4]) : 200;
  Gen G = generate(radius, atoms, ball);
  const Csr& A = G.A;
  const int n = A.n;
  const int64_t nnz = A.rp[n];
  Layout Ly = build(G);
  const double alg = 12.0 * nnz + 4.0 * (n + 1) + 32.0 * n * R;
  const double streamed = 4.0 * Ly.cols.size() + 8.0 * (Ly.uvval.size() + Ly.gval.size() + Ly.diag.size()) +
                          8.0 * Ly.dval.size() + 32.0 * n * R;
  std::printf("n=%d nnz=%lld (%.1f/row) blocks=%zu dense tasks=%zu | entries: dense %lld uv %lld g %lld "
              "partial %lld | positions/slice uv %.1f g %.1f p %.2f | algorithmic %.1f MB streamed %.1f MB\n",
              n, (long long)nnz, (double)nnz / n, G.balls.size(), Ly.dtasks.size(),
              (long long)Ly.dense_entries, (long long)Ly.uv_entries, (long long)Ly.g_entries,
              (long long)Ly.p_entries, (double)Ly.uv_pos / Ly.nslices, (double)Ly.g_pos / Ly.nslices,
              (double)Ly.p_pos / Ly.nslices, alg / 1e6, streamed / 1e6);

  const int nbt = (Ly.nslices + 3) / 4;

  View V{};
  V.n = n;
  V.ld = Ly.ld;
  V.nslices = Ly.nslices;
  V.ldp = Ly.ldp;
  V.ndtasks = (int)Ly.dtasks.size();
  V.hdr = upload(Ly.hdr);
  V.cols = upload(Ly.cols);
  V.uvval = upload(Ly.uvval);
  V.gval = upload(Ly.gval);
  V.diag = upload(Ly.diag);
  V.dtasks = upload(Ly.dtasks);
  V.dcols = upload(Ly.dcols);
  V.dval = upload(Ly.dval);
  V.nbtasks = nbt;
  int maxcols = 2;
  for (auto& T : Ly.dtasks) maxcols = std::max(maxcols, T.ncols);
  V.maxcols = maxcols;
  const size_t dsmem = (size_t)maxcols * 32 + 3 * DH * R * 32 * 8;
  std::printf("dense smem per CTA %zu B\n", dsmem);
  CK(cudaMalloc(&V.P, (size_t)Ly.ldp * R * 16));
  CK(cudaMemset(V.P, 0, (size_t)Ly.ldp * R * 16));
  unsigned* tickets;
  CK(cudaMalloc(&tickets, 4 * 4096));
  double epoch = 0;
  const size_t vecb = (size_t)Ly.ld * R * 8;
  std::vector<double> hy1((size_t)Ly.ld * R, 0.0), hy2(hy1), hx(hy1);
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  for (int k = 0; k < R; ++k)
    for (int i = 0; i < n; ++i) {
      hy1[(size_t)k * Ly.ld + i] = nd(rng);
      hy2[(size_t)k * Ly.ld + i] = nd(rng);
      hx[(size_t)k * Ly.ld + i] = nd(rng);
    }
  double *Y1, *Y2, *X;
  CK(cudaMalloc(&Y1, vecb));
  CK(cudaMalloc(&Y2, vecb));
  CK(cudaMalloc(&X, vecb));
  CK(cudaMemcpy(X, hx.data(), vecb, cudaMemcpyHostToDevice));
  const double s1 = 0.11, s2 = -0.07, bb = 0.3;

  // reference: one step on the CPU
  std::vector<double> ref(hy2);
  for (int k = 0; k < R; ++k)
    for (int i = 0; i < n; ++i) {
      double w = 0;
      for (int64_t e = A.rp[i]; e < A.rp[i + 1]; ++e) w += A.va[e] * hy1[(size_t)k * Ly.ld + A.ci[e]];
      const size_t o = (size_t)k * Ly.ld + i;
      ref[o] = s1 * w + s2 * hy1[o] - hy2[o] + bb * hx[o];
    }
  auto check = [&](const char* what) {
    std::vector<double> got(hy2.size());
    CK(cudaMemcpy(got.data(), Y2, vecb, cudaMemcpyDeviceToHost));
    double err = 0, mx = 0;
    for (size_t i = 0; i < got.size(); ++i) {
      err = std::max(err, std::abs(got[i] - ref[i]));
      mx = std::max(mx, std::abs(ref[i]));
    }
    std::printf("%-28s max err %.2e (rel %.2e)\n", what, err, err / mx);
  };
  auto reset = [&] {
    CK(cudaMemcpy(Y1, hy1.data(), vecb, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(Y2, hy2.data(), vecb, cudaMemcpyHostToDevice));
  };
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int dev_sms = 0;
  CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, 0));

  const int sdiv = std::getenv("HY_SDIV") ? std::atoi(std::getenv("HY_SDIV")) : 1;
  const int f2grid = dev_sms * F2_CTAS;
  const int spw = (Ly.nslices + f2grid * 4 - 1) / (f2grid * 4);
  auto launch = [&](auto kern, int grid, int block, size_t smem, auto... args) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(block);
    cfg.gridDim = dim3(grid);
    cfg.dynamicSmemBytes = smem;
    CK(cudaLaunchKernelEx(&cfg, kern, args...));
  };
  auto run = [&](int mode, int count) {  // 0: separate, 1: fused, 2: dense only, 3: slices only, 4: fused2
    double *a = Y1, *b2 = Y2;
    int slot = 0;
    for (int i = 0; i < count; ++i) {
      if (mode == 0 || mode == 2) launch(dense_kernel, V.ndtasks, 128, dsmem, V, (const double*)a);
      if (mode == 0 || mode == 3)
        launch(slice_kernel<BATCH>, nbt / sdiv, 128, 0, V, s1, s2, bb, (const double*)a, b2, (const double*)X);
      if (mode == 1) {
        if (slot == 0) CK(cudaMemsetAsync(tickets, 0, 4 * 4096, st));
        View W = V;
        W.tickets = tickets + slot;
        W.epoch = (epoch += 1.0);
        slot = (slot + 1) % 4096;
        launch(fused_kernel<BATCH>, dev_sms * SLICE_CTAS, 128, dsmem, W, s1, s2, bb, (const double*)a, b2, (const double*)X);
      }
      if (mode == 5) {
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t cfg{};
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.blockDim = dim3(128);
        cfg.gridDim = dim3(V.ndtasks);
        cfg.dynamicSmemBytes = dsmem;
        CK(cudaLaunchKernelEx(&cfg, dense_kernel_pdl, V, (const double*)a));
        cfg.gridDim = dim3(nbt);
        cfg.dynamicSmemBytes = 0;
        CK(cudaLaunchKernelEx(&cfg, slice_kernel_pdl<BATCH>, V, s1, s2, bb, (const double*)a, b2, (const double*)X));
      }
      if (mode == 4) {
        View W = V;
        W.epoch = (epoch += 1.0);
        launch(fused2_kernel<BATCH>, f2grid, 256, dsmem, W, s1, s2, bb, (const double*)a, b2, (const double*)X, spw);
      }
      std::swap(a, b2);
    }
  };
  const char* names[] = {"separate (dense, slices)", "fused (tickets)", "dense tasks only", "slice tasks only", "fused2 (static, warp-spec)", "separate + PDL"};
  for (int mode = 0; mode < 5; ++mode) {
    if (mode == 4 && !std::getenv("HY_F2")) continue;
    if (mode < 2 || mode >= 4) {
      reset();
      run(mode, 1);
      CK(cudaStreamSynchronize(st));
      check(names[mode]);
    }
    reset();
    run(mode, 20);
    CK(cudaStreamSynchronize(st));
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(e0, st));
      run(mode, steps);
      CK(cudaEventRecord(e1, st));
      CK(cudaStreamSynchronize(st));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    const double us = best * 1e3 / steps;
    std::printf("%-28s %7.2f us/step   algorithmic %.0f GB/s (%.2f of 6551)   streamed %.0f GB/s\n",
                names[mode], us, alg / us / 1e3, alg / us / 1e3 / 6551.4, streamed / us / 1e3);
  }
  if (std::getenv("HY_TRACE2")) {
    unsigned long long* tr;
    CK(cudaMalloc(&tr, 64 * 8 * 8));
    CK(cudaMemset(tr, 0, 64 * 8 * 8));
    View W = V;
    W.trace = tr;
    for (int i = 0; i < 6; ++i)
      launch(slice_kernel<BATCH>, nbt, 128, 0, W, s1, s2, bb, (const double*)(i & 1 ? Y2 : Y1), (i & 1 ? Y1 : Y2), (const double*)X);
    CK(cudaStreamSynchronize(st));
    std::vector<unsigned long long> h(64 * 8);
    CK(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost));
    for (int q = 0; q * 500 < Ly.nslices; ++q) {
      std::printf("slice %5d:", q * 500);
      for (int i = 1; i < 6; ++i) std::printf(" %6.2f", (double)(h[q * 8 + i] - h[q * 8]) / 1e3);
      std::printf("   (us after entry: hdr+cols | wait done | uv done | own rows | stored)\n");
    }
  }
  if (std::getenv("HY_TRACE")) {
    const int total = V.ndtasks + V.nbtasks;
    unsigned long long* tr;
    CK(cudaMalloc(&tr, (size_t)total * 24));
    View W = V;
    W.trace = tr;
    CK(cudaMemsetAsync(tickets, 0, 4 * 4096, st));
    for (int i = 0; i < 3; ++i) {
      W.tickets = tickets + i;
      W.epoch = (epoch += 1.0);
      fused_kernel<BATCH><<<dev_sms * SLICE_CTAS, 128, dsmem, st>>>(W, s1, s2, bb, Y1, Y2, X);
    }
    CK(cudaStreamSynchronize(st));
    std::vector<unsigned long long> h((size_t)total * 3);
    CK(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (int t = 0; t < total; ++t) t0 = std::min(t0, h[3 * t]);
    FILE* f = std::fopen(std::getenv("HY_TRACE"), "w");
    for (int t = 0; t < total; ++t)
      std::fprintf(f, "%d %c %llu %llu %llu\n", t, t < V.ndtasks ? 'D' : 'S', h[3 * t] - t0, h[3 * t + 1] - t0, h[3 * t + 2]);
    std::fclose(f);
  }
  CK(cudaGetLastError());
  return 0;
}
