// HBM ceilings for K1-like traffic mixes (round-1 investigation; not part of the product).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("%s: %s\n",#x,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) b[i] = a[i];
}
__global__ void read_k(const double2* __restrict__ a, double* out, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (; i < n; i += s) { double2 v = a[i]; acc += v.x + v.y; }
  if (acc == 1.2345) out[0] = acc;
}
// per "row": 7 doubles + 7 ints of matrix, 3 doubles from each of y1,y2,x, 3 doubles out; no gather
__global__ void mix_k(const double* __restrict__ val, const int* __restrict__ col, const double* __restrict__ y1,
                      double* __restrict__ y2, const double* __restrict__ x, size_t nrows) {
  size_t row = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  size_t slice = row >> 5, lane = row & 31;
  const double* v = val + slice * 7 * 32 + lane; const int* c = col + slice * 7 * 32 + lane;
  double acc[3] = {0,0,0};
#pragma unroll
  for (int p = 0; p < 7; ++p) { double a = v[p*32]; int cc = c[p*32]; acc[0] += a * cc; acc[1] += a; acc[2] -= a; }
#pragma unroll
  for (int k = 0; k < 3; ++k) y2[row*3+k] = acc[k] + y1[row*3+k] - y2[row*3+k] + x[k*nrows + row];
}
int main() {
  size_t n = (size_t)1 << 27;  // doubles: 1 GiB
  double *a, *b; CK(cudaMalloc(&a, n*8)); CK(cudaMalloc(&b, n*8)); CK(cudaMemset(a, 0, n*8)); CK(cudaMemset(b,0,n*8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int blocks : {148*8, 148*16, 148*32}) {
    copy_k<<<blocks, 512>>>((double2*)a, (double2*)b, n/2); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int i=0;i<5;i++) copy_k<<<blocks, 512>>>((double2*)a, (double2*)b, n/2); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("copy  blocks=%5d: %.0f GB/s\n", blocks, 5*2.0*n*8/ms/1e6);
    cudaEventRecord(e0); for (int i=0;i<5;i++) read_k<<<blocks, 512>>>((double2*)a, b, n/2); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("read  blocks=%5d: %.0f GB/s\n", blocks, 5*1.0*n*8/ms/1e6);
  }
  // small-footprint copy like one K1 step (183 MB total traffic), cold-ish L2 by alternating buffers
  for (size_t m : {(size_t)12000000, (size_t)48000000}) {
    cudaEventRecord(e0); for (int i=0;i<20;i++) copy_k<<<148*16, 512>>>((double2*)(a + (i%(n/m))*m), (double2*)(b + (i%(n/m))*m), m/2); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("copy of %zu MB per launch: %.1f us/launch %.0f GB/s\n", m*16/1000000, ms/20*1e3, 20*2.0*m*8/ms/1e6);
  }
  size_t rows = 1000000;
  double *val, *y1, *y2, *x; int* col;
  CK(cudaMalloc(&val, rows*7*8)); CK(cudaMalloc(&col, rows*7*4)); CK(cudaMalloc(&y1, rows*24)); CK(cudaMalloc(&y2, rows*24)); CK(cudaMalloc(&x, rows*24));
  cudaMemset(val,0,rows*56); cudaMemset(col,0,rows*28); cudaMemset(y1,0,rows*24); cudaMemset(y2,0,rows*24); cudaMemset(x,0,rows*24);
  for (int bs : {128, 256, 512}) {
    mix_k<<<(rows+bs-1)/bs, bs>>>(val, col, y1, y2, x, rows); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int i=0;i<50;i++) { mix_k<<<(rows+bs-1)/bs, bs>>>(val, col, y1, y2, x, rows); double* t=y1; y1=y2; y2=t; } cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("mix (K1 traffic, no gather) bs=%d: %.1f us/step  %.0f GB/s\n", bs, ms/50*1e3, 50.0*rows*(84+96)/ms/1e6);
  }
  return 0;
}
