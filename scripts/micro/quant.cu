// Is the back-to-back kernel time on this box quantized?  Spin kernels of growing duration.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void spin(long long cycles, int* sink) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
  if (cycles < 0) *sink = 1;
}
__global__ void spin_pdl(long long cycles, int* sink) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
  if (cycles < 0) *sink = 1;
}
int main() {
  int* sink; cudaMalloc(&sink, 4);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int pdl = 0; pdl < 2; ++pdl)
  for (int grid : {148, 888})
  for (long long us10 = 20; us10 <= 140; us10 += 5) {   // 2.0 .. 14.0 us
    const long long cyc = (long long)(us10 * 0.1 * 1965.0);
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0, st);
      for (int i = 0; i < 300; ++i) {
        if (!pdl) spin<<<grid, 128, 0, st>>>(cyc, sink);
        else {
          cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
          cudaLaunchConfig_t cfg{}; cfg.stream = st; cfg.attrs = at; cfg.numAttrs = 1; cfg.blockDim = dim3(128); cfg.gridDim = dim3(grid);
          cudaLaunchKernelEx(&cfg, spin_pdl, cyc, sink);
        }
      }
      cudaEventRecord(e1, st); cudaStreamSynchronize(st);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("pdl=%d grid=%d spin %.1f us -> %.2f us/launch\n", pdl, grid, us10 * 0.1, best * 1e3 / 300);
  }
  return 0;
}
