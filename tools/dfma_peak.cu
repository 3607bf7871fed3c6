// fp64 FMA (DFMA, non-tensor) throughput on the box: the denominator of the assembly and
// gradient fp64 rooflines (bench.py fp64_peak_tflops).  Every thread runs 8 independent FMA
// chains; grids of 8 CTAs x 256 threads per SM.  Prints one JSON line.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dfma_peak.cu -o /tmp/dfma && /tmp/dfma
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int grid = sms * 8, iters = 1 << 16;
  dfma_kernel<<<grid, 256>>>(out, 1024, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<grid, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8.0 * iters * (double)grid * 256.0;
  printf("{\"tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"sm_clock_khz_attr\": %d, \"how\": \"%d CTAs x 256 threads x 8 "
         "independent DFMA chains x %d iterations, best of 5 (CUDA events)\", \"error\": \"%s\"}\n",
         flops / (best * 1e-3) / 1e12, best, sms, clk, grid, iters, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
