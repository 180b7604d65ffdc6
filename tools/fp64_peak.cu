// FP64 roofline denominator: DFMA throughput of this B200 (MEASURED_PEAKS.json
// has no FP64 entry).  Many independent DFMA chains per thread, full grid,
// CUDA-event timed, best of 10.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* out;
  cudaMalloc(&out, 8);
  const int CH = 8, iters = 20000, block = 256;
  int grid = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 12; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<CH><<<grid, block>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2 && ms < best) best = ms;
  }
  double flops = 2.0 * CH * (double)iters * grid * block;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp64_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"clock_khz_attr\": %d, \"dfma_per_sm_per_clk_at_attr_clock\": %.2f}\n",
         flops / best / 1e9, best, sms, clk, flops / (best * 1e-3) / sms / (clk * 1e3) / 2.0);
  return 0;
}
