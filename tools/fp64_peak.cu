// FP64 roofline denominator: DFMA throughput of this B200 (MEASURED_PEAKS.json
// has no FP64 entry).  Independent DFMA chains per thread, full grid, CUDA-event
// timed, best over launch shapes (chains per thread x block size x blocks per
// SM) and repetitions; prints the best.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
static float run(int grid, int block, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 8; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<CH><<<grid, block>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  double* out;
  cudaMalloc(&out, 8);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double best_tf = 0, best_ms = 0;
  int best_cfg[3] = {0, 0, 0};
  const int iters = 5000;
  for (int block : {128, 256, 512})
    for (int per_sm : {1, 2, 4, 8})
      for (int ch : {4, 8, 16}) {
        if (block * per_sm > 2048) continue;
        const int grid = sms * per_sm;
        float ms = ch == 4 ? run<4>(grid, block, iters, out) : ch == 8 ? run<8>(grid, block, iters, out)
                                                                       : run<16>(grid, block, iters, out);
        const double flops = 2.0 * 4 * ch * (double)iters * grid * block;
        const double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best_tf) { best_tf = tf; best_ms = ms; best_cfg[0] = block; best_cfg[1] = per_sm; best_cfg[2] = ch; }
      }
  printf("{\"fp64_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"clock_khz_attr\": %d, "
         "\"dfma_per_sm_per_clk_at_attr_clock\": %.2f, \"block\": %d, \"blocks_per_sm\": %d, \"chains\": %d}\n",
         best_tf, best_ms, sms, clk, best_tf * 1e12 / sms / (clk * 1e3) / 2.0, best_cfg[0], best_cfg[1], best_cfg[2]);
  return 0;
}
