// fp64 FMA peak of this B200: independent DFMA chains, full occupancy, CUDA-event timed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;  // independent chains per thread

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains alive
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dfma, 256, 0);
  double* out;
  cudaMalloc(&out, 256 * sizeof(double));
  const int blocks = sms * occ, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, 256>>>(out, 100, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dfma = (double)blocks * 256 * iters * CH;
  const double rate = dfma / (best * 1e-3);
  printf("{\"fp64_tflops\": %.3f, \"dfma_per_clk_per_sm_at_max_clock\": %.2f, \"sms\": %d, \"blocks\": %d, "
         "\"max_clock_mhz\": %d, \"ms\": %.3f, \"how\": \"%d chains x %d iters DFMA per thread, 256 x %d blocks, best of 5\"}\n",
         2.0 * rate / 1e12, rate / sms / (clk * 1e3), sms, blocks, clk / 1000, best, CH, iters, blocks);
  return 0;
}
