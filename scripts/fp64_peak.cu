// fp64_peak.cu — measured FP64 FMA throughput of this B200: the roofline denominator of the
// FP64-bound applies (MEASURED_PEAKS.json has no FP64 entry).  8 independent DFMA chains per
// thread, 148*16 CTAs of 256 threads, CUDA events after 3 warm-up launches.
//   burst:     best of 10 single launches (~10 ms each: a kernel timed alone)
//   sustained: back-to-back launches for ~4 s (a kernel inside a long step; power/clock settle)
// Prints one JSON object.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = sms * 16, threads = 256, iters = 2000;
  const double flop = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t s, e;
  cudaEventCreate(&s); cudaEventCreate(&e);
  for (int w = 0; w < 3; ++w) dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(s);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    if (ms < best) best = ms;
  }
  // sustained: enough launches for ~4 s at the burst rate
  const int nl = (int)(4000.0f / best) + 1;
  cudaEventRecord(s);
  for (int r = 0; r < nl; ++r) dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float tot; cudaEventElapsedTime(&tot, s, e);
  const double burst = flop / (best * 1e-3) / 1e12, sust = flop * nl / (tot * 1e-3) / 1e12;
  const double nominal = sms * 64.0 * 2.0 * (clk * 1e3) / 1e12;
  printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_dfma_tflops_sustained\": %.3f, \"nominal_tflops_at_max_clock\": %.3f, "
         "\"sms\": %d, \"max_clock_mhz\": %.0f, \"sustained_launches\": %d, \"sustained_s\": %.2f, "
         "\"how\": \"8 DFMA chains x 256 threads x %d CTAs, 2 flop/FMA; burst = best of 10 launches, sustained = %d back-to-back launches\"}\n",
         burst, sust, nominal, sms, clk / 1e3, nl, tot / 1e3, blocks, nl);
  return 0;
}
