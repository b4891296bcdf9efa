// dmma_dfma_mix.cu — do DMMA (FP64 tensor) and DFMA (FP64 CUDA cores) share one pipe on B200?
// Half of the warps of every CTA run m8n8k4 DMMA chains, the other half DFMA chains; the
// combined FLOP rate is compared with each alone.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__global__ void mix(double* out, int iters, int mode) {   // mode 0: dmma only, 1: dfma only, 2: half/half
  const int w = threadIdx.x / 32;
  const bool do_mma = mode == 0 || (mode == 2 && (w & 1) == 0);
  double s = 0;
  if (do_mma) {
    double c[8][2];
    double a = threadIdx.x * 1e-3, b = 0.5;
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) mma884(c[j], a, b);
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  } else {
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    // 8 DFMA per lane per j-step = 256 FMA per warp = one m8n8k4
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int r = 0; r < 8; ++r) x[r] = fma(x[r], 0.999999, 1e-7);
    for (int j = 0; j < 8; ++j) s += x[j];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  const int blocks = 148 * 8, threads = 256, iters = 2000;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    for (int w = 0; w < 2; ++w) mix<<<blocks, threads>>>(out, iters, mode);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      mix<<<blocks, threads>>>(out, iters, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    // every warp does 8*iters units of 256 FMA = 512 flop
    const double flops = 512.0 * 8 * iters * (double)blocks * threads / 32;
    printf("{\"mode\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f}\n", mode == 0 ? "dmma" : mode == 1 ? "dfma" : "half_dmma_half_dfma",
           flops / (best * 1e-3) / 1e12, best);
  }
  return 0;
}
