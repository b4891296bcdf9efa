// dmma_peak.cu — measured FP64 tensor-core (mma.sync f64) throughput on this B200, to decide
// whether the small sum-factorisation contractions can gain from DMMA (north_star: "tensor
// cores only if ncu shows ... gain").  8 independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double (&c)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma1688(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__global__ void k884(double* out, int iters) {
  double c[8][2];
  double a = threadIdx.x * 1e-3, b = 0.5;
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) mma884(c[j], a, b);
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k1684(double* out, int iters) {
  double c[8][4];
  double a = threadIdx.x * 1e-3, b = 0.5;
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) mma1684(c[j], a, a + 1, b);
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k1688(double* out, int iters) {
  double c[8][4];
  double a[4] = {threadIdx.x * 1e-3, 1, 2, 3}, b[2] = {0.5, 0.25};
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) mma1688(c[j], a, b);
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class K>
void run(const char* name, K kern, double fma_per_mma, int threads) {
  const int blocks = 148 * 8, iters = 2000;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t s, e;
  cudaEventCreate(&s); cudaEventCreate(&e);
  for (int w = 0; w < 2; ++w) kern<<<blocks, threads>>>(out, iters);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(s);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    if (ms < best) best = ms;
  }
  const double warps = (double)blocks * threads / 32;
  const double flops = 2.0 * fma_per_mma * 8 * (double)iters * warps;
  printf("{\"kernel\": \"%s\", \"threads\": %d, \"tflops\": %.3f, \"ms\": %.3f, \"err\": \"%s\"}\n", name, threads,
         flops / (best * 1e-3) / 1e12, best, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}
int main() {
  for (int t : {128, 256, 512}) {
    run("m8n8k4", k884, 8 * 8 * 4, t);
    run("m16n8k4", k1684, 16 * 8 * 4, t);
    run("m16n8k8", k1688, 16 * 8 * 8, t);
  }
  return 0;
}
