// lds_patterns.cu — shared-memory load cost (L1 wavefronts per warp instruction) of the access
// patterns the apply kernel uses, measured with ncu (l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld
// / smsp__inst_executed_op_shared_ld).  One kernel per pattern; each warp issues ITER loads.
#include <cstdio>
#include <cuda_runtime.h>
#define ITER 4096
template <int P>
__global__ void lds_kernel(double* out, int sel) {
  __shared__ __align__(16) double sm[4096 + 1024];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31, a = lane & 3, b = (lane >> 2) & 3, cell = lane >> 4;
  int off;
  double acc = 0.0;
  // P0: LDS.128 all lanes one address; P1: LDS.128 8 distinct rows, groups of 4 consecutive lanes,
  // contiguous (row = lane/4); P2: as P1 but the two half-warps 1 KB apart (2 cells, row = b);
  // P3: LDS.128 8 distinct, interleaved (row = lane % 8); P4: LDS.128 16 distinct (pairs);
  // P5: LDS.128 32 distinct contiguous; P6: LDS.64 column pattern (addr = cell*CS + k*RS + a, 8 distinct);
  // P7: LDS.64 32 distinct contiguous; P8: LDS.64 8 distinct, groups of 4 consecutive lanes.
  if (P == 0) off = 0;
  else if (P == 1) off = 2 * (lane >> 2);
  else if (P == 2) off = cell * 128 + b * 4;
  else if (P == 3) off = 2 * (lane & 7);
  else if (P == 4) off = 2 * (lane >> 1);
  else if (P == 5) off = 2 * lane;
  else if (P == 6) off = cell * 128 + a;
  else if (P == 7) off = lane;
  else if (P == 8) off = lane >> 2;
  // P9: 8 distinct, groups of 4 consecutive lanes, group stride 9 doubles (distinct banks, not contiguous)
  else if (P == 9) off = 9 * (lane >> 2);
  // P10: the volume y-contraction pattern: a = lane & 3 (interleaved sharing), cells 840 doubles apart
  else if (P == 10) off = cell * 840 + a;
  // P11: consecutive-lane sharing within each cell (addr = b), cells 840 apart
  else if (P == 11) off = cell * 840 + b;
  // P12: interleaved sharing, cells adjacent (cell * 4 + a)
  else if (P == 12) off = cell * 4 + a;
  // P13: interleaved sharing in one cell only (all 32 lanes: addr = lane & 3)
  else if (P == 13) off = a;
  // P14: interleaved sharing, 8 distinct: addr = lane & 7
  else if (P == 14) off = lane & 7;
  // P15: all lanes one address (LDS.64)
  else off = 0;
#pragma unroll 4
  for (int it = 0; it < ITER; ++it) {
    const int o = (off + (it & 7) * 256 * sel) % 4096;
    if (P <= 5) {
      const double2 v = *reinterpret_cast<const double2*>(sm + (o & ~1));
      acc += v.x * v.y;
    } else {
      acc += sm[o];
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 256 * sizeof(double));
  lds_kernel<0><<<148, 256>>>(out, 1);
  lds_kernel<1><<<148, 256>>>(out, 1);
  lds_kernel<2><<<148, 256>>>(out, 1);
  lds_kernel<3><<<148, 256>>>(out, 1);
  lds_kernel<4><<<148, 256>>>(out, 1);
  lds_kernel<5><<<148, 256>>>(out, 1);
  lds_kernel<6><<<148, 256>>>(out, 1);
  lds_kernel<7><<<148, 256>>>(out, 1);
  lds_kernel<8><<<148, 256>>>(out, 1);
  lds_kernel<9><<<148, 256>>>(out, 1);
  lds_kernel<10><<<148, 256>>>(out, 1);
  lds_kernel<11><<<148, 256>>>(out, 1);
  lds_kernel<12><<<148, 256>>>(out, 1);
  lds_kernel<13><<<148, 256>>>(out, 1);
  lds_kernel<14><<<148, 256>>>(out, 1);
  lds_kernel<15><<<148, 256>>>(out, 1);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
