// k_cg.cu — §8(f) f3, the c-level of the cph hierarchy ("first the
// conversion from a discontinuous to a continuous polynomial space is performed"): the
// continuous Q1 space on the mesh of a degree-1 DG level (readings C1-C3).
//  * embedding P_c (C1): per cell the trilinear corner functions at the 2^3 Gauss points,
//    E(q, o) = prod_a E1[q_a][o_a], E1[i][o] = (1 - xi_i, xi_i)[o];
//  * its transpose as a vertex-centric gather over the (cell, corner) incidences of each vertex
//    (CSR built on the host): no atomics, deterministic;
//  * nested Q1 h-transfer (C3) and its transpose as CSR sparse matrices (host-built), applied
//    per component;
//  * probing kernels for the diagonal of A_c = P_c^T A_DG P_c (vertex colouring: vertices of one
//    colour share no cell, so (A_c s)_v = (A_c)_vv for the colour's indicator s);
//  * the Chebyshev vector update of the continuous level.
// Layouts: DG_1 vector [cell][c][q] (8 per cell and component), continuous vector [c][v].
#include "common.cuh"
#include "launch.h"
#include "tables.h"

#include <algorithm>

namespace dgvv {

struct E1Tab { double e[2][2]; };   // e[i][o] = value of corner function o at Gauss point i

__device__ __forceinline__ double e3(const E1Tab& E, int q, int o) {
  return E.e[q & 1][o & 1] * E.e[(q >> 1) & 1][(o >> 1) & 1] * E.e[(q >> 2) & 1][(o >> 2) & 1];
}

static inline int gblocks(long n) { return (int)std::min<long>(148L * 16, std::max<long>(1, (n + 255) / 256)); }

// dg[(cell * nc + c) * 8 + q] = sum_o E(q, o) cg[c * nv + vid[cell * 8 + o]] + beta dg[...]
__global__ void cg_embed_kernel(E1Tab E, const double* cg, double* dg, const int* vid, int n_cells, int nv, int nc,
                                double beta) {
  const long tot = (long)n_cells * nc * 8;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (long)gridDim.x * blockDim.x) {
    const int q = (int)(i & 7);
    const long cc = i >> 3;
    const int c = (int)(cc % nc);
    const int cell = (int)(cc / nc);
    double s = 0.0;
#pragma unroll
    for (int o = 0; o < 8; ++o) s = fma(e3(E, q, o), cg[(size_t)c * nv + vid[cell * 8 + o]], s);
    dg[i] = beta == 0.0 ? s : s + beta * dg[i];
  }
}

// cg[c * nv + v] = sum over incidences (cell, o) of v of sum_q E(q, o) dg[(cell * nc + c) * 8 + q]
__global__ void cg_embedT_kernel(E1Tab E, const double* dg, double* cg, const int* inc_ptr, const int* inc, int nv,
                                 int nc, double beta) {
  const long tot = (long)nv * nc;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i / nv), v = (int)(i % nv);
    double s = 0.0;
    for (int j = inc_ptr[v]; j < inc_ptr[v + 1]; ++j) {
      const int cell = inc[j] >> 3, o = inc[j] & 7;
      const double* d = dg + ((size_t)cell * nc + c) * 8;
#pragma unroll
      for (int q = 0; q < 8; ++q) s = fma(e3(E, q, o), d[q], s);
    }
    cg[i] = beta == 0.0 ? s : s + beta * cg[i];
  }
}

// y[c * nrows + r] = sum_j val[j] x[c * ncols + col[j]] + beta y[...]   (per component)
__global__ void csr_spmv_kernel(const int* ptr, const int* col, const double* val, const double* x, double* y,
                                int nrows, int ncols, int nc, double beta) {
  const long tot = (long)nrows * nc;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i / nrows), r = (int)(i % nrows);
    double s = 0.0;
    for (int j = ptr[r]; j < ptr[r + 1]; ++j) s = fma(val[j], x[(size_t)c * ncols + col[j]], s);
    y[i] = beta == 0.0 ? s : s + beta * y[i];
  }
}

// probe vector of colour k, component comp;  diag extraction of the same
__global__ void cg_probe_set_kernel(double* s, const int* color, int k, int comp, int nv, int nc) {
  const long tot = (long)nv * nc;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i / nv), v = (int)(i % nv);
    s[i] = (c == comp && color[v] == k) ? 1.0 : 0.0;
  }
}
__global__ void cg_probe_get_kernel(const double* y, double* diag, const int* color, int k, int comp, int nv) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x)
    if (color[v] == k) diag[(size_t)comp * nv + v] = y[(size_t)comp * nv + v];
}

// Chebyshev step on a plain vector: d = c_rho d + c_r dinv r;  x += d   (c_rho = 0: first step)
__global__ void cheb_vec_kernel(const double* r, const double* dinv, double c_rho, double c_r, double* d, double* x,
                                long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const double dn = c_r * dinv[i] * r[i] + (c_rho != 0.0 ? c_rho * d[i] : 0.0);
    d[i] = dn;
    x[i] += dn;
  }
}

static E1Tab make_e1() {
  E1Tab E;
  double x[DGVV_NMAX], w[DGVV_NMAX];
  gauss01(2, x, w);
  for (int i = 0; i < 2; ++i) {
    E.e[i][0] = 1.0 - x[i];
    E.e[i][1] = x[i];
  }
  return E;
}

cudaError_t launch_cg_embed(const double* cg, double* dg, const int* vid, int n_cells, int nv, int nc, double beta,
                            cudaStream_t s) {
  cg_embed_kernel<<<gblocks((long)n_cells * nc * 8), 256, 0, s>>>(make_e1(), cg, dg, vid, n_cells, nv, nc, beta);
  return cudaGetLastError();
}
cudaError_t launch_cg_embedT(const double* dg, double* cg, const int* inc_ptr, const int* inc, int nv, int nc,
                             double beta, cudaStream_t s) {
  cg_embedT_kernel<<<gblocks((long)nv * nc), 256, 0, s>>>(make_e1(), dg, cg, inc_ptr, inc, nv, nc, beta);
  return cudaGetLastError();
}
cudaError_t launch_csr_spmv(const int* ptr, const int* col, const double* val, const double* x, double* y, int nrows,
                            int ncols, int nc, double beta, cudaStream_t s) {
  csr_spmv_kernel<<<gblocks((long)nrows * nc), 256, 0, s>>>(ptr, col, val, x, y, nrows, ncols, nc, beta);
  return cudaGetLastError();
}
cudaError_t launch_cg_probe_set(double* sv, const int* color, int k, int comp, int nv, int nc, cudaStream_t s) {
  cg_probe_set_kernel<<<gblocks((long)nv * nc), 256, 0, s>>>(sv, color, k, comp, nv, nc);
  return cudaGetLastError();
}
// The same step from an operator product: r = b - Ax formed in the kernel (the penalty smoother's
// residual axpby and Chebyshev update in one pass: 7 instead of 9 vector streams per step)
__global__ void cheb_vec_resid_kernel(const double* __restrict__ Ax, const double* __restrict__ b,
                                      const double* __restrict__ dinv, double c_rho, double c_r, double* d, double* x,
                                      long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const double r = 1.0 * b[i] + (-1.0) * Ax[i];
    const double dn = c_r * dinv[i] * r + (c_rho != 0.0 ? c_rho * d[i] : 0.0);
    d[i] = dn;
    x[i] += dn;
  }
}
cudaError_t launch_cheb_vec_resid(const double* Ax, const double* b, const double* dinv, double c_rho, double c_r,
                                  double* d, double* x, long n, cudaStream_t s) {
  cheb_vec_resid_kernel<<<gblocks(n), 256, 0, s>>>(Ax, b, dinv, c_rho, c_r, d, x, n);
  return cudaGetLastError();
}
cudaError_t launch_cg_probe_get(const double* y, double* diag, const int* color, int k, int comp, int nv,
                                cudaStream_t s) {
  cg_probe_get_kernel<<<gblocks(nv), 256, 0, s>>>(y, diag, color, k, comp, nv);
  return cudaGetLastError();
}
cudaError_t launch_cheb_vec(const double* r, const double* dinv, double c_rho, double c_r, double* d, double* x,
                            long n, cudaStream_t s) {
  cheb_vec_kernel<<<gblocks(n), 256, 0, s>>>(r, dinv, c_rho, c_r, d, x, n);
  return cudaGetLastError();
}

}  // namespace dgvv
