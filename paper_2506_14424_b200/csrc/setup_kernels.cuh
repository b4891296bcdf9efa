// setup_kernels.cuh — geometry, coefficient evaluation (a2), alignment
// check, coefficient range checks.  Setup-time kernels; not on the per-apply path.
#pragma once
#include "common.cuh"
#include "tables.h"
#include "laws.cuh"

namespace dgvv {

// ----------------------------------------------------------------- Cartesian geometry
// cart[cell] = {1/hx, 1/hy, 1/hz, H, hx hy hz, x0, y0, z0} from corners 0 and 7.
// H_K = (sum_interior A_f / 2 + sum_boundary A_f) / V   (reading G3)
__global__ void cart_geom_kernel(const double* nodes, const int* nbr, int n_total, double* cart) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_total) return;
  const double* X = nodes + (size_t)c * 8 * 3;
  double h[3], x0[3];
  for (int d = 0; d < 3; ++d) { x0[d] = X[d]; h[d] = X[7 * 3 + d] - X[d]; }
  const double V = h[0] * h[1] * h[2];
  double num = 0.0;
  for (int f = 0; f < 6; ++f) {
    const int d = f / 2;
    const double A = V / h[d];
    const int nb = nbr[c * 6 + f];
    num += (nb == NB_DIRICHLET || nb == NB_NEUMANN) ? A : 0.5 * A;
  }
  double* o = cart + (size_t)c * CART_STRIDE;
  o[0] = 1.0 / h[0]; o[1] = 1.0 / h[1]; o[2] = 1.0 / h[2];
  o[3] = num / V; o[4] = V;
  o[5] = x0[0]; o[6] = x0[1]; o[7] = x0[2];
}

// per-face neighbour data of the Cartesian record (after cart_geom_kernel: reads the neighbours')
__global__ void cart_face_kernel(const int* nbr, int n_cells, double* cart) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  double* o = cart + (size_t)c * CART_STRIDE;
  for (int f = 0; f < 6; ++f) {
    const int nb = nbr[c * 6 + f];
    const double* q = cart + (size_t)(nb >= 0 ? nb : c) * CART_STRIDE;
    o[CART_FACE + 2 * f] = q[f / 2];
    o[CART_FACE + 2 * f + 1] = fmax(o[3], q[3]);
  }
}

// physical points for Cartesian cells: xq [cell][n^3][3], xf [cell][6][n^2][3]
__global__ void cart_points_kernel(const double* cart, int n_owned, int n_total, int n, Tab1D T,
                                   double* xq, double* xf) {
  const int n2 = n * n, n3 = n2 * n, P = n3 + 6 * n2;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)n_total * P) return;
  const int c = idx / P, r = idx % P;
  const double* g = cart + (size_t)c * CART_STRIDE;
  const double h[3] = {1.0 / g[0], 1.0 / g[1], 1.0 / g[2]};
  double xi[3];
  if (r < n3) {
    if (c >= n_owned) return;
    xi[0] = T.x[r % n]; xi[1] = T.x[(r / n) % n]; xi[2] = T.x[r / n2];
    for (int d = 0; d < 3; ++d) xq[((size_t)c * n3 + r) * 3 + d] = g[5 + d] + h[d] * xi[d];
  } else {
    const int f = (r - n3) / n2, p = (r - n3) % n2, d = f / 2, s = f % 2;
    xi[d] = s;
    xi[face_t1(d)] = T.x[p % n];
    xi[face_t2(d)] = T.x[p / n];
    for (int e = 0; e < 3; ++e) xf[(((size_t)c * 6 + f) * n2 + p) * 3 + e] = g[5 + e] + h[e] * xi[e];
  }
}

// ----------------------------------------------------------------- general geometry
// x(xi) = sum_a X_a L_a(xi) over the (m+1)^3 GLL nodes; J_{i,k} = d x_i / d xi_k.
// vJi[cell][9][n^3] (J^-1 row-major k,j), jxw; fJi[cell][6][9][n^2] (own J^-1 at face points),
// fdA = det J |J^-T N| w_a w_b (Nanson; the unit normal is recomputed from J^-1), xq, xf points.
__global__ void gen_geom_kernel(GeoTab G, const double* nodes, int n_total, double* vJi, double* jxw,
                                double* fJi, double* fdA, double* xq, double* xf, int* bad) {
  const int n = G.n, m1 = G.m + 1, n2 = n * n, n3 = n2 * n, P = n3 + 6 * n2;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)n_total * P) return;
  const int c = idx / P, r = idx % P;
  const double* Lx; const double* Ly; const double* Lz;
  const double* dLx; const double* dLy; const double* dLz;
  double w;
  int f = -1, p = 0, d = 0, s = 0;
  if (r < n3) {
    const int qx = r % n, qy = (r / n) % n, qz = r / n2;
    Lx = G.L[qx]; Ly = G.L[qy]; Lz = G.L[qz];
    dLx = G.dL[qx]; dLy = G.dL[qy]; dLz = G.dL[qz];
    w = G.w[qx] * G.w[qy] * G.w[qz];
  } else {
    f = (r - n3) / n2; p = (r - n3) % n2; d = f / 2; s = f % 2;
    const int ta = p % n, tb = p / n;
    const double* Lt[3]; const double* dLt[3];
    Lt[d] = G.E[s]; dLt[d] = G.dE[s];
    Lt[face_t1(d)] = G.L[ta]; dLt[face_t1(d)] = G.dL[ta];
    Lt[face_t2(d)] = G.L[tb]; dLt[face_t2(d)] = G.dL[tb];
    Lx = Lt[0]; Ly = Lt[1]; Lz = Lt[2]; dLx = dLt[0]; dLy = dLt[1]; dLz = dLt[2];
    w = G.w[ta] * G.w[tb];
  }
  const double* X = nodes + (size_t)c * m1 * m1 * m1 * 3;
  double x[3] = {0, 0, 0}, J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int az = 0; az < m1; ++az)
    for (int ay = 0; ay < m1; ++ay)
      for (int ax = 0; ax < m1; ++ax) {
        const double* Xa = X + ((az * m1 + ay) * m1 + ax) * 3;
        const double v = Lx[ax] * Ly[ay] * Lz[az];
        const double gx = dLx[ax] * Ly[ay] * Lz[az];
        const double gy = Lx[ax] * dLy[ay] * Lz[az];
        const double gz = Lx[ax] * Ly[ay] * dLz[az];
        for (int i = 0; i < 3; ++i) {
          x[i] += Xa[i] * v;
          J[i][0] += Xa[i] * gx;
          J[i][1] += Xa[i] * gy;
          J[i][2] += Xa[i] * gz;
        }
      }
  const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                     J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                     J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  if (!(det > 0.0)) atomicAdd(bad, 1);
  const double id = 1.0 / det;
  double Ji[9];   // Ji[k][j] = (J^-1)_{kj} = cofactor(J)_{jk} / det
  Ji[0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * id;
  Ji[1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
  Ji[2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
  Ji[3] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * id;
  Ji[4] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
  Ji[5] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
  Ji[6] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * id;
  Ji[7] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
  Ji[8] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
  if (f < 0) {
    double* o = vJi + (size_t)c * 9 * n3 + r;
    for (int k = 0; k < 9; ++k) o[k * n3] = Ji[k];
    jxw[(size_t)c * n3 + r] = det * w;
    for (int i = 0; i < 3; ++i) xq[((size_t)c * n3 + r) * 3 + i] = x[i];
  } else {
    const double v0 = Ji[3 * d], v1 = Ji[3 * d + 1], v2 = Ji[3 * d + 2];
    const double ln = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
    double* o = fJi + ((size_t)c * 6 + f) * 9 * n2 + p;
    for (int k = 0; k < 9; ++k) o[k * n2] = Ji[k];
    fdA[((size_t)c * 6 + f) * n2 + p] = det * ln * w;
    for (int i = 0; i < 3; ++i) xf[(((size_t)c * 6 + f) * n2 + p) * 3 + i] = x[i];
  }
}

// H_K from the streamed metric: V = sum JxW, A_f = sum dA  (G3)
__global__ void gen_H_kernel(const double* jxw, const double* fdA, const int* nbr, int n_total,
                             int n, double* H) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_total) return;
  const int n2 = n * n, n3 = n2 * n;
  double V = 0.0;
  for (int q = 0; q < n3; ++q) V += jxw[(size_t)c * n3 + q];
  double num = 0.0;
  for (int f = 0; f < 6; ++f) {
    double A = 0.0;
    for (int p = 0; p < n2; ++p) A += fdA[((size_t)c * 6 + f) * n2 + p];
    const int nb = nbr[c * 6 + f];
    num += (nb == NB_DIRICHLET || nb == NB_NEUMANN) ? A : 0.5 * A;
  }
  H[c] = num / V;
}

// Structured-alignment check: point p of face f of cell c must coincide with point p of face
// f^1 of its neighbour up to one translation per face (periodic shift).
__global__ void align_check_kernel(const double* xf, const int* nbr, int n_owned, int n, double tol,
                                   int* bad) {
  const int n2 = n * n;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)n_owned * 6) return;
  const int c = idx / 6, f = idx % 6;
  const int nb = nbr[c * 6 + f];
  if (nb < 0) return;
  const double* A = xf + ((size_t)c * 6 + f) * n2 * 3;
  const double* B = xf + ((size_t)nb * 6 + (f ^ 1)) * n2 * 3;
  const double s0 = A[0] - B[0], s1 = A[1] - B[1], s2 = A[2] - B[2];
  for (int p = 0; p < n2; ++p) {
    const double e0 = A[3 * p] - B[3 * p] - s0, e1 = A[3 * p + 1] - B[3 * p + 1] - s1,
                 e2 = A[3 * p + 2] - B[3 * p + 2] - s2;
    if (fabs(e0) + fabs(e1) + fabs(e2) > tol) { atomicAdd(bad, 1); return; }
  }
}

// ----------------------------------------------------------------- analytic coefficient
__global__ void law_points_kernel(int kind, const double* __restrict__ pp_unused, double p0,
                                  double p1, const double* x, long npts, double* out) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  const double p[2] = {p0, p1};
  out[i] = eval_law(kind, p, x[3 * i], x[3 * i + 1], x[3 * i + 2]);
}

// min / max / count of non-positive-or-non-finite over an array (per-block partials)
__global__ void range_kernel(const double* v, long n, double* bmin, double* bmax, int* bad) {
  __shared__ double smin[256], smax[256];
  double lo = INFINITY, hi = -INFINITY;
  int nb = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const double x = v[i];
    if (!(x > 0.0) || !isfinite(x)) ++nb;
    lo = fmin(lo, x);
    hi = fmax(hi, x);
  }
  if (nb) atomicAdd(bad, nb);
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { bmin[blockIdx.x] = smin[0]; bmax[blockIdx.x] = smax[0]; }
}

}  // namespace dgvv
