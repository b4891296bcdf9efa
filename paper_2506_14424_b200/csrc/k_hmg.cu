// k_hmg.cu — §8(f) f3: h-multigrid transfer between nested refinements and the dense direct
// coarse solver ("h-coarsening … the individual h-levels are created by
// refining an initial coarse grid"; "a direct solver if the system size falls below 2000 DoFs").
//
// Transfer (readings H1/H2): a fine cell is the octant (ox, oy, oz) of its parent's reference
// cube; P restricted to it is Ph[oz] (x) Ph[oy] (x) Ph[ox] with Ph[o][i][j] = l_j((xi_i + o)/2)
// (the parent's degree-k Lagrange basis at the child's Gauss points).  Prolongation is
// fine-centric (gather of the parent), restriction coarse-centric (sum over the 8 children in
// octant order): no atomics, deterministic.  Both are HBM-bound streams of (1 + 8 / 8) vectors.
//
// Direct solve (H3): the coarsest operator is assembled column by column from the matrix-free
// apply (A e_j), inverted once by Gauss-Jordan elimination without pivoting (the SIPG / Helmholtz
// operators are SPD), and applied as a dense matvec (one warp per row).
#include "common.cuh"
#include "launch.h"
#include "tables.h"

#include <algorithm>
#include <cstring>

namespace dgvv {

// x-fastest three-pass tensor contraction of one n^3 block with per-direction matrices
// (M?[i_out * n + j_in]); in/out in shared memory; t = thread index in the team of T threads
template <int n, int T, typename R>
__device__ inline void tensor3_dir(const R* Mx, const R* My, const R* Mz, const R* in, R* s1, R* s2, R* out,
                                   int t) {
  constexpr int n2 = n * n, n3 = n2 * n;
  for (int i = t; i < n3; i += T) {               // x
    const int xo = i % n, r = i / n;
    R acc = R(0);
#pragma unroll
    for (int k = 0; k < n; ++k) acc = fma(Mx[xo * n + k], in[r * n + k], acc);
    s1[i] = acc;
  }
  __syncwarp();
  __syncthreads();
  for (int i = t; i < n3; i += T) {               // y
    const int xo = i % n, yo = (i / n) % n, z = i / n2;
    R acc = R(0);
#pragma unroll
    for (int k = 0; k < n; ++k) acc = fma(My[yo * n + k], s1[z * n2 + k * n + xo], acc);
    s2[i] = acc;
  }
  __syncthreads();
  for (int i = t; i < n3; i += T) {               // z
    const int r = i % n2, zo = i / n2;
    R acc = R(0);
#pragma unroll
    for (int k = 0; k < n; ++k) acc = fma(Mz[zo * n + k], s2[k * n2 + r], acc);
    out[i] = acc;
  }
  __syncthreads();
}

struct HMats {
  double P[2][DGVV_NMAX * DGVV_NMAX];    // Ph[o][i_f * n + j_c]
  double PT[2][DGVV_NMAX * DGVV_NMAX];   // Ph[o]^T [j_c * n + i_f]
};

constexpr int HT = 64;   // threads per block (one (cell, component) block at a time)

// fine[f][c] = P_oct(f) coarse[parent[f]][c] + beta fine[f][c]
template <int n, typename R>
__global__ void __launch_bounds__(HT) hprolong_kernel(HMats M, const R* coarse, R* fine, const int* parent,
                                                      const signed char* octant, int nc, R beta, int n_fine) {
  constexpr int n3 = n * n * n;
  __shared__ R sin_[n3], s1[n3], s2[n3], sout[n3];
  __shared__ R sm[3][n * n];
  const int f = blockIdx.x;
  const int oc = octant[f];
  const int p = parent[f];
  for (int i = threadIdx.x; i < n * n; i += HT) {
    sm[0][i] = R(M.P[oc & 1][i]);
    sm[1][i] = R(M.P[(oc >> 1) & 1][i]);
    sm[2][i] = R(M.P[(oc >> 2) & 1][i]);
  }
  for (int c = 0; c < nc; ++c) {
    for (int i = threadIdx.x; i < n3; i += HT) sin_[i] = coarse[((size_t)p * nc + c) * n3 + i];
    __syncthreads();
    tensor3_dir<n, HT, R>(sm[0], sm[1], sm[2], sin_, s1, s2, sout, threadIdx.x);
    for (int i = threadIdx.x; i < n3; i += HT) {
      const size_t o = ((size_t)f * nc + c) * n3 + i;
      fine[o] = beta == R(0) ? sout[i] : sout[i] + beta * fine[o];
    }
    __syncthreads();
  }
}

// coarse[p][c] = sum_{oct} P_oct^T fine[child[p][oct]][c] + beta coarse[p][c]
template <int n, typename R>
__global__ void __launch_bounds__(HT) hrestrict_kernel(HMats M, const R* fine, R* coarse, const int* child,
                                                       int nc, R beta, int n_coarse) {
  constexpr int n3 = n * n * n;
  __shared__ R sin_[n3], s1[n3], s2[n3], sout[n3];
  __shared__ R sm[2][n * n];
  const int p = blockIdx.x;
  for (int i = threadIdx.x; i < n * n; i += HT) {
    sm[0][i] = R(M.PT[0][i]);
    sm[1][i] = R(M.PT[1][i]);
  }
  __syncthreads();
  for (int c = 0; c < nc; ++c) {
    R acc[(n3 + HT - 1) / HT];
#pragma unroll
    for (int r = 0; r < (n3 + HT - 1) / HT; ++r) acc[r] = R(0);
    for (int oc = 0; oc < 8; ++oc) {
      const int f = child[p * 8 + oc];
      for (int i = threadIdx.x; i < n3; i += HT) sin_[i] = fine[((size_t)f * nc + c) * n3 + i];
      __syncthreads();
      tensor3_dir<n, HT, R>(sm[oc & 1], sm[(oc >> 1) & 1], sm[(oc >> 2) & 1], sin_, s1, s2, sout, threadIdx.x);
#pragma unroll
      for (int r = 0; r < (n3 + HT - 1) / HT; ++r) {
        const int i = threadIdx.x + r * HT;
        if (i < n3) acc[r] += sout[i];
      }
    }
#pragma unroll
    for (int r = 0; r < (n3 + HT - 1) / HT; ++r) {
      const int i = threadIdx.x + r * HT;
      if (i < n3) {
        const size_t o = ((size_t)p * nc + c) * n3 + i;
        coarse[o] = beta == R(0) ? acc[r] : acc[r] + beta * coarse[o];
      }
    }
  }
}

static HMats make_hmats(int n) {
  HMats M;
  std::memset(&M, 0, sizeof(M));
  double x[DGVV_NMAX], w[DGVV_NMAX];
  gauss01(n, x, w);
  for (int o = 0; o < 2; ++o)
    for (int i = 0; i < n; ++i) {
      double v[DGVV_NMAX], d[DGVV_NMAX];
      lagrange_at(x, n, 0.5 * (x[i] + o), v, d);
      for (int j = 0; j < n; ++j) {
        M.P[o][i * n + j] = v[j];
        M.PT[o][j * n + i] = v[j];
      }
    }
  return M;
}

template <typename R>
static cudaError_t hprolong_t(int n, int nc, const R* coarse, R* fine, const int* parent, const signed char* octant,
                              double beta, int n_fine, cudaStream_t s) {
  if (n_fine <= 0) return cudaSuccess;
  const HMats M = make_hmats(n);
  switch (n) {
#define HP(N) case N: hprolong_kernel<N, R><<<n_fine, HT, 0, s>>>(M, coarse, fine, parent, octant, nc, R(beta), n_fine); break;
    HP(2) HP(3) HP(4) HP(5) HP(6)
#undef HP
    default: return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

template <typename R>
static cudaError_t hrestrict_t(int n, int nc, const R* fine, R* coarse, const int* child, double beta, int n_coarse,
                               cudaStream_t s) {
  if (n_coarse <= 0) return cudaSuccess;
  const HMats M = make_hmats(n);
  switch (n) {
#define HR(N) case N: hrestrict_kernel<N, R><<<n_coarse, HT, 0, s>>>(M, fine, coarse, child, nc, R(beta), n_coarse); break;
    HR(2) HR(3) HR(4) HR(5) HR(6)
#undef HR
    default: return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

cudaError_t launch_hprolongate(int n, int nc, const double* coarse, double* fine, const int* parent,
                               const signed char* octant, double beta, int n_fine, cudaStream_t s) {
  return hprolong_t<double>(n, nc, coarse, fine, parent, octant, beta, n_fine, s);
}
cudaError_t launch_hprolongate_f(int n, int nc, const float* coarse, float* fine, const int* parent,
                                 const signed char* octant, double beta, int n_fine, cudaStream_t s) {
  return hprolong_t<float>(n, nc, coarse, fine, parent, octant, beta, n_fine, s);
}
cudaError_t launch_hrestrict(int n, int nc, const double* fine, double* coarse, const int* child, double beta,
                             int n_coarse, cudaStream_t s) {
  return hrestrict_t<double>(n, nc, fine, coarse, child, beta, n_coarse, s);
}
cudaError_t launch_hrestrict_f(int n, int nc, const float* fine, float* coarse, const int* child, double beta,
                               int n_coarse, cudaStream_t s) {
  return hrestrict_t<float>(n, nc, fine, coarse, child, beta, n_coarse, s);
}

// ------------------------------------------------------------------ dense direct solver
__global__ void set_unit_kernel(double* v, long n, long j) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    v[i] = i == j ? 1.0 : 0.0;
}

// W[r][c] (row-major, N x 2N) = [A | I] with A[r][c] = cols[c * N + r] (cols[c] = A e_c)
__global__ void gj_init_kernel(const double* cols, double* W, int N) {
  const long tot = (long)N * 2 * N;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / (2 * N)), c = (int)(i % (2 * N));
    W[i] = c < N ? cols[(size_t)c * N + r] : (c - N == r ? 1.0 : 0.0);
  }
}

// step k: fac[r] = W[r][k] / W[k][k]; pivot check
__global__ void gj_factor_kernel(const double* W, double* fac, int N, int k, int* bad) {
  const double piv = W[(size_t)k * 2 * N + k];
  if (blockIdx.x == 0 && threadIdx.x == 0 && !(piv > 0.0)) atomicAdd(bad, 1);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x)
    fac[r] = W[(size_t)r * 2 * N + k] / piv;
}

// W[r][c] -= fac[r] W[k][c] for r != k, c in (k, N + k] (columns <= k of A are already reduced
// except column k itself, which becomes 0 and is never read again)
__global__ void gj_elim_kernel(double* W, const double* fac, int N, int k) {
  const int width = N;                            // columns k+1 .. N+k (right of N+k row k is 0)
  const long tot = (long)N * width;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / width), c = k + 1 + (int)(i % width);
    if (r == k) continue;
    W[(size_t)r * 2 * N + c] -= fac[r] * W[(size_t)k * 2 * N + c];
  }
}

__global__ void gj_scale_kernel(double* W, const double* fac, int N, int k) {
  const double inv = 1.0 / W[(size_t)k * 2 * N + k];
  for (int c = k + 1 + blockIdx.x * blockDim.x + threadIdx.x; c <= N + k; c += gridDim.x * blockDim.x)
    W[(size_t)k * 2 * N + c] *= inv;
}

// Ainv (row-major N x N) = right half of W
__global__ void gj_extract_kernel(const double* W, double* Ainv, int N) {
  const long tot = (long)N * N;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / N), c = (int)(i % N);
    Ainv[i] = W[(size_t)r * 2 * N + N + c];
  }
}

// x = Ainv b, one warp per row (row-major, coalesced); FP64 accumulation for FP32 vectors too
// (the paper's coarse solver runs in double precision)
// (multi-rank: rows = this rank's owned DoFs of the replicated inverse, b the gathered full vector)
template <typename RB, typename R>
__global__ void dense_matvec_kernel(const double* Ainv, const RB* b, R* x, int N, int rows) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const double* row = Ainv + (size_t)warp * N;
  double acc = 0.0;
  for (int c = lane; c < N; c += 32) acc = fma(row[c], (double)b[c], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) x[warp] = R(acc);
}

static inline int blocks_for(long n) { return (int)std::min<long>(148L * 16, std::max<long>(1, (n + 255) / 256)); }

cudaError_t launch_set_unit(double* v, long n, long j, cudaStream_t s) {
  set_unit_kernel<<<blocks_for(n), 256, 0, s>>>(v, n, j);
  return cudaGetLastError();
}

cudaError_t launch_gauss_jordan_inverse(const double* cols, double* W, double* fac, double* Ainv, int N, int* bad,
                                        cudaStream_t s) {
  gj_init_kernel<<<blocks_for(2L * N * N), 256, 0, s>>>(cols, W, N);
  for (int k = 0; k < N; ++k) {
    gj_factor_kernel<<<blocks_for(N), 256, 0, s>>>(W, fac, N, k, bad);
    gj_elim_kernel<<<blocks_for((long)N * N), 256, 0, s>>>(W, fac, N, k);
    gj_scale_kernel<<<blocks_for(N), 256, 0, s>>>(W, fac, N, k);
  }
  gj_extract_kernel<<<blocks_for((long)N * N), 256, 0, s>>>(W, Ainv, N);
  return cudaGetLastError();
}

cudaError_t launch_dense_matvec(const double* Ainv, const double* b, double* x, int N, cudaStream_t s, int rows) {
  if (rows < 0) rows = N;
  if (rows == 0) return cudaSuccess;
  dense_matvec_kernel<double, double><<<(rows * 32 + 255) / 256, 256, 0, s>>>(Ainv, b, x, N, rows);
  return cudaGetLastError();
}
cudaError_t launch_dense_matvec_df(const double* Ainv, const double* b, float* x, int N, cudaStream_t s, int rows) {
  if (rows < 0) rows = N;
  if (rows == 0) return cudaSuccess;
  dense_matvec_kernel<double, float><<<(rows * 32 + 255) / 256, 256, 0, s>>>(Ainv, b, x, N, rows);
  return cudaGetLastError();
}
cudaError_t launch_dense_matvec_f(const double* Ainv, const float* b, float* x, int N, cudaStream_t s, int rows) {
  if (rows < 0) rows = N;
  if (rows == 0) return cudaSuccess;
  dense_matvec_kernel<float, float><<<(rows * 32 + 255) / 256, 256, 0, s>>>(Ainv, b, x, N, rows);
  return cudaGetLastError();
}

}  // namespace dgvv
