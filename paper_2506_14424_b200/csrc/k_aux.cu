// k_aux.cu — setup kernels, Carreau viscosity (K3), inverse diagonal (K5), transfer (K7),
// vector kernels: launchers.
#include "tu_tables.cuh"
#include "aux_kernels.cuh"
#include "launch.h"

#include <algorithm>

namespace dgvv {

cudaError_t upload_tables_aux(const Tab1D* tabs) { return tu_upload_tables(tabs); }

static inline int nblk(long n, int bs = 256) { return (int)((n + bs - 1) / bs); }
static inline int gs_blocks(long n) {
  long b = (n + 255) / 256;
  return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

// ---------------------------------------------------------------- K3
template <int n, int GEO>
static cudaError_t carreau_run(const NuArgs& a, cudaStream_t s) {
  constexpr int CPB = (128 / (n * n)) > 0 ? (128 / (n * n)) : 1;
  const size_t smem = (size_t)CPB * (3 * n * n * n + 3 * n * n) * sizeof(double);
  auto k = carreau_nu_kernel<n, GEO, CPB>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_optin(attr, smem, k); e != cudaSuccess) return e;
  if (a.n_total <= 0) return cudaSuccess;
  k<<<(a.n_total + CPB - 1) / CPB, CPB * n * n, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_carreau(int n, int geo, const NuArgs& a, cudaStream_t s) {
  switch (n) {
    case 2: return geo ? carreau_run<2, 1>(a, s) : carreau_run<2, 0>(a, s);
    case 3: return geo ? carreau_run<3, 1>(a, s) : carreau_run<3, 0>(a, s);
    case 4: return geo ? carreau_run<4, 1>(a, s) : carreau_run<4, 0>(a, s);
    case 5: return geo ? carreau_run<5, 1>(a, s) : carreau_run<5, 0>(a, s);
    case 6: return geo ? carreau_run<6, 1>(a, s) : carreau_run<6, 0>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- K5
template <int n, int NC, int FORM, int GEO>
static cudaError_t diag_run(const DiagArgs& a, cudaStream_t s) {
  const long tot = (long)a.n_owned * NC * n * n * n;
  if (tot <= 0) return cudaSuccess;
  diag_kernel<n, NC, FORM, GEO><<<nblk(tot), 256, 0, s>>>(a);
  return cudaGetLastError();
}

template <int n>
static cudaError_t diag_n(int nc, int form, int geo, const DiagArgs& a, cudaStream_t s) {
  if (nc == 1) return geo ? diag_run<n, 1, 1, 1>(a, s) : diag_run<n, 1, 1, 0>(a, s);
  if (form == 0) return geo ? diag_run<n, 3, 0, 1>(a, s) : diag_run<n, 3, 0, 0>(a, s);
  return geo ? diag_run<n, 3, 1, 1>(a, s) : diag_run<n, 3, 1, 0>(a, s);
}

cudaError_t launch_diag(int nc, int n, int form, int geo, const DiagArgs& a, cudaStream_t s) {
  switch (n) {
    case 2: return diag_n<2>(nc, form, geo, a, s);
    case 3: return diag_n<3>(nc, form, geo, a, s);
    case 4: return diag_n<4>(nc, form, geo, a, s);
    case 5: return diag_n<5>(nc, form, geo, a, s);
    case 6: return diag_n<6>(nc, form, geo, a, s);
    case 7: return diag_n<7>(nc, form, geo, a, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- K7
template <typename R, int nin, int nout>
static cudaError_t t3_run(int nc, const Mat8& M, const R* in, R* out, const R* add, double beta, int ncells, cudaStream_t s) {
  using Cf = T3Cfg<nin, nout>;
  constexpr int CPB = Cf::CPB;   // cells per CTA (teams of max(nin, nout)^2 threads)
  const size_t smem = (size_t)CPB * Cf::CS * sizeof(R);
  if (ncells <= 0) return cudaSuccess;
  const int grid = (ncells + CPB - 1) / CPB;
  if (nc == 3) tensor3_kernel<R, nin, nout, 3, CPB><<<grid, CPB * Cf::TS, smem, s>>>(M, in, out, add, (R)beta, ncells);
  else tensor3_kernel<R, nin, nout, 1, CPB><<<grid, CPB * Cf::TS, smem, s>>>(M, in, out, add, (R)beta, ncells);
  return cudaGetLastError();
}

template <typename R, int nin>
static cudaError_t t3_in(int nout, int nc, const Mat8& M, const R* in, R* out, const R* add, double beta,
                         int ncells, cudaStream_t s) {
  switch (nout) {
    case 2: return t3_run<R, nin, 2>(nc, M, in, out, add, beta, ncells, s);
    case 3: return t3_run<R, nin, 3>(nc, M, in, out, add, beta, ncells, s);
    case 4: return t3_run<R, nin, 4>(nc, M, in, out, add, beta, ncells, s);
    case 5: return t3_run<R, nin, 5>(nc, M, in, out, add, beta, ncells, s);
    case 6: return t3_run<R, nin, 6>(nc, M, in, out, add, beta, ncells, s);
    case 7: return t3_run<R, nin, 7>(nc, M, in, out, add, beta, ncells, s);
    default: return cudaErrorInvalidValue;
  }
}

template <typename R>
static cudaError_t tensor3_t(int nin, int nout, int nc, const double* M, const R* in, R* out, double beta,
                             int ncells, cudaStream_t s, const R* add) {
  if (!add) add = out;
  Mat8 m;
  for (int i = 0; i < DGVV_NMAX * DGVV_NMAX; ++i) m.m[i] = 0.0;
  for (int i = 0; i < nin * nout; ++i) m.m[i] = M[i];
  switch (nin) {
    case 2: return t3_in<R, 2>(nout, nc, m, in, out, add, beta, ncells, s);
    case 3: return t3_in<R, 3>(nout, nc, m, in, out, add, beta, ncells, s);
    case 4: return t3_in<R, 4>(nout, nc, m, in, out, add, beta, ncells, s);
    case 5: return t3_in<R, 5>(nout, nc, m, in, out, add, beta, ncells, s);
    case 6: return t3_in<R, 6>(nout, nc, m, in, out, add, beta, ncells, s);
    case 7: return t3_in<R, 7>(nout, nc, m, in, out, add, beta, ncells, s);
    default: return cudaErrorInvalidValue;
  }
}
cudaError_t launch_tensor3(int nin, int nout, int nc, const double* M, const double* in, double* out,
                           double beta, int ncells, cudaStream_t s, const double* add) {
  return tensor3_t<double>(nin, nout, nc, M, in, out, beta, ncells, s, add);
}
cudaError_t launch_tensor3_f(int nin, int nout, int nc, const double* M, const float* in, float* out,
                             double beta, int ncells, cudaStream_t s, const float* add) {
  return tensor3_t<float>(nin, nout, nc, M, in, out, beta, ncells, s, add);
}

// ---------------------------------------------------------------- setup
cudaError_t launch_cart_geom(const double* nodes, const int* nbr, int n_total, double* cart, cudaStream_t s) {
  cart_geom_kernel<<<nblk(n_total), 256, 0, s>>>(nodes, nbr, n_total, cart);
  return cudaGetLastError();
}

cudaError_t launch_cart_face(const int* nbr, int n_cells, double* cart, cudaStream_t s) {
  if (n_cells <= 0) return cudaSuccess;
  cart_face_kernel<<<nblk(n_cells), 256, 0, s>>>(nbr, n_cells, cart);
  return cudaGetLastError();
}

cudaError_t launch_cart_points(const double* cart, int n_owned, int n_total, int n, double* xq, double* xf,
                               cudaStream_t s) {
  Tab1D T;
  make_tab(n, &T);
  const long tot = (long)n_total * (n * n * n + 6 * n * n);
  cart_points_kernel<<<nblk(tot), 256, 0, s>>>(cart, n_owned, n_total, n, T, xq, xf);
  return cudaGetLastError();
}

cudaError_t launch_gen_geom(const GeoTab& g, const double* nodes, int n_total, double* vJi, double* jxw,
                            double* fJi, double* fdA, double* xq, double* xf, int* bad, cudaStream_t s) {
  const int n = g.n;
  const long tot = (long)n_total * (n * n * n + 6 * n * n);
  gen_geom_kernel<<<nblk(tot, 128), 128, 0, s>>>(g, nodes, n_total, vJi, jxw, fJi, fdA, xq, xf, bad);
  return cudaGetLastError();
}

cudaError_t launch_gen_H(const double* jxw, const double* fdA, const int* nbr, int n_total, int n, double* H,
                         cudaStream_t s) {
  gen_H_kernel<<<nblk(n_total), 256, 0, s>>>(jxw, fdA, nbr, n_total, n, H);
  return cudaGetLastError();
}

cudaError_t launch_align_check(const double* xf, const int* nbr, int n_owned, int n, double tol, int* bad,
                               cudaStream_t s) {
  align_check_kernel<<<nblk((long)n_owned * 6), 256, 0, s>>>(xf, nbr, n_owned, n, tol, bad);
  return cudaGetLastError();
}

cudaError_t launch_law_points(int kind, const double* p, const double* x, long npts, double* out, cudaStream_t s) {
  if (npts <= 0) return cudaSuccess;
  law_points_kernel<<<nblk(npts), 256, 0, s>>>(kind, nullptr, p[0], p[1], x, npts, out);
  return cudaGetLastError();
}

cudaError_t launch_range(const double* v, long n, double* bmin, double* bmax, int* bad, int nblocks,
                         cudaStream_t s) {
  range_kernel<<<nblocks, 256, 0, s>>>(v, n, bmin, bmax, bad);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- vectors
// thread-group allreduce: out[i] = sum over ranks (in rank order) of ranks[r][i] — every rank sums
// the same operands in the same order, so every rank holds the same bits
struct RankPtrs { const double* p[64]; };
__global__ void sum_ranks_kernel(RankPtrs P, int R, long count, double* out) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < R; ++r) s += P.p[r][i];     // rank order: the same sum on every rank
    out[i] = s;
  }
}
cudaError_t launch_sum_ranks(const double* const* ranks, int R, long count, double* out, cudaStream_t s) {
  RankPtrs P;
  for (int r = 0; r < R && r < 64; ++r) P.p[r] = ranks[r];
  const int blocks = (int)std::min<long>(148L * 8, std::max<long>(1, (count + 255) / 256));
  sum_ranks_kernel<<<blocks, 256, 0, s>>>(P, R, count, out);
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* a, const double* b, long n, double* part, int nblocks, double* out,
                       cudaStream_t s) {
  dot_partial_kernel<<<nblocks, 256, 0, s>>>(a, b, n, part);
  sum_partials_kernel<<<1, 256, 0, s>>>(part, nblocks, out);
  return cudaGetLastError();
}

cudaError_t launch_cheb_first(const double* b, const double* dinv, double c_r, double* d, double* x, long n,
                              cudaStream_t s) {
  cheb_first_kernel<double><<<gs_blocks(n), 256, 0, s>>>(b, dinv, c_r, d, x, n);
  return cudaGetLastError();
}
cudaError_t launch_cheb_first_f(const float* b, const float* dinv, double c_r, float* d, float* x, long n,
                                cudaStream_t s) {
  cheb_first_kernel<float><<<gs_blocks(n), 256, 0, s>>>(b, dinv, (float)c_r, d, x, n);
  return cudaGetLastError();
}
cudaError_t launch_d2f(const double* a, float* out, long n, cudaStream_t s) {
  d2f_kernel<<<gs_blocks(n), 256, 0, s>>>(a, out, n);
  return cudaGetLastError();
}
cudaError_t launch_f2d(const float* a, double* out, long n, cudaStream_t s) {
  f2d_kernel<<<gs_blocks(n), 256, 0, s>>>(a, out, n);
  return cudaGetLastError();
}
cudaError_t launch_ew_mul(const double* a, const double* b, double* out, long n, cudaStream_t s) {
  ew_mul_kernel<<<gs_blocks(n), 256, 0, s>>>(a, b, out, n);
  return cudaGetLastError();
}
cudaError_t launch_axpby(double alpha, const double* x, double beta, double* y, long n, cudaStream_t s) {
  axpby_kernel<<<gs_blocks(n), 256, 0, s>>>(alpha, x, beta, y, n);
  return cudaGetLastError();
}
cudaError_t launch_ew_sqrt(const double* a, double* out, long n, cudaStream_t s) {
  ew_sqrt_kernel<<<gs_blocks(n), 256, 0, s>>>(a, out, n);
  return cudaGetLastError();
}
cudaError_t launch_ew_div(const double* a, const double* b, double* out, long n, cudaStream_t s) {
  ew_div_kernel<<<gs_blocks(n), 256, 0, s>>>(a, b, out, n);
  return cudaGetLastError();
}
cudaError_t launch_lanczos_update(double* w, const double* q, const double* qprev, const double* alpha,
                                  const double* beta_prev, long n, cudaStream_t s) {
  lanczos_update_kernel<<<gs_blocks(n), 256, 0, s>>>(w, q, qprev, alpha, beta_prev, n);
  return cudaGetLastError();
}
cudaError_t launch_axpy_dev(const double* coef, double sgn, const double* x, double* y, long n, cudaStream_t s) {
  axpy_dev_kernel<<<gs_blocks(n), 256, 0, s>>>(coef, sgn, x, y, n);
  return cudaGetLastError();
}
cudaError_t launch_scale_by_inv(const double* w, const double* s2, double* q, long n, cudaStream_t s) {
  scale_by_inv_kernel<<<gs_blocks(n), 256, 0, s>>>(w, s2, q, n);
  return cudaGetLastError();
}
cudaError_t launch_gather_cells(const double* src, const int* list, int ncells, int len, double* out,
                                cudaStream_t s) {
  if ((long)ncells * len <= 0) return cudaSuccess;
  gather_cells_kernel<double><<<nblk((long)ncells * len), 256, 0, s>>>(src, list, ncells, len, out);
  return cudaGetLastError();
}
cudaError_t launch_gather_cells_f(const float* src, const int* list, int ncells, int len, float* out,
                                  cudaStream_t s) {
  if ((long)ncells * len <= 0) return cudaSuccess;
  gather_cells_kernel<float><<<nblk((long)ncells * len), 256, 0, s>>>(src, list, ncells, len, out);
  return cudaGetLastError();
}

}  // namespace dgvv
