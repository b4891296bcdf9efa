// k_pen.cu — instantiations of the penalty-step operator (§8(f) f2): apply and inverse diagonal.
#include "tu_tables.cuh"
#include "penalty_apply.cuh"
#include "convective_apply.cuh"
#include "launch.h"

#include <algorithm>

namespace dgvv {

cudaError_t upload_tables_pen(const Tab1D* tabs) { return tu_upload_tables(tabs); }

template <int n> constexpr int cpb_pen() { return n == 2 ? 32 : n == 3 ? 14 : n == 4 ? 8 : n == 5 ? 5 : 3; }

template <int n, int GEO>
static cudaError_t pen_run(const PenaltyArgs& a, bool diag, cudaStream_t s) {
  if (diag) {
    const long tot = (long)a.n_owned * 3 * n * n * n;
    if (tot <= 0) return cudaSuccess;
    penalty_diag_kernel<n, GEO><<<(int)((tot + 255) / 256), 256, 0, s>>>(a);
    return cudaGetLastError();
  }
  constexpr int CPB = cpb_pen<n>();
  const size_t smem = (size_t)CPB * PenaltyCfg<n, GEO>::CS * sizeof(double);
  auto k = penalty_apply_kernel<n, GEO, CPB>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_optin(attr, smem, k); e != cudaSuccess) return e;
  if (a.n_proc <= 0) return cudaSuccess;
  k<<<(a.n_proc + CPB - 1) / CPB, CPB * n * n, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_penalty(int n, int geo, const PenaltyArgs& a, bool diag, cudaStream_t s) {
  switch (n) {
    case 2: return geo ? pen_run<2, 1>(a, diag, s) : pen_run<2, 0>(a, diag, s);
    case 3: return geo ? pen_run<3, 1>(a, diag, s) : pen_run<3, 0>(a, diag, s);
    case 4: return geo ? pen_run<4, 1>(a, diag, s) : pen_run<4, 0>(a, diag, s);
    case 5: return geo ? pen_run<5, 1>(a, diag, s) : pen_run<5, 0>(a, diag, s);
    case 6: return geo ? pen_run<6, 1>(a, diag, s) : pen_run<6, 0>(a, diag, s);
    default: return cudaErrorNotSupported;
  }
}

// f4: upwind convective term
template <int n, int GEO>
static cudaError_t conv_pd_run(const ConvArgs& a, double* wref, double* wface, cudaStream_t s) {
  const long tot = (long)a.n_owned * (n * n * n + 6 * n * n);
  if (tot <= 0) return cudaSuccess;
  const int blocks = (int)std::min<long>(148L * 16, (tot + 255) / 256);
  conv_pointdata_kernel<n, GEO><<<blocks, 256, 0, s>>>(a, wref, wface);
  return cudaGetLastError();
}

cudaError_t launch_conv_pointdata(int n, int geo, const ConvArgs& a, double* wref, double* wface, cudaStream_t s) {
  switch (n) {
    case 2: return geo ? conv_pd_run<2, 1>(a, wref, wface, s) : conv_pd_run<2, 0>(a, wref, wface, s);
    case 3: return geo ? conv_pd_run<3, 1>(a, wref, wface, s) : conv_pd_run<3, 0>(a, wref, wface, s);
    case 4: return geo ? conv_pd_run<4, 1>(a, wref, wface, s) : conv_pd_run<4, 0>(a, wref, wface, s);
    case 5: return geo ? conv_pd_run<5, 1>(a, wref, wface, s) : conv_pd_run<5, 0>(a, wref, wface, s);
    case 6: return geo ? conv_pd_run<6, 1>(a, wref, wface, s) : conv_pd_run<6, 0>(a, wref, wface, s);
    default: return cudaErrorNotSupported;
  }
}

template <int n>
static cudaError_t conv_pd_apply(const ConvArgs& a, const double* wref, const double* wface, cudaStream_t s) {
  constexpr int CPB = cpb_pen<n>();
  const size_t smem = (size_t)CPB * 2 * 3 * Lay<n>::CST * sizeof(double);
  auto k = convective_pd_kernel<n, CPB>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_optin(attr, smem, k); e != cudaSuccess) return e;
  if (a.n_proc <= 0) return cudaSuccess;
  k<<<(a.n_proc + CPB - 1) / CPB, CPB * n * n, smem, s>>>(a, wref, wface);
  return cudaGetLastError();
}

cudaError_t launch_convective_pd(int n, const ConvArgs& a, const double* wref, const double* wface, cudaStream_t s) {
  switch (n) {
    case 2: return conv_pd_apply<2>(a, wref, wface, s);
    case 3: return conv_pd_apply<3>(a, wref, wface, s);
    case 4: return conv_pd_apply<4>(a, wref, wface, s);
    case 5: return conv_pd_apply<5>(a, wref, wface, s);
    case 6: return conv_pd_apply<6>(a, wref, wface, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace dgvv
