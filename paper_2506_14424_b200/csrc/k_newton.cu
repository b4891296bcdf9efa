// k_newton.cu — instantiations of the Newton-linearised viscous apply (K2).
#include "tu_tables.cuh"
#include "newton_apply.cuh"
#include "newton_apply3.cuh"
#include "launch.h"

#include <algorithm>

namespace dgvv {

cudaError_t upload_tables_newton(const Tab1D* tabs) { return tu_upload_tables(tabs); }

template <int n> constexpr int cpb_newton() { return n == 2 ? 16 : n == 3 ? 8 : n == 4 ? 4 : n == 5 ? 3 : 2; }

#ifndef NCPB5
#define NCPB5 1
#endif
#ifndef NMINB5
#define NMINB5 10
#endif
// Cartesian cells: newton_apply3_kernel from stored point data of u0 (the v2 kernel that
// recomputed u0's gradients every apply was 5.21 ms vs 3.92 ms on C3; removed)
template <int n> constexpr int cpb_newton2() { return n == 2 ? 16 : n == 3 ? 6 : n == 4 ? 2 : n == 5 ? NCPB5 : 1; }
template <int n> constexpr int minb_newton2() { return n == 5 ? NMINB5 : n == 4 ? 4 : 2; }

template <int n>
static cudaError_t run2(const ApplyArgs& a, cudaStream_t s) {
  constexpr int CPB = cpb_newton2<n>();
  const size_t smem = (size_t)CPB * Newton3Cfg<n>::CS * sizeof(double);
  auto k = newton_apply3_kernel<n, CPB, minb_newton2<n>()>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_optin(attr, smem, k); e != cudaSuccess) return e;
  if (a.n_proc <= 0) return cudaSuccess;
  k<<<(a.n_proc + CPB - 1) / CPB, CPB * n * n, smem, s>>>(a);
  return cudaGetLastError();
}

template <int n, int GEO>
static cudaError_t run(const ApplyArgs& a, cudaStream_t s) {
  if constexpr (GEO == 0) return run2<n>(a, s);
  constexpr int CPB = cpb_newton<n>();
  const size_t smem = (size_t)CPB * NewtonCfg<n, GEO>::CS * sizeof(double);
  auto k = newton_apply_kernel<n, GEO, CPB, 1>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_optin(attr, smem, k); e != cudaSuccess) return e;
  if (a.n_proc <= 0) return cudaSuccess;
  k<<<(a.n_proc + CPB - 1) / CPB, CPB * n * n, smem, s>>>(a);
  return cudaGetLastError();
}

bool newton_uses_pointdata(int geo) { return geo == 0; }

template <int n>
static cudaError_t npd_run(const ApplyArgs& a, int n_total, double* pc, double* pf, cudaStream_t s) {
  const long tot = (long)a.n_owned * n * n * n + (long)n_total * 6 * n * n;
  if (tot <= 0) return cudaSuccess;
  const int blocks = (int)std::min<long>(148L * 16, (tot + 255) / 256);
  newton_pointdata_kernel<n><<<blocks, 256, 0, s>>>(a, n_total, pc, pf);
  return cudaGetLastError();
}

cudaError_t launch_newton_pointdata(int n, const ApplyArgs& a, int n_total, double* pc, double* pf, cudaStream_t s) {
  switch (n) {
    case 2: return npd_run<2>(a, n_total, pc, pf, s);
    case 3: return npd_run<3>(a, n_total, pc, pf, s);
    case 4: return npd_run<4>(a, n_total, pc, pf, s);
    case 5: return npd_run<5>(a, n_total, pc, pf, s);
    case 6: return npd_run<6>(a, n_total, pc, pf, s);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t launch_newton(int n, int geo, const ApplyArgs& a, cudaStream_t s) {
  switch (n) {
    case 2: return geo ? run<2, 1>(a, s) : run<2, 0>(a, s);
    case 3: return geo ? run<3, 1>(a, s) : run<3, 0>(a, s);
    case 4: return geo ? run<4, 1>(a, s) : run<4, 0>(a, s);
    case 5: return geo ? run<5, 1>(a, s) : run<5, 0>(a, s);
    case 6: return geo ? run<6, 1>(a, s) : run<6, 0>(a, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace dgvv
