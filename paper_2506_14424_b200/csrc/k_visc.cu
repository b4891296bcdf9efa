// k_visc.cu — instantiations of the vector SIPG viscous apply (K1, with K6 epilogues).
#include "tu_tables.cuh"
#include "sipg_apply.cuh"
#include "launch.h"

namespace dgvv {

cudaError_t upload_tables_visc(const Tab1D* tabs) { return tu_upload_tables(tabs); }

template <int n> constexpr int cpb_visc() { return (128 / (n * n)) > 0 ? (128 / (n * n)) : 1; }

template <int n, int FORM, int GEO>
static cudaError_t run(const ApplyArgs& a, cudaStream_t s) {
  constexpr int CPB = cpb_visc<n>();
  constexpr int NC = 3;
  const size_t smem = (size_t)CPB * 4 * NC * n * n * n * sizeof(double);
  auto k = sipg_apply_kernel<n, NC, FORM, GEO, CPB>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (a.n_proc <= 0) return cudaSuccess;
  const int grid = (a.n_proc + CPB - 1) / CPB;
  k<<<grid, CPB * n * n, smem, s>>>(a);
  return cudaGetLastError();
}

template <int n>
static cudaError_t run_n(int form, int geo, const ApplyArgs& a, cudaStream_t s) {
  if (form == 0) return geo == 0 ? run<n, 0, 0>(a, s) : run<n, 0, 1>(a, s);
  return geo == 0 ? run<n, 1, 0>(a, s) : run<n, 1, 1>(a, s);
}

cudaError_t launch_apply_visc(int n, int form, int geo, const ApplyArgs& a, cudaStream_t s) {
  switch (n) {
    case 2: return run_n<2>(form, geo, a, s);
    case 3: return run_n<3>(form, geo, a, s);
    case 4: return run_n<4>(form, geo, a, s);
    case 5: return run_n<5>(form, geo, a, s);
    case 6: return run_n<6>(form, geo, a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dgvv
