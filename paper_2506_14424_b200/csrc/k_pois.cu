// k_pois.cu — instantiations of the scalar SIPG Poisson apply (K4, with K6 epilogues).
#include "tu_tables.cuh"
#include "sipg_apply2.cuh"
#include "launch.h"

namespace dgvv {

cudaError_t launch_apply_visc(int n, int form, int geo, const ApplyArgs& a, cudaStream_t s);
cudaError_t launch_apply_visc_f(int n, int form, int geo, const ApplyArgsT<float>& a, cudaStream_t s);

cudaError_t upload_tables_pois(const Tab1D* tabs) { return tu_upload_tables(tabs); }

// n = 6 (C4, k = 5) FP64: 4 cells x 4 CTAs/SM.  With the Chebyshev epilogue's loads issued together
// (sipg_apply2.cuh) the smaller CTA wins everywhere: apply 1.110 -> 1.057 ms, Chebyshev(5) 5.72 ->
// 5.25 ms, V-cycle 19.98 -> 18.67 ms against 6 x 4 (5 x 4: 1.111 / 5.66 / 19.8); before that fix its
// apply-only gain was lost in the epilogue
#ifndef PCPB6
#define PCPB6 4
#endif
#ifndef PMINB6
#define PMINB6 4
#endif
#ifndef PCPB4
#define PCPB4 8
#endif
#ifndef PCPB3
#define PCPB3 14
#endif
template <int n> constexpr int cpb_pois() { return n == 2 ? 32 : n == 3 ? PCPB3 : n == 4 ? PCPB4 : n == 5 ? 5 : n == 6 ? PCPB6 : 3; }
#ifndef PCPB4F
#define PCPB4F 16
#endif
#ifndef PCPB6F
#define PCPB6F 8
#endif
template <typename R, int n> constexpr int cpb_pois_t() {
  return sizeof(R) == 4 ? (n == 4 ? PCPB4F : n == 6 ? PCPB6F : cpb_pois<n>()) : cpb_pois<n>();
}
#ifndef PMINB4
#define PMINB4 6
#endif
#ifndef PMINB3
#define PMINB3 5
#endif
#ifndef PMINB2
#define PMINB2 6
#endif
template <int n> constexpr int minb_pois() { return n == 2 ? PMINB2 : n == 3 ? PMINB3 : n == 6 ? PMINB6 : n == 4 ? PMINB4 : 4; }
// FP32 multigrid levels (half the registers and shared memory per cell)
#ifndef PMINB6F
#define PMINB6F 4
#endif
#ifndef PMINB4F
#define PMINB4F 4
#endif
#ifndef PMINB3F
#define PMINB3F 4
#endif
#ifndef PMINB2F
#define PMINB2F 4
#endif
template <typename R, int n> constexpr int minb_pois_t() {
  if constexpr (sizeof(R) == 4) return n == 2 ? PMINB2F : n == 3 ? PMINB3F : n == 4 ? PMINB4F : n == 6 ? PMINB6F : minb_pois<n>();
  else return minb_pois<n>();
}

template <typename R, int n, int GEO>
static cudaError_t run(const ApplyArgsT<R>& a, cudaStream_t s) {
  constexpr int CPB = cpb_pois_t<R, n>();
  const size_t smem = (size_t)CPB * Apply2Cfg<n, 1, 1, GEO>::CS * sizeof(R);
  auto k0 = sipg_apply2_kernel<R, n, 1, 1, GEO, CPB, minb_pois_t<R, n>(), false>;
  auto k1 = sipg_apply2_kernel<R, n, 1, 1, GEO, CPB, minb_pois_t<R, n>(), true>;
  auto k0t = sipg_apply2_kernel<R, n, 1, 1, GEO, CPB, minb_pois_t<R, n>(), false, false, true>;
  auto k1t = sipg_apply2_kernel<R, n, 1, 1, GEO, CPB, minb_pois_t<R, n>(), true, false, true>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_optin(attr, smem, k0, k1, k0t, k1t); e != cudaSuccess) return e;
  if (a.n_proc <= 0) return cudaSuccess;
  const int grid = (a.n_proc + CPB - 1) / CPB;
  if (a.gtr) (a.mass != 0.0 ? k1t : k0t)<<<grid, CPB * n * n, smem, s>>>(a);
  else if (a.mass != 0.0) k1<<<grid, CPB * n * n, smem, s>>>(a);
  else k0<<<grid, CPB * n * n, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename R>
static cudaError_t launch_pois_t(int n, int geo, const ApplyArgsT<R>& a, cudaStream_t s) {
  switch (n) {
    case 2: return geo ? run<R, 2, 1>(a, s) : run<R, 2, 0>(a, s);
    case 3: return geo ? run<R, 3, 1>(a, s) : run<R, 3, 0>(a, s);
    case 4: return geo ? run<R, 4, 1>(a, s) : run<R, 4, 0>(a, s);
    case 5: return geo ? run<R, 5, 1>(a, s) : run<R, 5, 0>(a, s);
    case 6: return geo ? run<R, 6, 1>(a, s) : run<R, 6, 0>(a, s);
    case 7: return geo ? run<R, 7, 1>(a, s) : run<R, 7, 0>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_apply(int nc, int n, int form, int geo, const ApplyArgs& a, cudaStream_t s) {
  if (nc == 3) return launch_apply_visc(n, form, geo, a, s);
  return launch_pois_t<double>(n, geo, a, s);
}
cudaError_t launch_apply_f(int nc, int n, int form, int geo, const ApplyArgsT<float>& a, cudaStream_t s) {
  if (nc == 3) return launch_apply_visc_f(n, form, geo, a, s);
  return launch_pois_t<float>(n, geo, a, s);
}

}  // namespace dgvv
