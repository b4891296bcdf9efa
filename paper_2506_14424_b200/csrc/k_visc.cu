// k_visc.cu — instantiations of the vector SIPG viscous apply (K1, with K6 epilogues).
#include "tu_tables.cuh"
#include "sipg_apply2.cuh"
#include "launch.h"

namespace dgvv {

cudaError_t upload_tables_visc(const Tab1D* tabs) { return tu_upload_tables(tabs); }

// cells per CTA and min resident CTAs per SM (register cap), chosen by measurement (DESIGN.md
// §11): n = 4 general geometry (C2) 2 cells x 8 CTAs (smem-bound by the TMA face stage; 4 x 4:
// +2 %);
// n = 4 Cartesian (C5) 4 x 6 (r02; r01: 4 x 8, 8 x 4: +2 %, 2 x 16: +3 %); n = 5 Cartesian (C3) 5 x 3 (125 threads: 98 % lane use).
#ifndef CPB4G
#define CPB4G 2
#endif
#ifndef MINB4G
#define MINB4G 8
#endif
#ifndef CPB4
#define CPB4 4
#endif
#ifndef MINB4
#define MINB4 6   // with the 2x2 lane-quad swizzle and early coefficient loads (r02): 6 > 7 = 8 (C5 2848 / 2897 / 2897 us)
#endif
#ifndef CPB5
#define CPB5 5
#endif
#ifndef MINB5
#define MINB5 3
#endif
#ifndef CPB3
#define CPB3 7
#endif
#ifndef CPB2
#define CPB2 32
#endif
template <int n, int GEO> constexpr int cpb_visc() {
  return n == 2 ? (GEO ? 32 : CPB2) : n == 3 ? (GEO ? 14 : CPB3) : n == 4 ? (GEO ? CPB4G : CPB4) : n == 5 ? CPB5 : 3;
}
#ifndef MINB2
#define MINB2 4
#endif
#ifndef MINB3
#define MINB3 8
#endif
#ifndef MINB23G
#define MINB23G 3   // general geometry n = 2, 3 (0: as Cartesian); 2 / 6 measured slower
#endif
template <int n, int GEO> constexpr int minb_visc() {
  return (GEO && (n == 2 || n == 3) && MINB23G > 0) ? MINB23G
         : n == 2 ? MINB2 : n == 3 ? MINB3 : n == 4 ? (GEO ? MINB4G : MINB4) : n == 5 ? MINB5 : 2;
}
// FP32 multigrid levels (half the registers and shared memory per cell)
#ifndef MINB5F
#define MINB5F 5
#endif
#ifndef MINB4F
#define MINB4F 6
#endif
#ifndef MINB2F
#define MINB2F 6
#endif
#ifndef MINB3F
#define MINB3F 5
#endif
#ifndef CPB4F
#define CPB4F 8
#endif
#ifndef CPB4GF
#define CPB4GF 4   // FP32 general geometry n = 4 (tuned with MINB4GF = 6)
#endif
#ifndef CPB3F
#define CPB3F 14
#endif
template <typename R, int n, int GEO> constexpr int cpb_visc_t() {
  return (sizeof(R) == 4 && n == 4) ? (GEO ? CPB4GF : CPB4F) : (sizeof(R) == 4 && n == 3) ? CPB3F
         : (sizeof(R) == 4 && n == 2) ? 32 : cpb_visc<n, GEO>();
}
#ifndef MINB4GF
#define MINB4GF 6
#endif
#ifndef MINBGF_COARSE
#define MINBGF_COARSE 6   // 0: as FP64
#endif
template <typename R, int n, int GEO> constexpr int minb_visc_t() {
  if constexpr (sizeof(R) == 4 && GEO == 0)
    return n == 2 ? MINB2F : n == 3 ? MINB3F : n == 4 ? MINB4F : n == 5 ? MINB5F : minb_visc<n, GEO>();
  else if constexpr (sizeof(R) == 4 && GEO == 1)
    return n == 4 ? MINB4GF : ((n == 2 || n == 3) && MINBGF_COARSE > 0) ? MINBGF_COARSE : minb_visc<n, GEO>();
  else
    return minb_visc<n, GEO>();
}

template <typename R, int n, int FORM, int GEO>
static cudaError_t run(const ApplyArgsT<R>& a, cudaStream_t s) {
  constexpr int CPB = cpb_visc_t<R, n, GEO>();
  constexpr int NC = 3;
  const size_t smem = (size_t)CPB * Apply2Cfg<n, NC, FORM, GEO>::CS * sizeof(R);
  // the Helmholtz mass term is a separate instantiation: the plain operator pays nothing for it
  auto k0 = sipg_apply2_kernel<R, n, NC, FORM, GEO, CPB, minb_visc_t<R, n, GEO>(), false>;
  auto k1 = sipg_apply2_kernel<R, n, NC, FORM, GEO, CPB, minb_visc_t<R, n, GEO>(), true>;
  // ghost face traces (communicator mode, boundary cells): a separate instantiation, so the
  // single-GPU / interior kernel carries no branch for them (measured: +4 % at C5 otherwise)
  auto k0t = sipg_apply2_kernel<R, n, NC, FORM, GEO, CPB, minb_visc_t<R, n, GEO>(), false, false, true>;
  auto k1t = sipg_apply2_kernel<R, n, NC, FORM, GEO, CPB, minb_visc_t<R, n, GEO>(), true, false, true>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_optin(attr, smem, k0, k1, k0t, k1t); e != cudaSuccess) return e;
#ifdef DGVV_CARVEOUT
  static std::atomic<uint64_t> attr_co{0};
  if (!(attr_co.load() & current_device_bit())) {
    cudaFuncSetAttribute(k0, cudaFuncAttributePreferredSharedMemoryCarveout, DGVV_CARVEOUT);
    attr_co.fetch_or(current_device_bit());
  }
#endif
  if (a.n_proc <= 0) return cudaSuccess;
  const int grid = (a.n_proc + CPB - 1) / CPB;
  if (a.gtr) (a.mass != 0.0 ? k1t : k0t)<<<grid, CPB * n * n, smem, s>>>(a);
  else if (a.mass != 0.0) k1<<<grid, CPB * n * n, smem, s>>>(a);
  else k0<<<grid, CPB * n * n, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename R, int n>
static cudaError_t run_n(int form, int geo, const ApplyArgsT<R>& a, cudaStream_t s) {
  if (form == 0) return geo == 0 ? run<R, n, 0, 0>(a, s) : run<R, n, 0, 1>(a, s);
  return geo == 0 ? run<R, n, 1, 0>(a, s) : run<R, n, 1, 1>(a, s);
}

template <typename R>
static cudaError_t launch_visc_t(int n, int form, int geo, const ApplyArgsT<R>& a, cudaStream_t s) {
  switch (n) {
    case 2: return run_n<R, 2>(form, geo, a, s);
    case 3: return run_n<R, 3>(form, geo, a, s);
    case 4: return run_n<R, 4>(form, geo, a, s);
    case 5: return run_n<R, 5>(form, geo, a, s);
    case 6: return run_n<R, 6>(form, geo, a, s);
    default: return cudaErrorInvalidValue;
  }
}

// f4: viscous apply with the convective term fused (divergence form, FP64, mass term included)
template <int n, int GEO>
static cudaError_t run_oseen(const ApplyArgs& a, cudaStream_t s) {
  constexpr int CPB = cpb_visc<n, GEO>();
  const size_t smem = (size_t)CPB * Apply2Cfg<n, 3, 0, GEO>::CS * sizeof(double);
  auto k = sipg_apply2_kernel<double, n, 3, 0, GEO, CPB, minb_visc<n, GEO>(), true, true>;
  auto kt = sipg_apply2_kernel<double, n, 3, 0, GEO, CPB, minb_visc<n, GEO>(), true, true, true>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_optin(attr, smem, k, kt); e != cudaSuccess) return e;
  if (a.n_proc <= 0) return cudaSuccess;
  (a.gtr ? kt : k)<<<(a.n_proc + CPB - 1) / CPB, CPB * n * n, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_apply_oseen(int n, int geo, const ApplyArgs& a, cudaStream_t s) {
  switch (n) {
    case 2: return geo ? run_oseen<2, 1>(a, s) : run_oseen<2, 0>(a, s);
    case 3: return geo ? run_oseen<3, 1>(a, s) : run_oseen<3, 0>(a, s);
    case 4: return geo ? run_oseen<4, 1>(a, s) : run_oseen<4, 0>(a, s);
    case 5: return geo ? run_oseen<5, 1>(a, s) : run_oseen<5, 0>(a, s);
    case 6: return geo ? run_oseen<6, 1>(a, s) : run_oseen<6, 0>(a, s);
    default: return cudaErrorNotSupported;
  }
}

// Face traces of owned cells for the ghost exchange: for every listed
// (cell, face) item the value and the reference normal derivative of each component at the face's
// n^2 points, out[((item * NC + c) * 2 + {0, 1}) * n^2 + p].  The line of point p = a + n b and the
// fma order are those of the apply kernel's own neighbour-trace loop, so a rank that reads these
// traces computes bit for bit what a single context computes from the neighbour's cell data.
template <typename R, int n, int NC>
__global__ void pack_traces_kernel(const R* __restrict__ src, const int* __restrict__ cells,
                                   const int* __restrict__ faces, int n_items, R* __restrict__ out) {
  constexpr int n2 = n * n, n3 = n * n * n;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)n_items * NC * n2) return;
  const int p = (int)(t % n2);
  const int c = (int)((t / n2) % NC);
  const int it = (int)(t / ((long)n2 * NC));
  const int f = faces[it], d = f >> 1;
  const int a = p % n, b = p / n;
  const R* u = src + (size_t)cells[it] * NC * n3 + c * n3;
  const Tab1D& T = c_tab[n];
  const double* lO = (f & 1) ? T.l1 : T.l0;
  const double* dO = (f & 1) ? T.d1 : T.d0;
  R x[n];
#pragma unroll
  for (int i = 0; i < n; ++i)
    x[i] = d == 0 ? u[b * n2 + a * n + i] : d == 1 ? u[b * n2 + i * n + a] : u[i * n2 + p];
  R v = R(0.0), g = R(0.0);
#pragma unroll
  for (int i = 0; i < n; ++i) { v = fma(R(lO[i]), x[i], v); g = fma(R(dO[i]), x[i], g); }
  out[((size_t)(it * NC + c) * 2) * n2 + p] = v;
  out[((size_t)(it * NC + c) * 2 + 1) * n2 + p] = g;
}

template <typename R>
static cudaError_t pack_traces_t(int nc, int n, const R* src, const int* cells, const int* faces, int n_items,
                                 R* out, cudaStream_t s) {
  if (n_items <= 0) return cudaSuccess;
  const long tot = (long)n_items * nc * n * n;
  const int blocks = (int)((tot + 255) / 256);
#define DGVV_PT(N)                                                                                      \
  case N:                                                                                               \
    if (nc == 3) pack_traces_kernel<R, N, 3><<<blocks, 256, 0, s>>>(src, cells, faces, n_items, out);   \
    else pack_traces_kernel<R, N, 1><<<blocks, 256, 0, s>>>(src, cells, faces, n_items, out);           \
    break;
  switch (n) {
    DGVV_PT(2) DGVV_PT(3) DGVV_PT(4) DGVV_PT(5) DGVV_PT(6) DGVV_PT(7)
    default: return cudaErrorNotSupported;
  }
#undef DGVV_PT
  return cudaGetLastError();
}
cudaError_t launch_pack_traces(int nc, int n, const double* src, const int* cells, const int* faces, int n_items,
                               double* out, cudaStream_t s) {
  return pack_traces_t<double>(nc, n, src, cells, faces, n_items, out, s);
}
cudaError_t launch_pack_traces_f(int nc, int n, const float* src, const int* cells, const int* faces, int n_items,
                                 float* out, cudaStream_t s) {
  return pack_traces_t<float>(nc, n, src, cells, faces, n_items, out, s);
}

cudaError_t launch_apply_visc(int n, int form, int geo, const ApplyArgs& a, cudaStream_t s) {
  return launch_visc_t<double>(n, form, geo, a, s);
}
// FP32 levels of the multigrid preconditioner
cudaError_t launch_apply_visc_f(int n, int form, int geo, const ApplyArgsT<float>& a, cudaStream_t s) {
  return launch_visc_t<float>(n, form, geo, a, s);
}

}  // namespace dgvv
