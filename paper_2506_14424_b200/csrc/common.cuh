// common.cuh — shared definitions of the dgvv CUDA library (sm_100a, FP64).
// Included by every translation unit; each TU owns a private copy of the 1D tables in
// __constant__ memory (uploaded by that TU's upload function, see tables.cpp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#ifndef __CUDACC_RTC__
#include <atomic>
#endif

#define DGVV_NMAX 8        // max points per direction (degree <= 7)
#ifndef DGVV_MINB
#define DGVV_MINB 1        // min resident CTAs per SM requested from ptxas for the apply kernel
#endif

// 1D tables of the degree-(n-1) Lagrange basis on the n Gauss-Legendre points of [0,1]
// (readings G1/G2).  Computed on the host by tables.cpp (Newton iteration on P_n and the
// barycentric formulas) — independent of the oracle.
struct Tab1D {
  double D[DGVV_NMAX * DGVV_NMAX];   // D[q*NMAX + i] = l_i'(x_q)
  double x[DGVV_NMAX];               // Gauss points on [0,1]
  double w[DGVV_NMAX];               // Gauss weights on [0,1]
  double l0[DGVV_NMAX], l1[DGVV_NMAX];   // l_i(0), l_i(1)
  double d0[DGVV_NMAX], d1[DGVV_NMAX];   // l_i'(0), l_i'(1)
};

// Boundary codes in the device neighbour table (int32): >= 0 local cell index
#define NB_DIRICHLET (-2)
#define NB_NEUMANN (-3)
#define NB_REMOTE (-100)   // neighbour of a ghost row that is not present locally (H only)

// Per-cell geometry of the Cartesian fast path (axis-aligned boxes):
//   [0..2] 1/h_x,1/h_y,1/h_z  [3] H_K  [4] h_x h_y h_z  [5..7] x0   (8 doubles)
// Cartesian cell record: [1/hx 1/hy 1/hz H V x0 y0 z0 | per face f: 1/h_d of the neighbour across f,
// max(H, H_neighbour)] (own values on boundary faces): the face terms read their neighbour data
// from the cell's own record instead of chasing the neighbour's (ncu: 3 % of stall samples)
#define CART_STRIDE 20
#define CART_FACE 8

// Streamed metric terms of the general (iso-parametric) path, per level:
//   vJi[cell][9][n^3]     : Ji[k][j] = d xi_k / d x_j at cell points (row-major k,j)
//   fJi[cell][6][9][n^2]  : own-side Ji at face points; the outward unit normal is
//                           n = s J^-T e_d / |J^-T e_d| (recomputed), dA = JxW-like weight
//   jxw[cell][n^3], fdA[cell][6][n^2]: JxW and dA (setup; premultiplied by nu for the apply)

enum { MODE_APPLY = 0, MODE_RESID = 1, MODE_CHEB = 2 };

template <typename R>
struct ApplyArgsT {  // R = double (operators) or float (FP32 multigrid levels)
  const R* src;        // owned cells [n_owned][NC][n^3]
  const R* ghost;      // ghost cells [n_ghost][NC][n^3] (may be null)
  R* dst;
  const int* nbr;           // [n_total][6]
  const int* cell_list;     // cells to process (null: cell_base .. cell_base+n_proc-1)
  int n_proc;
  int cell_base;
  int n_owned;
  // coefficient at quadrature points.  Cartesian: nu itself; general geometry:
  // premultiplied weights nu*JxW (cells) and nu*dA (own face points).
  const R* nu_cell;    // [n_owned][n^3]
  const R* nu_face;    // [n_total][6][n^2]
  const R* cart;       // [n_total][CART_STRIDE]      (Cartesian)
  const R* vJi;        // [n_total][9][n^3]  J^-1 at cell points        (general)
  const R* fJi;        // [n_total][6][9][n^2] own J^-1 at face points  (general)
  const R* Hcell;      // [n_total]                   (general)
  double pen;               // IP (k+1)^2
  double mass;              // Helmholtz: + mass * M (diagonal, M_ii = JxW_i per component)
  // epilogue
  int mode;
  const R* b;          // RESID / CHEB
  const R* dinv;       // CHEB
  R* dvec;             // CHEB: d in/out
  R* xout;             // CHEB: x_{j+1}
  double c_rho, c_r;        // CHEB: d = c_rho d + c_r Dinv r
  // Newton (linearised) extras
  const R* ulin;       // owned u_lin
  const R* ulin_ghost; // ghost u_lin
  const R* jxw;        // general geometry: JxW [n_owned][n^3]
  const R* fdA;        // general geometry: dA  [n_total][6][n^2]
  double law[4];            // eta0, eta_inf, lambda, n
  // f4 fused convective term (CONV instantiation): + alpha_c C(w) src
  const R* wref;       // JxW J^-1 w at cell points [n_owned][3][n^3] (convective_apply.cuh)
  const R* wface;      // min({{w}}.n, 0) dA at own face points [n_owned][6][n^2]
  // K2 v3 (newton_apply3.cuh): point data of the linearisation point (Cartesian)
  const R* npc;        // [n_owned][7][n^3]  S0 (6), g at cell points
  const R* npf;        // [n_total][6][10][n^2]  S0 (6), g, u0 trace (3) at own face points
  double alpha_c;
  // multi-rank with a communicator: ghost neighbours' face traces instead of whole ghost cells.
  // gtr[((item * NC + c) * 2 + {0: value, 1: d/dxi_n}) * n^2 + face point], item = gslot[g * 6 + f]
  // for ghost g's face f (null: traces computed from the ghost cells in `ghost`)
  const R* gtr;
  const int* gslot;
};
using ApplyArgs = ApplyArgsT<double>;

// f2 penalty-step operator (penalty_apply.cuh)
struct PenaltyArgs {
  const double* src;
  const double* ghost;
  double* dst;
  const int* nbr;
  int n_proc, n_owned, cell_base;
  const double* cart;       // Cartesian geometry
  const double* vJi;        // general: J^-1 at cell points
  const double* jxw;        // general: JxW at cell points
  const double* fJi;        // general: own J^-1 at face points (normal)
  const double* fdA;        // general: dA at own face points
  const double* tau_div;    // [n_total]
  const double* tau_cont;   // [n_total]
};

// f4 convective term (convective_apply.cuh): dst += alpha C(w) src
struct ConvArgs {
  const double* src;
  const double* ghost;
  const double* w;
  const double* wghost;
  double* dst;
  const int* nbr;
  int n_proc, n_owned, cell_base;
  const double* cart;
  const double* vJi;
  const double* jxw;
  const double* fJi;
  const double* fdA;
  double alpha;
  int accumulate;           // 1: dst += alpha C src, 0: dst = alpha C src
};

struct NuArgs {
  const double* u;          // owned [n_owned][3][n^3]
  const double* ughost;     // ghost [n_ghost][3][n^3]
  int n_owned, n_total;
  const double* cart;
  const double* vJi;        // general: [n_total][9][n^3]
  const double* fJi;        // general: [n_total][6][9][n^2]
  double law[4];
  double* nu_cell;          // [n_owned][n^3]
  double* nu_face;          // [n_total][6][n^2]
  int* bad;                 // counts points with nu <= 0 or non-finite (domain check)
};

struct DiagArgs {
  const int* nbr;
  int n_owned;
  const double* nu_cell;    // Cartesian: nu; general: nu*JxW
  const double* nu_face;    // Cartesian: nu; general: nu*dA
  const double* cart;
  const double* vJi;
  const double* fJi;
  const double* Hcell;
  double pen;
  double mass;              // + mass * JxW_i on the diagonal (Helmholtz operator)
  const double* jxw;        // general geometry: JxW [n_owned][n^3]
  double* out;              // 1 / D
};

#define DGVV_CUDA_TRY(expr)                                                        \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "%s: %s (%s:%d)", #expr,   \
                                            cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

__host__ __device__ inline int face_t1(int d) { return d == 0 ? 1 : 0; }
__host__ __device__ inline int face_t2(int d) { return d == 2 ? 1 : 2; }

#ifndef __CUDACC_RTC__
namespace dgvv {
// Per-DEVICE one-time host setup: bit d of `done` is set once device d (the current
// device) has the dynamic shared-memory opt-in of the kernels `ks`.  A second device in the same
// process gets its own opt-in; concurrent first calls at worst set the attribute twice.
inline uint64_t current_device_bit() {
  int d = 0;
  cudaGetDevice(&d);
  return 1ull << (d & 63);
}
// SM count of the current device (persistent launches), cached per device
inline int sm_count() {
  static std::atomic<int> cache[64];
  int d = 0;
  cudaGetDevice(&d);
  int v = cache[d & 63].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) v = 148;
    cache[d & 63].store(v, std::memory_order_relaxed);
  }
  return v;
}
template <typename... K>
inline cudaError_t smem_optin(std::atomic<uint64_t>& done, size_t smem, K... ks) {
  const uint64_t bit = current_device_bit();
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  ((e = (e == cudaSuccess) ? cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) : e), ...);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}
}  // namespace dgvv
#endif
