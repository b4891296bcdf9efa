// launch.h — host-side launchers exported by the kernel translation units.
#pragma once
#include "common.cuh"
#include "tables.h"

namespace dgvv {


// each kernel TU owns a private __constant__ copy of the tables
cudaError_t upload_tables_visc(const Tab1D* tabs);
cudaError_t upload_tables_pois(const Tab1D* tabs);
cudaError_t upload_tables_aux(const Tab1D* tabs);
cudaError_t upload_tables_newton(const Tab1D* tabs);
cudaError_t upload_tables_pen(const Tab1D* tabs);

// K1 / K4 / K6: SIPG apply with epilogue (nc = 3 viscous, 1 Poisson)
cudaError_t launch_apply(int nc, int n, int form, int geo, const ApplyArgs& a, cudaStream_t s);
// FP32 variant (multigrid preconditioner levels)
cudaError_t launch_apply_f(int nc, int n, int form, int geo, const ApplyArgsT<float>& a, cudaStream_t s);
// f2: divergence/continuity penalty operator (apply, or inverse diagonal when diag = true)
cudaError_t launch_penalty(int n, int geo, const PenaltyArgs& a, bool diag, cudaStream_t s);
// f4: viscous apply (divergence form, + mass M) with the convective term alpha_c C(w) fused in
cudaError_t launch_apply_oseen(int n, int geo, const ApplyArgs& a, cudaStream_t s);
// f4: quadrature-point data of the convective term for the fused apply (wref, wface)
cudaError_t launch_conv_pointdata(int n, int geo, const ConvArgs& a, double* wref, double* wface, cudaStream_t s);
// f4: dst (+)= alpha C(w) src from the stored point data
cudaError_t launch_convective_pd(int n, const ConvArgs& a, const double* wref, const double* wface, cudaStream_t s);
// f3: h-transfer between nested refinements (octant = ox + 2 oy + 4 oz; child[p * 8 + octant])
cudaError_t launch_hprolongate(int n, int nc, const double* coarse, double* fine, const int* parent,
                               const signed char* octant, double beta, int n_fine, cudaStream_t s);
cudaError_t launch_hrestrict(int n, int nc, const double* fine, double* coarse, const int* child, double beta,
                             int n_coarse, cudaStream_t s);
cudaError_t launch_hprolongate_f(int n, int nc, const float* coarse, float* fine, const int* parent,
                                 const signed char* octant, double beta, int n_fine, cudaStream_t s);
cudaError_t launch_hrestrict_f(int n, int nc, const float* fine, float* coarse, const int* child, double beta,
                               int n_coarse, cudaStream_t s);
// f3: dense direct coarse solver (Gauss-Jordan inverse of the assembled operator, dense matvec)
cudaError_t launch_set_unit(double* v, long n, long j, cudaStream_t s);
cudaError_t launch_gauss_jordan_inverse(const double* cols, double* W, double* fac, double* Ainv, int N, int* bad,
                                        cudaStream_t s);
// x[0:rows] = Ainv[0:rows][0:N] b  (rows < 0: N)
cudaError_t launch_dense_matvec(const double* Ainv, const double* b, double* x, int N, cudaStream_t s, int rows = -1);
cudaError_t launch_dense_matvec_f(const double* Ainv, const float* b, float* x, int N, cudaStream_t s, int rows = -1);
cudaError_t launch_dense_matvec_df(const double* Ainv, const double* b, float* x, int N, cudaStream_t s, int rows = -1);
// f3 c-level: continuous Q1 level (embedding, transpose, CSR transfers, diagonal probing, Chebyshev)
cudaError_t launch_cg_embed(const double* cg, double* dg, const int* vid, int n_cells, int nv, int nc, double beta,
                            cudaStream_t s);
cudaError_t launch_cg_embedT(const double* dg, double* cg, const int* inc_ptr, const int* inc, int nv, int nc,
                             double beta, cudaStream_t s);
cudaError_t launch_csr_spmv(const int* ptr, const int* col, const double* val, const double* x, double* y, int nrows,
                            int ncols, int nc, double beta, cudaStream_t s);
cudaError_t launch_cg_probe_set(double* sv, const int* color, int k, int comp, int nv, int nc, cudaStream_t s);
cudaError_t launch_cg_probe_get(const double* y, double* diag, const int* color, int k, int comp, int nv,
                                cudaStream_t s);
cudaError_t launch_cheb_vec(const double* r, const double* dinv, double c_rho, double c_r, double* d, double* x,
                            long n, cudaStream_t s);
// K2 v3: point data of the linearisation point (Cartesian), derived once per update_viscosity
bool newton_uses_pointdata(int geo);
cudaError_t launch_newton_pointdata(int n, const ApplyArgs& a, int n_total, double* pc, double* pf, cudaStream_t s);
// K2: Newton-linearised viscous apply
cudaError_t launch_newton(int n, int geo, const ApplyArgs& a, cudaStream_t s);
// K3: Carreau viscosity at all points
cudaError_t launch_carreau(int n, int geo, const NuArgs& a, cudaStream_t s);
// K5: inverse diagonal
cudaError_t launch_diag(int nc, int n, int form, int geo, const DiagArgs& a, cudaStream_t s);
// K7: out = (M x M x M) in + beta add  (add = out when null)
cudaError_t launch_tensor3(int nin, int nout, int nc, const double* M, const double* in, double* out,
                           double beta, int ncells, cudaStream_t s, const double* add = nullptr);
cudaError_t launch_tensor3_f(int nin, int nout, int nc, const double* M, const float* in, float* out,
                             double beta, int ncells, cudaStream_t s, const float* add = nullptr);

// setup kernels
cudaError_t launch_cart_geom(const double* nodes, const int* nbr, int n_total, double* cart, cudaStream_t s);
cudaError_t launch_cart_face(const int* nbr, int n_cells, double* cart, cudaStream_t s);
cudaError_t launch_cart_points(const double* cart, int n_owned, int n_total, int n, double* xq, double* xf,
                               cudaStream_t s);
cudaError_t launch_gen_geom(const GeoTab& g, const double* nodes, int n_total, double* vJi, double* jxw,
                            double* fJi, double* fdA, double* xq, double* xf, int* bad, cudaStream_t s);
cudaError_t launch_gen_H(const double* jxw, const double* fdA, const int* nbr, int n_total, int n, double* H,
                         cudaStream_t s);
cudaError_t launch_align_check(const double* xf, const int* nbr, int n_owned, int n, double tol, int* bad,
                               cudaStream_t s);
cudaError_t launch_law_points(int kind, const double* p, const double* x, long npts, double* out, cudaStream_t s);
cudaError_t launch_range(const double* v, long n, double* bmin, double* bmax, int* bad, int nblocks,
                         cudaStream_t s);

// vector kernels
cudaError_t launch_sum_ranks(const double* const* ranks, int R, long count, double* out, cudaStream_t s);
cudaError_t launch_dot(const double* a, const double* b, long n, double* part, int nblocks, double* out,
                       cudaStream_t s);
cudaError_t launch_cheb_first(const double* b, const double* dinv, double c_r, double* d, double* x, long n,
                              cudaStream_t s);
cudaError_t launch_cheb_first_f(const float* b, const float* dinv, double c_r, float* d, float* x, long n,
                                cudaStream_t s);
cudaError_t launch_d2f(const double* a, float* out, long n, cudaStream_t s);
cudaError_t launch_f2d(const float* a, double* out, long n, cudaStream_t s);
cudaError_t launch_ew_mul(const double* a, const double* b, double* out, long n, cudaStream_t s);
cudaError_t launch_axpby(double alpha, const double* x, double beta, double* y, long n, cudaStream_t s);
cudaError_t launch_ew_sqrt(const double* a, double* out, long n, cudaStream_t s);
cudaError_t launch_ew_div(const double* a, const double* b, double* out, long n, cudaStream_t s);
cudaError_t launch_lanczos_update(double* w, const double* q, const double* qprev, const double* alpha,
                                  const double* beta_prev, long n, cudaStream_t s);
cudaError_t launch_axpy_dev(const double* coef, double sgn, const double* x, double* y, long n, cudaStream_t s);
cudaError_t launch_scale_by_inv(const double* w, const double* s2, double* q, long n, cudaStream_t s);
// a5: face traces (value, d/dxi_n) of listed (cell, face) items for the ghost exchange
cudaError_t launch_pack_traces(int nc, int n, const double* src, const int* cells, const int* faces, int n_items,
                               double* out, cudaStream_t s);
cudaError_t launch_pack_traces_f(int nc, int n, const float* src, const int* cells, const int* faces, int n_items,
                                 float* out, cudaStream_t s);
cudaError_t launch_gather_cells_f(const float* src, const int* list, int ncells, int len, float* out,
                                  cudaStream_t s);
cudaError_t launch_gather_cells(const double* src, const int* list, int ncells, int len, double* out,
                                cudaStream_t s);

}  // namespace dgvv
