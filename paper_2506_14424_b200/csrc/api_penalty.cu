// api_penalty.cu — C ABI: the divergence/continuity penalty-step operator and its multigrid (f2).
#include "api_internal.cuh"

namespace dgvv {
cudaError_t launch_cheb_vec_resid(const double* Ax, const double* b, const double* dinv, double c_rho, double c_r,
                                  double* d, double* x, long n, cudaStream_t s);   // k_cg.cu
}

extern "C" {

// ------------------------------------------------------------------ f2: penalty-step operator
DGVV_INTERNAL PenaltyArgs penalty_args(dgvv_ctx* c, int l) {
  PenaltyArgs a;
  std::memset(&a, 0, sizeof(a));
  Level& L = c->L[l];
  a.nbr = c->d_nbr;
  a.n_proc = c->n_owned;
  a.n_owned = c->n_owned;
  a.cart = c->d_cart;
  a.vJi = L.vJi;
  a.jxw = L.jxw;
  a.fJi = L.fJi;
  a.fdA = L.fdA;
  a.tau_div = c->d_tau_div;
  a.tau_cont = c->d_tau_cont;
  a.ghost = L.ghost[0];
  return a;
}

// the penalty-step operator on level l (the level's degree and geometry, the same per-cell tau)
DGVV_INTERNAL dgvv_status apply_penalty_impl(dgvv_ctx* c, int l, const double* src, double* dst, cudaStream_t s) {
  PenaltyArgs a = penalty_args(c, l);
  a.src = src;
  a.dst = dst;
  Level& L = c->L[l];
  if (c->n_ghost) {
    if (!L.ghost[0]) TRY(dalloc(c, &L.ghost[0], (size_t)c->n_ghost * 3 * L.n * L.n * L.n));
    a.ghost = L.ghost[0];
    TRY(exchange_sync(c, l, 3, src, L.ghost[0], s));
  }
  cudaError_t e = launch_penalty(L.n, c->geo, a, false, s);
  if (e == cudaErrorNotSupported) return dgvv_fail(DGVV_EUNSUPPORTED, "penalty kernel not built for degree %d", L.k);
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "penalty kernel: %s", cudaGetErrorString(e));
  return DGVV_OK;
}

DGVV_INTERNAL dgvv_status ensure_dinv_pen(dgvv_ctx* c, int l, cudaStream_t s) {
  Level& L = c->L[l];
  if (L.dinv_pen && L.dinv_pen_ok) return DGVV_OK;
  if (!L.dinv_pen) TRY(dalloc(c, &L.dinv_pen, (size_t)3 * level_dofs(c, l)));
  PenaltyArgs a = penalty_args(c, l);
  a.dst = L.dinv_pen;
  cudaError_t e = launch_penalty(L.n, c->geo, a, true, s);
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "penalty diagonal: %s", cudaGetErrorString(e));
  L.dinv_pen_ok = true;
  return DGVV_OK;
}

// Chebyshev-Jacobi smoother of SURVEY §8(c) c1.6 for the penalty operator on level l:
// A x by the penalty kernel, then r = b - A x, d = c_rho d + c_r D^-1 r, x += d in one vector kernel.
// work holds 2 N doubles (r | d).
DGVV_INTERNAL dgvv_status cheb_pen(dgvv_ctx* c, int l, double* x, const double* b, int degree, double lo, double hi,
                            int x_is_zero, double* work, cudaStream_t s) {
  const long N = 3L * level_dofs(c, l);
  TRY(ensure_dinv_pen(c, l, s));
  const double* dinv = c->L[l].dinv_pen;
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
  double rho = 1.0 / sigma;
  double *r = work, *d = work + N;
  if (x_is_zero) {
    DGVV_CUDA_TRY(launch_cheb_first(b, dinv, 1.0 / theta, d, x, N, s));
  } else {
    TRY(apply_penalty_impl(c, l, x, r, s));                       // r = A x; b - A x in the update kernel
    DGVV_CUDA_TRY(launch_cheb_vec_resid(r, b, dinv, 0.0, 1.0 / theta, d, x, N, s));
  }
  for (int j = 1; j < degree; ++j) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    TRY(apply_penalty_impl(c, l, x, r, s));
    DGVV_CUDA_TRY(launch_cheb_vec_resid(r, b, dinv, rho_new * rho, 2.0 * rho_new / delta, d, x, N, s));
    rho = rho_new;
  }
  return DGVV_OK;
}

DGVV_INTERNAL dgvv_status ensure_pen_scratch(dgvv_ctx* c) {
  for (size_t l = 0; l < c->L.size(); ++l) {
    auto& S = c->L[l].scratch_pen;
    if (!S.empty()) continue;
    const size_t Nl = 3 * (size_t)level_dofs(c, (int)l);
    S.resize(5, nullptr);
    TRY(dalloc(c, &S[0], Nl));
    TRY(dalloc(c, &S[1], 2 * Nl));
    if (l > 0) { TRY(dalloc(c, &S[3], Nl)); TRY(dalloc(c, &S[4], Nl)); }
  }
  return DGVV_OK;
}

// f2 ("a multigrid preconditioner is necessary for the penalty step"): the
// V-cycle of SURVEY §8(c) c1.7 over the context's p-levels for the penalty operator — Chebyshev(5)
// pre/post smoothing, residual, p-restriction R = P^T, recursion, prolongation; coarsest level
// Chebyshev(5) from zero (G15).  h-levels / the c-level of the viscous hierarchy are not used.
DGVV_INTERNAL dgvv_status vcycle_pen_rec(dgvv_ctx* c, int l, const double* b, double* x, const double* his,
                                  cudaStream_t s) {
  auto& S = c->L[l].scratch_pen;
  const int last = (int)c->L.size() - 1;
  const long N = 3L * level_dofs(c, l);
  const double hi = his[l], lo = hi / 20.0;
  TRY(cheb_pen(c, l, x, b, 5, lo, hi, 1, S[1], s));
  if (l == last) return DGVV_OK;
  TRY(apply_penalty_impl(c, l, x, S[0], s));
  DGVV_CUDA_TRY(launch_axpby(1.0, b, -1.0, S[0], N, s));         // r = b - A x
  auto& C = c->L[l + 1].scratch_pen;
  TRY(transfer(c, DGVV_OP_VISCOUS, l, S[0], C[3], 0.0, false, s));
  TRY(vcycle_pen_rec(c, l + 1, C[3], C[4], his, s));
  TRY(transfer(c, DGVV_OP_VISCOUS, l, C[4], x, 1.0, true, s));
  TRY(cheb_pen(c, l, x, b, 5, lo, hi, 0, S[1], s));
  return DGVV_OK;
}

dgvv_status dgvv_set_penalty_parameters(dgvv_ctx* c, const double* tau_div, const double* tau_cont) {
  DGVV_RANGE();
  if (!c || !tau_div || !tau_cont) return dgvv_fail(DGVV_EINVAL, "null argument");
  const int nt = c->n_total;
  std::vector<double> td(nt), tc(nt);
  for (int i = 0; i < nt; ++i) {
    const int r = i < c->n_owned ? i : c->n_owned + c->h_gperm[i - c->n_owned];
    td[i] = tau_div[r];
    tc[i] = tau_cont[r];
    if (!std::isfinite(td[i]) || !std::isfinite(tc[i]) || td[i] < 0.0 || tc[i] < 0.0)
      return dgvv_fail(DGVV_EDOMAIN, "penalty parameters must be finite and >= 0 (cell row %d)", r);
  }
  if (!c->d_tau_div) TRY(dalloc(c, &c->d_tau_div, (size_t)nt));
  if (!c->d_tau_cont) TRY(dalloc(c, &c->d_tau_cont, (size_t)nt));
  DGVV_CUDA_TRY(cudaMemcpy(c->d_tau_div, td.data(), nt * sizeof(double), cudaMemcpyHostToDevice));
  DGVV_CUDA_TRY(cudaMemcpy(c->d_tau_cont, tc.data(), nt * sizeof(double), cudaMemcpyHostToDevice));
  for (auto& L : c->L) L.dinv_pen_ok = false;   // recomputed lazily in the same buffers
  c->has_pen = true;
  return DGVV_OK;
}

dgvv_status dgvv_apply_penalty(dgvv_ctx* c, const double* src, double* dst, dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (src == dst) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  TRY(op_ready(c, DGVV_OP_PENALTY));
  return apply_penalty_impl(c, 0, src, dst, (cudaStream_t)stream);
}

dgvv_status dgvv_apply_penalty_level(dgvv_ctx* c, int32_t level, const double* src, double* dst,
                                     dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  if (!src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (src == dst) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  TRY(op_ready(c, DGVV_OP_PENALTY));
  return apply_penalty_impl(c, level, src, dst, (cudaStream_t)stream);
}

}  // extern "C"
