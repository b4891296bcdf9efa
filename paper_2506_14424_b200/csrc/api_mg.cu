// api_mg.cu — C ABI: inverse diagonal (a8), Chebyshev smoother (a9), p-transfer (a10), V-cycles in
// FP64 and FP32 (a11, f1), Lanczos lambda_max, preconditioned CG (f1).
#include "api_internal.cuh"

extern "C" {

dgvv_status dgvv_inverse_diagonal(dgvv_ctx* c, int32_t op, int32_t level, double* dst, dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  TRY(op_ready(c, op));
  if (!dst) return dgvv_fail(DGVV_EINVAL, "null dst");
  cudaStream_t s = (cudaStream_t)stream;
  if (op == DGVV_OP_PENALTY) {
    TRY(ensure_dinv_pen(c, level, s));
    DGVV_CUDA_TRY(cudaMemcpyAsync(dst, c->L[level].dinv_pen, (size_t)3 * level_dofs(c, level) * sizeof(double),
                                  cudaMemcpyDeviceToDevice, s));
    return DGVV_OK;
  }
  TRY(ensure_dinv(c, op, level, s));
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  DGVV_CUDA_TRY(cudaMemcpyAsync(dst, c->L[level].dinv[op == DGVV_OP_VISCOUS ? 0 : 1],
                                (size_t)nc * level_dofs(c, level) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return DGVV_OK;
}

DGVV_INTERNAL dgvv_status cheb_impl(dgvv_ctx* c, int op, int l, double* x, const double* b, int degree, double lo,
                             double hi, int x_is_zero, double* work, cudaStream_t s,
                             int start_in_work) {
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  const long N = (long)nc * level_dofs(c, l);
  TRY(ensure_dinv(c, op, l, s));
  const double* dinv = c->L[l].dinv[op == DGVV_OP_VISCOUS ? 0 : 1];
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
  double rho = 1.0 / sigma;
  double* bufs[2] = {x, work};
  double* d = work + N;
  int cur;
  if (x_is_zero) {
    DGVV_CUDA_TRY(launch_cheb_first(b, dinv, 1.0 / theta, d, x, N, s));
    cur = 0;
  } else {
    ApplyArgs a = base_args(c, l, op);
    cur = start_in_work ? 1 : 0;         // the start iterate is in work (out-of-place prolongation-add)
    a.src = bufs[cur]; a.b = b; a.dinv = dinv; a.dvec = d; a.xout = bufs[1 - cur];
    a.mode = MODE_CHEB; a.c_rho = 0.0; a.c_r = 1.0 / theta;
    TRY(run_apply(c, op, l, a, s));
    cur = 1 - cur;
  }
  for (int j = 1; j < degree; ++j) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    ApplyArgs a = base_args(c, l, op);
    a.src = bufs[cur]; a.b = b; a.dinv = dinv; a.dvec = d; a.xout = bufs[1 - cur];
    a.mode = MODE_CHEB; a.c_rho = rho_new * rho; a.c_r = 2.0 * rho_new / delta;
    TRY(run_apply(c, op, l, a, s));
    cur = 1 - cur;
    rho = rho_new;
  }
  if (cur != 0) DGVV_CUDA_TRY(cudaMemcpyAsync(x, work, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return DGVV_OK;
}

dgvv_status dgvv_chebyshev_smooth(dgvv_ctx* c, int32_t op, int32_t level, double* x, const double* b,
                                  int32_t degree, double lambda_lo, double lambda_hi, int32_t x_is_zero,
                                  double* work, dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  TRY(op_ready(c, op));
  if (!x || !b || !work) return dgvv_fail(DGVV_EINVAL, "null vector");
  if (degree < 1) return dgvv_fail(DGVV_EINVAL, "degree %d < 1", degree);
  if (!(lambda_hi > lambda_lo) || !(lambda_lo > 0.0)) return dgvv_fail(DGVV_EDOMAIN, "need 0 < lambda_lo < lambda_hi");
  if (op == DGVV_OP_PENALTY)
    return cheb_pen(c, level, x, b, degree, lambda_lo, lambda_hi, x_is_zero, work, (cudaStream_t)stream);
  return cheb_impl(c, op, level, x, b, degree, lambda_lo, lambda_hi, x_is_zero, work, (cudaStream_t)stream);
}

DGVV_INTERNAL dgvv_status transfer(dgvv_ctx* c, int op, int fl, const double* in, double* out, double beta, bool prol,
                            cudaStream_t s, const double* add) {
  if (fl < 0 || fl + 1 >= (int)c->L.size()) return dgvv_fail(DGVV_EINVAL, "fine_level %d has no coarser level", fl);
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "op");
  const int nf = c->L[fl].n, ncs = c->L[fl + 1].n;
  std::vector<double> P1((size_t)nf * ncs), M((size_t)nf * ncs);
  transfer_matrix(nf, ncs, P1.data());
  if (prol) {
    M = P1;   // nout = nf, nin = nc
    DGVV_CUDA_TRY(launch_tensor3(ncs, nf, nc, M.data(), in, out, beta, c->n_owned, s, add));
  } else {
    for (int i = 0; i < nf; ++i)
      for (int j = 0; j < ncs; ++j) M[(size_t)j * nf + i] = P1[(size_t)i * ncs + j];
    DGVV_CUDA_TRY(launch_tensor3(nf, ncs, nc, M.data(), in, out, beta, c->n_owned, s));
  }
  return DGVV_OK;
}

dgvv_status dgvv_prolongate(dgvv_ctx* c, int32_t op, int32_t fine_level, const double* coarse, double* fine,
                            double beta, dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !coarse || !fine) return dgvv_fail(DGVV_EINVAL, "null argument");
  return transfer(c, op, fine_level, coarse, fine, beta, true, (cudaStream_t)stream);
}

dgvv_status dgvv_restrict(dgvv_ctx* c, int32_t op, int32_t fine_level, const double* fine, double* coarse,
                          double beta, dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !coarse || !fine) return dgvv_fail(DGVV_EINVAL, "null argument");
  return transfer(c, op, fine_level, fine, coarse, beta, false, (cudaStream_t)stream);
}


// V(l, b) of SURVEY §8(c) c1.7 over the chain of contexts (p-levels of c, then — f3 — the levels
// of c->coarse after an h-transfer); the coarsest level of the chain is either Chebyshev(5) from
// 0 (G15) or, after dgvv_setup_coarse_solver, the direct solve (reading H3).
DGVV_INTERNAL dgvv_status vcycle_rec(dgvv_ctx* c, int op, int l, const double* b, double* x, const double* his,
                              cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  auto& S = c->L[l].scratch[oi];   // [0] r, [1..2] work, (l>0: [3] b, [4] x of coarser handled by caller)
  const int last = (int)c->L.size() - 1;
  if (l == last && !c->coarse && !c->cg.on && c->Ainv[oi]) {   // the c-level, when enabled, comes first
    if (c->direct_epoch[oi] != c->coef_epoch)
      return dgvv_fail(DGVV_ESTATE, "direct coarse solver is stale (coefficients or mass changed): call dgvv_setup_coarse_solver again");
    return direct_solve(c, oi, b, x, s);
  }
  const double hi = his[l], lo = hi / 20.0;
  TRY(cheb_impl(c, op, l, x, b, 5, lo, hi, 1, S[1], s));
  if (l == last && !c->coarse && !c->cg.on) return DGVV_OK;
  ApplyArgs a = base_args(c, l, op);
  a.src = x; a.dst = S[0]; a.b = b; a.mode = MODE_RESID;
  TRY(run_apply(c, op, l, a, s));
  if (l == last && c->cg.on) {                 // c-level: DG_1 -> continuous Q1 (reading C1)
    TRY(cg_enter(c, op, S[0], x, his + c->L.size(), s));
  } else if (l < last) {
    auto& C = c->L[l + 1].scratch[oi];
    TRY(transfer(c, op, l, S[0], C[3], 0.0, false, s));
    TRY(vcycle_rec(c, op, l + 1, C[3], C[4], his, s));
    // post-smoothing starts from x + P x_c written out of place into the work buffer: its 5
    // ping-pong sweeps then end in x (no closing copy)
    TRY(transfer(c, op, l, C[4], S[1], 1.0, true, s, x));
    TRY(cheb_impl(c, op, l, x, b, 5, lo, hi, 0, S[1], s, 1));
    return DGVV_OK;
  } else {                                     // h-coarsening into the coarser context
    TRY(hrestrict_impl(c, op, S[0], c->hb[oi], 0.0, s));
    TRY(vcycle_rec(c->coarse, op, 0, c->hb[oi], c->hx[oi], his + c->L.size(), s));
    TRY(hprolong_impl(c, op, c->hx[oi], x, 1.0, s));
  }
  TRY(cheb_impl(c, op, l, x, b, 5, lo, hi, 0, S[1], s));
  return DGVV_OK;
}

// ------------------------------------------------------------------ FP32 multigrid (f1)
DGVV_INTERNAL dgvv_status d2f_alloc(dgvv_ctx* c, float** dst, const double* src, long n, cudaStream_t s) {
  if (!*dst) TRY(dalloc(c, dst, (size_t)n));
  DGVV_CUDA_TRY(launch_d2f(src, *dst, n, s));
  return DGVV_OK;
}

DGVV_INTERNAL dgvv_status ensure_fp32(dgvv_ctx* c, int op, cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  if (c->LF.size() != c->L.size()) c->LF.resize(c->L.size());
  if (c->geo == 0 && !c->d_cart_f) TRY(d2f_alloc(c, &c->d_cart_f, c->d_cart, (long)c->n_total * CART_STRIDE, s));
  for (size_t l = 0; l < c->L.size(); ++l) {
    Level& L = c->L[l];
    LevelF& F = c->LF[l];
    const long n3 = (long)L.n * L.n * L.n, n2 = (long)L.n * L.n;
    if (c->geo == 1 && !F.vJi) {
      TRY(d2f_alloc(c, &F.vJi, L.vJi, (long)c->n_total * 9 * n3, s));
      TRY(d2f_alloc(c, &F.fJi, L.fJi, (long)c->n_total * 6 * 9 * n2, s));
      TRY(d2f_alloc(c, &F.Hc, L.Hc, (long)c->n_total, s));
      TRY(d2f_alloc(c, &F.jxw, L.jxw, (long)c->n_owned * n3, s));
    }
    if (F.epoch[oi] != c->coef_epoch) {
      const double* nuc = c->geo == 0 ? (oi == 0 ? L.nu_cell : L.c_cell) : (oi == 0 ? L.wv_cell : L.wc_cell);
      const double* nuf = c->geo == 0 ? (oi == 0 ? L.nu_face : L.c_face) : (oi == 0 ? L.wv_face : L.wc_face);
      TRY(d2f_alloc(c, &F.nu_cell[oi], nuc, (long)c->n_owned * n3, s));
      TRY(d2f_alloc(c, &F.nu_face[oi], nuf, (long)c->n_total * 6 * n2, s));
      TRY(ensure_dinv(c, op, (int)l, s));
      TRY(d2f_alloc(c, &F.dinv[oi], L.dinv[oi], (long)nc * c->n_owned * n3, s));
      F.epoch[oi] = c->coef_epoch;
    }
    if (c->n_ghost && !F.ghost[oi]) TRY(dalloc(c, &F.ghost[oi], (size_t)nc * c->n_ghost * n3));
    auto& S = F.scratch[oi];
    if (S.empty()) {
      const size_t N = (size_t)nc * c->n_owned * n3;
      S.resize(5, nullptr);
      TRY(dalloc(c, &S[0], N));
      TRY(dalloc(c, &S[1], 2 * N));
      S[2] = S[1] + N;
      TRY(dalloc(c, &S[3], N));
      TRY(dalloc(c, &S[4], N));
    }
  }
  if (c->coarse) {                              // f3: FP32 levels of the coarser contexts too
    TRY(op_ready(c->coarse, op));
    const size_t Nc = (size_t)nc * level_dofs(c->coarse, 0);
    if (!c->hbf[oi]) TRY(dalloc(c, &c->hbf[oi], Nc));
    if (!c->hxf[oi]) TRY(dalloc(c, &c->hxf[oi], Nc));
    TRY(ensure_fp32(c->coarse, op, s));
  }
  return DGVV_OK;
}

DGVV_INTERNAL ApplyArgsT<float> base_args_f(dgvv_ctx* c, int l, int op) {
  ApplyArgsT<float> a;
  std::memset(&a, 0, sizeof(a));
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  LevelF& F = c->LF[l];
  a.nbr = c->d_nbr;
  a.n_proc = c->n_owned;
  a.n_owned = c->n_owned;
  a.nu_cell = F.nu_cell[oi];
  a.nu_face = F.nu_face[oi];
  a.cart = c->d_cart_f;
  a.vJi = F.vJi;
  a.fJi = F.fJi;
  a.jxw = F.jxw;
  a.Hcell = F.Hc;
  a.pen = c->ip * (double)(c->L[l].k + 1) * (double)(c->L[l].k + 1);
  a.mass = c->mass[oi];
  a.ghost = F.ghost[oi];
  a.mode = MODE_APPLY;
  return a;
}

// FP32 levels across ranks: the ghost face traces travel in single precision, packed by the trace
// kernel and moved by the same collective as the FP64 exchange; interior cells run while they move
DGVV_INTERNAL dgvv_status run_apply_f(dgvv_ctx* c, int op, int l, const ApplyArgsT<float>& a, cudaStream_t s) {
  if (reinterpret_cast<uintptr_t>(a.src) & 15)    // float4 neighbour rows (internal FP32 buffers are aligned)
    return dgvv_fail(DGVV_EINVAL, "FP32 source vector %p is not 16-byte aligned", (const void*)a.src);
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  const int form = op == DGVV_OP_VISCOUS ? c->form : DGVV_FORM_LAPLACE;
  auto launch = [&](const ApplyArgsT<float>& x) -> dgvv_status {
    cudaError_t e = launch_apply_f(nc, c->L[l].n, form, c->geo, x, s);
    if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "FP32 apply kernel: %s", cudaGetErrorString(e));
    return DGVV_OK;
  };
  if (!c->comm || c->peers.empty()) return launch(a);
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  TRY(exchange_traces(c, l, nc, a.src, &c->LF[l].gtr[oi], s));   // FP32 face traces
  ApplyArgsT<float> a2 = a;
  a2.gtr = c->LF[l].gtr[oi];
  a2.gslot = c->d_gslot;
  ApplyArgsT<float> ai = a2;
  ai.cell_list = c->d_interior;
  ai.n_proc = c->n_interior;
  ai.gtr = nullptr;
  TRY(launch(ai));
  DGVV_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_comm, 0));
  ApplyArgsT<float> ab = a2;
  ab.cell_list = c->d_boundary;
  ab.n_proc = c->n_boundary;
  return launch(ab);
}

DGVV_INTERNAL dgvv_status cheb_impl_f(dgvv_ctx* c, int op, int l, float* x, const float* b, int degree, double lo,
                               double hi, int x_is_zero, float* work, cudaStream_t s,
                             int start_in_work) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  const long N = (long)nc * level_dofs(c, l);
  const float* dinv = c->LF[l].dinv[oi];
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
  double rho = 1.0 / sigma;
  float* bufs[2] = {x, work};
  float* d = work + N;
  int cur;
  if (x_is_zero) {
    DGVV_CUDA_TRY(launch_cheb_first_f(b, dinv, 1.0 / theta, d, x, N, s));
    cur = 0;
  } else {
    ApplyArgsT<float> a = base_args_f(c, l, op);
    cur = start_in_work ? 1 : 0;
    a.src = bufs[cur]; a.b = b; a.dinv = dinv; a.dvec = d; a.xout = bufs[1 - cur];
    a.mode = MODE_CHEB; a.c_rho = 0.0; a.c_r = 1.0 / theta;
    TRY(run_apply_f(c, op, l, a, s));
    cur = 1 - cur;
  }
  for (int j = 1; j < degree; ++j) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    ApplyArgsT<float> a = base_args_f(c, l, op);
    a.src = bufs[cur]; a.b = b; a.dinv = dinv; a.dvec = d; a.xout = bufs[1 - cur];
    a.mode = MODE_CHEB; a.c_rho = rho_new * rho; a.c_r = 2.0 * rho_new / delta;
    TRY(run_apply_f(c, op, l, a, s));
    cur = 1 - cur;
    rho = rho_new;
  }
  if (cur != 0) DGVV_CUDA_TRY(cudaMemcpyAsync(x, work, N * sizeof(float), cudaMemcpyDeviceToDevice, s));
  return DGVV_OK;
}

DGVV_INTERNAL dgvv_status transfer_f(dgvv_ctx* c, int op, int fl, const float* in, float* out, double beta, bool prol,
                              cudaStream_t s, const float* add) {
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  const int nf = c->L[fl].n, ncs = c->L[fl + 1].n;
  std::vector<double> P1((size_t)nf * ncs), M((size_t)nf * ncs);
  transfer_matrix(nf, ncs, P1.data());
  if (prol) {
    DGVV_CUDA_TRY(launch_tensor3_f(ncs, nf, nc, P1.data(), in, out, beta, c->n_owned, s, add));
  } else {
    for (int i = 0; i < nf; ++i)
      for (int j = 0; j < ncs; ++j) M[(size_t)j * nf + i] = P1[(size_t)i * ncs + j];
    DGVV_CUDA_TRY(launch_tensor3_f(nf, ncs, nc, M.data(), in, out, beta, c->n_owned, s));
  }
  return DGVV_OK;
}

// the V-cycle of vcycle_rec with every level in FP32
DGVV_INTERNAL dgvv_status vcycle_rec_f(dgvv_ctx* c, int op, int l, const float* b, float* x, const double* his,
                                cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  auto& S = c->LF[l].scratch[oi];
  const int last = (int)c->L.size() - 1;
  if (l == last && !c->coarse && !c->cg.on && c->Ainv[oi]) {   // direct coarse solve, FP64 arithmetic; the c-level, when enabled, comes first
    if (c->direct_epoch[oi] != c->coef_epoch)
      return dgvv_fail(DGVV_ESTATE, "direct coarse solver is stale (coefficients or mass changed): call dgvv_setup_coarse_solver again");
    return direct_solve(c, oi, b, x, s);
  }
  const double hi = his[l], lo = hi / 20.0;
  TRY(cheb_impl_f(c, op, l, x, b, 5, lo, hi, 1, S[1], s));
  if (l == last && !c->coarse) return DGVV_OK;
  ApplyArgsT<float> a = base_args_f(c, l, op);
  a.src = x; a.dst = S[0]; a.b = b; a.mode = MODE_RESID;
  TRY(run_apply_f(c, op, l, a, s));
  if (l < last) {
    auto& C = c->LF[l + 1].scratch[oi];
    TRY(transfer_f(c, op, l, S[0], C[3], 0.0, false, s));
    TRY(vcycle_rec_f(c, op, l + 1, C[3], C[4], his, s));
    TRY(transfer_f(c, op, l, C[4], S[1], 1.0, true, s, x));   // out of place, as vcycle_rec
    TRY(cheb_impl_f(c, op, l, x, b, 5, lo, hi, 0, S[1], s, 1));
    return DGVV_OK;
  } else {                                     // h-coarsening into the coarser context (f3)
    const int n = c->L.back().n;
    DGVV_CUDA_TRY(launch_hrestrict_f(n, nc, S[0], c->hbf[oi], c->d_child, 0.0, c->coarse->n_owned, s));
    TRY(vcycle_rec_f(c->coarse, op, 0, c->hbf[oi], c->hxf[oi], his + c->L.size(), s));
    DGVV_CUDA_TRY(launch_hprolongate_f(n, nc, c->hxf[oi], x, c->d_parent, c->d_octant, 1.0, c->n_owned, s));
  }
  TRY(cheb_impl_f(c, op, l, x, b, 5, lo, hi, 0, S[1], s));
  return DGVV_OK;
}

// z = V_fp32(r) for FP64 vectors (conversion in and out)
DGVV_INTERNAL dgvv_status vcycle_fp32_d(dgvv_ctx* c, int op, const double* r, double* z, const double* his, cudaStream_t s) {
  for (dgvv_ctx* q = c; q; q = q->coarse)
    if (q->cg.on) return dgvv_fail(DGVV_EUNSUPPORTED, "FP32 V-cycle: the continuous (c-) level is FP64 only");
  TRY(ensure_fp32(c, op, s));
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const long N = (long)(op == DGVV_OP_VISCOUS ? 3 : 1) * level_dofs(c, 0);
  auto& S = c->LF[0].scratch[oi];
  DGVV_CUDA_TRY(launch_d2f(r, S[3], N, s));
  TRY(vcycle_rec_f(c, op, 0, S[3], S[4], his, s));
  DGVV_CUDA_TRY(launch_f2d(S[4], z, N, s));
  return DGVV_OK;
}

dgvv_status dgvv_vcycle_fp32(dgvv_ctx* c, int32_t op, const double* b, double* x, const double* his,
                             dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !b || !x || !his) return dgvv_fail(DGVV_EINVAL, "null argument");
  TRY(op_ready(c, op));
  return vcycle_fp32_d(c, op, b, x, his, (cudaStream_t)stream);
}


dgvv_status dgvv_vcycle(dgvv_ctx* c, int32_t op, const double* b, double* x, const double* his,
                        dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !b || !x || !his) return dgvv_fail(DGVV_EINVAL, "null argument");
  TRY(op_ready(c, op));
  if (op == DGVV_OP_PENALTY) {                 // f2: p-levels of this context
    TRY(ensure_pen_scratch(c));
    return vcycle_pen_rec(c, 0, b, x, his, (cudaStream_t)stream);
  }
  TRY(ensure_vcycle_scratch(c, op));
  return vcycle_rec(c, op, 0, b, x, his, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ f1: preconditioned CG
// V-cycle scratch of every level (as dgvv_vcycle)
DGVV_INTERNAL dgvv_status ensure_vcycle_scratch(dgvv_ctx* c, int op) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  for (size_t l = 0; l < c->L.size(); ++l) {
    auto& S = c->L[l].scratch[oi];
    if (S.empty()) {
      const size_t Nl = (size_t)nc * level_dofs(c, (int)l);
      S.resize(5, nullptr);
      TRY(dalloc(c, &S[0], Nl));
      TRY(dalloc(c, &S[1], 2 * Nl));
      S[2] = S[1] + Nl;
      if (l > 0) { TRY(dalloc(c, &S[3], Nl)); TRY(dalloc(c, &S[4], Nl)); }
    }
  }
  if (c->cg.on) {                               // f3 c-level: continuous levels below
    for (dgvv_ctx* q = c; q; q = q->coarse) {
      if (!q->cg.on) return dgvv_fail(DGVV_ESTATE, "continuous level: every context below the c-level needs dgvv_set_continuous_level");
      TRY(op_ready(q, op));
      auto& G = q->cg;
      const size_t Nv = (size_t)nc * G.nv, Nd = (size_t)nc * q->n_owned * 8;
      if (!G.xdg[oi]) { TRY(dalloc(q, &G.xdg[oi], Nd)); TRY(dalloc(q, &G.ydg[oi], Nd)); }
      if (!G.r[oi]) { TRY(dalloc(q, &G.r[oi], Nv)); TRY(dalloc(q, &G.d[oi], Nv)); }
      if (!G.b0[oi]) { TRY(dalloc(q, &G.b0[oi], Nv)); TRY(dalloc(q, &G.x0[oi], Nv)); }
      if (q->coarse) {
        const size_t Nc = (size_t)nc * q->coarse->cg.nv;
        if (!q->coarse->cg.on) return dgvv_fail(DGVV_ESTATE, "continuous level: the coarse context needs dgvv_set_continuous_level");
        if (!G.hb[oi]) { TRY(dalloc(q, &G.hb[oi], Nc)); TRY(dalloc(q, &G.hx[oi], Nc)); }
      }
    }
    return DGVV_OK;
  }
  if (c->coarse) {                              // f3: the chain continues in the coarser context
    TRY(op_ready(c->coarse, op));
    const size_t Nc = (size_t)nc * level_dofs(c->coarse, 0);
    if (!c->hb[oi]) TRY(dalloc(c, &c->hb[oi], Nc));
    if (!c->hx[oi]) TRY(dalloc(c, &c->hx[oi], Nc));
    TRY(ensure_vcycle_scratch(c->coarse, op));
  }
  return DGVV_OK;
}

DGVV_INTERNAL dgvv_status dot_host(dgvv_ctx* c, const double* a, const double* b, long n, double* out, cudaStream_t s) {
  TRY(dot_dev(c, a, b, n, c->d_scal + 5, s));
  DGVV_CUDA_TRY(cudaMemcpyAsync(out, c->d_scal + 5, sizeof(double), cudaMemcpyDeviceToHost, s));
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  return DGVV_OK;
}

dgvv_status dgvv_cg_solve(dgvv_ctx* c, int32_t op, const double* b, double* x, double rtol, int32_t maxit,
                          int32_t precond, const double* lambda_hi_per_level, int32_t* iters, double* relres,
                          dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !b || !x) return dgvv_fail(DGVV_EINVAL, "null argument");
  TRY(op_ready(c, op));
  if (b == x) return dgvv_fail(DGVV_EINVAL, "b and x alias");
  if (!(rtol >= 0.0) || maxit < 0) return dgvv_fail(DGVV_EINVAL, "rtol >= 0 and maxit >= 0 required");
  if (precond < DGVV_PRECOND_NONE || precond > DGVV_PRECOND_VCYCLE_FP32)
    return dgvv_fail(DGVV_EINVAL, "unknown preconditioner %d", precond);
  if ((precond == DGVV_PRECOND_VCYCLE || precond == DGVV_PRECOND_VCYCLE_FP32) && !lambda_hi_per_level)
    return dgvv_fail(DGVV_EINVAL, "V-cycle preconditioner needs lambda_hi_per_level");
  cudaStream_t s = (cudaStream_t)stream;
  const bool pen = op == DGVV_OP_PENALTY;
  if (pen && precond == DGVV_PRECOND_VCYCLE_FP32)
    return dgvv_fail(DGVV_EUNSUPPORTED, "penalty operator: FP64 V-cycle, Jacobi or none");
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_POISSON ? 1 : 3;
  const long N = (long)nc * level_dofs(c, 0);
  auto& W = c->cg_work[pen ? 2 : oi];
  if (!W) TRY(dalloc(c, &W, (size_t)4 * N));
  double *r = W, *z = W + N, *pv = W + 2 * N, *q = W + 3 * N;
  if (precond == DGVV_PRECOND_JACOBI) TRY(pen ? ensure_dinv_pen(c, 0, s) : ensure_dinv(c, op, 0, s));
  if (precond == DGVV_PRECOND_VCYCLE) TRY(pen ? ensure_pen_scratch(c) : ensure_vcycle_scratch(c, op));
  auto apply_A = [&](const double* src, double* dst, const double* rhs) -> dgvv_status {
    if (pen) {
      TRY(apply_penalty_impl(c, 0, src, dst, s));
      if (rhs) DGVV_CUDA_TRY(launch_axpby(1.0, rhs, -1.0, dst, N, s));   // dst = rhs - A src
      return DGVV_OK;
    }
    ApplyArgs a = base_args(c, 0, op);
    a.src = src; a.dst = dst;
    if (rhs) { a.b = rhs; a.mode = MODE_RESID; }
    return run_apply(c, op, 0, a, s);
  };
  auto prec = [&](const double* rr, double* zz) -> dgvv_status {
    if (precond == DGVV_PRECOND_JACOBI) {
      DGVV_CUDA_TRY(launch_ew_mul(pen ? c->L[0].dinv_pen : c->L[0].dinv[oi], rr, zz, N, s));
    } else if (precond == DGVV_PRECOND_VCYCLE) {
      TRY(pen ? vcycle_pen_rec(c, 0, rr, zz, lambda_hi_per_level, s) : vcycle_rec(c, op, 0, rr, zz, lambda_hi_per_level, s));
    } else if (precond == DGVV_PRECOND_VCYCLE_FP32) {
      TRY(vcycle_fp32_d(c, op, rr, zz, lambda_hi_per_level, s));
    } else {
      DGVV_CUDA_TRY(cudaMemcpyAsync(zz, rr, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    return DGVV_OK;
  };
  double bb, rr, rz, pq;
  TRY(dot_host(c, b, b, N, &bb, s));
  TRY(apply_A(x, r, b));                      // r = b - A x
  TRY(dot_host(c, r, r, N, &rr, s));
  const double bn = std::sqrt(bb);
  int it = 0;
  if (bn > 0.0 && std::sqrt(rr) > rtol * bn && maxit > 0) {
    TRY(prec(r, z));
    DGVV_CUDA_TRY(cudaMemcpyAsync(pv, z, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    TRY(dot_host(c, r, z, N, &rz, s));
    while (it < maxit) {
      ++it;
      TRY(apply_A(pv, q, nullptr));           // q = A p
      TRY(dot_host(c, pv, q, N, &pq, s));
      const double alpha = rz / pq;
      DGVV_CUDA_TRY(launch_axpby(alpha, pv, 1.0, x, N, s));
      DGVV_CUDA_TRY(launch_axpby(-alpha, q, 1.0, r, N, s));
      TRY(dot_host(c, r, r, N, &rr, s));
      if (std::sqrt(rr) <= rtol * bn) break;
      TRY(prec(r, z));
      double rz_new;
      TRY(dot_host(c, r, z, N, &rz_new, s));
      DGVV_CUDA_TRY(launch_axpby(1.0, z, rz_new / rz, pv, N, s));
      rz = rz_new;
    }
  }
  if (iters) *iters = it;
  if (relres) *relres = bn > 0.0 ? std::sqrt(rr) / bn : 0.0;
  return DGVV_OK;
}


dgvv_status dgvv_estimate_lambda_max(dgvv_ctx* c, int32_t op, int32_t level, int32_t steps, const double* v0,
                                     double* out, dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_ctx(c));
  const bool cgl = c->cg.on && level == (int)c->L.size();      // the continuous (c-) level
  if (!cgl) TRY(check_level(c, level));
  TRY(op_ready(c, op));
  if (cgl && op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  if (!v0 || !out || steps < 1) return dgvv_fail(DGVV_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  const bool pen = op == DGVV_OP_PENALTY;
  const int nc = op == DGVV_OP_POISSON ? 1 : 3;
  const long N = cgl ? (long)nc * c->cg.nv : (long)nc * level_dofs(c, level);
  const double* dinv;
  if (pen) {
    TRY(ensure_dinv_pen(c, level, s));
    dinv = c->L[level].dinv_pen;
  } else if (cgl) {
    TRY(ensure_vcycle_scratch(c, op));
    TRY(cg_ensure_dinv(c, op, s));
    dinv = c->cg.dinv[op == DGVV_OP_VISCOUS ? 0 : 1];
  } else {
    TRY(ensure_dinv(c, op, level, s));
    dinv = c->L[level].dinv[op == DGVV_OP_VISCOUS ? 0 : 1];
  }
  auto apply_op = [&](const double* src, double* dst) -> dgvv_status {
    if (cgl) return cg_apply(c, op, src, dst, s);
    if (pen) return apply_penalty_impl(c, level, src, dst, s);
    ApplyArgs a = base_args(c, level, op);
    a.src = src; a.dst = dst;
    return run_apply(c, op, level, a, s);
  };
  if (c->lz_len < (size_t)(5 * N)) {           // work vectors kept by the context (grow-only)
    if (c->lz_buf) {
      cudaFree(c->lz_buf);
      c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), (void*)c->lz_buf), c->allocs.end());
      c->lz_buf = nullptr;
    }
    TRY(dalloc(c, &c->lz_buf, (size_t)(5 * N)));
    c->lz_len = (size_t)(5 * N);
  }
  double* buf = c->lz_buf;
  double *sq = buf, *q = buf + N, *qp = buf + 2 * N, *w = buf + 3 * N, *t = buf + 4 * N;
  double* d_alpha = c->d_scal;
  double* d_beta = c->d_scal + 1;
  double* d_nrm = c->d_scal + 2;
  DGVV_CUDA_TRY(launch_ew_sqrt(dinv, sq, N, s));
  DGVV_CUDA_TRY(launch_ew_div(v0, sq, t, N, s));            // q = v0 / s
  TRY(dot_dev(c, t, t, N, d_nrm, s));
  DGVV_CUDA_TRY(launch_scale_by_inv(t, d_nrm, q, N, s));
  DGVV_CUDA_TRY(cudaMemsetAsync(qp, 0, N * sizeof(double), s));
  DGVV_CUDA_TRY(cudaMemsetAsync(d_beta, 0, sizeof(double), s));
  std::vector<double> al, be;
  for (int it = 0; it < steps; ++it) {
    DGVV_CUDA_TRY(launch_ew_mul(sq, q, t, N, s));
    TRY(apply_op(t, w));
    DGVV_CUDA_TRY(launch_ew_mul(sq, w, w, N, s));
    TRY(dot_dev(c, q, w, N, d_alpha, s));
    DGVV_CUDA_TRY(launch_lanczos_update(w, q, qp, d_alpha, d_beta, N, s));
    TRY(dot_dev(c, w, w, N, d_nrm, s));
    double h[2];
    DGVV_CUDA_TRY(cudaMemcpyAsync(&h[0], d_alpha, sizeof(double), cudaMemcpyDeviceToHost, s));
    DGVV_CUDA_TRY(cudaMemcpyAsync(&h[1], d_nrm, sizeof(double), cudaMemcpyDeviceToHost, s));
    DGVV_CUDA_TRY(cudaStreamSynchronize(s));
    al.push_back(h[0]);
    const double bn = std::sqrt(h[1]);
    if (bn == 0.0) break;
    be.push_back(bn);
    std::swap(q, qp);                                          // qp <- q
    DGVV_CUDA_TRY(launch_scale_by_inv(w, d_nrm, q, N, s));     // q <- w / |w|
    DGVV_CUDA_TRY(cudaMemcpyAsync(d_beta, &bn, sizeof(double), cudaMemcpyHostToDevice, s));
    DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  }
  be.resize(al.size() > 0 ? al.size() - 1 : 0);
  *out = tridiag_max_eig(al, be);
  return DGVV_OK;
}

}  // extern "C"
