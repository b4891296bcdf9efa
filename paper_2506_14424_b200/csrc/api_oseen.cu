// api_oseen.cu — C ABI: upwind convective term, Oseen-type viscous step, GMRES (f4).
#include "api_internal.cuh"

extern "C" {

// ------------------------------------------------------------------ f4: convective term + GMRES
DGVV_INTERNAL ConvArgs conv_args(dgvv_ctx* c) {
  ConvArgs a;
  std::memset(&a, 0, sizeof(a));
  Level& L = c->L[0];
  a.nbr = c->d_nbr;
  a.n_proc = c->n_owned;
  a.n_owned = c->n_owned;
  a.cart = c->d_cart;
  a.vJi = L.vJi;
  a.jxw = L.jxw;
  a.fJi = L.fJi;
  a.fdA = L.fdA;
  a.w = c->d_wtr;
  a.wghost = c->wtr_ghost;
  a.ghost = L.ghost[0];
  return a;
}

// quadrature-point data of w (JxW J^-1 w, min({{w}}.n, 0) dA), derived at the first use after
// dgvv_set_transport (external-exchange mode: after the caller filled the transport ghosts)
DGVV_INTERNAL dgvv_status ensure_conv_pointdata(dgvv_ctx* c, cudaStream_t s) {
  if (!c->wq_stale) return DGVV_OK;
  const size_t n3 = (size_t)c->L[0].n * c->L[0].n * c->L[0].n, n2 = (size_t)c->L[0].n * c->L[0].n;
  if (!c->d_wref) TRY(dalloc(c, &c->d_wref, (size_t)c->n_owned * 3 * n3));
  if (!c->d_wface) TRY(dalloc(c, &c->d_wface, (size_t)c->n_owned * 6 * n2));
  cudaError_t e = launch_conv_pointdata(c->L[0].n, c->geo, conv_args(c), c->d_wref, c->d_wface, s);
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "convective point data: %s", cudaGetErrorString(e));
  c->wq_stale = false;
  return DGVV_OK;
}

// dst (+)= alpha C(w) src; the ghosts of src must already be in L[0].ghost[0]
DGVV_INTERNAL dgvv_status launch_conv(dgvv_ctx* c, const double* src, double* dst, double alpha, int accumulate,
                               cudaStream_t s) {
  ConvArgs a = conv_args(c);
  a.src = src;
  a.dst = dst;
  a.alpha = alpha;
  a.accumulate = accumulate;
  TRY(ensure_conv_pointdata(c, s));
  cudaError_t e = launch_convective_pd(c->L[0].n, a, c->d_wref, c->d_wface, s);
  if (e == cudaErrorNotSupported) return dgvv_fail(DGVV_EUNSUPPORTED, "convective kernel not built for degree %d", c->L[0].k);
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "convective kernel: %s", cudaGetErrorString(e));
  return DGVV_OK;
}

dgvv_status dgvv_set_transport(dgvv_ctx* c, const double* w, dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !w) return dgvv_fail(DGVV_EINVAL, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t N = (size_t)3 * level_dofs(c, 0);
  if (!c->d_wtr) TRY(dalloc(c, &c->d_wtr, N));
  if (c->n_ghost && !c->wtr_ghost) {
    const size_t n3 = (size_t)c->L[0].n * c->L[0].n * c->L[0].n;
    TRY(dalloc(c, &c->wtr_ghost, (size_t)c->n_ghost * 3 * n3));
  }
  DGVV_CUDA_TRY(cudaMemcpyAsync(c->d_wtr, w, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  double ww;
  TRY(dot_host(c, c->d_wtr, c->d_wtr, (long)N, &ww, s));        // synchronous; NaN/Inf propagate
  if (!std::isfinite(ww)) return dgvv_fail(DGVV_EDOMAIN, "transport field has non-finite entries");
  if (c->n_ghost) TRY(exchange_sync(c, 0, 3, c->d_wtr, c->wtr_ghost, s));
  c->has_wtr = true;
  c->wq_stale = true;                        // point data derived at the next fused apply (after the
                                             // caller filled external-mode transport ghosts)
  return DGVV_OK;
}

dgvv_status dgvv_apply_convective(dgvv_ctx* c, const double* src, double* dst, dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (src == dst) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  if (!c->has_wtr) return dgvv_fail(DGVV_ESTATE, "convective term: call dgvv_set_transport first");
  cudaStream_t s = (cudaStream_t)stream;
  if (c->n_ghost) TRY(exchange_sync(c, 0, 3, src, c->L[0].ghost[0], s));
  return launch_conv(c, src, dst, 1.0, 0, s);
}

// dst = (mass M + A(nu) + alpha_c C(w)) src [rhs given: dst = rhs - (...) src]
DGVV_INTERNAL dgvv_status apply_oseen(dgvv_ctx* c, double alpha_c, const double* src, double* dst, const double* rhs,
                               cudaStream_t s) {
  ApplyArgs a = base_args(c, 0, DGVV_OP_VISCOUS);
  a.src = src;
  a.dst = dst;
  if (rhs) { a.b = rhs; a.mode = MODE_RESID; }
  if (alpha_c != 0.0 && c->form == DGVV_FORM_DIVERGENCE) {   // one fused kernel (viscous + mass + convective)
    TRY(ensure_conv_pointdata(c, s));
    a.wref = c->d_wref;
    a.wface = c->d_wface;
    a.alpha_c = alpha_c;
    return run_apply(c, DGVV_OP_VISCOUS, 0, a, s, 2);
  }
  TRY(run_apply(c, DGVV_OP_VISCOUS, 0, a, s));     // leaves the ghosts of src in L[0].ghost[0]
  if (alpha_c != 0.0) TRY(launch_conv(c, src, dst, rhs ? -alpha_c : alpha_c, 1, s));
  return DGVV_OK;
}

dgvv_status dgvv_apply_oseen(dgvv_ctx* c, double alpha_c, const double* src, double* dst, dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (src == dst) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  if (!std::isfinite(alpha_c)) return dgvv_fail(DGVV_EINVAL, "alpha_c must be finite");
  TRY(op_ready(c, DGVV_OP_VISCOUS));
  if (alpha_c != 0.0 && !c->has_wtr) return dgvv_fail(DGVV_ESTATE, "convective term: call dgvv_set_transport first");
  return apply_oseen(c, alpha_c, src, dst, nullptr, (cudaStream_t)stream);
}

dgvv_status dgvv_gmres_solve(dgvv_ctx* c, double alpha_c, const double* b, double* x, double rtol,
                             int32_t restart, int32_t maxit, int32_t precond, const double* lambda_hi_per_level,
                             int32_t* iters, double* relres, dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !b || !x) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (b == x) return dgvv_fail(DGVV_EINVAL, "b and x alias");
  TRY(op_ready(c, DGVV_OP_VISCOUS));
  if (!std::isfinite(alpha_c)) return dgvv_fail(DGVV_EINVAL, "alpha_c must be finite");
  if (alpha_c != 0.0 && !c->has_wtr) return dgvv_fail(DGVV_ESTATE, "convective term: call dgvv_set_transport first");
  if (!(rtol >= 0.0) || maxit < 0 || restart < 1 || restart > 200)
    return dgvv_fail(DGVV_EINVAL, "rtol >= 0, maxit >= 0 and 1 <= restart <= 200 required");
  if (precond < DGVV_PRECOND_NONE || precond > DGVV_PRECOND_VCYCLE_FP32)
    return dgvv_fail(DGVV_EINVAL, "unknown preconditioner %d", precond);
  if ((precond == DGVV_PRECOND_VCYCLE || precond == DGVV_PRECOND_VCYCLE_FP32) && !lambda_hi_per_level)
    return dgvv_fail(DGVV_EINVAL, "V-cycle preconditioner needs lambda_hi_per_level");
  cudaStream_t s = (cudaStream_t)stream;
  const long N = 3L * level_dofs(c, 0);
  const int m = restart;
  if (c->gm_restart < m) {
    if (c->gm_work) {
      cudaFree(c->gm_work);
      c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), (void*)c->gm_work), c->allocs.end());
      c->gm_work = nullptr;
    }
    TRY(dalloc(c, &c->gm_work, (size_t)(2 * m + 3) * N));
    c->gm_restart = m;
  }
  double* r = c->gm_work;
  double* V = r + N;                           // V[0..m]
  double* Z = V + (size_t)(m + 1) * N;         // Z[0..m-1]
  if (!c->gm_H) TRY(dalloc(c, &c->gm_H, 256));
  double* dH = c->gm_H;                        // device column of H (m + 2 <= 202 entries)
  if (precond == DGVV_PRECOND_JACOBI) TRY(ensure_dinv(c, DGVV_OP_VISCOUS, 0, s));
  if (precond == DGVV_PRECOND_VCYCLE) TRY(ensure_vcycle_scratch(c, DGVV_OP_VISCOUS));
  auto prec = [&](const double* rr, double* zz) -> dgvv_status {
    if (precond == DGVV_PRECOND_JACOBI) {
      DGVV_CUDA_TRY(launch_ew_mul(c->L[0].dinv[0], rr, zz, N, s));
    } else if (precond == DGVV_PRECOND_VCYCLE) {
      TRY(vcycle_rec(c, DGVV_OP_VISCOUS, 0, rr, zz, lambda_hi_per_level, s));
    } else if (precond == DGVV_PRECOND_VCYCLE_FP32) {
      TRY(vcycle_fp32_d(c, DGVV_OP_VISCOUS, rr, zz, lambda_hi_per_level, s));
    } else {
      DGVV_CUDA_TRY(cudaMemcpyAsync(zz, rr, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    return DGVV_OK;
  };
  double bb, rr;
  TRY(dot_host(c, b, b, N, &bb, s));
  const double bn = std::sqrt(bb);
  TRY(apply_oseen(c, alpha_c, x, r, b, s));    // r = b - A x
  TRY(dot_host(c, r, r, N, &rr, s));
  double rn = std::sqrt(rr);
  int total = 0;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), yk(m), col(m + 2);
  auto Hij = [&](int i, int j) -> double& { return H[(size_t)i * m + j]; };
  while (bn > 0.0 && rn > rtol * bn && total < maxit) {
    const int mm = std::min(m, maxit - total);
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = rn;
    DGVV_CUDA_TRY(launch_axpby(1.0 / rn, r, 0.0, V, N, s));     // V_0 = r / ||r||
    int jd = 0;
    for (int j = 0; j < mm; ++j) {
      double* Vj = V + (size_t)j * N;
      double* Vn = V + (size_t)(j + 1) * N;
      double* Zj = Z + (size_t)j * N;
      TRY(prec(Vj, Zj));
      TRY(apply_oseen(c, alpha_c, Zj, Vn, nullptr, s));       // w = A z_j (in V_{j+1})
      for (int i = 0; i <= j; ++i) {                           // modified Gram-Schmidt, scalars on device
        TRY(dot_dev(c, Vn, V + (size_t)i * N, N, dH + i, s));
        DGVV_CUDA_TRY(launch_axpy_dev(dH + i, -1.0, V + (size_t)i * N, Vn, N, s));
      }
      TRY(dot_dev(c, Vn, Vn, N, dH + j + 1, s));
      DGVV_CUDA_TRY(cudaMemcpyAsync(col.data(), dH, (size_t)(j + 2) * sizeof(double), cudaMemcpyDeviceToHost, s));
      DGVV_CUDA_TRY(cudaStreamSynchronize(s));
      const double hn = std::sqrt(col[j + 1]);
      if (hn > 0.0) DGVV_CUDA_TRY(launch_axpby(1.0 / hn, Vn, 0.0, Vn, N, s));
      for (int i = 0; i <= j; ++i) Hij(i, j) = col[i];
      Hij(j + 1, j) = hn;
      for (int i = 0; i < j; ++i) {                            // previous Givens rotations
        const double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double den = std::hypot(Hij(j, j), Hij(j + 1, j));
      cs[j] = Hij(j, j) / den;
      sn[j] = Hij(j + 1, j) / den;
      Hij(j, j) = den;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++total;
      jd = j + 1;
      if (std::fabs(g[j + 1]) <= rtol * bn || hn == 0.0) break;
    }
    for (int i = jd - 1; i >= 0; --i) {
      double t = g[i];
      for (int l = i + 1; l < jd; ++l) t -= Hij(i, l) * yk[l];
      yk[i] = t / Hij(i, i);
    }
    for (int i = 0; i < jd; ++i) DGVV_CUDA_TRY(launch_axpby(yk[i], Z + (size_t)i * N, 1.0, x, N, s));
    TRY(apply_oseen(c, alpha_c, x, r, b, s));
    TRY(dot_host(c, r, r, N, &rr, s));
    rn = std::sqrt(rr);
  }
  if (iters) *iters = total;
  if (relres) *relres = bn > 0.0 ? rn / bn : 0.0;
  return DGVV_OK;
}

}  // extern "C"
