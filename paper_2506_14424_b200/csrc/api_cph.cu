// api_cph.cu — C ABI: continuous (c-) level, h-levels and the direct coarse solver (f3).
#include "api_internal.cuh"

extern "C" {

// ------------------------------------------------------------------ f3 c-level (continuous Q1)
DGVV_INTERNAL dgvv_status cg_apply(dgvv_ctx* c, int op, const double* x, double* y, cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  auto& G = c->cg;
  const int l = (int)c->L.size() - 1;
  DGVV_CUDA_TRY(launch_cg_embed(x, G.xdg[oi], G.d_vid, c->n_owned, G.nv, nc, 0.0, s));
  ApplyArgs a = base_args(c, l, op);
  a.src = G.xdg[oi];
  a.dst = G.ydg[oi];
  TRY(run_apply(c, op, l, a, s));
  DGVV_CUDA_TRY(launch_cg_embedT(G.ydg[oi], y, G.d_inc_ptr, G.d_inc, G.nv, nc, 0.0, s));
  return DGVV_OK;
}

// 1 / diag(P_c^T A P_c) by probing with the vertex colouring (vertices of one colour share no cell)
DGVV_INTERNAL dgvv_status cg_ensure_dinv(dgvv_ctx* c, int op, cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  auto& G = c->cg;
  if (G.dinv[oi] && G.dinv_epoch[oi] == c->coef_epoch) return DGVV_OK;
  const long Nv = (long)nc * G.nv;
  if (!G.dinv[oi]) TRY(dalloc(c, &G.dinv[oi], Nv));
  double *sv = nullptr, *yv = nullptr;
  DGVV_CUDA_TRY(cudaMalloc(&sv, 2 * Nv * sizeof(double)));
  struct F { double* p; ~F() { cudaFree(p); } } fr{sv};
  yv = sv + Nv;
  for (int k = 0; k < G.ncolors; ++k)
    for (int comp = 0; comp < nc; ++comp) {
      DGVV_CUDA_TRY(launch_cg_probe_set(sv, G.d_color, k, comp, G.nv, nc, s));
      TRY(cg_apply(c, op, sv, yv, s));
      DGVV_CUDA_TRY(launch_cg_probe_get(yv, G.dinv[oi], G.d_color, k, comp, G.nv, s));
    }
  std::vector<double> h(Nv);
  DGVV_CUDA_TRY(cudaMemcpyAsync(h.data(), G.dinv[oi], Nv * sizeof(double), cudaMemcpyDeviceToHost, s));
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  for (long i = 0; i < Nv; ++i) {
    if (!(h[i] > 0.0)) return dgvv_fail(DGVV_EDOMAIN, "continuous level: non-positive diagonal entry %ld", i);
    h[i] = 1.0 / h[i];
  }
  DGVV_CUDA_TRY(cudaMemcpyAsync(G.dinv[oi], h.data(), Nv * sizeof(double), cudaMemcpyHostToDevice, s));
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  G.dinv_epoch[oi] = c->coef_epoch;
  return DGVV_OK;
}

// Chebyshev(degree) on the continuous level (SURVEY §8(c) c1.6 with the level's diagonal)
DGVV_INTERNAL dgvv_status cg_cheb(dgvv_ctx* c, int op, double* x, const double* b, int degree, double lo, double hi,
                           bool x_is_zero, cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  auto& G = c->cg;
  const long Nv = (long)nc * G.nv;
  TRY(cg_ensure_dinv(c, op, s));
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
  double rho = 1.0 / sigma;
  if (x_is_zero) {
    DGVV_CUDA_TRY(cudaMemsetAsync(x, 0, Nv * sizeof(double), s));
    DGVV_CUDA_TRY(launch_cheb_vec(b, G.dinv[oi], 0.0, 1.0 / theta, G.d[oi], x, Nv, s));
  } else {
    TRY(cg_apply(c, op, x, G.r[oi], s));
    DGVV_CUDA_TRY(launch_axpby(1.0, b, -1.0, G.r[oi], Nv, s));                 // r = b - A x
    DGVV_CUDA_TRY(launch_cheb_vec(G.r[oi], G.dinv[oi], 0.0, 1.0 / theta, G.d[oi], x, Nv, s));
  }
  for (int j = 1; j < degree; ++j) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    TRY(cg_apply(c, op, x, G.r[oi], s));
    DGVV_CUDA_TRY(launch_axpby(1.0, b, -1.0, G.r[oi], Nv, s));
    DGVV_CUDA_TRY(launch_cheb_vec(G.r[oi], G.dinv[oi], rho_new * rho, 2.0 * rho_new / delta, G.d[oi], x, Nv, s));
    rho = rho_new;
  }
  return DGVV_OK;
}

// nested Q1 prolongation (reading C3) from c->coarse's continuous level to c's, as CSR; R = P^T
DGVV_INTERNAL dgvv_status cg_build_transfer(dgvv_ctx* c) {
  dgvv_ctx* cc = c->coarse;
  auto& G = c->cg;
  if (G.transfer_to == cc) return DGVV_OK;
  if ((int)c->h_parent.size() != c->n_owned) return dgvv_fail(DGVV_ESTATE, "continuous level: no parent map");
  const int nvf = G.nv, nvc = cc->cg.nv;
  std::vector<std::vector<std::pair<int, double>>> rows(nvf);
  std::vector<char> done(nvf, 0);
  for (int f = 0; f < c->n_owned; ++f)
    for (int o = 0; o < 8; ++o) {
      const int v = G.h_vid[(size_t)f * 8 + o];
      if (done[v]) continue;
      done[v] = 1;
      const int p = c->h_parent[f], oc = c->h_octant[f];
      double t[3];
      for (int a = 0; a < 3; ++a) t[a] = 0.5 * ((o >> a) & 1) + 0.5 * ((oc >> a) & 1);
      for (int co = 0; co < 8; ++co) {
        double w = 1.0;
        for (int a = 0; a < 3; ++a) w *= ((co >> a) & 1) ? t[a] : 1.0 - t[a];
        if (w == 0.0) continue;
        const int vc = cc->cg.h_vid[(size_t)p * 8 + co];
        bool merged = false;
        for (auto& e : rows[v])
          if (e.first == vc) { e.second += w; merged = true; }
        if (!merged) rows[v].push_back({vc, w});
      }
    }
  std::vector<int> pp(nvf + 1, 0), pc, rp(nvc + 1, 0), rc;
  std::vector<double> pv, rv;
  for (int v = 0; v < nvf; ++v) {
    for (auto& e : rows[v]) { pc.push_back(e.first); pv.push_back(e.second); ++rp[e.first + 1]; }
    pp[v + 1] = (int)pc.size();
  }
  for (int v = 0; v < nvc; ++v) rp[v + 1] += rp[v];
  rc.resize(pc.size());
  rv.resize(pc.size());
  std::vector<int> fill(rp.begin(), rp.end() - 1);
  for (int v = 0; v < nvf; ++v)
    for (int j = pp[v]; j < pp[v + 1]; ++j) { rc[fill[pc[j]]] = v; rv[fill[pc[j]]++] = pv[j]; }
  auto up_i = [&](int** d, const std::vector<int>& h) -> dgvv_status {
    if (*d) { cudaFree(*d); c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), (void*)*d), c->allocs.end()); }
    TRY(dalloc(c, d, h.size()));
    DGVV_CUDA_TRY(cudaMemcpy(*d, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice));
    return DGVV_OK;
  };
  auto up_d = [&](double** d, const std::vector<double>& h) -> dgvv_status {
    if (*d) { cudaFree(*d); c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), (void*)*d), c->allocs.end()); }
    TRY(dalloc(c, d, h.size()));
    DGVV_CUDA_TRY(cudaMemcpy(*d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
    return DGVV_OK;
  };
  TRY(up_i(&G.pp, pp)); TRY(up_i(&G.pc, pc)); TRY(up_d(&G.pv, pv));
  TRY(up_i(&G.rp, rp)); TRY(up_i(&G.rc, rc)); TRY(up_d(&G.rv, rv));
  G.transfer_to = cc;
  return DGVV_OK;
}

// V-cycle over the continuous levels: this context's, then (nested Q1) its coarse contexts'
DGVV_INTERNAL dgvv_status cg_vcycle(dgvv_ctx* c, int op, const double* b, double* x, const double* his, cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  auto& G = c->cg;
  if (!c->coarse && G.Ainv[oi]) {
    if (G.direct_epoch[oi] != c->coef_epoch)
      return dgvv_fail(DGVV_ESTATE, "direct coarse solver is stale (coefficients or mass changed): call dgvv_setup_coarse_solver again");
    DGVV_CUDA_TRY(launch_dense_matvec(G.Ainv[oi], b, x, G.direct_n[oi], s));
    return DGVV_OK;
  }
  const double hi = his[0], lo = hi / 20.0;
  TRY(cg_cheb(c, op, x, b, 5, lo, hi, true, s));
  if (!c->coarse) return DGVV_OK;
  TRY(cg_build_transfer(c));
  const long Nv = (long)nc * G.nv;
  TRY(cg_apply(c, op, x, G.r[oi], s));
  DGVV_CUDA_TRY(launch_axpby(1.0, b, -1.0, G.r[oi], Nv, s));
  DGVV_CUDA_TRY(launch_csr_spmv(G.rp, G.rc, G.rv, G.r[oi], G.hb[oi], c->coarse->cg.nv, G.nv, nc, 0.0, s));
  TRY(cg_vcycle(c->coarse, op, G.hb[oi], G.hx[oi], his + 1, s));
  DGVV_CUDA_TRY(launch_csr_spmv(G.pp, G.pc, G.pv, G.hx[oi], x, G.nv, c->coarse->cg.nv, nc, 1.0, s));
  TRY(cg_cheb(c, op, x, b, 5, lo, hi, false, s));
  return DGVV_OK;
}

// from the DG_1 residual r_dg of c's last level: x_dg += P_c V_c(P_c^T r_dg)
DGVV_INTERNAL dgvv_status cg_enter(dgvv_ctx* c, int op, const double* r_dg, double* x_dg, const double* his, cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  auto& G = c->cg;
  DGVV_CUDA_TRY(launch_cg_embedT(r_dg, G.b0[oi], G.d_inc_ptr, G.d_inc, G.nv, nc, 0.0, s));
  TRY(cg_vcycle(c, op, G.b0[oi], G.x0[oi], his, s));
  DGVV_CUDA_TRY(launch_cg_embed(G.x0[oi], x_dg, G.d_vid, c->n_owned, G.nv, nc, 1.0, s));
  return DGVV_OK;
}

DGVV_INTERNAL dgvv_status cg_setup_direct(dgvv_ctx* c, int op, int32_t* n_dofs) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  auto& G = c->cg;
  const long N = (long)nc * G.nv;
  if (N > 4096) return dgvv_fail(DGVV_EINVAL, "direct coarse solver: %ld continuous DoFs (max 4096)", N);
  cudaStream_t s = 0;
  TRY(ensure_vcycle_scratch(c, op));
  double *cols = nullptr, *W = nullptr, *fac = nullptr, *e = nullptr;
  struct Tmp { double** p[4]; ~Tmp() { for (auto q : p) if (*q) cudaFree(*q); } } tmp{{&cols, &W, &fac, &e}};
  DGVV_CUDA_TRY(cudaMalloc(&cols, (size_t)N * N * sizeof(double)));
  DGVV_CUDA_TRY(cudaMalloc(&W, (size_t)2 * N * N * sizeof(double)));
  DGVV_CUDA_TRY(cudaMalloc(&fac, (size_t)N * sizeof(double)));
  DGVV_CUDA_TRY(cudaMalloc(&e, (size_t)N * sizeof(double)));
  for (long j = 0; j < N; ++j) {
    DGVV_CUDA_TRY(launch_set_unit(e, N, j, s));
    TRY(cg_apply(c, op, e, cols + (size_t)j * N, s));
  }
  if (!G.Ainv[oi]) TRY(dalloc(c, &G.Ainv[oi], (size_t)N * N));
  DGVV_CUDA_TRY(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
  DGVV_CUDA_TRY(launch_gauss_jordan_inverse(cols, W, fac, G.Ainv[oi], (int)N, c->d_flag, s));
  int bad = 0;
  DGVV_CUDA_TRY(cudaMemcpyAsync(&bad, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  if (bad) {                                  // drop the inverse: later V-cycles fall back to Chebyshev
    cudaFree(G.Ainv[oi]);
    c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), (void*)G.Ainv[oi]), c->allocs.end());
    G.Ainv[oi] = nullptr;
    G.direct_epoch[oi] = -1;
    return dgvv_fail(DGVV_EDOMAIN, "direct coarse solver: %d non-positive pivots (operator not SPD?)", bad);
  }
  G.direct_n[oi] = (int)N;
  G.direct_epoch[oi] = c->coef_epoch;
  if (n_dofs) *n_dofs = (int32_t)N;
  return DGVV_OK;
}

dgvv_status dgvv_set_continuous_level(dgvv_ctx* c, int32_t enable) {
  DGVV_RANGE();
  TRY(check_ctx(c));
  if (!enable) { c->cg.on = false; return DGVV_OK; }
  if (c->L.back().k != 1) return dgvv_fail(DGVV_EINVAL, "continuous level: the coarsest degree must be 1 (is %d)", c->L.back().k);
  if (c->n_ghost || c->comm) return dgvv_fail(DGVV_EUNSUPPORTED, "continuous level: single-GPU contexts only");
  auto& G = c->cg;
  if (G.nv == 0) {
    const int nc8 = c->n_owned * 8;
    std::vector<int> par(nc8);
    for (int i = 0; i < nc8; ++i) par[i] = i;
    auto find = [&](int x) { while (par[x] != x) { par[x] = par[par[x]]; x = par[x]; } return x; };
    for (int K = 0; K < c->n_owned; ++K)
      for (int f = 0; f < 6; ++f) {
        const int nb = c->h_nbr[(size_t)K * 6 + f];
        if (nb < 0 || nb >= c->n_owned) continue;
        const int d = f >> 1, sd = f & 1;
        for (int o = 0; o < 8; ++o) {
          if (((o >> d) & 1) != sd) continue;
          const int a = find(K * 8 + o), b = find(nb * 8 + (o ^ (1 << d)));
          if (a != b) par[std::max(a, b)] = std::min(a, b);
        }
      }
    std::vector<int> id(nc8, -1);
    G.h_vid.assign(nc8, 0);
    int nv = 0;
    for (int i = 0; i < nc8; ++i) {
      const int r = find(i);
      if (id[r] < 0) id[r] = nv++;
      G.h_vid[i] = id[r];
    }
    std::vector<int> ptr(nv + 1, 0), inc(nc8);
    for (int i = 0; i < nc8; ++i) ++ptr[G.h_vid[i] + 1];
    for (int v = 0; v < nv; ++v) ptr[v + 1] += ptr[v];
    std::vector<int> fill(ptr.begin(), ptr.end() - 1);
    for (int i = 0; i < nc8; ++i) inc[fill[G.h_vid[i]]++] = i;
    std::vector<int> color(nv, -1);                 // greedy colouring of the "shares a cell" graph
    int ncol = 0;
    std::vector<int> mark;
    for (int v = 0; v < nv; ++v) {
      mark.assign(ncol + 1, 0);
      for (int j = ptr[v]; j < ptr[v + 1]; ++j) {
        const int K = inc[j] >> 3;
        for (int o = 0; o < 8; ++o) {
          const int w = G.h_vid[(size_t)K * 8 + o];
          if (color[w] >= 0) mark[color[w]] = 1;
        }
      }
      int col = 0;
      while (mark[col]) ++col;
      color[v] = col;
      ncol = std::max(ncol, col + 1);
    }
    TRY(dalloc(c, &G.d_vid, (size_t)nc8));
    TRY(dalloc(c, &G.d_inc_ptr, (size_t)nv + 1));
    TRY(dalloc(c, &G.d_inc, (size_t)nc8));
    TRY(dalloc(c, &G.d_color, (size_t)nv));
    DGVV_CUDA_TRY(cudaMemcpy(G.d_vid, G.h_vid.data(), nc8 * sizeof(int), cudaMemcpyHostToDevice));
    DGVV_CUDA_TRY(cudaMemcpy(G.d_inc_ptr, ptr.data(), (nv + 1) * sizeof(int), cudaMemcpyHostToDevice));
    DGVV_CUDA_TRY(cudaMemcpy(G.d_inc, inc.data(), nc8 * sizeof(int), cudaMemcpyHostToDevice));
    DGVV_CUDA_TRY(cudaMemcpy(G.d_color, color.data(), nv * sizeof(int), cudaMemcpyHostToDevice));
    G.nv = nv;
    G.ncolors = ncol;
  }
  G.on = true;
  return DGVV_OK;
}

dgvv_status dgvv_continuous_level_info(const dgvv_ctx* c, int32_t* n_vertices, int32_t* n_colors) {
  DGVV_RANGE();
  TRY(check_ctx(c));
  if (!c->cg.on) return dgvv_fail(DGVV_ESTATE, "continuous level not enabled");
  if (n_vertices) *n_vertices = c->cg.nv;
  if (n_colors) *n_colors = c->cg.ncolors;
  return DGVV_OK;
}

dgvv_status dgvv_apply_continuous(dgvv_ctx* c, int32_t op, const double* src, double* dst, dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (!c->cg.on) return dgvv_fail(DGVV_ESTATE, "continuous level not enabled");
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  TRY(op_ready(c, op));
  TRY(ensure_vcycle_scratch(c, op));
  return cg_apply(c, op, src, dst, (cudaStream_t)stream);
}

dgvv_status dgvv_embed_continuous(dgvv_ctx* c, int32_t op, int32_t transpose, const double* src, double* dst,
                                  double beta, dgvv_stream stream) {
  DGVV_RANGE();
  if (!c || !src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (!c->cg.on) return dgvv_fail(DGVV_ESTATE, "continuous level not enabled");
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  cudaStream_t s = (cudaStream_t)stream;
  if (transpose) DGVV_CUDA_TRY(launch_cg_embedT(src, dst, c->cg.d_inc_ptr, c->cg.d_inc, c->cg.nv, nc, beta, s));
  else DGVV_CUDA_TRY(launch_cg_embed(src, dst, c->cg.d_vid, c->n_owned, c->cg.nv, nc, beta, s));
  return DGVV_OK;
}

// ------------------------------------------------------------------ f3: h-levels, direct coarse solve
DGVV_INTERNAL dgvv_status hprolong_impl(dgvv_ctx* c, int op, const double* coarse, double* fine, double beta,
                                 cudaStream_t s) {
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  cudaError_t e = launch_hprolongate(c->L.back().n, nc, coarse, fine, c->d_parent, c->d_octant, beta, c->n_owned, s);
  if (e == cudaErrorNotSupported) return dgvv_fail(DGVV_EUNSUPPORTED, "h-transfer not built for degree %d", c->L.back().k);
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "h-prolongation: %s", cudaGetErrorString(e));
  return DGVV_OK;
}

DGVV_INTERNAL dgvv_status hrestrict_impl(dgvv_ctx* c, int op, const double* fine, double* coarse, double beta,
                                  cudaStream_t s) {
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  cudaError_t e = launch_hrestrict(c->L.back().n, nc, fine, coarse, c->d_child, beta, c->coarse->n_owned, s);
  if (e == cudaErrorNotSupported) return dgvv_fail(DGVV_EUNSUPPORTED, "h-transfer not built for degree %d", c->L.back().k);
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "h-restriction: %s", cudaGetErrorString(e));
  return DGVV_OK;
}

dgvv_status dgvv_set_coarse_context(dgvv_ctx* c, dgvv_ctx* cc, const int32_t* parent, const int8_t* octant) {
  DGVV_RANGE();
  if (!c || !cc || !parent || !octant) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (c == cc) return dgvv_fail(DGVV_EINVAL, "a context cannot be its own coarse level");
  for (dgvv_ctx* q = cc; q; q = q->coarse)
    if (q == c) return dgvv_fail(DGVV_EINVAL, "coarse-context chain would form a cycle");
  // across ranks: both contexts on the communicator, partitions nested (every owned fine cell's
  // parent is an owned coarse cell, checked below), so the h-transfers stay rank-local and the
  // coarse levels exchange their own ghosts
  if ((c->comm == nullptr) != (cc->comm == nullptr) || (c->n_ghost && !c->comm) || (cc->n_ghost && !cc->comm))
    return dgvv_fail(DGVV_EUNSUPPORTED, "h-levels across ranks need a communicator on both contexts");
  if (cc->L[0].k != c->L.back().k)
    return dgvv_fail(DGVV_EINVAL, "coarse context degree %d != coarsest level degree %d", cc->L[0].k, c->L.back().k);
  const int nf = c->n_owned, ncs = cc->n_owned;
  if ((long)ncs * 8 != (long)nf) return dgvv_fail(DGVV_EINVAL, "fine cells (%d) != 8 x coarse cells (%d)", nf, ncs);
  std::vector<int> child((size_t)ncs * 8, -1);
  for (int f = 0; f < nf; ++f) {
    const int p = parent[f], o = octant[f];
    if (p < 0 || p >= ncs || o < 0 || o > 7) return dgvv_fail(DGVV_EINVAL, "fine cell %d: parent %d / octant %d out of range", f, p, o);
    if (child[(size_t)p * 8 + o] >= 0) return dgvv_fail(DGVV_EINVAL, "coarse cell %d has two children in octant %d", p, o);
    child[(size_t)p * 8 + o] = f;
  }
  if (!c->d_parent) TRY(dalloc(c, &c->d_parent, (size_t)nf));
  if (!c->d_octant) TRY(dalloc(c, &c->d_octant, (size_t)nf));
  if (!c->d_child) TRY(dalloc(c, &c->d_child, (size_t)ncs * 8));
  DGVV_CUDA_TRY(cudaMemcpy(c->d_parent, parent, nf * sizeof(int), cudaMemcpyHostToDevice));
  DGVV_CUDA_TRY(cudaMemcpy(c->d_octant, octant, nf, cudaMemcpyHostToDevice));
  DGVV_CUDA_TRY(cudaMemcpy(c->d_child, child.data(), child.size() * sizeof(int), cudaMemcpyHostToDevice));
  c->h_parent.assign(parent, parent + nf);
  c->h_octant.assign(octant, octant + nf);
  c->cg.transfer_to = nullptr;               // continuous-level transfers rebuilt on demand
  if (c->coarse != cc) {                     // buffers sized by the previous coarse context
    auto drop = [&](void** pp) {
      if (*pp) {
        cudaFree(*pp);
        c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), *pp), c->allocs.end());
        *pp = nullptr;
      }
    };
    for (int o = 0; o < 2; ++o) {
      drop((void**)&c->hb[o]);
      drop((void**)&c->hx[o]);
      drop((void**)&c->hbf[o]);
      drop((void**)&c->hxf[o]);
      drop((void**)&c->cg.hb[o]);
      drop((void**)&c->cg.hx[o]);
    }
  }
  c->coarse = cc;
  return DGVV_OK;
}

DGVV_INTERNAL dgvv_status h_ready(dgvv_ctx* c, int op) {
  TRY(check_ctx(c));
  if (!c->coarse) return dgvv_fail(DGVV_ESTATE, "no coarse context: call dgvv_set_coarse_context first");
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  return DGVV_OK;
}

dgvv_status dgvv_prolongate_h(dgvv_ctx* c, int32_t op, const double* coarse, double* fine, double beta,
                              dgvv_stream stream) {
  DGVV_RANGE();
  TRY(h_ready(c, op));
  if (!coarse || !fine) return dgvv_fail(DGVV_EINVAL, "null vector");
  return hprolong_impl(c, op, coarse, fine, beta, (cudaStream_t)stream);
}

dgvv_status dgvv_restrict_h(dgvv_ctx* c, int32_t op, const double* fine, double* coarse, double beta,
                            dgvv_stream stream) {
  DGVV_RANGE();
  TRY(h_ready(c, op));
  if (!coarse || !fine) return dgvv_fail(DGVV_EINVAL, "null vector");
  return hrestrict_impl(c, op, fine, coarse, beta, (cudaStream_t)stream);
}

dgvv_status dgvv_setup_coarse_solver(dgvv_ctx* c, int32_t op, int32_t* n_dofs) {
  DGVV_RANGE();
  TRY(check_ctx(c));
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  TRY(op_ready(c, op));
  if (c->n_ghost && !c->comm)
    return dgvv_fail(DGVV_EUNSUPPORTED, "direct coarse solver: external-exchange contexts (no communicator) are not supported");
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  const int l = (int)c->L.size() - 1;
  if (c->cg.on) return cg_setup_direct(c, op, n_dofs);
  // multi-rank (communicator): every rank assembles its owned rows of every global column with the
  // distributed apply (ghost exchange included), the columns are gathered (exact zero-padded sum)
  // and every rank inverts the same matrix; a solve applies this rank's rows to the gathered b
  const bool mr = c->comm != nullptr;
  const long Nown = (long)nc * level_dofs(c, l);
  const long len = c->n_owned ? Nown / c->n_owned : 0;
  const long N = mr ? (long)nc * (long)c->n_global * ((long)c->L[l].n * c->L[l].n * c->L[l].n) : Nown;
  const long off = mr ? (long)c->first * (len ? len : (long)nc * c->L[l].n * c->L[l].n * c->L[l].n) : 0;
  if (N > 4096) return dgvv_fail(DGVV_EINVAL, "direct coarse solver: %ld DoFs on the coarsest level (max 4096)", N);
  cudaStream_t s = 0;
  double *cols = nullptr, *W = nullptr, *fac = nullptr, *e = nullptr;
  struct Tmp { double** p[4]; ~Tmp() { for (auto q : p) if (*q) cudaFree(*q); } } tmp{{&cols, &W, &fac, &e}};
  DGVV_CUDA_TRY(cudaMalloc(&cols, (size_t)N * N * sizeof(double)));
  DGVV_CUDA_TRY(cudaMalloc(&W, (size_t)2 * N * N * sizeof(double)));
  DGVV_CUDA_TRY(cudaMalloc(&fac, (size_t)N * sizeof(double)));
  DGVV_CUDA_TRY(cudaMalloc(&e, (size_t)(Nown > 0 ? Nown : 1) * sizeof(double)));
  if (mr) DGVV_CUDA_TRY(cudaMemsetAsync(cols, 0, (size_t)N * N * sizeof(double), s));
  for (long j = 0; j < N; ++j) {               // column j = A e_j (the level's matrix-free apply)
    DGVV_CUDA_TRY(launch_set_unit(e, Nown, j - off, s));
    ApplyArgs a = base_args(c, l, op);
    a.src = e;
    a.dst = cols + (size_t)j * N + off;        // this rank's rows of column j
    TRY(run_apply(c, op, l, a, s));
  }
  if (mr) TRY(comm_allreduce(c, cols, N * N, s));
  if (!c->Ainv[oi]) TRY(dalloc(c, &c->Ainv[oi], (size_t)N * N));
  DGVV_CUDA_TRY(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
  DGVV_CUDA_TRY(launch_gauss_jordan_inverse(cols, W, fac, c->Ainv[oi], (int)N, c->d_flag, s));
  int bad = 0;
  DGVV_CUDA_TRY(cudaMemcpyAsync(&bad, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  if (bad) {
    cudaFree(c->Ainv[oi]);
    c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), (void*)c->Ainv[oi]), c->allocs.end());
    c->Ainv[oi] = nullptr;
    return dgvv_fail(DGVV_EDOMAIN, "direct coarse solver: %d non-positive pivots (operator not SPD?)", bad);
  }
  c->direct_n[oi] = (int)N;
  c->direct_off[oi] = off;
  c->direct_rows[oi] = (int)Nown;
  if (mr && !c->direct_bf[oi]) TRY(dalloc(c, &c->direct_bf[oi], (size_t)4096));
  c->direct_epoch[oi] = c->coef_epoch;
  if (n_dofs) *n_dofs = (int32_t)N;
  return DGVV_OK;
}

}  // extern "C"
