// api_core.cu — C ABI: errors, communicators, context setup/destroy,
// viscosity update (a2), operator applies (a3-a7, incl. the host-buffer pipeline), dots, sizes, ghosts.
#include "api_internal.cuh"

extern "C" {

const char* dgvv_last_error(void) { return g_err.c_str(); }
const char* dgvv_version(void) { return "dgvv 0.1 (sm_100a, fp64)"; }

dgvv_status dgvv_nccl_get_unique_id(char out_id[128]) {
  DGVV_RANGE();
  TRY(nccl_load());
  ncclUniqueId id;
  NCCL_TRY(g_nccl.getUniqueId(&id));
  std::memcpy(out_id, id.internal, 128);
  return DGVV_OK;
}

dgvv_status dgvv_nccl_comm_init(const char id_bytes[128], int32_t nranks, int32_t rank, void** comm) {
  DGVV_RANGE();
  TRY(nccl_load());
  ncclUniqueId id;
  std::memcpy(id.internal, id_bytes, 128);
  ncclComm_t nc;
  NCCL_TRY(g_nccl.commInitRank(&nc, nranks, id, rank));
  DgvvComm* cm = new DgvvComm;
  cm->kind = COMM_NCCL;
  cm->nccl = nc;
  cm->rank = rank;
  *comm = (void*)cm;
  return DGVV_OK;
}

dgvv_status dgvv_nccl_comm_destroy(void* comm) {
  DGVV_RANGE();
  if (!comm) return DGVV_OK;
  DgvvComm* cm = (DgvvComm*)comm;
  if (cm->kind != COMM_NCCL) return dgvv_fail(DGVV_EINVAL, "not an NCCL communicator");
  TRY(nccl_load());
  NCCL_TRY(g_nccl.commDestroy(cm->nccl));
  delete cm;
  return DGVV_OK;
}

dgvv_status dgvv_thread_group_create(int32_t nranks, void** group) {
  DGVV_RANGE();
  if (nranks < 1 || nranks > 64 || !group) return dgvv_fail(DGVV_EINVAL, "thread group: 1 <= nranks <= 64");
  ThreadGroup* g = new ThreadGroup;
  g->R = nranks;
  g->sptr.assign(nranks, std::vector<const void*>(nranks, nullptr));
  g->sbytes.assign(nranks, std::vector<size_t>(nranks, 0));
  g->ev_a.assign(nranks, nullptr);
  g->ev_b.assign(nranks, nullptr);
  g->red.assign(nranks, nullptr);
  g->hval.assign(nranks, 0);
  g->comms.resize(nranks);
  for (int r = 0; r < nranks; ++r) {
    g->comms[r].kind = COMM_THREADS;
    g->comms[r].tg = g;
    g->comms[r].rank = r;
  }
  *group = (void*)g;
  return DGVV_OK;
}

dgvv_status dgvv_thread_group_comm(void* group, int32_t rank, void** comm) {
  DGVV_RANGE();
  ThreadGroup* g = (ThreadGroup*)group;
  if (!g || !comm || rank < 0 || rank >= g->R) return dgvv_fail(DGVV_EINVAL, "thread group: bad rank %d", rank);
  *comm = (void*)&g->comms[rank];
  return DGVV_OK;
}

dgvv_status dgvv_thread_group_destroy(void* group) {
  DGVV_RANGE();
  delete (ThreadGroup*)group;
  return DGVV_OK;
}

void dgvv_destroy(dgvv_ctx* c) {
  if (!c) return;
  for (auto& L : c->L)
    for (int o = 0; o < 2; ++o) L.scratch[o].clear();
  for (void* p : c->allocs) cudaFree(p);
  for (cudaEvent_t e : c->hp.ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : c->hp.ev_out) cudaEventDestroy(e);
  if (c->hp.ev_start) cudaEventDestroy(c->hp.ev_start);
  if (c->hp.ev_done) cudaEventDestroy(c->hp.ev_done);
  for (int i = 0; i < 2; ++i)
    if (c->hp.cs[i]) cudaStreamDestroy(c->hp.cs[i]);
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  if (c->ev_red) cudaEventDestroy(c->ev_red);
  if (c->ev_red2) cudaEventDestroy(c->ev_red2);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  delete c;
}

DGVV_INTERNAL dgvv_status setup_impl(const dgvv_mesh* m, int32_t degree, const dgvv_law* vl, const dgvv_law* pl,
                              const dgvv_options* opt, cudaStream_t s, dgvv_ctx* c) {
  if (!m || !m->neighbor || !m->nodes) return dgvv_fail(DGVV_EINVAL, "mesh, neighbor and nodes are required");
  if (m->n_cells <= 0 || m->n_ghost < 0) return dgvv_fail(DGVV_EINVAL, "n_cells must be > 0");
  if (m->n_ghost > 0 && (!m->ghost_global_id || !m->ghost_owner))
    return dgvv_fail(DGVV_EINVAL, "ghost ids/owners required when n_ghost > 0");
  if (m->map_degree < 1 || m->map_degree > 7) return dgvv_fail(DGVV_EUNSUPPORTED, "map_degree %d not in 1..7", m->map_degree);
  if (!vl && !pl) return dgvv_fail(DGVV_EINVAL, "at least one of visc_law / poisson_law is required");
  TRY(upload_tables());
  DGVV_CUDA_TRY(cudaGetDevice(&c->device));

  c->n_owned = m->n_cells;
  c->n_ghost = m->n_ghost;
  c->n_total = m->n_cells + m->n_ghost;
  c->first = m->first_global_cell;
  c->map_degree = m->map_degree;
  c->ip = (opt && opt->ip_factor > 0.0) ? opt->ip_factor : 1.0;
  c->form = opt ? opt->formulation : DGVV_FORM_DIVERGENCE;
  if (c->form != DGVV_FORM_DIVERGENCE && c->form != DGVV_FORM_LAPLACE)
    return dgvv_fail(DGVV_EINVAL, "formulation %d", c->form);

  // levels
  std::vector<int> degs;
  if (opt && opt->n_levels > 0 && opt->degrees) degs.assign(opt->degrees, opt->degrees + opt->n_levels);
  else degs.push_back(degree);
  if (degs[0] != degree) return dgvv_fail(DGVV_EINVAL, "degrees[0] (%d) must equal degree (%d)", degs[0], degree);
  for (int k : degs) {
    if (k < 1) return dgvv_fail(DGVV_EDOMAIN, "degree %d < 1", k);
    if (vl && k > 5) return dgvv_fail(DGVV_EUNSUPPORTED, "viscous operator: degree %d > 5", k);
    if (k > 6) return dgvv_fail(DGVV_EUNSUPPORTED, "degree %d > 6", k);
  }
  c->L.resize(degs.size());
  for (size_t l = 0; l < degs.size(); ++l) { c->L[l].k = degs[l]; c->L[l].n = degs[l] + 1; }
  if (vl) {
    c->visc = *vl;
    c->has_visc = true;
    if (vl->kind == DGVV_LAW_CARREAU) c->carreau = true;
    else if (vl->kind < 0 || vl->kind > 2) return dgvv_fail(DGVV_EINVAL, "unknown law kind %d", vl->kind);
  }
  if (pl) {
    c->pois = *pl;
    c->has_pois = true;
    if (pl->kind < 0 || pl->kind > 2) return dgvv_fail(DGVV_EUNSUPPORTED, "Poisson coefficient law kind %d (analytic only)", pl->kind);
  }

  // ---- local numbering: owned [0, n_owned), ghosts sorted by (owner, global id)
  std::vector<int> gperm(c->n_ghost);
  for (int i = 0; i < c->n_ghost; ++i) gperm[i] = i;
  std::sort(gperm.begin(), gperm.end(), [&](int x, int y) {
    if (m->ghost_owner[x] != m->ghost_owner[y]) return m->ghost_owner[x] < m->ghost_owner[y];
    return m->ghost_global_id[x] < m->ghost_global_id[y];
  });
  std::unordered_map<long long, int> gmap;
  for (int i = 0; i < c->n_ghost; ++i) gmap[m->ghost_global_id[gperm[i]]] = c->n_owned + i;
  auto row_of = [&](int local) -> int { return local < c->n_owned ? local : c->n_owned + gperm[local - c->n_owned]; };
  c->h_gperm = gperm;
  std::vector<int> nbr((size_t)c->n_total * 6);
  for (int lc = 0; lc < c->n_total; ++lc) {
    const int r = row_of(lc);
    for (int f = 0; f < 6; ++f) {
      const long long g = m->neighbor[(size_t)r * 6 + f];
      int v;
      if (g == -1 - DGVV_BC_DIRICHLET) v = NB_DIRICHLET;
      else if (g == -1 - DGVV_BC_NEUMANN) v = NB_NEUMANN;
      else if (g < 0) return dgvv_fail(DGVV_EINVAL, "cell %d face %d: bad neighbour code %lld", lc, f, g);
      else if (g >= c->first && g < c->first + c->n_owned) v = (int)(g - c->first);
      else {
        auto it = gmap.find(g);
        if (it != gmap.end()) v = it->second;
        else if (lc >= c->n_owned) v = NB_REMOTE;
        else return dgvv_fail(DGVV_EINVAL, "owned cell %d: neighbour %lld is neither owned nor a ghost", lc, g);
      }
      nbr[(size_t)lc * 6 + f] = v;
    }
  }
  // reciprocity inside the local set
  for (int lc = 0; lc < c->n_owned; ++lc)
    for (int f = 0; f < 6; ++f) {
      const int v = nbr[(size_t)lc * 6 + f];
      if (v >= 0 && v < c->n_owned && nbr[(size_t)v * 6 + (f ^ 1)] != lc)
        return dgvv_fail(DGVV_EUNSUPPORTED, "cell %d face %d: neighbour does not point back through the opposite face (unaligned mesh)", lc, f);
    }

  // ---- geometry input (reordered rows)
  const int m1 = m->map_degree + 1;
  const size_t row_len = (size_t)m1 * m1 * m1 * 3;
  std::vector<double> nodes((size_t)c->n_total * row_len);
  for (int lc = 0; lc < c->n_total; ++lc)
    std::memcpy(&nodes[(size_t)lc * row_len], m->nodes + (size_t)row_of(lc) * row_len, row_len * sizeof(double));
  // Cartesian fast path: every cell an axis-aligned box given by its 8 corners
  bool cart = (m->map_degree == 1);
  for (int lc = 0; cart && lc < c->n_total; ++lc) {
    const double* X = &nodes[(size_t)lc * row_len];
    double h[3];
    for (int d = 0; d < 3; ++d) h[d] = X[7 * 3 + d] - X[d];
    const double sc = std::fabs(h[0]) + std::fabs(h[1]) + std::fabs(h[2]);
    for (int d = 0; d < 3; ++d) if (!(h[d] > 0.0)) cart = false;
    for (int v = 0; cart && v < 8; ++v) {
      const int b[3] = {v & 1, (v >> 1) & 1, (v >> 2) & 1};
      for (int d = 0; d < 3; ++d)
        if (std::fabs(X[v * 3 + d] - (X[d] + b[d] * h[d])) > 1e-13 * sc) cart = false;
    }
  }
  c->geo = cart ? 0 : 1;

  TRY(dalloc(c, &c->d_part, 2 * kPartials));
  TRY(dalloc(c, &c->d_scal, 16));
  TRY(dalloc(c, &c->d_flag, 4));
  TRY(dalloc(c, &c->d_nbr, nbr.size()));
  c->h_nbr = nbr;
  DGVV_CUDA_TRY(cudaMemcpyAsync(c->d_nbr, c->h_nbr.data(), nbr.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  TRY(dalloc(c, &c->d_nodes, nodes.size()));
  DGVV_CUDA_TRY(cudaMemcpyAsync(c->d_nodes, nodes.data(), nodes.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  if (c->geo == 0) {
    TRY(dalloc(c, &c->d_cart, (size_t)c->n_total * CART_STRIDE));
    DGVV_CUDA_TRY(launch_cart_geom(c->d_nodes, c->d_nbr, c->n_total, c->d_cart, s));
    DGVV_CUDA_TRY(launch_cart_face(c->d_nbr, c->n_owned, c->d_cart, s));
  }

  // ---- per level: geometry, points, coefficients
  for (size_t l = 0; l < c->L.size(); ++l) {
    Level& L = c->L[l];
    const int n = L.n, n2 = n * n, n3 = n2 * n;
    double *xq = nullptr, *xf = nullptr;
    DGVV_CUDA_TRY(cudaMalloc(&xq, (size_t)c->n_total * n3 * 3 * sizeof(double)));
    DGVV_CUDA_TRY(cudaMalloc(&xf, (size_t)c->n_total * 6 * n2 * 3 * sizeof(double)));
    struct Tmp { double* a; double* b; ~Tmp() { cudaFree(a); cudaFree(b); } } tmp{xq, xf};
    if (c->geo == 0) {
      DGVV_CUDA_TRY(launch_cart_points(c->d_cart, c->n_total, c->n_total, n, xq, xf, s));
    } else {
      TRY(dalloc(c, &L.vJi, (size_t)c->n_total * 9 * n3));
      TRY(dalloc(c, &L.fJi, (size_t)c->n_total * 6 * 9 * n2));
      TRY(dalloc(c, &L.jxw, (size_t)c->n_total * n3));
      TRY(dalloc(c, &L.fdA, (size_t)c->n_total * 6 * n2));
      TRY(dalloc(c, &L.Hc, (size_t)c->n_total));
      GeoTab g;
      make_geotab(m->map_degree, n, &g);
      DGVV_CUDA_TRY(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
      DGVV_CUDA_TRY(launch_gen_geom(g, c->d_nodes, c->n_total, L.vJi, L.jxw, L.fJi, L.fdA, xq, xf, c->d_flag, s));
      int bad = 0;
      DGVV_CUDA_TRY(cudaMemcpyAsync(&bad, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
      DGVV_CUDA_TRY(cudaStreamSynchronize(s));
      if (bad) return dgvv_fail(DGVV_EDOMAIN, "level %zu: %d points with non-positive Jacobian", l, bad);
      DGVV_CUDA_TRY(launch_gen_H(L.jxw, L.fdA, c->d_nbr, c->n_total, n, L.Hc, s));
    }
    if (l == 0) {   // structured alignment of face quadrature points (needed by the kernels)
      double sc = 0.0;
      for (int d = 0; d < 3; ++d) sc = std::max(sc, std::fabs(nodes[(m1 * m1 * m1 - 1) * 3 + d] - nodes[d]));
      DGVV_CUDA_TRY(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
      DGVV_CUDA_TRY(launch_align_check(xf, c->d_nbr, c->n_owned, n, 1e-9 * std::max(sc, 1e-300), c->d_flag, s));
      int bad = 0;
      DGVV_CUDA_TRY(cudaMemcpyAsync(&bad, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
      DGVV_CUDA_TRY(cudaStreamSynchronize(s));
      if (bad) return dgvv_fail(DGVV_EUNSUPPORTED, "%d faces whose quadrature points do not match their neighbour's (mesh not structured/aligned)", bad);
    }
    if (c->has_visc) {
      TRY(dalloc(c, &L.nu_cell, (size_t)c->n_owned * n3));
      TRY(dalloc(c, &L.nu_face, (size_t)c->n_total * 6 * n2));
      if (c->geo == 1) {
        TRY(dalloc(c, &L.wv_cell, (size_t)c->n_owned * n3));
        TRY(dalloc(c, &L.wv_face, (size_t)c->n_total * 6 * n2));
      }
      if (!c->carreau) {
        TRY(eval_analytic(c, &c->visc, (int)l, xq, xf, L.nu_cell, L.nu_face, s));
        TRY(check_positive(c, L.nu_cell, (long)c->n_owned * n3, s, "viscosity (cells)"));
        TRY(check_positive(c, L.nu_face, (long)c->n_total * 6 * n2, s, "viscosity (faces)"));
        TRY(premultiply(c, (int)l, L.nu_cell, L.nu_face, L.wv_cell, L.wv_face, s));
      }
      if (c->n_ghost) {
        TRY(dalloc(c, &L.ghost[0], (size_t)c->n_ghost * 3 * n3));
        if (c->carreau) TRY(dalloc(c, &L.ulin_ghost, (size_t)c->n_ghost * 3 * n3));
      }
      if (c->carreau && l > 0) TRY(dalloc(c, &L.ulin, (size_t)c->n_owned * 3 * n3));
    }
    if (c->has_pois) {
      TRY(dalloc(c, &L.c_cell, (size_t)c->n_owned * n3));
      TRY(dalloc(c, &L.c_face, (size_t)c->n_total * 6 * n2));
      TRY(eval_analytic(c, &c->pois, (int)l, xq, xf, L.c_cell, L.c_face, s));
      TRY(check_positive(c, L.c_cell, (long)c->n_owned * n3, s, "Poisson coefficient (cells)"));
      TRY(check_positive(c, L.c_face, (long)c->n_total * 6 * n2, s, "Poisson coefficient (faces)"));
      if (c->geo == 1) {
        TRY(dalloc(c, &L.wc_cell, (size_t)c->n_owned * n3));
        TRY(dalloc(c, &L.wc_face, (size_t)c->n_total * 6 * n2));
        TRY(premultiply(c, (int)l, L.c_cell, L.c_face, L.wc_cell, L.wc_face, s));
      }
      if (c->n_ghost) TRY(dalloc(c, &L.ghost[1], (size_t)c->n_ghost * n3));
    }
    DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  }

  // ---- communication plan: peers from the ghost owners (sorted), send lists by the rule of
  // partition.py (owned cells with a face neighbour owned by the peer, ascending id)
  if (c->n_ghost > 0) {
    std::vector<int> owners;
    for (int i = 0; i < c->n_ghost; ++i) owners.push_back(m->ghost_owner[gperm[i]]);
    std::vector<int> uniq = owners;
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    size_t total_send = 0, total_send_f = 0;
    for (int r : uniq) {
      Peer P;
      P.rank = r;
      P.recv_off = (int)(std::lower_bound(owners.begin(), owners.end(), r) - owners.begin());
      P.n_recv = (int)(std::upper_bound(owners.begin(), owners.end(), r) - owners.begin()) - P.recv_off;
      std::vector<int> send;
      for (int lc = 0; lc < c->n_owned; ++lc)
        for (int f = 0; f < 6; ++f) {
          const int v = nbr[(size_t)lc * 6 + f];
          if (v >= c->n_owned && owners[v - c->n_owned] == r) { send.push_back(lc); break; }
        }
      P.n_send = (int)send.size();
      TRY(dalloc(c, &P.d_send, send.size()));
      DGVV_CUDA_TRY(cudaMemcpy(P.d_send, send.data(), send.size() * sizeof(int), cudaMemcpyHostToDevice));
      total_send += send.size();
      // face-trace items: (owned cell, face) with the neighbour owned by r, ascending
      std::vector<int> fc, ff;
      for (int lc = 0; lc < c->n_owned; ++lc)
        for (int f = 0; f < 6; ++f) {
          const int v = nbr[(size_t)lc * 6 + f];
          if (v >= c->n_owned && owners[v - c->n_owned] == r) { fc.push_back(lc); ff.push_back(f); }
        }
      P.n_send_f = (int)fc.size();
      TRY(dalloc(c, &P.d_fcell, fc.size()));
      TRY(dalloc(c, &P.d_fface, ff.size()));
      DGVV_CUDA_TRY(cudaMemcpy(P.d_fcell, fc.data(), fc.size() * sizeof(int), cudaMemcpyHostToDevice));
      DGVV_CUDA_TRY(cudaMemcpy(P.d_fface, ff.data(), ff.size() * sizeof(int), cudaMemcpyHostToDevice));
      total_send_f += fc.size();
      c->peers.push_back(P);
    }
    // received items: the faces of each peer's ghosts that touch an owned cell, in ghost order
    std::vector<int> gslot((size_t)c->n_ghost * 6, -1);
    int item = 0;
    for (auto& P : c->peers) {
      P.recv_off_f = item;
      for (int g = P.recv_off; g < P.recv_off + P.n_recv; ++g)
        for (int f = 0; f < 6; ++f) {
          const int v = nbr[(size_t)(c->n_owned + g) * 6 + f];
          if (v >= 0 && v < c->n_owned) gslot[(size_t)g * 6 + f] = item++;
        }
      P.n_recv_f = item - P.recv_off_f;
    }
    c->n_recv_f = item;
    TRY(dalloc(c, &c->d_gslot, gslot.size()));
    DGVV_CUDA_TRY(cudaMemcpy(c->d_gslot, gslot.data(), gslot.size() * sizeof(int), cudaMemcpyHostToDevice));
    int nmax = 0;
    for (auto& L : c->L) nmax = std::max(nmax, L.n);
    c->sendbuf_len = std::max(total_send * 3 * nmax * nmax * nmax, total_send_f * 2 * 3 * nmax * nmax);
    TRY(dalloc(c, &c->d_sendbuf, c->sendbuf_len));
    std::vector<int> inner, bnd;
    for (int lc = 0; lc < c->n_owned; ++lc) {
      bool g = false;
      for (int f = 0; f < 6; ++f) g |= nbr[(size_t)lc * 6 + f] >= c->n_owned;
      (g ? bnd : inner).push_back(lc);
    }
    c->n_interior = (int)inner.size();
    c->n_boundary = (int)bnd.size();
    TRY(dalloc(c, &c->d_interior, inner.size()));
    TRY(dalloc(c, &c->d_boundary, bnd.size()));
    DGVV_CUDA_TRY(cudaMemcpy(c->d_interior, inner.data(), inner.size() * sizeof(int), cudaMemcpyHostToDevice));
    DGVV_CUDA_TRY(cudaMemcpy(c->d_boundary, bnd.data(), bnd.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  if (opt && opt->nccl_comm) {
    DgvvComm* cm = (DgvvComm*)opt->nccl_comm;
    if (cm->kind != COMM_NCCL && cm->kind != COMM_THREADS) return dgvv_fail(DGVV_EINVAL, "not a dgvv communicator");
    if (cm->kind == COMM_NCCL) TRY(nccl_load());
    c->comm = opt->nccl_comm;
    DGVV_CUDA_TRY(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    DGVV_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
    DGVV_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));
    DGVV_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_red, cudaEventDisableTiming));
    DGVV_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_red2, cudaEventDisableTiming));
    TRY(dalloc(c, &c->tg_red, 8));
    c->tg_red_cap = 8;
    if (cm->kind == COMM_THREADS) {               // handshake: send counts vs listed ghosts
      ThreadGroup* g = cm->tg;
      {
        std::lock_guard<std::mutex> lk(g->mu);
        for (int q = 0; q < g->R; ++q) g->sbytes[cm->rank][q] = 0;
        for (auto& P : c->peers) g->sbytes[cm->rank][P.rank] = (size_t)P.n_send + ((size_t)P.n_send_f << 32);
      }
      tg_barrier(g);
      std::string bad;
      for (auto& P : c->peers)
        if (g->sbytes[P.rank][cm->rank] != (size_t)P.n_recv + ((size_t)P.n_recv_f << 32)) bad = "peer count mismatch";
      tg_barrier(g);
      if (!bad.empty()) return dgvv_fail(DGVV_EINVAL, "thread group: a peer sends a different number of cells than the ghosts listed");
    } else if (!c->peers.empty()) {
      // handshake: every peer's send counts (cells, trace items) must equal what is listed here
      const size_t np = c->peers.size();
      int* d_cnt = nullptr;
      TRY(dalloc(c, &d_cnt, 4 * np));
      std::vector<int> hs(2 * np);
      for (size_t i = 0; i < np; ++i) { hs[2 * i] = c->peers[i].n_send; hs[2 * i + 1] = c->peers[i].n_send_f; }
      DGVV_CUDA_TRY(cudaMemcpy(d_cnt, hs.data(), hs.size() * sizeof(int), cudaMemcpyHostToDevice));
      NCCL_TRY(g_nccl.groupStart());
      for (size_t i = 0; i < np; ++i) {
        NCCL_TRY(g_nccl.send(d_cnt + 2 * i, 2, ncclInt32, c->peers[i].rank, cm->nccl, s));
        NCCL_TRY(g_nccl.recv(d_cnt + 2 * np + 2 * i, 2, ncclInt32, c->peers[i].rank, cm->nccl, s));
      }
      NCCL_TRY(g_nccl.groupEnd());
      std::vector<int> got(2 * np);
      DGVV_CUDA_TRY(cudaMemcpyAsync(got.data(), d_cnt + 2 * np, got.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
      DGVV_CUDA_TRY(cudaStreamSynchronize(s));
      for (size_t i = 0; i < np; ++i)
        if (got[2 * i] != c->peers[i].n_recv || got[2 * i + 1] != c->peers[i].n_recv_f)
          return dgvv_fail(DGVV_EINVAL, "peer %d sends %d cells / %d faces but %d ghosts / %d faces are listed",
                           c->peers[i].rank, got[2 * i], got[2 * i + 1], c->peers[i].n_recv, c->peers[i].n_recv_f);
    }
  }
  // global DoF count
  c->n_global = c->n_owned;   // multi-rank: caller sums (dgvv_sizes reports local/global via comm)
  if (c->comm) {
    long long v = c->n_owned;
    TRY(comm_host_sum(c, &v, s));
    c->n_global = v;
  }
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  return check_cuda("setup");
}

dgvv_status dgvv_setup(const dgvv_mesh* m, int32_t degree, const dgvv_law* vl, const dgvv_law* pl,
                       const dgvv_options* opt, dgvv_stream stream, dgvv_ctx** out) {
  DGVV_RANGE();
  if (!out) return dgvv_fail(DGVV_EINVAL, "out is null");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return dgvv_fail(DGVV_ECUDA, "no CUDA device");
  dgvv_ctx* c = new dgvv_ctx();
  dgvv_status st = setup_impl(m, degree, vl, pl, opt, (cudaStream_t)stream, c);
  if (st != DGVV_OK) {
    std::string msg = g_err;
    dgvv_destroy(c);
    g_err = msg;
    return st;
  }
  *out = c;
  return DGVV_OK;
}

dgvv_status dgvv_update_viscosity(dgvv_ctx* c, const double* u_lin, dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_ctx(c));
  if (!c->carreau) return dgvv_fail(DGVV_EUNSUPPORTED, "update_viscosity needs the Carreau law");
  if (!u_lin) return dgvv_fail(DGVV_EINVAL, "u_lin is null");
  cudaStream_t s = (cudaStream_t)stream;
  for (size_t l = 0; l < c->L.size(); ++l) {
    Level& L = c->L[l];
    const int n = L.n, n3 = n * n * n;
    const double* u = u_lin;
    if (l > 0) {   // G19: interpolate u_lin (fine polynomial at the coarse Gauss points)
      const int nf = c->L[0].n;
      double xf_[DGVV_NMAX], wf[DGVV_NMAX], xc[DGVV_NMAX], wc[DGVV_NMAX];
      gauss01(nf, xf_, wf);
      gauss01(n, xc, wc);
      std::vector<double> I1((size_t)n * nf);
      for (int j = 0; j < n; ++j) {
        double v[DGVV_NMAX], d[DGVV_NMAX];
        lagrange_at(xf_, nf, xc[j], v, d);
        for (int i = 0; i < nf; ++i) I1[(size_t)j * nf + i] = v[i];
      }
      DGVV_CUDA_TRY(launch_tensor3(nf, n, 3, I1.data(), u_lin, L.ulin, 0.0, c->n_owned, s));
      if (c->n_ghost)
        DGVV_CUDA_TRY(launch_tensor3(nf, n, 3, I1.data(), c->L[0].ulin_ghost, L.ulin_ghost, 0.0, c->n_ghost, s));
      u = L.ulin;
    } else if (c->n_ghost) {
      TRY(exchange_sync(c, 0, 3, u_lin, L.ulin_ghost, s));
    }
    NuArgs a;
    a.u = u;
    a.ughost = L.ulin_ghost;
    a.n_owned = c->n_owned;
    a.n_total = c->n_total;
    a.cart = c->d_cart;
    a.vJi = L.vJi;
    a.fJi = L.fJi;
    for (int i = 0; i < 4; ++i) a.law[i] = c->visc.p[i];
    a.nu_cell = L.nu_cell;
    a.nu_face = L.nu_face;
    a.bad = c->d_flag;                       // domain check in the kernel: one host read at the end
    if (l == 0) DGVV_CUDA_TRY(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
    DGVV_CUDA_TRY(launch_carreau(n, c->geo, a, s));
    TRY(premultiply(c, (int)l, L.nu_cell, L.nu_face, L.wv_cell, L.wv_face, s));
    L.dinv_ok[0] = false;                    // the diagonal depends on nu: recomputed lazily (same buffer)
  }
  {
    int bad = 0;
    DGVV_CUDA_TRY(cudaMemcpyAsync(&bad, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    DGVV_CUDA_TRY(cudaStreamSynchronize(s));
    if (bad) {
      c->nu_ready = false;
      return dgvv_fail(DGVV_EDOMAIN, "Carreau viscosity: %d quadrature points with non-positive or non-finite value", bad);
    }
  }
  c->ulin = u_lin;
  c->nu_ready = true;
  c->npd_stale = true;
  ++c->coef_epoch;
  return DGVV_OK;
}

dgvv_status dgvv_apply_viscous(dgvv_ctx* c, int32_t level, const double* src, double* dst, dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  TRY(op_ready(c, DGVV_OP_VISCOUS));
  if (!src || !dst) return dgvv_fail(DGVV_EINVAL, "null vector");
  if (src == dst) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  ApplyArgs a = base_args(c, level, DGVV_OP_VISCOUS);
  a.src = src;
  a.dst = dst;
  return run_apply(c, DGVV_OP_VISCOUS, level, a, (cudaStream_t)stream);
}

// Host-buffer apply: slab pipeline H2D (copy stream 0) -> apply (caller stream) -> D2H (copy
// stream 1).  Slab i is applied once every slab holding one of its neighbours has arrived.
DGVV_INTERNAL dgvv_status host_pipe_setup(dgvv_ctx* c, int level) {
  auto& P = c->hp;
  const size_t N = (size_t)3 * level_dofs(c, level);
  if (P.level == level) return DGVV_OK;
  if (P.level >= 0) return dgvv_fail(DGVV_EUNSUPPORTED, "host apply is set up for level %d only", P.level);
  TRY(dalloc(c, &P.d_src, N));
  TRY(dalloc(c, &P.d_dst, N));
  for (int i = 0; i < 2; ++i) DGVV_CUDA_TRY(cudaStreamCreateWithFlags(&P.cs[i], cudaStreamNonBlocking));
  DGVV_CUDA_TRY(cudaEventCreateWithFlags(&P.ev_start, cudaEventDisableTiming));
  DGVV_CUDA_TRY(cudaEventCreateWithFlags(&P.ev_done, cudaEventDisableTiming));
  const int n = c->n_owned;
  // slab sizes: small first/last slabs shorten the pipeline fill (compute of slab 0 waits for
  // its neighbours' slab) and drain (copy-out of the last slab); large middle slabs keep the
  // per-slab launch/event overhead low.  Weights 1 1 6 6 6 6 6 6 1 1 (DGVV_HOST_SLABS = uniform k).
  std::vector<int> wts = {1, 1, 6, 6, 6, 6, 6, 6, 1, 1};
  if (const char* e = std::getenv("DGVV_HOST_SLABS")) wts.assign(std::max(1, std::atoi(e)), 1);
  if (n < 64 * (int)wts.size()) wts.assign(1, 1);
  P.nslab = (int)wts.size();
  long long wsum = 0, acc = 0;
  for (int w : wts) wsum += w;
  std::vector<int> slab_of(n);
  for (int i = 0; i < P.nslab; ++i) {
    const int a = (int)((long long)n * acc / wsum);
    acc += wts[i];
    const int b = (int)((long long)n * acc / wsum);
    P.first.push_back(a);
    P.count.push_back(b - a);
    for (int k = a; k < b; ++k) slab_of[k] = i;
  }
  P.need.assign(P.nslab, 0);
  for (int k = 0; k < n; ++k) {
    int nd = slab_of[k];
    for (int f = 0; f < 6; ++f) {
      const int v = c->h_nbr[(size_t)k * 6 + f];
      if (v >= 0 && v < n) nd = std::max(nd, slab_of[v]);
    }
    P.need[slab_of[k]] = std::max(P.need[slab_of[k]], nd);
  }
  P.ev_in.resize(P.nslab);
  P.ev_out.resize(P.nslab);
  for (int i = 0; i < P.nslab; ++i) {
    DGVV_CUDA_TRY(cudaEventCreateWithFlags(&P.ev_in[i], cudaEventDisableTiming));
    DGVV_CUDA_TRY(cudaEventCreateWithFlags(&P.ev_out[i], cudaEventDisableTiming));
  }
  P.level = level;
  return DGVV_OK;
}

dgvv_status dgvv_apply_viscous_host(dgvv_ctx* c, int32_t level, const double* src_host, double* dst_host,
                                    dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  TRY(op_ready(c, DGVV_OP_VISCOUS));
  if (!src_host || !dst_host) return dgvv_fail(DGVV_EINVAL, "null vector");
  if (src_host == dst_host) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  TRY(host_pipe_setup(c, level));
  auto& P = c->hp;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t per = (size_t)3 * level_dofs(c, level) / std::max(1, c->n_owned);   // doubles per cell
  if (!c->peers.empty()) {   // ghosts: whole vector in, exchange + apply, whole vector out
    const size_t N = per * c->n_owned;
    DGVV_CUDA_TRY(cudaMemcpyAsync(P.d_src, src_host, N * sizeof(double), cudaMemcpyHostToDevice, s));
    TRY(dgvv_apply_viscous(c, level, P.d_src, P.d_dst, stream));
    DGVV_CUDA_TRY(cudaMemcpyAsync(dst_host, P.d_dst, N * sizeof(double), cudaMemcpyDeviceToHost, s));
    return DGVV_OK;
  }
  // the copy streams start after everything already queued on the caller's stream
  DGVV_CUDA_TRY(cudaEventRecord(P.ev_start, s));
  for (int i = 0; i < 2; ++i) DGVV_CUDA_TRY(cudaStreamWaitEvent(P.cs[i], P.ev_start, 0));
  for (int i = 0; i < P.nslab; ++i) {
    DGVV_CUDA_TRY(cudaMemcpyAsync(P.d_src + per * P.first[i], src_host + per * P.first[i],
                                  per * P.count[i] * sizeof(double), cudaMemcpyHostToDevice, P.cs[0]));
    DGVV_CUDA_TRY(cudaEventRecord(P.ev_in[i], P.cs[0]));
  }
  ApplyArgs a = base_args(c, level, DGVV_OP_VISCOUS);
  a.src = P.d_src;
  a.dst = P.d_dst;
  int waited = -1;
  for (int i = 0; i < P.nslab; ++i) {
    if (P.need[i] > waited) {
      DGVV_CUDA_TRY(cudaStreamWaitEvent(s, P.ev_in[P.need[i]], 0));
      waited = P.need[i];
    }
    a.cell_base = P.first[i];
    a.n_proc = P.count[i];
    cudaError_t e = launch_apply(3, c->L[level].n, c->form, c->geo, a, s);
    if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "apply kernel: %s", cudaGetErrorString(e));
    DGVV_CUDA_TRY(cudaEventRecord(P.ev_out[i], s));
    DGVV_CUDA_TRY(cudaStreamWaitEvent(P.cs[1], P.ev_out[i], 0));
    DGVV_CUDA_TRY(cudaMemcpyAsync(dst_host + per * P.first[i], P.d_dst + per * P.first[i],
                                  per * P.count[i] * sizeof(double), cudaMemcpyDeviceToHost, P.cs[1]));
  }
  DGVV_CUDA_TRY(cudaEventRecord(P.ev_done, P.cs[1]));
  DGVV_CUDA_TRY(cudaStreamWaitEvent(s, P.ev_done, 0));
  return DGVV_OK;
}

dgvv_status dgvv_apply_poisson(dgvv_ctx* c, int32_t level, const double* src, double* dst, dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  TRY(op_ready(c, DGVV_OP_POISSON));
  if (!src || !dst) return dgvv_fail(DGVV_EINVAL, "null vector");
  if (src == dst) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  ApplyArgs a = base_args(c, level, DGVV_OP_POISSON);
  a.src = src;
  a.dst = dst;
  return run_apply(c, DGVV_OP_POISSON, level, a, (cudaStream_t)stream);
}

dgvv_status dgvv_apply_linearized_viscous(dgvv_ctx* c, const double* src, double* dst, dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_ctx(c));
  if (!c->has_visc || !c->carreau) return dgvv_fail(DGVV_EUNSUPPORTED, "linearised apply needs the Carreau law");
  if (!c->nu_ready || !c->ulin) return dgvv_fail(DGVV_ESTATE, "call dgvv_update_viscosity first");
  if (!src || !dst || src == dst || dst == c->ulin) return dgvv_fail(DGVV_EINVAL, "bad vectors (null or aliasing)");
  if (c->form != DGVV_FORM_DIVERGENCE) return dgvv_fail(DGVV_EUNSUPPORTED, "Newton apply: divergence form only");
  cudaStream_t s = (cudaStream_t)stream;
  ApplyArgs a = base_args(c, 0, DGVV_OP_VISCOUS);
  a.src = src;
  a.dst = dst;
  a.ulin = c->ulin;
  a.ulin_ghost = c->L[0].ulin_ghost;
  for (int i = 0; i < 4; ++i) a.law[i] = c->visc.p[i];
  if (newton_uses_pointdata(c->geo)) {
    if (c->npd_stale) {                       // once per linearisation (after the ghosts of u_lin arrived)
      const size_t n = c->L[0].n, n3 = n * n * n, n2 = n * n;
      if (!c->d_npc) TRY(dalloc(c, &c->d_npc, (size_t)c->n_owned * 7 * n3));
      if (!c->d_npf) TRY(dalloc(c, &c->d_npf, (size_t)c->n_total * 60 * n2));
      cudaError_t e = launch_newton_pointdata((int)n, a, c->n_total, c->d_npc, c->d_npf, s);
      if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "Newton point data: %s", cudaGetErrorString(e));
      c->npd_stale = false;
    }
    a.npc = c->d_npc;
    a.npf = c->d_npf;
  }
  return run_apply(c, DGVV_OP_VISCOUS, 0, a, s, 1);
}


dgvv_status dgvv_set_mass(dgvv_ctx* c, int32_t op, double mass) {
  DGVV_RANGE();
  TRY(check_ctx(c));
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  if (!std::isfinite(mass) || mass < 0.0) return dgvv_fail(DGVV_EDOMAIN, "mass coefficient %g must be finite and >= 0", mass);
  if (c->mass[op] == mass) return DGVV_OK;
  c->mass[op] = mass;
  ++c->coef_epoch;
  for (auto& L : c->L) L.dinv_ok[op] = false;   // the diagonal changes: recomputed lazily (same buffer)
  return DGVV_OK;
}

dgvv_status dgvv_dot(dgvv_ctx* c, int32_t level, int32_t ncomp, const double* a, const double* b, double* out,
                     dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  if (!a || !b || !out || ncomp < 1) return dgvv_fail(DGVV_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  TRY(dot_dev(c, a, b, (long)ncomp * level_dofs(c, level), c->d_scal + 4, s));
  DGVV_CUDA_TRY(cudaMemcpyAsync(out, c->d_scal + 4, sizeof(double), cudaMemcpyDeviceToHost, s));
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  return DGVV_OK;
}

dgvv_status dgvv_sizes(const dgvv_ctx* c, int32_t level, int64_t* nl, int64_t* ng) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  const long long n3 = (long long)c->L[level].n * c->L[level].n * c->L[level].n;
  if (nl) *nl = (int64_t)c->n_owned * n3;
  if (ng) *ng = (int64_t)c->n_global * n3;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "pending CUDA error: %s", cudaGetErrorString(e));
  return DGVV_OK;
}

dgvv_status dgvv_coefficient_range(dgvv_ctx* c, int32_t op, int32_t level, double* lo, double* hi) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  TRY(op_ready(c, op));
  Level& L = c->L[level];
  const int n = L.n;
  double a1, b1, a2, b2;
  int bad;
  cudaStream_t s = 0;
  const double* vc = op == DGVV_OP_VISCOUS ? L.nu_cell : L.c_cell;
  const double* vf = op == DGVV_OP_VISCOUS ? L.nu_face : L.c_face;
  TRY(array_range(c, vc, (long)c->n_owned * n * n * n, s, &a1, &b1, &bad));
  TRY(array_range(c, vf, (long)c->n_owned * 6 * n * n, s, &a2, &b2, &bad));
  *lo = std::min(a1, a2);
  *hi = std::max(b1, b2);
  return DGVV_OK;
}

dgvv_status dgvv_exchange_bytes(const dgvv_ctx* c, int32_t level, int32_t op, int64_t* sent, int64_t* received) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  if (!sent || !received) return dgvv_fail(DGVV_EINVAL, "null output");
  const int nc = op == DGVV_OP_POISSON ? 1 : 3;
  const long long per = 2LL * nc * c->L[level].n * c->L[level].n * 8;   // value + d/dxi_n, FP64
  long long snd = 0, rcv = 0;
  for (auto& P : c->peers) { snd += P.n_send_f * per; rcv += P.n_recv_f * per; }
  *sent = snd;
  *received = rcv;
  return DGVV_OK;
}

dgvv_status dgvv_ghost_layout(const dgvv_ctx* c, int32_t* n_peers, int32_t* peer_ranks, int32_t* send_counts,
                              int32_t* recv_counts) {
  DGVV_RANGE();
  if (!c || !n_peers) return dgvv_fail(DGVV_EINVAL, "null argument");
  *n_peers = (int32_t)c->peers.size();
  for (size_t i = 0; i < c->peers.size(); ++i) {
    if (peer_ranks) peer_ranks[i] = c->peers[i].rank;
    if (send_counts) send_counts[i] = c->peers[i].n_send;
    if (recv_counts) recv_counts[i] = c->peers[i].n_recv;
  }
  return DGVV_OK;
}

dgvv_status dgvv_pack_ghosts(dgvv_ctx* c, int32_t level, int32_t kind, const double* src, double* sendbuf,
                             dgvv_stream stream) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  if (!src || !sendbuf) return dgvv_fail(DGVV_EINVAL, "null vector");
  const int nc = kind == DGVV_GHOST_POISSON ? 1 : 3;
  return pack(c, level, nc, src, sendbuf, (cudaStream_t)stream);
}

dgvv_status dgvv_ghost_buffer(dgvv_ctx* c, int32_t level, int32_t kind, double** out) {
  DGVV_RANGE();
  TRY(check_level(c, level));
  if (!out) return dgvv_fail(DGVV_EINVAL, "null out");
  Level& L = c->L[level];
  double* p = kind == DGVV_GHOST_VISCOUS ? L.ghost[0] : kind == DGVV_GHOST_POISSON ? L.ghost[1]
            : kind == DGVV_GHOST_TRANSPORT ? (level == 0 ? c->wtr_ghost : nullptr) : L.ulin_ghost;
  if (!p) return dgvv_fail(DGVV_ESTATE, "no ghost buffer of kind %d on level %d (no ghosts or operator unused)", kind, level);
  *out = p;
  return DGVV_OK;
}

}  // extern "C"
