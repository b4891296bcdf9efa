// api.cu — the C ABI (include/dgvv.h): context, setup, operator
// applies, smoother, transfer, V-cycle, Lanczos, dot, NCCL plumbing.  Host orchestration
// only: every arithmetic step of the path runs in the kernels of k_*.cu.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dgvv.h"
#include "launch.h"

using namespace dgvv;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static dgvv_status dgvv_fail(dgvv_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define TRY(expr)                         \
  do {                                    \
    dgvv_status st_ = (expr);             \
    if (st_ != DGVV_OK) return st_;       \
  } while (0)

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

dgvv_status nccl_load() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.ok) return DGVV_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return dgvv_fail(DGVV_ENCCL, "cannot load libnccl.so.2: %s", dlerror());
#define LD(field, name)                                                          \
  g_nccl.field = (decltype(g_nccl.field))dlsym(h, name);                         \
  if (!g_nccl.field) return dgvv_fail(DGVV_ENCCL, "libnccl: missing %s", name);
  LD(getUniqueId, "ncclGetUniqueId");
  LD(commInitRank, "ncclCommInitRank");
  LD(commDestroy, "ncclCommDestroy");
  LD(groupStart, "ncclGroupStart");
  LD(groupEnd, "ncclGroupEnd");
  LD(send, "ncclSend");
  LD(recv, "ncclRecv");
  LD(allReduce, "ncclAllReduce");
  LD(errStr, "ncclGetErrorString");
#undef LD
  g_nccl.ok = true;
  return DGVV_OK;
}

#define NCCL_TRY(expr)                                                                     \
  do {                                                                                     \
    ncclResult_t r_ = (expr);                                                              \
    if (r_ != ncclSuccess) return dgvv_fail(DGVV_ENCCL, "%s: %s", #expr, g_nccl.errStr(r_)); \
  } while (0)

// ------------------------------------------------------------------ communicators
// A dgvv communicator (the void* of dgvv_options.nccl_comm) is either an NCCL communicator (one
// process per GPU, the production transport) or one rank of an in-process thread group: R host
// threads, each driving its own context and CUDA stream, exchanging through device-to-device copies
// ordered by CUDA events (no kernel ever waits on another rank's kernel: the dependencies are
// stream/event edges recorded before a host barrier).  The thread group runs the whole multi-rank
// library path — grouped ghost exchange overlapped with the interior cells, allreduced dots,
// multi-rank V-cycles and Krylov solvers — on one GPU, so it can be tested where NCCL cannot run
// (NCCL refuses two ranks on one device).
enum { COMM_NCCL = 1, COMM_THREADS = 2 };
struct ThreadGroup;
struct DgvvComm {
  int kind = 0;
  ncclComm_t nccl = nullptr;
  ThreadGroup* tg = nullptr;
  int rank = 0;
};
struct ThreadGroup {
  int R = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long gen = 0;
  std::vector<std::vector<const void*>> sptr;   // [from][to] send segment
  std::vector<std::vector<size_t>> sbytes;
  std::vector<cudaEvent_t> ev_a, ev_b;          // per rank events of the current collective
  std::vector<const double*> red;               // per rank allreduce staging
  std::vector<long long> hval;                  // per rank host values
  std::vector<DgvvComm> comms;
};
void tg_barrier(ThreadGroup* g) {
  std::unique_lock<std::mutex> lk(g->mu);
  const unsigned long my = g->gen;
  if (++g->arrived == g->R) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->gen != my; });
  }
}

// ------------------------------------------------------------------ tables
// each TU's __constant__ tables live per device: uploaded once per DEVICE, not once
// per process — a context created later on another device would otherwise read zero tables
std::mutex g_tab_mu;
uint64_t g_tab_done = 0;     // bit d: tables uploaded to device d

dgvv_status upload_tables() {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  const uint64_t bit = current_device_bit();
  if (g_tab_done & bit) return DGVV_OK;
  std::vector<Tab1D> tabs(DGVV_NMAX + 1);
  std::memset(tabs.data(), 0, sizeof(Tab1D) * tabs.size());
  for (int n = 1; n <= DGVV_NMAX; ++n) make_tab(n, &tabs[n]);
  DGVV_CUDA_TRY(upload_tables_visc(tabs.data()));
  DGVV_CUDA_TRY(upload_tables_pois(tabs.data()));
  DGVV_CUDA_TRY(upload_tables_aux(tabs.data()));
  DGVV_CUDA_TRY(upload_tables_newton(tabs.data()));
  DGVV_CUDA_TRY(upload_tables_pen(tabs.data()));
  g_tab_done |= bit;
  return DGVV_OK;
}
}  // namespace

// ------------------------------------------------------------------ context
struct Level {
  int k = 0, n = 0;
  double* vJi = nullptr;      // general geometry: J^-1 at cell points [n_total][9][n^3]
  double* fJi = nullptr;      //                   J^-1 at own face points [n_total][6][9][n^2]
  double* jxw = nullptr;      //                   JxW [n_total][n^3]
  double* fdA = nullptr;      //                   dA  [n_total][6][n^2]
  double* Hc = nullptr;
  double* nu_cell = nullptr;  // viscous coefficient at points (raw nu)
  double* nu_face = nullptr;
  double* wv_cell = nullptr;  // general geometry: nu*JxW, nu*dA
  double* wv_face = nullptr;
  double* c_cell = nullptr;   // Poisson coefficient (raw c)
  double* c_face = nullptr;
  double* wc_cell = nullptr;  // general geometry: c*JxW, c*dA
  double* wc_face = nullptr;
  double* dinv[2] = {nullptr, nullptr};
  bool dinv_ok[2] = {false, false};          // buffer kept across coefficient changes; recomputed when false
  double* ulin = nullptr;     // u_lin interpolated to this level (levels >= 1), owned
  double* ghost[2] = {nullptr, nullptr};   // ghost src buffers (NC = 3 / 1)
  double* ulin_ghost = nullptr;
  std::vector<double*> scratch[2];         // V-cycle scratch per op
  // f2 penalty-step operator on this level (same per-cell tau on every level): inverse diagonal
  // and V-cycle scratch [0] r, [1] Chebyshev work (r | d), [3] b, [4] x (levels >= 1)
  double* dinv_pen = nullptr;
  bool dinv_pen_ok = false;
  std::vector<double*> scratch_pen;
};

// FP32 mirror of a level for the single-precision multigrid preconditioner (PAPER.md:1546-1551,
// SURVEY §8(f) f1): coefficient/geometry arrays converted from the FP64 level, per-op epochs.
struct LevelF {
  float* nu_cell[2] = {nullptr, nullptr};   // per op: raw (Cartesian) or premultiplied (general)
  float* nu_face[2] = {nullptr, nullptr};
  float* dinv[2] = {nullptr, nullptr};
  int epoch[2] = {-1, -1};
  float* vJi = nullptr;
  float* fJi = nullptr;
  float* Hc = nullptr;
  float* jxw = nullptr;
  float* ghost[2] = {nullptr, nullptr};     // FP32 ghost cells per op (multi-rank)
  std::vector<float*> scratch[2];           // [0] r, [1] work (2N), [3] b, [4] x
};

struct Peer {
  int rank;
  int* d_send = nullptr;      // owned local cells to send (sorted by global id)
  int n_send = 0;
  int recv_off = 0, n_recv = 0;   // ghost index range received from this peer
};

struct dgvv_ctx {
  int device = 0;               // CUDA device the context was set up on (every call must run there)
  int n_owned = 0, n_ghost = 0, n_total = 0;
  long long first = 0, n_global = 0;
  int geo = 0;                  // 0 Cartesian fast path, 1 general iso-parametric
  int map_degree = 1;
  int* d_nbr = nullptr;
  double* d_nodes = nullptr;
  double* d_cart = nullptr;
  std::vector<Level> L;
  dgvv_law visc{}, pois{};
  bool has_visc = false, has_pois = false, carreau = false, nu_ready = false;
  int form = 0;
  double ip = 1.0;
  double mass[2] = {0.0, 0.0};  // Helmholtz mass coefficient per op (dgvv_set_mass)
  double* cg_work[3] = {nullptr, nullptr, nullptr};   // CG vectors r, z, p, q per op (level 0)
  // f2 penalty-step operator: per-cell parameters (owned then ghosts, internal order)
  double* d_tau_div = nullptr;
  double* d_tau_cont = nullptr;
  bool has_pen = false;
  // f4 convective term: transport field w (level 0, owned + ghosts), GMRES work
  double* d_wtr = nullptr;
  double* wtr_ghost = nullptr;
  bool has_wtr = false;
  double* d_npc = nullptr;                   // Newton point data of the linearisation point (lazy)
  double* d_npf = nullptr;
  bool npd_stale = true;
  double* d_wref = nullptr;                  // convective point data for the fused apply (lazy)
  double* d_wface = nullptr;
  bool wq_stale = true;
  double* gm_work = nullptr;                 // r, w, V[0..m], Z[0..m-1]
  int gm_restart = 0;
  double* gm_H = nullptr;                    // device Hessenberg column
  double* lz_buf = nullptr;                  // Lanczos work vectors (dgvv_estimate_lambda_max)
  size_t lz_len = 0;
  // f3: h-levels (a coarser context below the coarsest p-level) and the direct coarse solver
  dgvv_ctx* coarse = nullptr;
  int* d_parent = nullptr;                   // [n_owned] coarse cell of each fine cell
  signed char* d_octant = nullptr;           // [n_owned] ox + 2 oy + 4 oz
  int* d_child = nullptr;                    // [coarse n_owned][8]
  double* hb[2] = {nullptr, nullptr};        // coarse-level right-hand side / solution per op
  double* hx[2] = {nullptr, nullptr};
  double* Ainv[2] = {nullptr, nullptr};      // dense inverse of the coarsest level per op
  int direct_n[2] = {0, 0};
  int direct_epoch[2] = {-1, -1};            // coef_epoch the inverse was built at
  float* hbf[2] = {nullptr, nullptr};        // FP32 V-cycle: coarse-level b / x per op
  float* hxf[2] = {nullptr, nullptr};
  std::vector<int> h_parent;                 // host copies of the h-maps (c-level transfers)
  std::vector<signed char> h_octant;
  // f3 c-level: continuous Q1 level on this context's degree-1 mesh (readings C1-C3)
  struct CGLevel {
    bool on = false;
    int nv = 0, ncolors = 0;
    int *d_vid = nullptr, *d_inc_ptr = nullptr, *d_inc = nullptr, *d_color = nullptr;
    std::vector<int> h_vid;                  // [n_owned][8]
    double* dinv[2] = {nullptr, nullptr};
    int dinv_epoch[2] = {-1, -1};
    double *xdg[2] = {nullptr, nullptr}, *ydg[2] = {nullptr, nullptr};        // DG_1 temps
    double *r[2] = {nullptr, nullptr}, *d[2] = {nullptr, nullptr};            // CG temps
    double *b0[2] = {nullptr, nullptr}, *x0[2] = {nullptr, nullptr};          // c-level b / x
    double *hb[2] = {nullptr, nullptr}, *hx[2] = {nullptr, nullptr};          // next CG level b / x
    int *pp = nullptr, *pc = nullptr, *rp = nullptr, *rc = nullptr;           // CSR P (fine rows), R = P^T
    double *pv = nullptr, *rv = nullptr;
    dgvv_ctx* transfer_to = nullptr;         // coarse context the CSR transfers were built for
    double* Ainv[2] = {nullptr, nullptr};
    int direct_n[2] = {0, 0};
    int direct_epoch[2] = {-1, -1};
  } cg;
  std::vector<int> h_gperm;                  // internal ghost i -> mesh ghost row
  std::vector<LevelF> LF;                    // FP32 levels (lazily built)
  float* d_cart_f = nullptr;
  int coef_epoch = 0;                        // bumped whenever coefficients or the mass change
  const double* ulin = nullptr;
  // comm: peers exist whenever there are ghosts; NCCL transport only with a communicator
  // (without one the caller fills the ghost buffers: external-exchange mode, used by tests)
  void* comm = nullptr;                      // DgvvComm*
  std::vector<Peer> peers;
  double* tg_red = nullptr;                  // thread group: allreduce staging (8 doubles)
  cudaEvent_t ev_red = nullptr, ev_red2 = nullptr;
  double* d_sendbuf = nullptr;
  size_t sendbuf_len = 0;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_comm = nullptr;
  int* d_interior = nullptr;      // owned cells without a ghost neighbour
  int* d_boundary = nullptr;      // owned cells with a ghost neighbour
  int n_interior = 0, n_boundary = 0;
  // scratch
  double* d_part = nullptr;     // 1024 partials
  double* d_scal = nullptr;     // 16 scalars
  int* d_flag = nullptr;
  std::vector<void*> allocs;
  // host-buffer pipelined apply (dgvv_apply_viscous_host)
  std::vector<int> h_nbr;           // local neighbour table [n_total][6] (host copy)
  struct HostPipe {
    int level = -1, nslab = 0;
    double* d_src = nullptr;
    double* d_dst = nullptr;
    std::vector<int> first, count, need;
    cudaStream_t cs[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev_in, ev_out;
    cudaEvent_t ev_start = nullptr, ev_done = nullptr;
  } hp;
};

namespace {

const int kPartials = 1024;

template <typename T>
dgvv_status dalloc(dgvv_ctx* c, T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) return dgvv_fail(DGVV_ENOMEM, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
  c->allocs.push_back((void*)*p);
  return DGVV_OK;
}

dgvv_status check_cuda(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return DGVV_OK;
}

inline long level_dofs(const dgvv_ctx* c, int l) {
  const int n = c->L[l].n;
  return (long)c->n_owned * n * n * n;
}

// null context, or a call made while another device is current (device memory and
// the per-device tables / kernel attributes of the context belong to its setup device)
dgvv_status check_ctx(const dgvv_ctx* c) {
  if (!c) return dgvv_fail(DGVV_EINVAL, "null context");
  int d = -1;
  cudaGetDevice(&d);
  if (d != c->device)
    return dgvv_fail(DGVV_ESTATE, "context was set up on device %d but device %d is current", c->device, d);
  return DGVV_OK;
}

dgvv_status check_level(const dgvv_ctx* c, int level) {
  TRY(check_ctx(c));
  if (level < 0 || level >= (int)c->L.size()) return dgvv_fail(DGVV_EINVAL, "level %d out of range", level);
  return DGVV_OK;
}

// min/max/bad over an array (synchronous)
dgvv_status array_range(dgvv_ctx* c, const double* v, long n, cudaStream_t s, double* lo, double* hi,
                        int* nbad) {
  const int nb = 256;
  DGVV_CUDA_TRY(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
  DGVV_CUDA_TRY(launch_range(v, n, c->d_part, c->d_part + nb, c->d_flag, nb, s));
  std::vector<double> h(2 * nb);
  DGVV_CUDA_TRY(cudaMemcpyAsync(h.data(), c->d_part, 2 * nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  int bad = 0;
  DGVV_CUDA_TRY(cudaMemcpyAsync(&bad, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  double a = INFINITY, b = -INFINITY;
  for (int i = 0; i < nb; ++i) { a = std::min(a, h[i]); b = std::max(b, h[nb + i]); }
  *lo = a; *hi = b; *nbad = bad;
  return DGVV_OK;
}

// pack the owned cells every peer needs into the send buffer (peer-rank order)
dgvv_status pack(dgvv_ctx* c, int l, int nc, const double* src, double* sendbuf, cudaStream_t s) {
  const int n = c->L[l].n;
  const int len = nc * n * n * n;
  size_t off = 0;
  for (auto& P : c->peers) {
    DGVV_CUDA_TRY(launch_gather_cells(src, P.d_send, P.n_send, len, sendbuf + off, s));
    off += (size_t)P.n_send * len;
  }
  return DGVV_OK;
}

// ghost exchange of a level vector (NC components): pack on s, grouped ncclSend/ncclRecv on
// the comm stream into `ghost`; ev_comm marks completion (the caller's stream must wait on it
// before reading ghosts).  No-op without ghosts or without a communicator.
// grouped point-to-point exchange of packed cells (len elements of esz bytes per cell) with every
// peer, on the comm stream after ev_pack; ev_comm marks completion
dgvv_status comm_sendrecv(dgvv_ctx* c, const void* sendbuf, void* ghost, int len, size_t esz, cudaStream_t s) {
  DgvvComm* cm = (DgvvComm*)c->comm;
  DGVV_CUDA_TRY(cudaEventRecord(c->ev_pack, s));
  if (cm->kind == COMM_NCCL) {
    DGVV_CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_pack, 0));
    const ncclDataType_t dt = esz == 8 ? ncclDouble : ncclFloat;
    NCCL_TRY(g_nccl.groupStart());
    size_t off = 0;
    for (auto& P : c->peers) {
      if (P.n_send) NCCL_TRY(g_nccl.send((const char*)sendbuf + off * esz, (size_t)P.n_send * len, dt, P.rank, cm->nccl, c->comm_stream));
      if (P.n_recv) NCCL_TRY(g_nccl.recv((char*)ghost + (size_t)P.recv_off * len * esz, (size_t)P.n_recv * len, dt, P.rank, cm->nccl, c->comm_stream));
      off += (size_t)P.n_send * len;
    }
    NCCL_TRY(g_nccl.groupEnd());
    DGVV_CUDA_TRY(cudaEventRecord(c->ev_comm, c->comm_stream));
    return DGVV_OK;
  }
  ThreadGroup* g = cm->tg;
  const int r = cm->rank;
  {
    std::lock_guard<std::mutex> lk(g->mu);
    size_t off = 0;
    for (int q = 0; q < g->R; ++q) { g->sptr[r][q] = nullptr; g->sbytes[r][q] = 0; }
    for (auto& P : c->peers) {
      g->sptr[r][P.rank] = (const char*)sendbuf + off * esz;
      g->sbytes[r][P.rank] = (size_t)P.n_send * len * esz;
      off += (size_t)P.n_send * len;
    }
    g->ev_a[r] = c->ev_pack;
  }
  tg_barrier(g);
  // our ghost buffer is rewritten only after our own earlier kernels that read it (ordered before
  // ev_pack on s), and after each peer has packed
  DGVV_CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_pack, 0));
  for (auto& P : c->peers) {
    const size_t want = (size_t)P.n_recv * len * esz;
    if (g->sbytes[P.rank][r] != want)
      return dgvv_fail(DGVV_EINVAL, "thread group: rank %d sends %zu bytes, rank %d expects %zu", P.rank, g->sbytes[P.rank][r], r, want);
    if (!want) continue;
    DGVV_CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, g->ev_a[P.rank], 0));
    DGVV_CUDA_TRY(cudaMemcpyAsync((char*)ghost + (size_t)P.recv_off * len * esz, g->sptr[P.rank][r], want,
                                  cudaMemcpyDeviceToDevice, c->comm_stream));
  }
  DGVV_CUDA_TRY(cudaEventRecord(c->ev_comm, c->comm_stream));
  {
    std::lock_guard<std::mutex> lk(g->mu);
    g->ev_b[r] = c->ev_comm;
  }
  tg_barrier(g);
  // the peers copy from our send buffer: later work on s (the next pack) waits for their copies
  for (auto& P : c->peers) DGVV_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_b[P.rank], 0));
  tg_barrier(g);                               // ev_b is not re-recorded before every rank has waited
  return DGVV_OK;
}

// sum-allreduce of `count` doubles in place (device pointer, stream-ordered on s)
dgvv_status comm_allreduce(dgvv_ctx* c, double* ptr, int count, cudaStream_t s) {
  DgvvComm* cm = (DgvvComm*)c->comm;
  if (!cm) return DGVV_OK;
  if (cm->kind == COMM_NCCL) {
    NCCL_TRY(g_nccl.allReduce(ptr, ptr, count, ncclDouble, ncclSum, cm->nccl, s));
    return DGVV_OK;
  }
  ThreadGroup* g = cm->tg;
  const int r = cm->rank;
  if (count > 8) return dgvv_fail(DGVV_EINVAL, "thread group allreduce: count %d > 8", count);
  DGVV_CUDA_TRY(cudaMemcpyAsync(c->tg_red, ptr, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
  DGVV_CUDA_TRY(cudaEventRecord(c->ev_red, s));
  {
    std::lock_guard<std::mutex> lk(g->mu);
    g->red[r] = c->tg_red;
    g->ev_a[r] = c->ev_red;
  }
  tg_barrier(g);
  for (int q = 0; q < g->R; ++q) DGVV_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_a[q], 0));
  DGVV_CUDA_TRY(launch_sum_ranks(g->red.data(), g->R, count, ptr, s));   // ranks summed in rank order
  DGVV_CUDA_TRY(cudaEventRecord(c->ev_red2, s));
  {
    std::lock_guard<std::mutex> lk(g->mu);
    g->ev_b[r] = c->ev_red2;
  }
  tg_barrier(g);
  for (int q = 0; q < g->R; ++q) DGVV_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_b[q], 0));   // staging reusable
  tg_barrier(g);
  return DGVV_OK;
}

// host-side sum over the ranks (setup: global sizes)
dgvv_status comm_host_sum(dgvv_ctx* c, long long* v, cudaStream_t s) {
  DgvvComm* cm = (DgvvComm*)c->comm;
  if (!cm) return DGVV_OK;
  if (cm->kind == COMM_NCCL) {
    long long* d = nullptr;
    TRY(dalloc(c, &d, 1));
    DGVV_CUDA_TRY(cudaMemcpy(d, v, sizeof(long long), cudaMemcpyHostToDevice));
    NCCL_TRY(g_nccl.allReduce(d, d, 1, ncclInt64, ncclSum, cm->nccl, s));
    DGVV_CUDA_TRY(cudaMemcpyAsync(v, d, sizeof(long long), cudaMemcpyDeviceToHost, s));
    DGVV_CUDA_TRY(cudaStreamSynchronize(s));
    return DGVV_OK;
  }
  ThreadGroup* g = cm->tg;
  {
    std::lock_guard<std::mutex> lk(g->mu);
    g->hval[cm->rank] = *v;
  }
  tg_barrier(g);
  long long t = 0;
  for (int q = 0; q < g->R; ++q) t += g->hval[q];
  tg_barrier(g);
  *v = t;
  return DGVV_OK;
}

dgvv_status exchange(dgvv_ctx* c, int l, int nc, const double* src, double* ghost, cudaStream_t s) {
  if (!c->comm || c->peers.empty()) return DGVV_OK;
  const int n = c->L[l].n;
  const int len = nc * n * n * n;
  TRY(pack(c, l, nc, src, c->d_sendbuf, s));
  return comm_sendrecv(c, c->d_sendbuf, ghost, len, sizeof(double), s);
}

dgvv_status exchange_sync(dgvv_ctx* c, int l, int nc, const double* src, double* ghost, cudaStream_t s) {
  TRY(exchange(c, l, nc, src, ghost, s));
  if (c->comm && !c->peers.empty()) DGVV_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_comm, 0));
  return DGVV_OK;
}

ApplyArgs base_args(dgvv_ctx* c, int l, int op) {
  ApplyArgs a;
  std::memset(&a, 0, sizeof(a));
  Level& L = c->L[l];
  a.nbr = c->d_nbr;
  a.cell_list = nullptr;
  a.n_proc = c->n_owned;
  a.n_owned = c->n_owned;
  if (c->geo == 0) {
    a.nu_cell = op == DGVV_OP_VISCOUS ? L.nu_cell : L.c_cell;
    a.nu_face = op == DGVV_OP_VISCOUS ? L.nu_face : L.c_face;
  } else {
    a.nu_cell = op == DGVV_OP_VISCOUS ? L.wv_cell : L.wc_cell;
    a.nu_face = op == DGVV_OP_VISCOUS ? L.wv_face : L.wc_face;
  }
  a.cart = c->d_cart;
  a.vJi = L.vJi;
  a.fJi = L.fJi;
  a.jxw = L.jxw;
  a.fdA = L.fdA;
  a.Hcell = L.Hc;
  a.pen = c->ip * (double)(L.k + 1) * (double)(L.k + 1);
  a.mass = (op == DGVV_OP_VISCOUS || op == DGVV_OP_POISSON) ? c->mass[op] : 0.0;
  a.ghost = L.ghost[op == DGVV_OP_VISCOUS ? 0 : 1];
  a.mode = MODE_APPLY;
  return a;
}

dgvv_status op_ready(dgvv_ctx* c, int op) {
  TRY(check_ctx(c));
  if (op == DGVV_OP_VISCOUS) {
    if (!c->has_visc) return dgvv_fail(DGVV_ESTATE, "no viscosity law given at setup");
    if (c->carreau && !c->nu_ready) return dgvv_fail(DGVV_ESTATE, "Carreau law: call dgvv_update_viscosity first");
  } else if (op == DGVV_OP_POISSON) {
    if (!c->has_pois) return dgvv_fail(DGVV_ESTATE, "no Poisson coefficient law given at setup");
  } else if (op == DGVV_OP_PENALTY) {
    if (!c->has_pen) return dgvv_fail(DGVV_ESTATE, "penalty operator: call dgvv_set_penalty_parameters first");
  } else {
    return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  }
  return DGVV_OK;
}

// launch one apply in a given mode.  Multi-GPU: interior cells run while NCCL moves the
// ghost cells on the comm stream; cells with a ghost neighbour run after the exchange event.
// kind: 0 plain operator, 1 Newton-linearised (K2), 2 viscous + fused convective term (f4)
dgvv_status run_apply(dgvv_ctx* c, int op, int l, ApplyArgs a, cudaStream_t s, int kind = 0) {
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  const int form = op == DGVV_OP_VISCOUS ? c->form : DGVV_FORM_LAPLACE;
  auto launch = [&](const ApplyArgs& x) -> dgvv_status {
    cudaError_t e = kind == 1 ? launch_newton(c->L[l].n, c->geo, x, s)
                  : kind == 2 ? launch_apply_oseen(c->L[l].n, c->geo, x, s)
                              : launch_apply(nc, c->L[l].n, form, c->geo, x, s);
    if (e == cudaErrorNotSupported) return dgvv_fail(DGVV_EUNSUPPORTED, "kernel not built for degree %d", c->L[l].k);
    if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "apply kernel: %s", cudaGetErrorString(e));
    return DGVV_OK;
  };
  if (!c->comm || c->peers.empty()) return launch(a);
  TRY(exchange(c, l, nc, a.src, const_cast<double*>(a.ghost), s));
  ApplyArgs ai = a;
  ai.cell_list = c->d_interior;
  ai.n_proc = c->n_interior;
  TRY(launch(ai));
  DGVV_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_comm, 0));
  ApplyArgs ab = a;
  ab.cell_list = c->d_boundary;
  ab.n_proc = c->n_boundary;
  return launch(ab);
}

dgvv_status ensure_dinv(dgvv_ctx* c, int op, int l, cudaStream_t s) {
  Level& L = c->L[l];
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  if (L.dinv[oi] && L.dinv_ok[oi]) return DGVV_OK;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  if (!L.dinv[oi]) TRY(dalloc(c, &L.dinv[oi], (size_t)nc * level_dofs(c, l)));
  DiagArgs d;
  d.nbr = c->d_nbr;
  d.n_owned = c->n_owned;
  if (c->geo == 0) {
    d.nu_cell = oi == 0 ? L.nu_cell : L.c_cell;
    d.nu_face = oi == 0 ? L.nu_face : L.c_face;
  } else {
    d.nu_cell = oi == 0 ? L.wv_cell : L.wc_cell;
    d.nu_face = oi == 0 ? L.wv_face : L.wc_face;
  }
  d.cart = c->d_cart;
  d.vJi = L.vJi;
  d.fJi = L.fJi;
  d.Hcell = L.Hc;
  d.pen = c->ip * (double)(L.k + 1) * (double)(L.k + 1);
  d.mass = c->mass[oi];
  d.jxw = L.jxw;
  d.out = L.dinv[oi];
  const int form = op == DGVV_OP_VISCOUS ? c->form : DGVV_FORM_LAPLACE;
  cudaError_t e = launch_diag(nc, L.n, form, c->geo, d, s);
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "diag kernel: %s", cudaGetErrorString(e));
  L.dinv_ok[oi] = true;
  return DGVV_OK;
}

dgvv_status dot_dev(dgvv_ctx* c, const double* a, const double* b, long n, double* dout, cudaStream_t s) {
  const int nb = (int)std::max(1L, std::min((long)kPartials, (n + 255) / 256));
  DGVV_CUDA_TRY(launch_dot(a, b, n, c->d_part, nb, dout, s));
  if (c->comm) TRY(comm_allreduce(c, dout, 1, s));
  return DGVV_OK;
}

// analytic coefficient at all points of a level
dgvv_status eval_analytic(dgvv_ctx* c, const dgvv_law* law, int l, double* xq, double* xf, double* cell_out,
                          double* face_out, cudaStream_t s) {
  const int n = c->L[l].n;
  double p[2] = {law->p[0], law->p[1]};
  DGVV_CUDA_TRY(launch_law_points(law->kind, p, xq, (long)c->n_owned * n * n * n, cell_out, s));
  DGVV_CUDA_TRY(launch_law_points(law->kind, p, xf, (long)c->n_total * 6 * n * n, face_out, s));
  return DGVV_OK;
}

// general geometry: w_cell = nu * JxW, w_face = nu * dA (the apply and diagonal kernels read
// these; the normal and dA are otherwise recomputed from J^-1)
dgvv_status premultiply(dgvv_ctx* c, int l, const double* nc, const double* nf, double* wc, double* wf,
                        cudaStream_t s) {
  if (c->geo != 1) return DGVV_OK;
  Level& L = c->L[l];
  const long n3 = (long)L.n * L.n * L.n, n2 = (long)L.n * L.n;
  DGVV_CUDA_TRY(launch_ew_mul(nc, L.jxw, wc, (long)c->n_owned * n3, s));
  DGVV_CUDA_TRY(launch_ew_mul(nf, L.fdA, wf, (long)c->n_total * 6 * n2, s));
  return DGVV_OK;
}

dgvv_status check_positive(dgvv_ctx* c, const double* v, long n, cudaStream_t s, const char* what) {
  double lo, hi;
  int bad;
  TRY(array_range(c, v, n, s, &lo, &hi, &bad));
  if (bad) return dgvv_fail(DGVV_EDOMAIN, "%s: %d quadrature points with non-positive or non-finite value (min %g)", what, bad, lo);
  return DGVV_OK;
}

double tridiag_max_eig(const std::vector<double>& al, const std::vector<double>& be) {
  // bisection with Sturm sequence counts on the symmetric tridiagonal matrix
  const int k = (int)al.size();
  double lo = INFINITY, hi = -INFINITY;
  for (int i = 0; i < k; ++i) {
    double r = (i > 0 ? std::fabs(be[i - 1]) : 0.0) + (i + 1 < k ? std::fabs(be[i]) : 0.0);
    lo = std::min(lo, al[i] - r);
    hi = std::max(hi, al[i] + r);
  }
  auto count_below = [&](double x) {
    int cnt = 0;
    double d = 1.0;
    for (int i = 0; i < k; ++i) {
      const double b2 = i > 0 ? be[i - 1] * be[i - 1] : 0.0;
      d = al[i] - x - (i > 0 ? b2 / d : 0.0);
      if (d == 0.0) d = -1e-300;
      if (d < 0.0) ++cnt;
    }
    return cnt;
  };
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (count_below(mid) >= k) hi = mid;   // all eigenvalues below mid
    else lo = mid;
  }
  return 0.5 * (lo + hi);
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char* dgvv_last_error(void) { return g_err.c_str(); }
const char* dgvv_version(void) { return "dgvv 0.1 (sm_100a, fp64)"; }

dgvv_status dgvv_nccl_get_unique_id(char out_id[128]) {
  TRY(nccl_load());
  ncclUniqueId id;
  NCCL_TRY(g_nccl.getUniqueId(&id));
  std::memcpy(out_id, id.internal, 128);
  return DGVV_OK;
}

dgvv_status dgvv_nccl_comm_init(const char id_bytes[128], int32_t nranks, int32_t rank, void** comm) {
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
  if (!comm) return DGVV_OK;
  DgvvComm* cm = (DgvvComm*)comm;
  if (cm->kind != COMM_NCCL) return dgvv_fail(DGVV_EINVAL, "not an NCCL communicator");
  TRY(nccl_load());
  NCCL_TRY(g_nccl.commDestroy(cm->nccl));
  delete cm;
  return DGVV_OK;
}

dgvv_status dgvv_thread_group_create(int32_t nranks, void** group) {
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
  ThreadGroup* g = (ThreadGroup*)group;
  if (!g || !comm || rank < 0 || rank >= g->R) return dgvv_fail(DGVV_EINVAL, "thread group: bad rank %d", rank);
  *comm = (void*)&g->comms[rank];
  return DGVV_OK;
}

dgvv_status dgvv_thread_group_destroy(void* group) {
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

static dgvv_status setup_impl(const dgvv_mesh* m, int32_t degree, const dgvv_law* vl, const dgvv_law* pl,
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
    size_t total_send = 0;
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
      c->peers.push_back(P);
    }
    int nmax = 0;
    for (auto& L : c->L) nmax = std::max(nmax, L.n);
    c->sendbuf_len = total_send * 3 * nmax * nmax * nmax;
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
    if (cm->kind == COMM_THREADS) {               // handshake: send counts vs listed ghosts
      ThreadGroup* g = cm->tg;
      {
        std::lock_guard<std::mutex> lk(g->mu);
        for (int q = 0; q < g->R; ++q) g->sbytes[cm->rank][q] = 0;
        for (auto& P : c->peers) g->sbytes[cm->rank][P.rank] = (size_t)P.n_send;
      }
      tg_barrier(g);
      std::string bad;
      for (auto& P : c->peers)
        if (g->sbytes[P.rank][cm->rank] != (size_t)P.n_recv) bad = "peer count mismatch";
      tg_barrier(g);
      if (!bad.empty()) return dgvv_fail(DGVV_EINVAL, "thread group: a peer sends a different number of cells than the ghosts listed");
    } else if (!c->peers.empty()) {
      // handshake: every peer's send count must equal the ghosts listed here
      int* d_cnt = nullptr;
      TRY(dalloc(c, &d_cnt, 2 * c->peers.size()));
      std::vector<int> hs(c->peers.size());
      for (size_t i = 0; i < c->peers.size(); ++i) hs[i] = c->peers[i].n_send;
      DGVV_CUDA_TRY(cudaMemcpy(d_cnt, hs.data(), hs.size() * sizeof(int), cudaMemcpyHostToDevice));
      NCCL_TRY(g_nccl.groupStart());
      for (size_t i = 0; i < c->peers.size(); ++i) {
        NCCL_TRY(g_nccl.send(d_cnt + i, 1, ncclInt32, c->peers[i].rank, cm->nccl, s));
        NCCL_TRY(g_nccl.recv(d_cnt + c->peers.size() + i, 1, ncclInt32, c->peers[i].rank, cm->nccl, s));
      }
      NCCL_TRY(g_nccl.groupEnd());
      std::vector<int> got(c->peers.size());
      DGVV_CUDA_TRY(cudaMemcpyAsync(got.data(), d_cnt + c->peers.size(), got.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
      DGVV_CUDA_TRY(cudaStreamSynchronize(s));
      for (size_t i = 0; i < c->peers.size(); ++i)
        if (got[i] != c->peers[i].n_recv)
          return dgvv_fail(DGVV_EINVAL, "peer %d sends %d cells but %d ghosts are listed", c->peers[i].rank, got[i], c->peers[i].n_recv);
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
static dgvv_status host_pipe_setup(dgvv_ctx* c, int level) {
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

static dgvv_status ensure_dinv_pen(dgvv_ctx* c, int l, cudaStream_t s);
static dgvv_status apply_penalty_impl(dgvv_ctx* c, int l, const double* src, double* dst, cudaStream_t s);
static dgvv_status cheb_pen(dgvv_ctx* c, int l, double* x, const double* b, int degree, double lo, double hi,
                            int x_is_zero, double* work, cudaStream_t s);
static dgvv_status ensure_pen_scratch(dgvv_ctx* c);
static dgvv_status vcycle_pen_rec(dgvv_ctx* c, int l, const double* b, double* x, const double* his,
                                  cudaStream_t s);

dgvv_status dgvv_set_mass(dgvv_ctx* c, int32_t op, double mass) {
  TRY(check_ctx(c));
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  if (!std::isfinite(mass) || mass < 0.0) return dgvv_fail(DGVV_EDOMAIN, "mass coefficient %g must be finite and >= 0", mass);
  if (c->mass[op] == mass) return DGVV_OK;
  c->mass[op] = mass;
  ++c->coef_epoch;
  for (auto& L : c->L) L.dinv_ok[op] = false;   // the diagonal changes: recomputed lazily (same buffer)
  return DGVV_OK;
}

dgvv_status dgvv_inverse_diagonal(dgvv_ctx* c, int32_t op, int32_t level, double* dst, dgvv_stream stream) {
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

static dgvv_status cheb_impl(dgvv_ctx* c, int op, int l, double* x, const double* b, int degree, double lo,
                             double hi, int x_is_zero, double* work, cudaStream_t s) {
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
    a.src = x; a.b = b; a.dinv = dinv; a.dvec = d; a.xout = work;
    a.mode = MODE_CHEB; a.c_rho = 0.0; a.c_r = 1.0 / theta;
    TRY(run_apply(c, op, l, a, s));
    cur = 1;
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
  TRY(check_level(c, level));
  TRY(op_ready(c, op));
  if (!x || !b || !work) return dgvv_fail(DGVV_EINVAL, "null vector");
  if (degree < 1) return dgvv_fail(DGVV_EINVAL, "degree %d < 1", degree);
  if (!(lambda_hi > lambda_lo) || !(lambda_lo > 0.0)) return dgvv_fail(DGVV_EDOMAIN, "need 0 < lambda_lo < lambda_hi");
  if (op == DGVV_OP_PENALTY)
    return cheb_pen(c, level, x, b, degree, lambda_lo, lambda_hi, x_is_zero, work, (cudaStream_t)stream);
  return cheb_impl(c, op, level, x, b, degree, lambda_lo, lambda_hi, x_is_zero, work, (cudaStream_t)stream);
}

static dgvv_status transfer(dgvv_ctx* c, int op, int fl, const double* in, double* out, double beta, bool prol,
                            cudaStream_t s) {
  if (fl < 0 || fl + 1 >= (int)c->L.size()) return dgvv_fail(DGVV_EINVAL, "fine_level %d has no coarser level", fl);
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "op");
  const int nf = c->L[fl].n, ncs = c->L[fl + 1].n;
  std::vector<double> P1((size_t)nf * ncs), M((size_t)nf * ncs);
  transfer_matrix(nf, ncs, P1.data());
  if (prol) {
    M = P1;   // nout = nf, nin = nc
    DGVV_CUDA_TRY(launch_tensor3(ncs, nf, nc, M.data(), in, out, beta, c->n_owned, s));
  } else {
    for (int i = 0; i < nf; ++i)
      for (int j = 0; j < ncs; ++j) M[(size_t)j * nf + i] = P1[(size_t)i * ncs + j];
    DGVV_CUDA_TRY(launch_tensor3(nf, ncs, nc, M.data(), in, out, beta, c->n_owned, s));
  }
  return DGVV_OK;
}

dgvv_status dgvv_prolongate(dgvv_ctx* c, int32_t op, int32_t fine_level, const double* coarse, double* fine,
                            double beta, dgvv_stream stream) {
  if (!c || !coarse || !fine) return dgvv_fail(DGVV_EINVAL, "null argument");
  return transfer(c, op, fine_level, coarse, fine, beta, true, (cudaStream_t)stream);
}

dgvv_status dgvv_restrict(dgvv_ctx* c, int32_t op, int32_t fine_level, const double* fine, double* coarse,
                          double beta, dgvv_stream stream) {
  if (!c || !coarse || !fine) return dgvv_fail(DGVV_EINVAL, "null argument");
  return transfer(c, op, fine_level, fine, coarse, beta, false, (cudaStream_t)stream);
}

static dgvv_status cg_vcycle(dgvv_ctx* c, int op, const double* b, double* x, const double* his, cudaStream_t s);
static dgvv_status cg_setup_direct(dgvv_ctx* c, int op, int32_t* n_dofs);
static dgvv_status cg_enter(dgvv_ctx* c, int op, const double* r_dg, double* x_dg, const double* his, cudaStream_t s);
static dgvv_status hprolong_impl(dgvv_ctx* c, int op, const double* coarse, double* fine, double beta,
                                 cudaStream_t s);
static dgvv_status hrestrict_impl(dgvv_ctx* c, int op, const double* fine, double* coarse, double beta,
                                  cudaStream_t s);

// V(l, b) of SURVEY §8(c) c1.7 over the chain of contexts (p-levels of c, then — f3 — the levels
// of c->coarse after an h-transfer); the coarsest level of the chain is either Chebyshev(5) from
// 0 (G15) or, after dgvv_setup_coarse_solver, the direct solve (reading H3).
static dgvv_status vcycle_rec(dgvv_ctx* c, int op, int l, const double* b, double* x, const double* his,
                              cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  auto& S = c->L[l].scratch[oi];   // [0] r, [1..2] work, (l>0: [3] b, [4] x of coarser handled by caller)
  const int last = (int)c->L.size() - 1;
  if (l == last && !c->coarse && !c->cg.on && c->Ainv[oi]) {   // the c-level, when enabled, comes first
    if (c->direct_epoch[oi] != c->coef_epoch)
      return dgvv_fail(DGVV_ESTATE, "direct coarse solver is stale (coefficients or mass changed): call dgvv_setup_coarse_solver again");
    DGVV_CUDA_TRY(launch_dense_matvec(c->Ainv[oi], b, x, c->direct_n[oi], s));
    return DGVV_OK;
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
    TRY(transfer(c, op, l, C[4], x, 1.0, true, s));
  } else {                                     // h-coarsening into the coarser context
    TRY(hrestrict_impl(c, op, S[0], c->hb[oi], 0.0, s));
    TRY(vcycle_rec(c->coarse, op, 0, c->hb[oi], c->hx[oi], his + c->L.size(), s));
    TRY(hprolong_impl(c, op, c->hx[oi], x, 1.0, s));
  }
  TRY(cheb_impl(c, op, l, x, b, 5, lo, hi, 0, S[1], s));
  return DGVV_OK;
}

// ------------------------------------------------------------------ FP32 multigrid (f1)
static dgvv_status d2f_alloc(dgvv_ctx* c, float** dst, const double* src, long n, cudaStream_t s) {
  if (!*dst) TRY(dalloc(c, dst, (size_t)n));
  DGVV_CUDA_TRY(launch_d2f(src, *dst, n, s));
  return DGVV_OK;
}

static dgvv_status ensure_fp32(dgvv_ctx* c, int op, cudaStream_t s) {
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

static ApplyArgsT<float> base_args_f(dgvv_ctx* c, int l, int op) {
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

// FP32 levels across ranks: the ghost cells travel in single precision (half the bytes), packed by
// the float gather kernel and moved by the same collective as the FP64 exchange; interior cells
// run while they move
static dgvv_status run_apply_f(dgvv_ctx* c, int op, int l, const ApplyArgsT<float>& a, cudaStream_t s) {
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  const int form = op == DGVV_OP_VISCOUS ? c->form : DGVV_FORM_LAPLACE;
  auto launch = [&](const ApplyArgsT<float>& x) -> dgvv_status {
    cudaError_t e = launch_apply_f(nc, c->L[l].n, form, c->geo, x, s);
    if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "FP32 apply kernel: %s", cudaGetErrorString(e));
    return DGVV_OK;
  };
  if (!c->comm || c->peers.empty()) return launch(a);
  const int n = c->L[l].n;
  const int len = nc * n * n * n;
  float* sb = reinterpret_cast<float*>(c->d_sendbuf);
  size_t off = 0;
  for (auto& P : c->peers) {
    DGVV_CUDA_TRY(launch_gather_cells_f(a.src, P.d_send, P.n_send, len, sb + off, s));
    off += (size_t)P.n_send * len;
  }
  TRY(comm_sendrecv(c, sb, const_cast<float*>(a.ghost), len, sizeof(float), s));
  ApplyArgsT<float> ai = a;
  ai.cell_list = c->d_interior;
  ai.n_proc = c->n_interior;
  TRY(launch(ai));
  DGVV_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_comm, 0));
  ApplyArgsT<float> ab = a;
  ab.cell_list = c->d_boundary;
  ab.n_proc = c->n_boundary;
  return launch(ab);
}

static dgvv_status cheb_impl_f(dgvv_ctx* c, int op, int l, float* x, const float* b, int degree, double lo,
                               double hi, int x_is_zero, float* work, cudaStream_t s) {
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
    a.src = x; a.b = b; a.dinv = dinv; a.dvec = d; a.xout = work;
    a.mode = MODE_CHEB; a.c_rho = 0.0; a.c_r = 1.0 / theta;
    TRY(run_apply_f(c, op, l, a, s));
    cur = 1;
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

static dgvv_status transfer_f(dgvv_ctx* c, int op, int fl, const float* in, float* out, double beta, bool prol,
                              cudaStream_t s) {
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  const int nf = c->L[fl].n, ncs = c->L[fl + 1].n;
  std::vector<double> P1((size_t)nf * ncs), M((size_t)nf * ncs);
  transfer_matrix(nf, ncs, P1.data());
  if (prol) {
    DGVV_CUDA_TRY(launch_tensor3_f(ncs, nf, nc, P1.data(), in, out, beta, c->n_owned, s));
  } else {
    for (int i = 0; i < nf; ++i)
      for (int j = 0; j < ncs; ++j) M[(size_t)j * nf + i] = P1[(size_t)i * ncs + j];
    DGVV_CUDA_TRY(launch_tensor3_f(nf, ncs, nc, M.data(), in, out, beta, c->n_owned, s));
  }
  return DGVV_OK;
}

// the V-cycle of vcycle_rec with every level in FP32
static dgvv_status vcycle_rec_f(dgvv_ctx* c, int op, int l, const float* b, float* x, const double* his,
                                cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  auto& S = c->LF[l].scratch[oi];
  const int last = (int)c->L.size() - 1;
  if (l == last && !c->coarse && !c->cg.on && c->Ainv[oi]) {   // direct coarse solve, FP64 arithmetic; the c-level, when enabled, comes first
    if (c->direct_epoch[oi] != c->coef_epoch)
      return dgvv_fail(DGVV_ESTATE, "direct coarse solver is stale (coefficients or mass changed): call dgvv_setup_coarse_solver again");
    DGVV_CUDA_TRY(launch_dense_matvec_f(c->Ainv[oi], b, x, c->direct_n[oi], s));
    return DGVV_OK;
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
    TRY(transfer_f(c, op, l, C[4], x, 1.0, true, s));
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
static dgvv_status vcycle_fp32_d(dgvv_ctx* c, int op, const double* r, double* z, const double* his, cudaStream_t s) {
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
  if (!c || !b || !x || !his) return dgvv_fail(DGVV_EINVAL, "null argument");
  TRY(op_ready(c, op));
  return vcycle_fp32_d(c, op, b, x, his, (cudaStream_t)stream);
}

static dgvv_status ensure_vcycle_scratch(dgvv_ctx* c, int op);

dgvv_status dgvv_vcycle(dgvv_ctx* c, int32_t op, const double* b, double* x, const double* his,
                        dgvv_stream stream) {
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
static dgvv_status ensure_vcycle_scratch(dgvv_ctx* c, int op) {
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

static dgvv_status dot_host(dgvv_ctx* c, const double* a, const double* b, long n, double* out, cudaStream_t s) {
  TRY(dot_dev(c, a, b, n, c->d_scal + 5, s));
  DGVV_CUDA_TRY(cudaMemcpyAsync(out, c->d_scal + 5, sizeof(double), cudaMemcpyDeviceToHost, s));
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  return DGVV_OK;
}

// ------------------------------------------------------------------ f2: penalty-step operator
static PenaltyArgs penalty_args(dgvv_ctx* c, int l) {
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
static dgvv_status apply_penalty_impl(dgvv_ctx* c, int l, const double* src, double* dst, cudaStream_t s) {
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

static dgvv_status ensure_dinv_pen(dgvv_ctx* c, int l, cudaStream_t s) {
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
// r = b - A x by the penalty kernel, then d = c_rho d + c_r D^-1 r, x += d (cheb_vec kernel).
// work holds 2 N doubles (r | d).
static dgvv_status cheb_pen(dgvv_ctx* c, int l, double* x, const double* b, int degree, double lo, double hi,
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
    TRY(apply_penalty_impl(c, l, x, r, s));
    DGVV_CUDA_TRY(launch_axpby(1.0, b, -1.0, r, N, s));          // r = b - A x
    DGVV_CUDA_TRY(launch_cheb_vec(r, dinv, 0.0, 1.0 / theta, d, x, N, s));
  }
  for (int j = 1; j < degree; ++j) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    TRY(apply_penalty_impl(c, l, x, r, s));
    DGVV_CUDA_TRY(launch_axpby(1.0, b, -1.0, r, N, s));
    DGVV_CUDA_TRY(launch_cheb_vec(r, dinv, rho_new * rho, 2.0 * rho_new / delta, d, x, N, s));
    rho = rho_new;
  }
  return DGVV_OK;
}

static dgvv_status ensure_pen_scratch(dgvv_ctx* c) {
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
static dgvv_status vcycle_pen_rec(dgvv_ctx* c, int l, const double* b, double* x, const double* his,
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
  if (!c || !src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (src == dst) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  TRY(op_ready(c, DGVV_OP_PENALTY));
  return apply_penalty_impl(c, 0, src, dst, (cudaStream_t)stream);
}

dgvv_status dgvv_apply_penalty_level(dgvv_ctx* c, int32_t level, const double* src, double* dst,
                                     dgvv_stream stream) {
  TRY(check_level(c, level));
  if (!src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (src == dst) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  TRY(op_ready(c, DGVV_OP_PENALTY));
  return apply_penalty_impl(c, level, src, dst, (cudaStream_t)stream);
}

dgvv_status dgvv_cg_solve(dgvv_ctx* c, int32_t op, const double* b, double* x, double rtol, int32_t maxit,
                          int32_t precond, const double* lambda_hi_per_level, int32_t* iters, double* relres,
                          dgvv_stream stream) {
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


// ------------------------------------------------------------------ f4: convective term + GMRES
static ConvArgs conv_args(dgvv_ctx* c) {
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
static dgvv_status ensure_conv_pointdata(dgvv_ctx* c, cudaStream_t s) {
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
static dgvv_status launch_conv(dgvv_ctx* c, const double* src, double* dst, double alpha, int accumulate,
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
  if (!c || !src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (src == dst) return dgvv_fail(DGVV_EINVAL, "src and dst alias");
  if (!c->has_wtr) return dgvv_fail(DGVV_ESTATE, "convective term: call dgvv_set_transport first");
  cudaStream_t s = (cudaStream_t)stream;
  if (c->n_ghost) TRY(exchange_sync(c, 0, 3, src, c->L[0].ghost[0], s));
  return launch_conv(c, src, dst, 1.0, 0, s);
}

// dst = (mass M + A(nu) + alpha_c C(w)) src [rhs given: dst = rhs - (...) src]
static dgvv_status apply_oseen(dgvv_ctx* c, double alpha_c, const double* src, double* dst, const double* rhs,
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

// ------------------------------------------------------------------ f3 c-level (continuous Q1)
static dgvv_status cg_apply(dgvv_ctx* c, int op, const double* x, double* y, cudaStream_t s) {
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
static dgvv_status cg_ensure_dinv(dgvv_ctx* c, int op, cudaStream_t s) {
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
static dgvv_status cg_cheb(dgvv_ctx* c, int op, double* x, const double* b, int degree, double lo, double hi,
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
static dgvv_status cg_build_transfer(dgvv_ctx* c) {
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
static dgvv_status cg_vcycle(dgvv_ctx* c, int op, const double* b, double* x, const double* his, cudaStream_t s) {
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
static dgvv_status cg_enter(dgvv_ctx* c, int op, const double* r_dg, double* x_dg, const double* his, cudaStream_t s) {
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  auto& G = c->cg;
  DGVV_CUDA_TRY(launch_cg_embedT(r_dg, G.b0[oi], G.d_inc_ptr, G.d_inc, G.nv, nc, 0.0, s));
  TRY(cg_vcycle(c, op, G.b0[oi], G.x0[oi], his, s));
  DGVV_CUDA_TRY(launch_cg_embed(G.x0[oi], x_dg, G.d_vid, c->n_owned, G.nv, nc, 1.0, s));
  return DGVV_OK;
}

static dgvv_status cg_setup_direct(dgvv_ctx* c, int op, int32_t* n_dofs) {
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
  TRY(check_ctx(c));
  if (!c->cg.on) return dgvv_fail(DGVV_ESTATE, "continuous level not enabled");
  if (n_vertices) *n_vertices = c->cg.nv;
  if (n_colors) *n_colors = c->cg.ncolors;
  return DGVV_OK;
}

dgvv_status dgvv_apply_continuous(dgvv_ctx* c, int32_t op, const double* src, double* dst, dgvv_stream stream) {
  if (!c || !src || !dst) return dgvv_fail(DGVV_EINVAL, "null argument");
  if (!c->cg.on) return dgvv_fail(DGVV_ESTATE, "continuous level not enabled");
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  TRY(op_ready(c, op));
  TRY(ensure_vcycle_scratch(c, op));
  return cg_apply(c, op, src, dst, (cudaStream_t)stream);
}

dgvv_status dgvv_embed_continuous(dgvv_ctx* c, int32_t op, int32_t transpose, const double* src, double* dst,
                                  double beta, dgvv_stream stream) {
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
static dgvv_status hprolong_impl(dgvv_ctx* c, int op, const double* coarse, double* fine, double beta,
                                 cudaStream_t s) {
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  cudaError_t e = launch_hprolongate(c->L.back().n, nc, coarse, fine, c->d_parent, c->d_octant, beta, c->n_owned, s);
  if (e == cudaErrorNotSupported) return dgvv_fail(DGVV_EUNSUPPORTED, "h-transfer not built for degree %d", c->L.back().k);
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "h-prolongation: %s", cudaGetErrorString(e));
  return DGVV_OK;
}

static dgvv_status hrestrict_impl(dgvv_ctx* c, int op, const double* fine, double* coarse, double beta,
                                  cudaStream_t s) {
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  cudaError_t e = launch_hrestrict(c->L.back().n, nc, fine, coarse, c->d_child, beta, c->coarse->n_owned, s);
  if (e == cudaErrorNotSupported) return dgvv_fail(DGVV_EUNSUPPORTED, "h-transfer not built for degree %d", c->L.back().k);
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "h-restriction: %s", cudaGetErrorString(e));
  return DGVV_OK;
}

dgvv_status dgvv_set_coarse_context(dgvv_ctx* c, dgvv_ctx* cc, const int32_t* parent, const int8_t* octant) {
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

static dgvv_status h_ready(dgvv_ctx* c, int op) {
  TRY(check_ctx(c));
  if (!c->coarse) return dgvv_fail(DGVV_ESTATE, "no coarse context: call dgvv_set_coarse_context first");
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  return DGVV_OK;
}

dgvv_status dgvv_prolongate_h(dgvv_ctx* c, int32_t op, const double* coarse, double* fine, double beta,
                              dgvv_stream stream) {
  TRY(h_ready(c, op));
  if (!coarse || !fine) return dgvv_fail(DGVV_EINVAL, "null vector");
  return hprolong_impl(c, op, coarse, fine, beta, (cudaStream_t)stream);
}

dgvv_status dgvv_restrict_h(dgvv_ctx* c, int32_t op, const double* fine, double* coarse, double beta,
                            dgvv_stream stream) {
  TRY(h_ready(c, op));
  if (!coarse || !fine) return dgvv_fail(DGVV_EINVAL, "null vector");
  return hrestrict_impl(c, op, fine, coarse, beta, (cudaStream_t)stream);
}

dgvv_status dgvv_setup_coarse_solver(dgvv_ctx* c, int32_t op, int32_t* n_dofs) {
  TRY(check_ctx(c));
  if (op != DGVV_OP_VISCOUS && op != DGVV_OP_POISSON) return dgvv_fail(DGVV_EINVAL, "unknown op %d", op);
  TRY(op_ready(c, op));
  if (c->n_ghost || c->comm) return dgvv_fail(DGVV_EUNSUPPORTED, "direct coarse solver: single-GPU contexts only");
  const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
  const int nc = op == DGVV_OP_VISCOUS ? 3 : 1;
  const int l = (int)c->L.size() - 1;
  if (c->cg.on) return cg_setup_direct(c, op, n_dofs);
  const long N = (long)nc * level_dofs(c, l);
  if (N > 4096) return dgvv_fail(DGVV_EINVAL, "direct coarse solver: %ld DoFs on the coarsest level (max 4096)", N);
  cudaStream_t s = 0;
  double *cols = nullptr, *W = nullptr, *fac = nullptr, *e = nullptr;
  struct Tmp { double** p[4]; ~Tmp() { for (auto q : p) if (*q) cudaFree(*q); } } tmp{{&cols, &W, &fac, &e}};
  DGVV_CUDA_TRY(cudaMalloc(&cols, (size_t)N * N * sizeof(double)));
  DGVV_CUDA_TRY(cudaMalloc(&W, (size_t)2 * N * N * sizeof(double)));
  DGVV_CUDA_TRY(cudaMalloc(&fac, (size_t)N * sizeof(double)));
  DGVV_CUDA_TRY(cudaMalloc(&e, (size_t)N * sizeof(double)));
  for (long j = 0; j < N; ++j) {               // column j = A e_j (the level's matrix-free apply)
    DGVV_CUDA_TRY(launch_set_unit(e, N, j, s));
    ApplyArgs a = base_args(c, l, op);
    a.src = e;
    a.dst = cols + (size_t)j * N;
    TRY(run_apply(c, op, l, a, s));
  }
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
  c->direct_epoch[oi] = c->coef_epoch;
  if (n_dofs) *n_dofs = (int32_t)N;
  return DGVV_OK;
}

dgvv_status dgvv_estimate_lambda_max(dgvv_ctx* c, int32_t op, int32_t level, int32_t steps, const double* v0,
                                     double* out, dgvv_stream stream) {
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

dgvv_status dgvv_dot(dgvv_ctx* c, int32_t level, int32_t ncomp, const double* a, const double* b, double* out,
                     dgvv_stream stream) {
  TRY(check_level(c, level));
  if (!a || !b || !out || ncomp < 1) return dgvv_fail(DGVV_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  TRY(dot_dev(c, a, b, (long)ncomp * level_dofs(c, level), c->d_scal + 4, s));
  DGVV_CUDA_TRY(cudaMemcpyAsync(out, c->d_scal + 4, sizeof(double), cudaMemcpyDeviceToHost, s));
  DGVV_CUDA_TRY(cudaStreamSynchronize(s));
  return DGVV_OK;
}

dgvv_status dgvv_sizes(const dgvv_ctx* c, int32_t level, int64_t* nl, int64_t* ng) {
  TRY(check_level(c, level));
  const long long n3 = (long long)c->L[level].n * c->L[level].n * c->L[level].n;
  if (nl) *nl = (int64_t)c->n_owned * n3;
  if (ng) *ng = (int64_t)c->n_global * n3;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "pending CUDA error: %s", cudaGetErrorString(e));
  return DGVV_OK;
}

dgvv_status dgvv_coefficient_range(dgvv_ctx* c, int32_t op, int32_t level, double* lo, double* hi) {
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

dgvv_status dgvv_ghost_layout(const dgvv_ctx* c, int32_t* n_peers, int32_t* peer_ranks, int32_t* send_counts,
                              int32_t* recv_counts) {
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
  TRY(check_level(c, level));
  if (!src || !sendbuf) return dgvv_fail(DGVV_EINVAL, "null vector");
  const int nc = kind == DGVV_GHOST_POISSON ? 1 : 3;
  return pack(c, level, nc, src, sendbuf, (cudaStream_t)stream);
}

dgvv_status dgvv_ghost_buffer(dgvv_ctx* c, int32_t level, int32_t kind, double** out) {
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
