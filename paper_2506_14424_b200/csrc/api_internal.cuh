// api_internal.cuh — shared state and helpers of the C ABI implementation (api_*.cu): the context
// (levels, FP32 mirrors, communication plan), errors, communicators (NCCL / in-process thread
// group), per-device tables, and the host helpers every row's orchestration uses.  Host
// orchestration only: every arithmetic step of the path runs in the kernels of k_*.cu.
//   api_core.cu  — context, setup (§8(a) a1/a2), applies (a3-a7), ghosts, dots, sizes
//   api_mg.cu    — inverse diagonal, Chebyshev, p-transfer, V-cycles FP64/FP32, Lanczos, CG (a8-a11, f1)
//   api_penalty.cu — penalty-step operator and its multigrid (f2)
//   api_oseen.cu — convective term, Oseen operator, GMRES (f4)
//   api_cph.cu   — c-level, h-levels, direct coarse solver (f3)
#pragma once
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

#include <nvtx3/nvToolsExt.h>

#include "../../include/dgvv.h"
#include "launch.h"

using namespace dgvv;

// ------------------------------------------------------------------ NVTX ranges
// Every C-ABI entry point opens a range named after itself, so a timeline tool (nsys, ncu
// --nvtx) shows which call launched which kernels.  NVTX v3 is header-only: without a tool
// attached a push/pop is a null function-pointer test.
struct DgvvNvtxRange {
  explicit DgvvNvtxRange(const char* name) { nvtxRangePushA(name); }
  ~DgvvNvtxRange() { nvtxRangePop(); }
  DgvvNvtxRange(const DgvvNvtxRange&) = delete;
  DgvvNvtxRange& operator=(const DgvvNvtxRange&) = delete;
};
#define DGVV_RANGE() DgvvNvtxRange dgvv_nvtx_range_(__func__)

// ------------------------------------------------------------------ errors
inline thread_local std::string g_err;

inline dgvv_status dgvv_fail(dgvv_status st, const char* fmt, ...) {
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
namespace dgvv_api {
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
inline NcclApi g_nccl;
inline std::mutex g_nccl_mu;

inline dgvv_status nccl_load() {
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
inline void tg_barrier(ThreadGroup* g) {
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
inline std::mutex g_tab_mu;
inline uint64_t g_tab_done = 0;     // bit d: tables uploaded to device d

inline dgvv_status upload_tables() {
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
}  // namespace dgvv_api
using namespace dgvv_api;

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
  double* gtr[2] = {nullptr, nullptr};     // received ghost face traces (communicator mode)
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
  float* gtr[2] = {nullptr, nullptr};       // FP32 ghost face traces per op (communicator mode)
  std::vector<float*> scratch[2];           // [0] r, [1] work (2N), [3] b, [4] x
};

struct Peer {
  int rank;
  int* d_send = nullptr;      // owned local cells to send (sorted by global id)
  int n_send = 0;
  int recv_off = 0, n_recv = 0;   // ghost index range received from this peer
  // face-trace exchange (communicator mode): (owned cell, face) items whose neighbour the peer
  // owns, ascending (cell, face); the peer receives them in the same order for its ghosts
  int* d_fcell = nullptr;
  int* d_fface = nullptr;
  int n_send_f = 0;
  int recv_off_f = 0, n_recv_f = 0;   // trace item range received from this peer
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
  // multi-rank direct solve: the inverse is replicated on every rank; this rank's owned DoFs are
  // rows [direct_off, direct_off + direct_rows) and b is gathered into direct_bf (global length)
  long direct_off[2] = {0, 0};
  int direct_rows[2] = {0, 0};
  double* direct_bf[2] = {nullptr, nullptr};
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
  int* d_gslot = nullptr;                    // [n_ghost][6] trace item of ghost g's face f (-1: none)
  int n_recv_f = 0;                          // trace items received in total
  double* tg_red = nullptr;                  // thread group: allreduce staging (tg_red_cap doubles)
  long tg_red_cap = 0;
  double* align_buf = nullptr;               // aligned copy of a misaligned apply source
  long align_cap = 0;
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
dgvv_status comm_sendrecv(dgvv_ctx* c, const void* sendbuf, void* ghost, int len, size_t esz, cudaStream_t s,
                          bool faces = false) {
  auto nsend = [&](const Peer& P) { return faces ? P.n_send_f : P.n_send; };
  auto nrecv = [&](const Peer& P) { return faces ? P.n_recv_f : P.n_recv; };
  auto roff = [&](const Peer& P) { return faces ? P.recv_off_f : P.recv_off; };
  DgvvComm* cm = (DgvvComm*)c->comm;
  DGVV_CUDA_TRY(cudaEventRecord(c->ev_pack, s));
  if (cm->kind == COMM_NCCL) {
    DGVV_CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_pack, 0));
    const ncclDataType_t dt = esz == 8 ? ncclDouble : ncclFloat;
    NCCL_TRY(g_nccl.groupStart());
    size_t off = 0;
    for (auto& P : c->peers) {
      if (nsend(P)) NCCL_TRY(g_nccl.send((const char*)sendbuf + off * esz, (size_t)nsend(P) * len, dt, P.rank, cm->nccl, c->comm_stream));
      if (nrecv(P)) NCCL_TRY(g_nccl.recv((char*)ghost + (size_t)roff(P) * len * esz, (size_t)nrecv(P) * len, dt, P.rank, cm->nccl, c->comm_stream));
      off += (size_t)nsend(P) * len;
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
      g->sbytes[r][P.rank] = (size_t)nsend(P) * len * esz;
      off += (size_t)nsend(P) * len;
    }
    g->ev_a[r] = c->ev_pack;
  }
  tg_barrier(g);
  // our ghost buffer is rewritten only after our own earlier kernels that read it (ordered before
  // ev_pack on s), and after each peer has packed
  DGVV_CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_pack, 0));
  for (auto& P : c->peers) {
    const size_t want = (size_t)nrecv(P) * len * esz;
    if (g->sbytes[P.rank][r] != want)
      return dgvv_fail(DGVV_EINVAL, "thread group: rank %d sends %zu bytes, rank %d expects %zu", P.rank, g->sbytes[P.rank][r], r, want);
    if (!want) continue;
    DGVV_CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, g->ev_a[P.rank], 0));
    DGVV_CUDA_TRY(cudaMemcpyAsync((char*)ghost + (size_t)roff(P) * len * esz, g->sptr[P.rank][r], want,
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
dgvv_status comm_allreduce(dgvv_ctx* c, double* ptr, long count, cudaStream_t s) {
  DgvvComm* cm = (DgvvComm*)c->comm;
  if (!cm) return DGVV_OK;
  if (cm->kind == COMM_NCCL) {
    NCCL_TRY(g_nccl.allReduce(ptr, ptr, (size_t)count, ncclDouble, ncclSum, cm->nccl, s));
    return DGVV_OK;
  }
  ThreadGroup* g = cm->tg;
  const int r = cm->rank;
  if (count > c->tg_red_cap) {                 // staging grows on demand (the coarse-solver gathers)
    DGVV_CUDA_TRY(cudaStreamSynchronize(s));
    double* nb = nullptr;
    TRY(dalloc(c, &nb, (size_t)count));
    c->tg_red = nb;                            // the old block stays in c->allocs until destroy
    c->tg_red_cap = count;
  }
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

// full[0:N] = every rank's owned segment (this rank's at `off`): a sum-allreduce over zero-padded
// copies, exact (each entry is one rank's value plus zeros) and identical on every rank
dgvv_status comm_gather_full(dgvv_ctx* c, const double* own, long n_own, long off, double* full, long N,
                             cudaStream_t s) {
  DGVV_CUDA_TRY(cudaMemsetAsync(full, 0, (size_t)N * sizeof(double), s));
  if (n_own > 0) DGVV_CUDA_TRY(cudaMemcpyAsync(full + off, own, (size_t)n_own * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return comm_allreduce(c, full, N, s);
}

// the coarsest level's direct solve x = A^-1 b (single context, or this rank's rows of the
// replicated inverse applied to the gathered b)
template <typename R>
dgvv_status direct_solve(dgvv_ctx* c, int oi, const R* b, R* x, cudaStream_t s) {
  const int N = c->direct_n[oi];
  if (!c->comm) {
    if constexpr (sizeof(R) == 8) DGVV_CUDA_TRY(launch_dense_matvec(c->Ainv[oi], b, x, N, s));
    else DGVV_CUDA_TRY(launch_dense_matvec_f(c->Ainv[oi], b, x, N, s));
    return DGVV_OK;
  }
  const long off = c->direct_off[oi], rows = c->direct_rows[oi];
  double* bf = c->direct_bf[oi];
  if constexpr (sizeof(R) == 8) {
    TRY(comm_gather_full(c, b, rows, off, bf, N, s));
    DGVV_CUDA_TRY(launch_dense_matvec(c->Ainv[oi] + (size_t)off * N, bf, x, N, s, (int)rows));
  } else {
    DGVV_CUDA_TRY(cudaMemsetAsync(bf, 0, (size_t)N * sizeof(double), s));
    if (rows) DGVV_CUDA_TRY(launch_f2d(b, bf + off, rows, s));
    TRY(comm_allreduce(c, bf, N, s));
    DGVV_CUDA_TRY(launch_dense_matvec_df(c->Ainv[oi] + (size_t)off * N, bf, x, N, s, (int)rows));
  }
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

// a5 in communicator mode: the face traces (value, d/dxi_n; 2 NC n^2 per cut face) of the owned
// cells next to each peer instead of whole ghost cells (NC n^3): pack kernel, then the collective
template <typename R>
dgvv_status exchange_traces(dgvv_ctx* c, int l, int nc, const R* src, R** gtr, cudaStream_t s) {
  const int n = c->L[l].n;
  const int len = 2 * nc * n * n;
  if (!*gtr) TRY(dalloc(c, gtr, (size_t)std::max(1, c->n_recv_f) * len));
  R* sb = reinterpret_cast<R*>(c->d_sendbuf);
  size_t off = 0;
  for (auto& P : c->peers) {
    cudaError_t e = sizeof(R) == 8
        ? launch_pack_traces(nc, n, (const double*)src, P.d_fcell, P.d_fface, P.n_send_f, (double*)(sb + off), s)
        : launch_pack_traces_f(nc, n, (const float*)src, P.d_fcell, P.d_fface, P.n_send_f, (float*)(sb + off), s);
    if (e != cudaSuccess) return dgvv_fail(DGVV_ECUDA, "trace pack: %s", cudaGetErrorString(e));
    off += (size_t)P.n_send_f * len;
  }
  return comm_sendrecv(c, sb, *gtr, len, sizeof(R), s, true);
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
  if (reinterpret_cast<uintptr_t>(a.src) & 31) {
    // the kernels read neighbour rows with 256-bit loads: a source vector that is not 32-byte
    // aligned (a slice of a larger tensor) is staged through an aligned copy (16 B/DoF extra)
    const size_t N = (size_t)(kind == 1 ? 3 : nc) * level_dofs(c, l);
    if ((long)N > c->align_cap) {
      DGVV_CUDA_TRY(cudaStreamSynchronize(s));
      double* nb = nullptr;
      TRY(dalloc(c, &nb, N));
      c->align_buf = nb;
      c->align_cap = (long)N;
    }
    DGVV_CUDA_TRY(cudaMemcpyAsync(c->align_buf, a.src, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    a.src = c->align_buf;
  }
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
  if (kind != 1) {                            // SIPG applies: face traces; Newton (K2): ghost cells
    const int oi = op == DGVV_OP_VISCOUS ? 0 : 1;
    TRY(exchange_traces(c, l, nc, a.src, &c->L[l].gtr[oi], s));
    a.gtr = c->L[l].gtr[oi];
    a.gslot = c->d_gslot;
  } else {
    TRY(exchange(c, l, nc, a.src, const_cast<double*>(a.ghost), s));
  }
  ApplyArgs ai = a;
  ai.cell_list = c->d_interior;
  ai.n_proc = c->n_interior;
  ai.gtr = nullptr;                           // interior cells never read a ghost: plain kernel
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

// ---- row orchestration shared across api_*.cu (C linkage, not exported from the library)
#define DGVV_INTERNAL __attribute__((visibility("hidden")))
extern "C" {
DGVV_INTERNAL dgvv_status setup_impl(const dgvv_mesh* m, int32_t degree, const dgvv_law* vl, const dgvv_law* pl,
                              const dgvv_options* opt, cudaStream_t s, dgvv_ctx* c);
DGVV_INTERNAL dgvv_status host_pipe_setup(dgvv_ctx* c, int level);
DGVV_INTERNAL dgvv_status cheb_impl(dgvv_ctx* c, int op, int l, double* x, const double* b, int degree, double lo,
                             double hi, int x_is_zero, double* work, cudaStream_t s, int start_in_work = 0);
DGVV_INTERNAL dgvv_status transfer(dgvv_ctx* c, int op, int fl, const double* in, double* out, double beta, bool prol,
                            cudaStream_t s, const double* add = nullptr);
DGVV_INTERNAL dgvv_status vcycle_rec(dgvv_ctx* c, int op, int l, const double* b, double* x, const double* his,
                              cudaStream_t s);
DGVV_INTERNAL dgvv_status d2f_alloc(dgvv_ctx* c, float** dst, const double* src, long n, cudaStream_t s);
DGVV_INTERNAL dgvv_status ensure_fp32(dgvv_ctx* c, int op, cudaStream_t s);
DGVV_INTERNAL ApplyArgsT<float> base_args_f(dgvv_ctx* c, int l, int op);
DGVV_INTERNAL dgvv_status run_apply_f(dgvv_ctx* c, int op, int l, const ApplyArgsT<float>& a, cudaStream_t s);
DGVV_INTERNAL dgvv_status cheb_impl_f(dgvv_ctx* c, int op, int l, float* x, const float* b, int degree, double lo,
                               double hi, int x_is_zero, float* work, cudaStream_t s, int start_in_work = 0);
DGVV_INTERNAL dgvv_status transfer_f(dgvv_ctx* c, int op, int fl, const float* in, float* out, double beta, bool prol,
                              cudaStream_t s, const float* add = nullptr);
DGVV_INTERNAL dgvv_status vcycle_rec_f(dgvv_ctx* c, int op, int l, const float* b, float* x, const double* his,
                                cudaStream_t s);
DGVV_INTERNAL dgvv_status vcycle_fp32_d(dgvv_ctx* c, int op, const double* r, double* z, const double* his, cudaStream_t s);
DGVV_INTERNAL dgvv_status ensure_vcycle_scratch(dgvv_ctx* c, int op);
DGVV_INTERNAL dgvv_status dot_host(dgvv_ctx* c, const double* a, const double* b, long n, double* out, cudaStream_t s);
DGVV_INTERNAL PenaltyArgs penalty_args(dgvv_ctx* c, int l);
DGVV_INTERNAL dgvv_status apply_penalty_impl(dgvv_ctx* c, int l, const double* src, double* dst, cudaStream_t s);
DGVV_INTERNAL dgvv_status ensure_dinv_pen(dgvv_ctx* c, int l, cudaStream_t s);
DGVV_INTERNAL dgvv_status cheb_pen(dgvv_ctx* c, int l, double* x, const double* b, int degree, double lo, double hi,
                            int x_is_zero, double* work, cudaStream_t s);
DGVV_INTERNAL dgvv_status ensure_pen_scratch(dgvv_ctx* c);
DGVV_INTERNAL dgvv_status vcycle_pen_rec(dgvv_ctx* c, int l, const double* b, double* x, const double* his,
                                  cudaStream_t s);
DGVV_INTERNAL ConvArgs conv_args(dgvv_ctx* c);
DGVV_INTERNAL dgvv_status ensure_conv_pointdata(dgvv_ctx* c, cudaStream_t s);
DGVV_INTERNAL dgvv_status launch_conv(dgvv_ctx* c, const double* src, double* dst, double alpha, int accumulate,
                               cudaStream_t s);
DGVV_INTERNAL dgvv_status apply_oseen(dgvv_ctx* c, double alpha_c, const double* src, double* dst, const double* rhs,
                               cudaStream_t s);
DGVV_INTERNAL dgvv_status cg_apply(dgvv_ctx* c, int op, const double* x, double* y, cudaStream_t s);
DGVV_INTERNAL dgvv_status cg_ensure_dinv(dgvv_ctx* c, int op, cudaStream_t s);
DGVV_INTERNAL dgvv_status cg_cheb(dgvv_ctx* c, int op, double* x, const double* b, int degree, double lo, double hi,
                           bool x_is_zero, cudaStream_t s);
DGVV_INTERNAL dgvv_status cg_build_transfer(dgvv_ctx* c);
DGVV_INTERNAL dgvv_status cg_vcycle(dgvv_ctx* c, int op, const double* b, double* x, const double* his, cudaStream_t s);
DGVV_INTERNAL dgvv_status cg_enter(dgvv_ctx* c, int op, const double* r_dg, double* x_dg, const double* his, cudaStream_t s);
DGVV_INTERNAL dgvv_status cg_setup_direct(dgvv_ctx* c, int op, int32_t* n_dofs);
DGVV_INTERNAL dgvv_status hprolong_impl(dgvv_ctx* c, int op, const double* coarse, double* fine, double beta,
                                 cudaStream_t s);
DGVV_INTERNAL dgvv_status hrestrict_impl(dgvv_ctx* c, int op, const double* fine, double* coarse, double beta,
                                  cudaStream_t s);
DGVV_INTERNAL dgvv_status h_ready(dgvv_ctx* c, int op);
}  // extern "C"
