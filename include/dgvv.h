/* dgvv.h — C ABI of the B200-native matrix-free SIPG viscous-operator hot path
 * (arXiv 2506.14424, "variable viscosity incompressible flow", §4-§5).
 *
 * Everything below is FP64 and runs in the library's own CUDA kernels (sm_100a).  The
 * library never falls back to the CPU: without a CUDA device every compute call returns
 * DGVV_ECUDA.
 *
 * Conventions shared by every call (readings of SURVEY.md §8(c), restated in DESIGN.md):
 *  - Reference cell [0,1]^3.  Degree-k DG space: tensor Lagrange basis on the k+1
 *    Gauss-Legendre points (G2), quadrature with the same k+1 Gauss points per direction
 *    (G1) — "collocation": coefficient = value at the quadrature point.
 *  - Vector layout (canonical, device, caller-owned, contiguous FP64):
 *        vector operator : [local_cell][component 0..2][z][y][x]   (3 (k+1)^3 per cell)
 *        scalar operator : [local_cell][z][y][x]                   ((k+1)^3 per cell)
 *  - Local faces are ordered (-x,+x,-y,+y,-z,+z); face quadrature points are lexicographic
 *    over the two tangential axes in increasing axis order, first axis fastest.  Meshes
 *    must be structured and aligned: point (a,b) of face +d of a cell coincides with point
 *    (a,b) of face -d of its neighbour (checked at setup, DGVV_EUNSUPPORTED otherwise).
 *  - Penalty (G3, G5, G6): tau = IP (k+1)^2 max(H-,H+) (nu- + nu+)/2,
 *    H_K = (A(dK\Gamma)/2 + A(dK cap Gamma)) / V(K); boundary faces use H_K and nu-.
 *  - Boundary conditions by the mirror principle (G7): Dirichlet
 *    faces u+ = -u-, grad u+ = grad u-, nu+ = nu-; Neumann faces contribute nothing;
 *    periodic faces are ordinary neighbours.
 *
 * Ownership: dgvv_setup copies every host array; vectors are borrowed device pointers the
 * library never frees or retains (except u_lin, see dgvv_update_viscosity).  The operator
 * kernels read source vectors with 256-bit loads: a source that is not 32-byte aligned (a slice
 * of a larger allocation) is first copied into an aligned library buffer (correct, 16 B/DoF of
 * extra traffic; cudaMalloc and PyTorch caching-allocator blocks are aligned).  All compute
 * calls are asynchronous on the caller's stream unless stated otherwise.  Status codes are
 * returned, never thrown; dgvv_last_error gives a message for the last failure.
 * One context is used by one host thread at a time; distinct contexts are independent.
 * Multi-GPU: every rank calls every function collectively with its local part.
 */
#ifndef DGVV_H
#define DGVV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dgvv_ctx dgvv_ctx;            /* opaque, owned by the library            */
typedef struct CUstream_st* dgvv_stream;     /* identical to cudaStream_t; NULL = legacy */

typedef enum {
  DGVV_OK = 0,
  DGVV_EINVAL = 1,        /* bad argument (null pointer, size, aliasing src/dst, ...)      */
  DGVV_EDOMAIN = 2,       /* nu <= 0 / non-finite at a quadrature point, bad degree, ...   */
  DGVV_ENOMEM = 3,        /* device allocation failed                                      */
  DGVV_ECUDA = 4,         /* CUDA error (sticky kernel errors surface at the next call)    */
  DGVV_ENCCL = 5,         /* NCCL error                                                    */
  DGVV_ESTATE = 6,        /* call order violated (e.g. Newton apply before update)         */
  DGVV_EUNSUPPORTED = 7   /* mesh / degree / option outside what the kernels implement     */
} dgvv_status;

enum { DGVV_BC_DIRICHLET = 1, DGVV_BC_NEUMANN = 2 };         /* neighbour entry = -1 - bc */

enum {                                  /* coefficient laws */
  DGVV_LAW_CONST = 0,     /* nu = p[0]                                                     */
  DGVV_LAW_SIN3 = 1,      /* nu = p[0] + p[1] sin(2 pi x) sin(2 pi y) sin(2 pi z)      (C1) */
  DGVV_LAW_EXP = 2,       /* nu = exp(p[0] (x + y + z))                           (C2, C4) */
  DGVV_LAW_CARREAU = 3    /* nu = eta(gd(eps(u_lin))), p = {eta0, eta_inf, lambda, n}:
                             eta = eta_inf + (eta0-eta_inf)(1+(lambda gd)^2)^((n-1)/2),
                             gd = sqrt(2 eps:eps)  (G9)  (C3, C5) */
};

enum { DGVV_OP_VISCOUS = 0, DGVV_OP_POISSON = 1, DGVV_OP_PENALTY = 2 };
enum { DGVV_FORM_DIVERGENCE = 0,   /* the paper's -div(2 nu eps(u)) (eqn:viscous_term_weak) */
       DGVV_FORM_LAPLACE = 1 };    /* tau_1 terms only: -div(nu grad u)  */

typedef struct {
  int32_t kind;           /* DGVV_LAW_*                                                    */
  double p[8];            /* parameters, see DGVV_LAW_*                                    */
} dgvv_law;

typedef struct {
  int32_t n_cells;            /* owned cells on this rank (> 0)                            */
  int32_t n_ghost;            /* ghost cells = off-rank face neighbours (0 on one GPU)     */
  int64_t first_global_cell;  /* owned cells are global ids [first, first + n_cells)       */
  const int64_t* neighbor;    /* host [n_cells + n_ghost][6]: global id across each face,
                                 or -1-bc for a boundary face.  Rows n_cells.. describe the
                                 ghosts (only their boundary flags are used, for H_K).      */
  const int64_t* ghost_global_id; /* host [n_ghost] global ids of the ghost rows           */
  const int32_t* ghost_owner;     /* host [n_ghost] rank owning each ghost                 */
  int32_t map_degree;         /* degree m of the geometry map (1 = trilinear corners)      */
  const double* nodes;        /* host [n_cells + n_ghost][(m+1)^3][3]: physical positions
                                 of the map's nodes on the Gauss-Lobatto points of [0,1],
                                 lexicographic x fastest (m = 1: the 8 corners vx+2vy+4vz) */
} dgvv_mesh;

typedef struct {
  int32_t n_levels;           /* >= 1; level 0 is the finest                              */
  const int32_t* degrees;     /* host [n_levels], e.g. {5,3,2,1}; NULL: single level       */
  double ip_factor;           /* IP in tau (default 1.0 if <= 0)                           */
  int32_t formulation;        /* DGVV_FORM_* of the viscous operator                       */
  void* nccl_comm;            /* ncclComm_t from dgvv_nccl_comm_init, or NULL (one GPU)    */
} dgvv_options;

/* Build the context: copies the mesh, computes geometry (Cartesian fast path when every
 * cell is an axis-aligned box, else iso-parametric metric terms streamed per quadrature
 * point), evaluates analytic laws at every level's quadrature points (G8) and checks
 * nu > 0.  visc_law / poisson_law may be NULL when that operator is not used.
 * Synchronous (returns after the device work on `stream` completed). */
dgvv_status dgvv_setup(const dgvv_mesh* mesh, int32_t degree, const dgvv_law* visc_law,
                       const dgvv_law* poisson_law, const dgvv_options* opt,
                       dgvv_stream stream, dgvv_ctx** out);

/* Carreau law only: nu at every cell and face quadrature point of every level from the
 * linearisation vector u_lin (fine level, vector layout);
 * face values per side from that side's own trace gradient (G8).  Coarse levels use u_lin
 * interpolated to their degree (G19).  u_lin is retained (borrowed) for
 * dgvv_apply_linearized_viscous until the next call.  Synchronous (checks nu > 0). */
dgvv_status dgvv_update_viscosity(dgvv_ctx* ctx, const double* u_lin, dgvv_stream stream);

/* dst = A_visc(nu) src on `level` (eqn:viscous_term_weak). */
dgvv_status dgvv_apply_viscous(dgvv_ctx* ctx, int32_t level, const double* src, double* dst,
                               dgvv_stream stream);

/* End-to-end variant of dgvv_apply_viscous with HOST buffers (src_host, dst_host: n_local
 * doubles, canonical layout; page-locked memory gives overlapped copies, pageable memory is
 * accepted but the copies then serialise).  The library stages them through its own device
 * vectors: on one GPU the owned cells are split into contiguous slabs; slab i is copied in on
 * a copy stream, applied on `stream` as soon as every slab holding one of its neighbours has
 * arrived, and copied out on a second copy stream, so host->device, compute and device->host
 * overlap (PCIe is full duplex).  With ghosts (multi-GPU) the whole vector is copied in, the
 * normal exchange + apply runs, and the result is copied out.  Asynchronous on `stream`: the
 * host buffers must stay valid (and src unchanged) until `stream` reaches this point. */
dgvv_status dgvv_apply_viscous_host(dgvv_ctx* ctx, int32_t level, const double* src_host,
                                    double* dst_host, dgvv_stream stream);

/* dst = J(u_lin) src = A(nu0) src + A(delta nu[src]) u_lin on level 0 (Newton derivative,
 * reading G10; delta nu = 2 eta'(gd)/gd eps(u_lin):eps(src) at every point, both sides).
 * DGVV_ESTATE before dgvv_update_viscosity; DGVV_EUNSUPPORTED for analytic laws. */
dgvv_status dgvv_apply_linearized_viscous(dgvv_ctx* ctx, const double* src, double* dst,
                                          dgvv_stream stream);

/* dst = A_P(c) src, scalar SIPG Poisson with coefficient c = poisson_law (Appendix A.2,
 * eqn:pressure_step_weak with the penalty sign of G4). */
dgvv_status dgvv_apply_poisson(dgvv_ctx* ctx, int32_t level, const double* src, double* dst,
                               dgvv_stream stream);

/* Helmholtz form of the operator: every later apply, diagonal, smoother,
 * V-cycle and CG of `op` uses  mass * M + A  with M the DG mass matrix (diagonal with the
 * collocation basis G2: M_ii = JxW_i, per component on every level) — the
 * (gamma_0 / dt) M + A(nu) operator of the viscous step.  mass = 0 (the
 * default) gives the plain operator.  DGVV_EDOMAIN for mass < 0 or non-finite. */
dgvv_status dgvv_set_mass(dgvv_ctx* ctx, int32_t op, double mass);

enum { DGVV_PRECOND_NONE = 0, DGVV_PRECOND_JACOBI = 1, DGVV_PRECOND_VCYCLE = 2, DGVV_PRECOND_VCYCLE_FP32 = 3 };

/* Divergence/continuity penalty-step operator (PAPER.md:1190-1224,
 * eqn:penalty_step), homogeneous part, on level 0:
 *   dst_e = (v, u)_e + (div v, tau_div^e div u)_e + (v.n, tau_F [[u]].n)_{boundary of e}
 * [[u]] = u(e) - u(neighbour) on interior/periodic faces (tau_F = (tau_cont^e + tau_cont^nb)/2),
 * [[u]] = u on Dirichlet faces (tau_F = tau_cont^e; the data g_u belongs to the right-hand
 * side), no term on Neumann faces.  The paper takes tau_div, tau_cont from Fehn2018b without
 * formulas: they are inputs here, one value per cell (host arrays of n_cells + n_ghost
 * entries, owned cells then ghosts in the dgvv_mesh ghost order; copied).  DGVV_EDOMAIN for
 * negative or non-finite values.
 * Multigrid for the penalty step ("a multigrid preconditioner is necessary
 * for the penalty step"): the operator is defined on every p-level of the context (the level's
 * degree and geometry, the same per-cell tau), so op = DGVV_OP_PENALTY works with
 * dgvv_inverse_diagonal, dgvv_estimate_lambda_max and dgvv_chebyshev_smooth on any level, with
 * dgvv_vcycle (p-levels of this context only: Chebyshev(5) pre/post smoothing with the
 * unfused smoother r = b - A x, d = c_rho d + c_r D^-1 r, x += d; R = P^T of the velocity
 * p-transfer; coarsest p-level Chebyshev(5) from zero; h-levels / the c-level are not used) and
 * dgvv_cg_solve with preconditioner none, Jacobi or the FP64 V-cycle (lambda_hi_per_level: one
 * value per p-level).  DGVV_ESTATE before dgvv_set_penalty_parameters.
 * dgvv_apply_penalty: level 0; dgvv_apply_penalty_level: any p-level (same semantics). */
dgvv_status dgvv_set_penalty_parameters(dgvv_ctx* ctx, const double* tau_div, const double* tau_cont);
dgvv_status dgvv_apply_penalty(dgvv_ctx* ctx, const double* src, double* dst, dgvv_stream stream);
dgvv_status dgvv_apply_penalty_level(dgvv_ctx* ctx, int32_t level, const double* src, double* dst,
                                     dgvv_stream stream);

/* Preconditioned conjugate gradients on (mass M +) A_op, level 0 (the Krylov solver of the
 * symmetric viscous and pressure steps):
 *   r = b - A x; z = P r; p = z;  repeat q = A p, alpha = (r,z)/(p,q), x += alpha p,
 *   r -= alpha q, stop when ||r|| <= rtol ||b||, z = P r, p = z + beta p.
 * x is the initial guess on entry, the solution on return.  P = identity, inverse diagonal
 * (Jacobi), one V-cycle (dgvv_vcycle) or one FP32 V-cycle (dgvv_vcycle_fp32); the V-cycles need
 * lambda_hi_per_level.  Synchronous (one host
 * read per dot product); *iters and *relres = ||r||/||b|| returned.  Work vectors are owned
 * by the library.  Multi-GPU: every rank calls collectively; dots are allreduced. */
dgvv_status dgvv_cg_solve(dgvv_ctx* ctx, int32_t op, const double* b, double* x, double rtol,
                          int32_t maxit, int32_t precond, const double* lambda_hi_per_level,
                          int32_t* iters, double* relres, dgvv_stream stream);

/* Upwind DG convective term (eqn:convective_term_weak),
 * homogeneous part on level 0, linear in u for the transport field w:
 *   c_h^e(v, u; w) = (v, (w.grad) u)_e + (v, min({{w}}.n, 0) (u(neighbour) - u(e)))_{boundary of e}
 * i.e. the central flux {{w}}.n u plus the upwind correction 1/2 |{{w}}.n| [[u]] (u^dag =
 * {{u}} + 1/2 sign({{w}}.n)[[u]]) written per cell side.  Readings F4a-F4c: the
 * (w.grad)u form; Dirichlet faces take the mirror states u+ = -u, w+ = -w (homogeneous data),
 * so {{w}}.n = 0 there; Neumann faces have no jump; both contribute nothing.
 * dgvv_set_transport copies w (device, level-0 vector layout [cell][3][n^3]; the library keeps
 * its own copy and, multi-GPU, exchanges its ghosts once; external-exchange mode: fill the
 * DGVV_GHOST_TRANSPORT buffer).  Synchronous; DGVV_EDOMAIN for non-finite entries.
 * dgvv_apply_convective: dst = C(w) src (DGVV_ESTATE before dgvv_set_transport). */
dgvv_status dgvv_set_transport(dgvv_ctx* ctx, const double* w, dgvv_stream stream);
dgvv_status dgvv_apply_convective(dgvv_ctx* ctx, const double* src, double* dst, dgvv_stream stream);

/* The viscous-step operator with linearly implicit convection (eqn:viscous_step_with_convection,
 * PAPER.md:525-554, variant ii with u* = w):  dst = (mass M + A(nu) + alpha_c C(w)) src on level 0,
 * mass from dgvv_set_mass(DGVV_OP_VISCOUS, gamma_0 / dt).  alpha_c = 0 gives the Helmholtz form. */
dgvv_status dgvv_apply_oseen(dgvv_ctx* ctx, double alpha_c, const double* src, double* dst,
                             dgvv_stream stream);

/* Right-preconditioned restarted GMRES(restart) on that non-symmetric operator (
 * Saad Alg. 9.5 with modified Gram-Schmidt):
 *   r = b - A x; V_1 = r/||r||; for j: z_j = P V_j, w = A z_j, h_ij = (w, V_i), w -= h_ij V_i,
 *   h_{j+1,j} = ||w||, Givens rotation, |g_{j+1}| = ||b - A x_j||, stop at rtol ||b||;
 *   x += Z y; restart.  P: none, Jacobi, or one (FP64 / FP32) V-cycle of the symmetric part
 *   mass M + A(nu) (the convective term is not in the preconditioner).  1 <= restart <= 200;
 *   the library owns 2 restart + 3 work vectors.  Synchronous (one host read per iteration);
 *   *iters = total inner iterations, *relres = ||b - A x|| / ||b|| (recomputed).  Multi-GPU:
 *   collective, dots allreduced. */
dgvv_status dgvv_gmres_solve(dgvv_ctx* ctx, double alpha_c, const double* b, double* x, double rtol,
                             int32_t restart, int32_t maxit, int32_t precond,
                             const double* lambda_hi_per_level, int32_t* iters, double* relres,
                             dgvv_stream stream);

/* dst = 1 / diag(A) for op = DGVV_OP_* on `level`. */
dgvv_status dgvv_inverse_diagonal(dgvv_ctx* ctx, int32_t op, int32_t level, double* dst,
                                  dgvv_stream stream);

/* x = V(b) with every multigrid level (smoother applies, Chebyshev updates, transfers,
 * coefficients, inverse diagonals) in single precision — the paper's choice for the
 * preconditioner; b and x are FP64 and converted at
 * entry and exit.  Same algorithm as dgvv_vcycle; FP32 mirrors of the level data are built on
 * first use and refreshed after dgvv_update_viscosity / dgvv_set_mass.  Multi-rank: every FP32
 * apply exchanges its ghost cells in single precision (half the bytes of the FP64 exchange),
 * overlapped with the interior cells; collective (all ranks call it).  Not with the c-level. */
dgvv_status dgvv_vcycle_fp32(dgvv_ctx* ctx, int32_t op, const double* b, double* x,
                             const double* lambda_hi_per_level, dgvv_stream stream);

/* lambda_max(D^-1 A) estimate (reading G12): `steps` Lanczos steps on D^-1/2 A D^-1/2 from
 * the caller's start vector v0 (device, level layout; random inputs are generated by the
 * caller, G20).  Synchronous; result on the host. */
dgvv_status dgvv_estimate_lambda_max(dgvv_ctx* ctx, int32_t op, int32_t level, int32_t steps,
                                     const double* v0, double* lambda_max_host,
                                     dgvv_stream stream);

/* Chebyshev-Jacobi smoother of `degree` iterations:
 * x <- x_m with bounds [lambda_lo, lambda_hi]; x_is_zero = 1 skips the first apply.
 * work: 2 level vectors (device, caller-owned scratch). */
dgvv_status dgvv_chebyshev_smooth(dgvv_ctx* ctx, int32_t op, int32_t level, double* x,
                                  const double* b, int32_t degree, double lambda_lo,
                                  double lambda_hi, int32_t x_is_zero, double* work,
                                  dgvv_stream stream);

/* fine = P coarse + beta fine, from level fine_level+1 to fine_level (G18: P = exact DG
 * embedding, per cell the tensor product of P1[i_f][j_c] = l^(kc)_j(xi^(kf)_i)). */
dgvv_status dgvv_prolongate(dgvv_ctx* ctx, int32_t op, int32_t fine_level, const double* coarse,
                            double* fine, double beta, dgvv_stream stream);

/* coarse = P^T fine + beta coarse (R = P^T). */
dgvv_status dgvv_restrict(dgvv_ctx* ctx, int32_t op, int32_t fine_level, const double* fine,
                          double* coarse, double beta, dgvv_stream stream);

/* x = V(b): one V-cycle over all levels: Chebyshev(5) from 0,
 * residual, restrict, recurse, prolongate-add, Chebyshev(5) post-smoothing; coarsest level
 * Chebyshev(5) from 0.  lambda_hi_per_level: host [n_levels]; lambda_lo = lambda_hi/20.
 * Scratch is owned by the context (allocated on first use). */
dgvv_status dgvv_vcycle(dgvv_ctx* ctx, int32_t op, const double* b, double* x,
                        const double* lambda_hi_per_level, dgvv_stream stream);

/* h-levels of the cph hierarchy (after p-coarsening,
 * "h-coarsening is performed … the individual h-levels are created by refining an initial coarse
 * grid").  `coarse` is a context on the mesh whose refinement is `fine`'s mesh (every coarse cell
 * split into 2 x 2 x 2 children); its finest degree must equal `fine`'s coarsest degree.
 * parent[f] (host, [fine n_cells]) = local id of the coarse cell containing fine cell f,
 * octant[f] = ox + 2 oy + 4 oz = which half of the parent's reference interval [0,1] the child
 * occupies along each reference axis; every coarse cell needs exactly one child per octant.
 * The transfer (reading H1) is the exact DG embedding in reference coordinates:
 * P|child = Ph[oz] (x) Ph[oy] (x) Ph[ox], Ph[o][i][j] = l_j((xi_i + o) / 2) (parent's Lagrange basis
 * at the child's Gauss points); R = P^T (H2).  After the call every V-cycle on `fine` (dgvv_vcycle,
 * the V-cycle preconditioners of dgvv_cg_solve / dgvv_gmres_solve) continues below fine's
 * coarsest p-level into `coarse`'s levels (recursively, if `coarse` has a coarse context), and
 * lambda_hi_per_level lists every level of that chain in order.  `coarse` is borrowed: keep it
 * alive while `fine` is used; its coefficients/mass are its own (set them consistently).
 * The FP32 V-cycle (dgvv_vcycle_fp32, DGVV_PRECOND_VCYCLE_FP32) follows the chain as well, with
 * the direct coarse solve in FP64 arithmetic.  Across ranks: both contexts
 * carry the communicator and the partitions are nested (every owned fine cell's parent is an owned
 * coarse cell: parent[] holds local coarse ids < coarse n_cells), so the h-transfers stay
 * rank-local and every coarse level exchanges its own ghosts (DGVV_EUNSUPPORTED if only one of the
 * two has a communicator).  The direct coarse solver and the c-level are single-rank only. */
dgvv_status dgvv_set_coarse_context(dgvv_ctx* fine, dgvv_ctx* coarse, const int32_t* parent,
                                    const int8_t* octant);
/* fine = P coarse + beta fine (fine's coarsest level <- coarse's level 0), op selects 3 or 1
 * components; coarse = P^T fine + beta coarse.  DGVV_ESTATE without a coarse context. */
dgvv_status dgvv_prolongate_h(dgvv_ctx* fine, int32_t op, const double* coarse_vec, double* fine_vec,
                              double beta, dgvv_stream stream);
dgvv_status dgvv_restrict_h(dgvv_ctx* fine, int32_t op, const double* fine_vec, double* coarse_vec,
                            double beta, dgvv_stream stream);

/* c-level of the cph hierarchy ("first the conversion from
 * a discontinuous to a continuous polynomial space is performed").  Readings C1-C3:
 * the continuous level is Q1 — one value per mesh vertex and component, vector layout [c][vertex]
 * — on the mesh of ctx's coarsest (degree-1) DG level; vertices are numbered topologically
 * (corners matched across every interior/periodic face, first appearance in (cell, corner)
 * order).  Its embedding P_c into DG_1 interpolates the trilinear corner functions at the Gauss
 * points; its operator is the Galerkin product P_c^T A_DG P_c (matrix-free: embed, DG apply,
 * transpose-gather; no atomics); the smoother diagonal is obtained by probing with a vertex
 * colouring.  With the level enabled, every V-cycle on ctx continues below its coarsest DG level
 * in the continuous space: residual restricted by P_c^T, V-cycle over the continuous levels of ctx
 * and — nested Q1 h-transfer (reading C3), CSR on the GPU — of its coarse contexts (all of which
 * need the level enabled), correction prolongated by P_c.  lambda_hi_per_level then lists ctx's DG
 * levels followed by one entry per continuous level; dgvv_estimate_lambda_max with level =
 * n_levels estimates the continuous level's; dgvv_setup_coarse_solver on the last context of the
 * chain builds the direct solve of its continuous level (<= 4096 DoFs).  FP64 only (the FP32
 * V-cycle returns DGVV_EUNSUPPORTED); single-GPU contexts only. */
dgvv_status dgvv_set_continuous_level(dgvv_ctx* ctx, int32_t enable);
dgvv_status dgvv_continuous_level_info(const dgvv_ctx* ctx, int32_t* n_vertices, int32_t* n_colors);
/* dst = P_c^T A_DG P_c src on the continuous level (op's component count). */
dgvv_status dgvv_apply_continuous(dgvv_ctx* ctx, int32_t op, const double* src, double* dst,
                                  dgvv_stream stream);
/* transpose = 0: dst (DG_1, ctx's coarsest level) = P_c src + beta dst;
 * transpose = 1: dst (continuous) = P_c^T src + beta dst. */
dgvv_status dgvv_embed_continuous(dgvv_ctx* ctx, int32_t op, int32_t transpose, const double* src,
                                  double* dst, double beta, dgvv_stream stream);

/* Direct coarse solver ("a direct solver if the system size falls below 2000
 * DoFs"; reading H3): assembles the operator of ctx's coarsest level (with its mass term) column
 * by column from the matrix-free apply, inverts it on the GPU by Gauss-Jordan elimination (SPD:
 * no pivoting; DGVV_EDOMAIN on a non-positive pivot) and from then on replaces the coarsest
 * level's Chebyshev smoothing in every V-cycle that ends on this context by x = A^-1 b (dense
 * matvec).  At most 4096 DoFs (ncomp x level DoFs).  Synchronous.  A later change of the
 * coefficients or mass makes it stale: V-cycles then fail with DGVV_ESTATE until it is set up
 * again.  *n_dofs (may be NULL) = the system size (global).  Multi-rank (communicator contexts,
 * a collective: every rank calls it): each rank assembles its owned rows of every global column
 * with the distributed apply, the columns are gathered on every rank (zero-padded sum-allreduce:
 * exact) and every rank inverts the same matrix; a solve gathers b the same way and applies the
 * rank's owned rows of the inverse.  DGVV_EUNSUPPORTED for external-exchange contexts (ghosts
 * without a communicator). */
dgvv_status dgvv_setup_coarse_solver(dgvv_ctx* ctx, int32_t op, int32_t* n_dofs);

/* out_host = sum over all ranks of a.b over `ncomp` * level-dofs entries. Synchronous. */
dgvv_status dgvv_dot(dgvv_ctx* ctx, int32_t level, int32_t ncomp, const double* a,
                     const double* b, double* out_host, dgvv_stream stream);

/* Local / global DoF counts of one component set on `level` (ncomp = 1). */
dgvv_status dgvv_sizes(const dgvv_ctx* ctx, int32_t level, int64_t* n_local_dofs,
                       int64_t* n_global_dofs);

/* Realised min/max of nu (op = VISCOUS) or c (op = POISSON) over all quadrature points of
 * `level` (host results).  Synchronous. */
dgvv_status dgvv_coefficient_range(dgvv_ctx* ctx, int32_t op, int32_t level, double* lo,
                                   double* hi);

/* Ghost cells (multi-GPU).  Each rank owns a contiguous range of global cell
 * ids; the off-rank face neighbours are its ghosts, stored in (owner rank, global id) order.
 * Per apply the library packs, for every peer, its owned cells that have a face neighbour
 * owned by that peer (ascending id) and exchanges them with grouped ncclSend/ncclRecv on an
 * internal stream while the interior cells are computed; the cells with a ghost neighbour
 * run after the exchange.  Without a communicator (external-exchange mode) the caller fills
 * the ghost buffers itself, using dgvv_pack_ghosts on the peer's context. */
enum { DGVV_GHOST_VISCOUS = 0, DGVV_GHOST_POISSON = 1, DGVV_GHOST_ULIN = 2, DGVV_GHOST_TRANSPORT = 3 };
/* Bytes one apply of `op` on `level` sends / receives in communicator mode (a5): the face traces
 * (value and reference normal derivative of every component at the n^2 points of every cut face,
 * FP64) of the owned cells next to each peer — 2 NC n^2 doubles per cut face instead of the
 * NC n^3 of a whole ghost cell.  The Newton apply (K2), the penalty and the standalone convective
 * operator still exchange whole ghost cells; the external-exchange mode (no communicator; tests)
 * fills whole ghost cells for every operator. */
dgvv_status dgvv_exchange_bytes(const dgvv_ctx* ctx, int32_t level, int32_t op, int64_t* sent,
                                int64_t* received);

/* Peers in ascending rank; arrays (may be NULL) sized by a first call that only reads n_peers. */
dgvv_status dgvv_ghost_layout(const dgvv_ctx* ctx, int32_t* n_peers, int32_t* peer_ranks,
                              int32_t* send_counts, int32_t* recv_counts);
/* sendbuf = the cells every peer needs from src, concatenated in peer order (device). */
dgvv_status dgvv_pack_ghosts(dgvv_ctx* ctx, int32_t level, int32_t kind, const double* src,
                             double* sendbuf, dgvv_stream stream);
/* Device pointer of the ghost buffer of `kind` on `level` ([n_ghost][comp][n^3], owned by the
 * library). */
dgvv_status dgvv_ghost_buffer(dgvv_ctx* ctx, int32_t level, int32_t kind, double** out);

/* NCCL plumbing (multi-GPU): 128-byte unique id on rank 0, broadcast by the caller, then a
 * communicator on every rank.  The library loads libnccl.so.2 at run time. */
dgvv_status dgvv_nccl_get_unique_id(char out_id[128]);
dgvv_status dgvv_nccl_comm_init(const char id[128], int32_t nranks, int32_t rank, void** comm);
dgvv_status dgvv_nccl_comm_destroy(void* comm);

/* In-process communicator for R ranks driven by R host threads in ONE process (one GPU is
 * enough): dgvv_thread_group_create makes the group, dgvv_thread_group_comm returns rank r's
 * communicator, to be passed as dgvv_options.nccl_comm exactly like an NCCL one.  Every
 * collective of the library (setup handshake, ghost exchange, allreduced dots) then runs as
 * device-to-device copies / a rank-ordered sum on the ranks' own streams, ordered by CUDA events
 * recorded before a host barrier: no kernel waits on another rank's kernel.  Each rank must run
 * on its own (non-legacy) stream and every rank must make the same sequence of collective calls
 * (as with NCCL).  The group owns the per-rank communicators; destroy it after the contexts. */
dgvv_status dgvv_thread_group_create(int32_t nranks, void** group);
dgvv_status dgvv_thread_group_comm(void* group, int32_t rank, void** comm);
dgvv_status dgvv_thread_group_destroy(void* group);

const char* dgvv_last_error(void);   /* thread-local message of the last failure          */
const char* dgvv_version(void);
void dgvv_destroy(dgvv_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* DGVV_H */
