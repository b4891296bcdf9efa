// aux_kernels.cuh — Carreau viscosity evaluator (K3), inverse diagonal (K5), tensor-product
// transfer (K7), vector kernels (dot, Chebyshev first step, Lanczos helpers), ghost pack.
#pragma once
#include "common.cuh"
#include "setup_kernels.cuh"

namespace dgvv {

// ============================================================ K3: Carreau viscosity
// nu = eta(gd(eps(u_lin))) at every cell point (owned cells) and, per side, at every face
// point from the cell's own trace gradient (PAPER.md:838-866 eqn:viscosity_pointwise; G8).
// NuArgs: see common.cuh

#ifndef DGVV_K3_MINB
#define DGVV_K3_MINB 0    // 0: compiler's register choice
#endif
#if DGVV_K3_MINB > 0
#define K3_BOUNDS(t) __launch_bounds__(t, DGVV_K3_MINB)
#else
#define K3_BOUNDS(t) __launch_bounds__(t)
#endif
template <int n, int GEO, int CPB>
__global__ void K3_BOUNDS(CPB * n * n) carreau_nu_kernel(const NuArgs A) {
  constexpr int n2 = n * n, n3 = n2 * n;
  constexpr int CS = 3 * n3 + 3 * n2;
  extern __shared__ double smem[];
  const Tab1D& T = c_tab[n];
  const int lc = threadIdx.x / n2;
  const int p = threadIdx.x - lc * n2;
  const int a = p % n, b = p / n;
  const int slot_raw = blockIdx.x * CPB + lc;
  const bool active = slot_raw < A.n_total;
  const int cell = active ? slot_raw : A.n_total - 1;
  double* su = smem + lc * CS;
  double* st = su + 3 * n3;
  double Da[n], Db[n];
#pragma unroll
  for (int k = 0; k < n; ++k) { Da[k] = T.D[a * DGVV_NMAX + k]; Db[k] = T.D[b * DGVV_NMAX + k]; }
  const double* g = (cell < A.n_owned) ? A.u + (size_t)cell * 3 * n3
                                       : A.ughost + (size_t)(cell - A.n_owned) * 3 * n3;
  for (int i = p; i < 3 * n3; i += n2) su[i] = g[i];
  double ih[3] = {0, 0, 0};
  if (GEO == 0) {
    const double* cg = A.cart + (size_t)cell * CART_STRIDE;
    ih[0] = cg[0]; ih[1] = cg[1]; ih[2] = cg[2];
  }
  __syncthreads();
  auto eta_of = [&](const double (&gx)[3][3], const double (&Ji)[9]) {
    double G[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        G[c][j] = (GEO == 0) ? gx[c][j] * ih[j] : gx[c][0] * Ji[j] + gx[c][1] * Ji[3 + j] + gx[c][2] * Ji[6 + j];
    double ee = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double e = 0.5 * (G[c][j] + G[j][c]);
        ee += e * e;
      }
    return carreau_eta(A.law, sqrt(2.0 * ee));
  };
  if (cell < A.n_owned) {
#pragma unroll
    for (int z = 0; z < n; ++z) {
      const int q = z * n2 + p;
      double gx[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double sx = 0, sy = 0, sz = 0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          sx += Da[k] * su[c * n3 + z * n2 + b * n + k];
          sy += Db[k] * su[c * n3 + z * n2 + k * n + a];
          sz += T.D[z * DGVV_NMAX + k] * su[c * n3 + k * n2 + p];
        }
        gx[c][0] = sx; gx[c][1] = sy; gx[c][2] = sz;
      }
      double Ji[9];
      if (GEO == 1) {
        const double* vm = A.vJi + (size_t)cell * 9 * n3 + q;
#pragma unroll
        for (int r = 0; r < 9; ++r) Ji[r] = __ldg(vm + r * n3);   // read-only path: may be hoisted above the nu stores
      }
      if (active) {
        const double e = eta_of(gx, Ji);
        A.nu_cell[(size_t)cell * n3 + q] = e;
        if (!(e > 0.0) || !isfinite(e)) atomicAdd(A.bad, 1);
      }
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int sd = (d == 0) ? 1 : (d == 1 ? n : n2);
    const int st1 = (d == 0) ? n : 1;
    const int st2 = (d == 2) ? n : n2;
    const int t1 = face_t1(d), t2 = face_t2(d);
    const int base = a * st1 + b * st2;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int f = 2 * d + s;
      const double* lS = s ? T.l1 : T.l0;
      const double* dS = s ? T.d1 : T.d0;
      double gx[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v = 0, gg = 0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const double x = su[c * n3 + base + i * sd];
          v += lS[i] * x;
          gg += dS[i] * x;
        }
        st[c * n2 + p] = v;
        gx[c][d] = gg;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double m1 = 0, m2 = 0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          m1 += Da[k] * st[c * n2 + b * n + k];
          m2 += Db[k] * st[c * n2 + k * n + a];
        }
        gx[c][t1] = m1; gx[c][t2] = m2;
      }
      double Ji[9];
      if (GEO == 1) {
        const double* fm = A.fJi + ((size_t)cell * 6 + f) * 9 * n2 + p;
#pragma unroll
        for (int r = 0; r < 9; ++r) Ji[r] = __ldg(fm + r * n2);
      }
      const double e = eta_of(gx, Ji);
      if (active) {
        A.nu_face[((size_t)cell * 6 + f) * n2 + p] = e;
        if (!(e > 0.0) || !isfinite(e)) atomicAdd(A.bad, 1);
      }
      __syncthreads();
    }
  }
}

// ============================================================ K5: inverse diagonal
// D_ii = a(phi_i e_c, phi_i e_c).  With the collocation basis grad phi_i is non-zero only on
// the three grid lines through node i (volume) and phi_i is non-zero at exactly one point of
// each face (the projection of i), so
//   D_vol  = sum_{q on lines} JxW nu (|g|^2 + [div] g_c^2),      g = grad phi_i(q)
//   D_face = dA kappa [ -2 nu phi (e_c . S(grad(phi e_c)) n) + tau phi^2 (1 + [div] n_c^2) ]
// kappa = 1 interior, 2 Dirichlet (mirror), 0 Neumann; S = sym (div) or 1/2 grad (laplace).
// DiagArgs: see common.cuh

template <int n, int NC, int FORM, int GEO>
__global__ void diag_kernel(const DiagArgs A) {
  constexpr int n2 = n * n, n3 = n2 * n;
  const Tab1D& T = c_tab[n];
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)A.n_owned * NC * n3) return;
  const int cell = idx / (NC * n3);
  const int rem = idx % (NC * n3);
  const int comp = rem / n3, i = rem % n3;
  const int iv[3] = {i % n, (i / n) % n, i / n2};
  double ih[3] = {0, 0, 0}, vol = 0, Hm;
  if (GEO == 0) {
    const double* cg = A.cart + (size_t)cell * CART_STRIDE;
    ih[0] = cg[0]; ih[1] = cg[1]; ih[2] = cg[2]; Hm = cg[3]; vol = cg[4];
  } else {
    Hm = A.Hcell[cell];
  }
  double Dv = 0.0;
  // volume: the point q = i (all three derivatives non-zero) plus the other points of the
  // three grid lines through i (one derivative non-zero each)
  auto add_point = [&](const int (&qv)[3], const double (&gxi)[3]) {
    const int q = qv[0] + n * qv[1] + n2 * qv[2];
    double g[3], w;
    if (GEO == 0) {
      for (int j = 0; j < 3; ++j) g[j] = gxi[j] * ih[j];
      w = T.w[qv[0]] * T.w[qv[1]] * T.w[qv[2]] * vol;
    } else {
      const double* vm = A.vJi + (size_t)cell * 9 * n3 + q;
      for (int j = 0; j < 3; ++j) g[j] = gxi[0] * vm[j * n3] + gxi[1] * vm[(3 + j) * n3] + gxi[2] * vm[(6 + j) * n3];
      w = 1.0;                                   // nu_cell holds nu*JxW
    }
    double gg = g[0] * g[0] + g[1] * g[1] + g[2] * g[2];
    if (FORM == 0) gg += g[comp] * g[comp];
    Dv += w * A.nu_cell[(size_t)cell * n3 + q] * gg;
  };
  {
    const double gxi[3] = {T.D[iv[0] * DGVV_NMAX + iv[0]], T.D[iv[1] * DGVV_NMAX + iv[1]],
                           T.D[iv[2] * DGVV_NMAX + iv[2]]};
    add_point(iv, gxi);
  }
  for (int line = 0; line < 3; ++line)
    for (int qq = 0; qq < n; ++qq) {
      if (qq == iv[line]) continue;
      int qv[3] = {iv[0], iv[1], iv[2]};
      qv[line] = qq;
      double gxi[3] = {0.0, 0.0, 0.0};
      gxi[line] = T.D[qq * DGVV_NMAX + iv[line]];
      add_point(qv, gxi);
    }
  // faces
  for (int f = 0; f < 6; ++f) {
    const int d = f / 2, s = f % 2;
    const int nb = A.nbr[cell * 6 + f];
    if (nb == NB_NEUMANN) continue;
    const double kappa = (nb == NB_DIRICHLET) ? 2.0 : 1.0;
    const int t1 = face_t1(d), t2 = face_t2(d);
    const int pa = iv[t1], pb = iv[t2];
    const int pidx = pa + n * pb;
    const double phi = s ? T.l1[iv[d]] : T.l0[iv[d]];
    double gxi[3];
    gxi[d] = s ? T.d1[iv[d]] : T.d0[iv[d]];
    gxi[t1] = phi * T.D[pa * DGVV_NMAX + pa];
    gxi[t2] = phi * T.D[pb * DGVV_NMAX + pb];
    double g[3], nrm[3] = {0, 0, 0}, dA;
    if (GEO == 0) {
      for (int j = 0; j < 3; ++j) g[j] = gxi[j] * ih[j];
      nrm[d] = s ? 1.0 : -1.0;
      dA = T.w[pa] * T.w[pb] * vol * ih[d];
    } else {                                     // nu_face holds nu*dA: dA folded in below
      const double* fm = A.fJi + ((size_t)cell * 6 + f) * 9 * n2 + pidx;
      for (int j = 0; j < 3; ++j) g[j] = gxi[0] * fm[j * n2] + gxi[1] * fm[(3 + j) * n2] + gxi[2] * fm[(6 + j) * n2];
      const double sg = s ? 1.0 : -1.0;
      const double v0 = fm[(3 * d) * n2], v1 = fm[(3 * d + 1) * n2], v2 = fm[(3 * d + 2) * n2];
      const double il = sg / sqrt(v0 * v0 + v1 * v1 + v2 * v2);
      nrm[0] = v0 * il; nrm[1] = v1 * il; nrm[2] = v2 * il;
      dA = 1.0;
    }
    const double num = A.nu_face[((size_t)cell * 6 + f) * n2 + pidx];
    double nup = num, Hp = Hm;
    if (nb >= 0) {
      nup = A.nu_face[((size_t)nb * 6 + (f ^ 1)) * n2 + pidx];
      Hp = (GEO == 0) ? A.cart[(size_t)nb * CART_STRIDE + 3] : A.Hcell[nb];
    }
    const double tau = A.pen * fmax(Hm, Hp) * 0.5 * (num + nup);
    const double gn = g[0] * nrm[0] + g[1] * nrm[1] + g[2] * nrm[2];
    const double eSn = (FORM == 0) ? 0.5 * (gn + g[comp] * nrm[comp]) : 0.5 * gn;
    const double pn = (FORM == 0) ? (1.0 + nrm[comp] * nrm[comp]) : 1.0;
    Dv += dA * kappa * (-2.0 * num * phi * eSn + tau * phi * phi * pn);
  }
  if (A.mass != 0.0)                               // Helmholtz: + mass * JxW_i
    Dv += A.mass * ((GEO == 0) ? T.w[iv[0]] * T.w[iv[1]] * T.w[iv[2]] * vol : A.jxw[(size_t)cell * n3 + i]);
  A.out[idx] = 1.0 / Dv;
}

// ============================================================ K7: tensor-product transfer
// out[cell][c] = (M (x) M (x) M) in[cell][c] + beta add[cell][c];  M is nout x nin; add is out
// (in place) or another vector (the V-cycle's out-of-place prolongation-add).
// prolongation: M = P1 (nf x nc); restriction: M = P1^T; u_lin interpolation: M = I1.
struct Mat8 { double m[DGVV_NMAX * DGVV_NMAX]; };

// One team of TS = max(nin, nout)^2 threads per cell, CPB cells per CTA.  HBM-bound (§8(d): read
// nin^3, write nout^3 [+ read nout^3 of add] per component), so the kernel is organised around the
// memory system: thread (x, y) reads its z-column with nin independent coalesced loads and
// contracts it in registers (z first, coefficients as immediate constant-bank operands); the y
// and x contractions go through two small shared arrays with the thread's row of M in registers;
// the output planes are written coalesced.  Two barriers per component.
template <int nin, int nout>
struct T3Cfg {
  static constexpr int NMAXIO = nin > nout ? nin : nout;
  static constexpr int TS = NMAXIO * NMAXIO;
  static constexpr int S1 = nout * nin * nin, S2 = nout * nout * nin;
  static constexpr int CS = S1 + S2;
  static constexpr int CPB = (256 / TS) < 1 ? 1 : ((256 / TS) > 16 ? 16 : (256 / TS));
};

template <typename R, int nin, int nout, int NC, int CPB>
__global__ void __launch_bounds__(CPB * T3Cfg<nin, nout>::TS) tensor3_kernel(Mat8 M, const R* in, R* out, const R* add, R beta, int n_cells) {
  using Cf = T3Cfg<nin, nout>;
  constexpr int ni2 = nin * nin, ni3 = ni2 * nin, no2 = nout * nout, no3 = no2 * nout, nio = nin * nout;
  constexpr int TS = Cf::TS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* smem = reinterpret_cast<R*>(smem_raw);
  const int lc = threadIdx.x / TS, t = threadIdx.x - lc * TS;
  const int cell = blockIdx.x * CPB + lc;
  const bool active = cell < n_cells;
  R* s1 = smem + lc * Cf::CS;      // [z_o][y_i][x_i]
  R* s2 = s1 + Cf::S1;             // [z_o][y_o][x_i]
  R my[nin], mx[nin];              // this thread's rows of M for the y (t < nin nout) and x (t < nout^2) steps
#pragma unroll
  for (int k = 0; k < nin; ++k) {
    my[k] = (t < nio) ? R(M.m[(t / nin) * nin + k]) : R(0);
    mx[k] = (t < no2) ? R(M.m[(t % nout) * nin + k]) : R(0);
  }
  for (int c = 0; c < NC; ++c) {
    if (t < ni2) {
      R col[nin];
      const R* g = in + ((size_t)(active ? cell : 0) * NC + c) * ni3 + t;
#pragma unroll
      for (int k = 0; k < nin; ++k) col[k] = g[k * ni2];
#pragma unroll
      for (int zo = 0; zo < nout; ++zo) {
        R acc = R(0);
#pragma unroll
        for (int k = 0; k < nin; ++k) acc += R(M.m[zo * nin + k]) * col[k];
        s1[zo * ni2 + t] = acc;
      }
    }
    __syncthreads();
    if (t < nio) {
      const int xi = t % nin;
#pragma unroll
      for (int zo = 0; zo < nout; ++zo) {
        R acc = R(0);
#pragma unroll
        for (int k = 0; k < nin; ++k) acc += my[k] * s1[(zo * nin + k) * nin + xi];
        s2[zo * nio + t] = acc;
      }
    }
    __syncthreads();
    if (t < no2 && active) {
      const int yo = t / nout;
      const size_t o = ((size_t)cell * NC + c) * no3 + t;
      R av[nout];
      if (beta != R(0)) {
#pragma unroll
        for (int zo = 0; zo < nout; ++zo) av[zo] = add[o + zo * no2];
      }
#pragma unroll
      for (int zo = 0; zo < nout; ++zo) {
        R acc = R(0);
#pragma unroll
        for (int k = 0; k < nin; ++k) acc += mx[k] * s2[(zo * nout + yo) * nin + k];
        out[o + zo * no2] = (beta == R(0)) ? acc : acc + beta * av[zo];
      }
    }
  }
}

// ============================================================ vector kernels
// deterministic two-pass dot product
__global__ void dot_partial_kernel(const double* a, const double* b, long n, double* part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    acc += a[i] * b[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void sum_partials_kernel(const double* part, int np, double* out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// Chebyshev iteration 0 from x0 = 0: r0 = b, d0 = D^-1 b / theta, x1 = d0
template <typename R>
__global__ void cheb_first_kernel(const R* b, const R* dinv, R c_r, R* d, R* x, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const R v = c_r * dinv[i] * b[i];
    d[i] = v;
    x[i] = v;
  }
}
// precision conversions for the FP32 multigrid preconditioner
__global__ void d2f_kernel(const double* a, float* out, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = (float)a[i];
}
__global__ void f2d_kernel(const float* a, double* out, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = (double)a[i];
}

// out = a .* b
__global__ void ew_mul_kernel(const double* a, const double* b, double* out, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}
// y = alpha x + beta y  (CG updates)
__global__ void axpby_kernel(double alpha, const double* x, double beta, double* y, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    y[i] = beta == 0.0 ? alpha * x[i] : alpha * x[i] + beta * y[i];   // beta = 0: y is not read (BLAS)
}
// out = sqrt(a)
__global__ void ew_sqrt_kernel(const double* a, double* out, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = sqrt(a[i]);
}
// out = a ./ b
__global__ void ew_div_kernel(const double* a, const double* b, double* out, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = a[i] / b[i];
}
// y = alpha x + beta y + gamma z   (alpha/beta/gamma from device scalars when given)
__global__ void lanczos_update_kernel(double* w, const double* q, const double* qprev,
                                      const double* alpha, const double* beta_prev, long n) {
  const double al = *alpha, be = *beta_prev;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    w[i] = w[i] - al * q[i] - be * qprev[i];
}
// y += sgn * coef[0] * x (coefficient read on the device: GMRES Gram-Schmidt without a host sync)
__global__ void axpy_dev_kernel(const double* coef, double sgn, const double* x, double* y, long n) {
  const double a = sgn * *coef;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}
// q_new = w / s (s = device scalar norm)
__global__ void scale_by_inv_kernel(const double* w, const double* s2, double* q, long n) {
  const double inv = 1.0 / sqrt(*s2);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    q[i] = w[i] * inv;
}

// gather cells (ghost exchange pack): out[k] = src[list[k]] (blocks of len doubles)
template <typename R>
__global__ void gather_cells_kernel(const R* src, const int* list, int ncells, int len, R* out) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)ncells * len) return;
  const int k = i / len, r = i % len;
  out[i] = src[(size_t)list[k] * len + r];
}

}  // namespace dgvv
