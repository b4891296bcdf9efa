// sipg_apply.cuh — the hot kernel: matrix-free, sum-factorised SIPG operator apply
// (vector viscous operator, PAPER.md:1055-1111 eqn:viscous_term_weak; scalar Poisson,
// PAPER.md:713-758 eqn:pressure_step_weak) with fused epilogues (plain apply, residual
// b - A x, Chebyshev-Jacobi update of SURVEY §8(c) c1.6).
//
// Design: cell-centric.  A CTA holds CPB cells; each cell is a team of
// n^2 threads.  Thread (a,b) owns the z-column (x=a, y=b): its values and its output
// entries live in registers for the whole kernel.  With the Gauss-collocation basis (G1/G2)
// values at quadrature points are the coefficients, so the volume needs only derivative
// contractions: d/dxi_z in registers along the column, d/dxi_x, d/dxi_y from the cell's
// shared-memory copy.  Faces are processed in opposite pairs (-d,+d) from this cell's side
// only (own test functions); the neighbour's normal lines are read from L2/global.  The z
// faces run entirely on the column registers; x/y face contributions go through a shared
// accumulator that each column owner folds in at the end.  No atomics: every dst entry is
// written once by its owner (deterministic; a multi-GPU run is bitwise equal to one GPU).
// Cartesian cells (n = +-e_d, diagonal J^-1) only need the tangential derivatives of the
// normal velocity component (divergence form) and none for the Laplace/Poisson form.
// Dirichlet faces use the mirror state (G7); Neumann faces are skipped.
#pragma once
#include "common.cuh"

namespace dgvv {

// Flux coefficients at one face point from the own side ("-"), general geometry.
// Gm/Gp: physical gradients G[c][j] = d u_c / d x_j; um/up values; wm/wp = nu-*dA, nu+*dA;
// returns fv[c] (coefficient of v_c) and gk[c][k] (coefficient of d v_c / d xi_k).
template <int NC, int FORM>
__device__ __forceinline__ void face_flux_gen(const double (&um)[NC], const double (&up)[NC],
                                              const double (&Gm)[NC][3], const double (&Gp)[NC][3],
                                              const double* nrm, double wm, double wp, double tau,
                                              const double (&Jim)[9], double (&fv)[NC], double (&gk)[NC][3]) {
  static_assert(FORM == 1 || NC == 3, "divergence form needs 3 components");
  double jmp[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) jmp[c] = um[c] - up[c];
  double jn = 0.0;
  if constexpr (FORM == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) jn += jmp[c] * nrm[c];
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double sm, sp;
      if constexpr (FORM == 0) {
        sm = 0.5 * (Gm[c][j] + Gm[j][c]);
        sp = 0.5 * (Gp[c][j] + Gp[j][c]);
      } else {
        sm = 0.5 * Gm[c][j];
        sp = 0.5 * Gp[c][j];
      }
      acc += (wm * sm + wp * sp) * nrm[j];
    }
    const double pv = (FORM == 0) ? (jmp[c] + nrm[c] * jn) : jmp[c];
    fv[c] = -acc + tau * pv;
    double Gc[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if constexpr (FORM == 0) Gc[j] = -wm * 0.5 * (jmp[c] * nrm[j] + jmp[j] * nrm[c]);
      else Gc[j] = -wm * 0.5 * jmp[c] * nrm[j];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) gk[c][k] = Gc[0] * Jim[3 * k] + Gc[1] * Jim[3 * k + 1] + Gc[2] * Jim[3 * k + 2];
  }
}

template <int n, int NC, int FORM, int GEO>
struct ApplyCfg {
  static constexpr int n2 = n * n, n3 = n * n * n;
  // components whose tangential derivatives enter the face terms
  static constexpr int NT = (GEO == 1) ? NC : (FORM == 0 ? 1 : 0);
  static constexpr int FB = 8 * NT * n2;                    // face buffers of one face pair
  static constexpr int WV = 2 * NC * n3;                    // volume fluxes F_x, F_y
  static constexpr int WF = NC * n3 + FB;                   // x/y face accumulator + face buffers
  static constexpr int WS = WV > WF ? WV : WF;
  static constexpr int CS = NC * n3 + WS;                   // doubles of smem per cell
};

template <int n, int NC, int FORM, int GEO, int CPB, int MINB>
__global__ void __launch_bounds__(CPB * n * n, MINB)
sipg_apply_kernel(const ApplyArgs A) {
  static_assert(FORM == 1 || NC == 3, "divergence form needs 3 components");
  using Cf = ApplyCfg<n, NC, FORM, GEO>;
  constexpr int n2 = Cf::n2, n3 = Cf::n3, NT = Cf::NT;
  constexpr int NTa = NT > 0 ? NT : 1;
  extern __shared__ double smem[];
  const Tab1D& T = c_tab[n];

  const int lc = threadIdx.x / n2;
  const int p = threadIdx.x - lc * n2;
  const int a = p % n, b = p / n;
  const int slot_raw = blockIdx.x * CPB + lc;
  const bool active = slot_raw < A.n_proc;
  const int slot = active ? slot_raw : (A.n_proc - 1);
  const int cell = A.cell_list ? A.cell_list[slot] : A.cell_base + slot;

  double* su = smem + lc * Cf::CS;      // own cell values [NC][n3]
  double* W = su + NC * n3;             // work region
  double* Y = W;                        // face phase: x/y accumulator [NC][n3]
  double* st = W + NC * n3;             // face phase: traces [2 faces][2 sides][NT][n2]
  double* sg = st + 4 * NT * n2;        // face phase: tangential coefficients [2 faces][2][NT][n2]

  double Da[n], Db[n], DTa[n], DTb[n];
#pragma unroll
  for (int k = 0; k < n; ++k) {
    Da[k] = T.D[a * DGVV_NMAX + k];
    Db[k] = T.D[b * DGVV_NMAX + k];
    DTa[k] = T.D[k * DGVV_NMAX + a];
    DTb[k] = T.D[k * DGVV_NMAX + b];
  }

  const double* gsrc = A.src + (size_t)cell * NC * n3;
#pragma unroll
  for (int i = p; i < NC * n3; i += n2) su[i] = __ldg(gsrc + i);

  double ih[3] = {0, 0, 0}, vol = 0.0, Hm;
  if constexpr (GEO == 0) {
    const double* cg = A.cart + (size_t)cell * CART_STRIDE;
    ih[0] = cg[0]; ih[1] = cg[1]; ih[2] = cg[2]; Hm = cg[3]; vol = cg[4];
  } else {
    Hm = A.Hcell[cell];
  }
  __syncthreads();

  double ucol[NC][n], y[NC][n];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int z = 0; z < n; ++z) { ucol[c][z] = su[c * n3 + z * n2 + p]; y[c][z] = 0.0; }

  // =============================================================== volume term
  {
    const double wab = T.w[a] * T.w[b];
#pragma unroll
    for (int z = 0; z < n; ++z) {
      const int q = z * n2 + p;
      double gxi[NC][3];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          sx += Da[k] * su[c * n3 + z * n2 + b * n + k];
          sy += Db[k] * su[c * n3 + z * n2 + k * n + a];
          sz += T.D[z * DGVV_NMAX + k] * ucol[c][k];
        }
        gxi[c][0] = sx; gxi[c][1] = sy; gxi[c][2] = sz;
      }
      double Ji[9], w;
      if constexpr (GEO == 0) {
        w = A.nu_cell[(size_t)cell * n3 + q] * wab * T.w[z] * vol;
      } else {
        const double* vm = A.vJi + (size_t)cell * 9 * n3 + q;
#pragma unroll
        for (int r = 0; r < 9; ++r) Ji[r] = __ldg(vm + r * n3);
        w = A.nu_cell[(size_t)cell * n3 + q];                  // nu * JxW
      }
      double G[NC][3];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          if constexpr (GEO == 0) G[c][j] = gxi[c][j] * ih[j];
          else G[c][j] = gxi[c][0] * Ji[j] + gxi[c][1] * Ji[3 + j] + gxi[c][2] * Ji[6 + j];
        }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double Tc[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          if constexpr (FORM == 0) Tc[j] = w * (G[c][j] + G[j][c]);
          else Tc[j] = w * G[c][j];
        }
        double F[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          if constexpr (GEO == 0) F[k] = Tc[k] * ih[k];
          else F[k] = Tc[0] * Ji[3 * k] + Tc[1] * Ji[3 * k + 1] + Tc[2] * Ji[3 * k + 2];
        }
        W[c * n3 + q] = F[0];
        W[(NC + c) * n3 + q] = F[1];
#pragma unroll
        for (int z2 = 0; z2 < n; ++z2) y[c][z2] += T.D[z * DGVV_NMAX + z2] * F[2];
      }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          acc += DTa[k] * W[c * n3 + z * n2 + b * n + k];
          acc += DTb[k] * W[(NC + c) * n3 + z * n2 + k * n + a];
        }
        y[c][z] += acc;
      }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) Y[c * n3 + z * n2 + p] = 0.0;
  }

  // =============================================================== face terms
  // order z, x, y: the z pair works on the column registers (and its barrier orders the Y
  // zeroing before the first x-face update)
#pragma unroll
  for (int dd = 0; dd < 3; ++dd) {
    const int d = (dd == 0) ? 2 : dd - 1;
    const int sd = (d == 0) ? 1 : (d == 1 ? n : n2);
    const int st1 = (d == 0) ? n : 1;
    const int st2 = (d == 2) ? n : n2;
    const int t1 = face_t1(d), t2 = face_t2(d);
    const int base = a * st1 + b * st2;

    int nbv[2];
    bool act[2], inter[2];
    double um[2][NC], up[2][NC], dm[2][NC], dp[2][NC];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      nbv[s] = A.nbr[cell * 6 + 2 * d + s];
      inter[s] = nbv[s] >= 0;
      act[s] = inter[s] || (nbv[s] == NB_DIRICHLET);
    }
    // own traces (both faces from one pass over the normal line)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double v0 = 0.0, g0 = 0.0, v1 = 0.0, g1 = 0.0;
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const double x = (d == 2) ? ucol[c][i] : su[c * n3 + base + i * sd];
        v0 += T.l0[i] * x; g0 += T.d0[i] * x;
        v1 += T.l1[i] * x; g1 += T.d1[i] * x;
      }
      um[0][c] = v0; dm[0][c] = g0; um[1][c] = v1; dm[1][c] = g1;
    }
    // neighbour traces
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double* lO = s ? T.l0 : T.l1;
      const double* dO = s ? T.d0 : T.d1;
      if (inter[s]) {
        const int nb = nbv[s];
        const double* pn = (nb < A.n_owned) ? A.src + (size_t)nb * NC * n3
                                            : A.ghost + (size_t)(nb - A.n_owned) * NC * n3;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          double v = 0.0, g = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) {
            const double x = __ldg(pn + c * n3 + base + i * sd);
            v += lO[i] * x;
            g += dO[i] * x;
          }
          up[s][c] = v; dp[s][c] = g;
        }
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) { up[s][c] = -um[s][c]; dp[s][c] = dm[s][c]; }
      }
    }
    if constexpr (NT > 0) {
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int c = (GEO == 1) ? t : d;
          st[((s * 2 + 0) * NT + t) * n2 + p] = um[s][c];
          st[((s * 2 + 1) * NT + t) * n2 + p] = up[s][c];
        }
      __syncthreads();
    }

    double fv[2][NC], gn[2][NC], gt1[2][NTa], gt2[2][NTa];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int f = 2 * d + s;
      const double sgn = s ? 1.0 : -1.0;
      // tangential reference derivatives of the traces (NT components)
      double tm1[NTa], tm2[NTa], tp1[NTa], tp2[NTa];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        double m1 = 0.0, m2 = 0.0, p1 = 0.0, p2 = 0.0;
        const double* sm_ = st + ((s * 2 + 0) * NT + t) * n2;
        const double* sp_ = st + ((s * 2 + 1) * NT + t) * n2;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          m1 += Da[k] * sm_[b * n + k];
          m2 += Db[k] * sm_[k * n + a];
          p1 += Da[k] * sp_[b * n + k];
          p2 += Db[k] * sp_[k * n + a];
        }
        tm1[t] = m1; tm2[t] = m2;
        if (inter[s]) { tp1[t] = p1; tp2[t] = p2; } else { tp1[t] = m1; tp2[t] = m2; }
      }
      if constexpr (GEO == 0) {
        // ---------------- Cartesian: n = sgn e_d, J^-1 = diag(1/h)
        const double num = A.nu_face[((size_t)cell * 6 + f) * n2 + p];
        double nup = num, Hp = Hm;
        double ihp[3] = {ih[0], ih[1], ih[2]};
        if (inter[s]) {
          const double* cg = A.cart + (size_t)nbv[s] * CART_STRIDE;
          ihp[0] = cg[0]; ihp[1] = cg[1]; ihp[2] = cg[2]; Hp = cg[3];
          nup = A.nu_face[((size_t)nbv[s] * 6 + (f ^ 1)) * n2 + p];
        }
        const double dA = T.w[a] * T.w[b] * vol * ih[d];
        const double tau = A.pen * fmax(Hm, Hp) * 0.5 * (num + nup);
        double Sm[NC], Sp[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double gnm = dm[s][c] * ih[d], gnp = dp[s][c] * ihp[d];
          if constexpr (FORM == 0) {
            if (c == d) { Sm[c] = gnm; Sp[c] = gnp; }
            else {
              const bool c_is_t1 = (c == t1);
              const double gtm = (c_is_t1 ? tm1[0] : tm2[0]) * ih[c];
              const double gtp = (c_is_t1 ? tp1[0] : tp2[0]) * ihp[c];
              Sm[c] = 0.5 * (gnm + gtm);
              Sp[c] = 0.5 * (gnp + gtp);
            }
          } else {
            Sm[c] = 0.5 * gnm;
            Sp[c] = 0.5 * gnp;
          }
        }
        double jmp[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) jmp[c] = um[s][c] - up[s][c];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double sbn = sgn * (num * Sm[c] + nup * Sp[c]);
          const double pv = (FORM == 0 && c == d) ? 2.0 * jmp[c] : jmp[c];
          fv[s][c] = dA * (-sbn + tau * pv);
          const double Gcd = (FORM == 0 && c == d) ? -num * jmp[c] * sgn : -0.5 * num * jmp[c] * sgn;
          gn[s][c] = dA * Gcd * ih[d];
        }
        if constexpr (NT > 0) {
          gt1[s][0] = dA * (-0.5 * num * jmp[t1] * sgn) * ih[t1];
          gt2[s][0] = dA * (-0.5 * num * jmp[t2] * sgn) * ih[t2];
        }
      } else {
        // ---------------- general geometry: own / neighbour J^-1 at the face point
        const double* fm = A.fJi + ((size_t)cell * 6 + f) * 9 * n2 + p;
        double Jim[9], Jip[9];
#pragma unroll
        for (int r = 0; r < 9; ++r) Jim[r] = __ldg(fm + r * n2);
        const double wm = A.nu_face[((size_t)cell * 6 + f) * n2 + p];      // nu * dA
        double wp = wm, Hp = Hm;
        if (inter[s]) {
          const double* fp = A.fJi + ((size_t)nbv[s] * 6 + (f ^ 1)) * 9 * n2 + p;
#pragma unroll
          for (int r = 0; r < 9; ++r) Jip[r] = __ldg(fp + r * n2);
          wp = A.nu_face[((size_t)nbv[s] * 6 + (f ^ 1)) * n2 + p];
          Hp = A.Hcell[nbv[s]];
        } else {
#pragma unroll
          for (int r = 0; r < 9; ++r) Jip[r] = Jim[r];
        }
        double nrm[3];
        {
          const double v0 = Jim[3 * d], v1 = Jim[3 * d + 1], v2 = Jim[3 * d + 2];
          const double il = sgn / sqrt(v0 * v0 + v1 * v1 + v2 * v2);
          nrm[0] = v0 * il; nrm[1] = v1 * il; nrm[2] = v2 * il;
        }
        double gxm[NC][3], gxp[NC][3];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          gxm[c][d] = dm[s][c]; gxm[c][t1] = tm1[c]; gxm[c][t2] = tm2[c];
          gxp[c][d] = dp[s][c]; gxp[c][t1] = tp1[c]; gxp[c][t2] = tp2[c];
        }
        double Gm[NC][3], Gp[NC][3];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            Gm[c][j] = gxm[c][0] * Jim[j] + gxm[c][1] * Jim[3 + j] + gxm[c][2] * Jim[6 + j];
            Gp[c][j] = gxp[c][0] * Jip[j] + gxp[c][1] * Jip[3 + j] + gxp[c][2] * Jip[6 + j];
          }
        const double tau = A.pen * fmax(Hm, Hp) * 0.5 * (wm + wp);
        double um_[NC], up_[NC], fv_[NC], gk[NC][3];
#pragma unroll
        for (int c = 0; c < NC; ++c) { um_[c] = um[s][c]; up_[c] = up[s][c]; }
        face_flux_gen<NC, FORM>(um_, up_, Gm, Gp, nrm, wm, wp, tau, Jim, fv_, gk);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          fv[s][c] = fv_[c];
          gn[s][c] = gk[c][d];
          if constexpr (NT > 0) { gt1[s][c] = gk[c][t1]; gt2[s][c] = gk[c][t2]; }
        }
      }
      if (!act[s]) {
#pragma unroll
        for (int c = 0; c < NC; ++c) { fv[s][c] = 0.0; gn[s][c] = 0.0; }
#pragma unroll
        for (int t = 0; t < NTa; ++t) { gt1[s][t] = 0.0; gt2[s][t] = 0.0; }
      }
      if constexpr (NT > 0) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          sg[((s * 2 + 0) * NT + t) * n2 + p] = gt1[s][t];
          sg[((s * 2 + 1) * NT + t) * n2 + p] = gt2[s][t];
        }
      }
    }
    if constexpr (NT > 0) __syncthreads();

    // value coefficient at this face node = fv + transposed tangential contributions
    double val[2][NC];
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int c = 0; c < NC; ++c) val[s][c] = fv[s][c];
    if constexpr (NT > 0) {
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int c = (GEO == 1) ? t : d;
          double acc = 0.0;
          const double* g1 = sg + ((s * 2 + 0) * NT + t) * n2;
          const double* g2 = sg + ((s * 2 + 1) * NT + t) * n2;
#pragma unroll
          for (int k = 0; k < n; ++k) acc += DTa[k] * g1[b * n + k] + DTb[k] * g2[k * n + a];
          val[s][c] += acc;
        }
    }
    // extrapolate both faces' coefficients along the normal line into the cell
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const double add = T.l0[i] * val[0][c] + T.d0[i] * gn[0][c] + T.l1[i] * val[1][c] + T.d1[i] * gn[1][c];
        if (d == 2) y[c][i] += add;
        else Y[c * n3 + base + i * sd] += add;
      }
    __syncthreads();
  }

  // =============================================================== epilogue
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int z = 0; z < n; ++z) y[c][z] += Y[c * n3 + z * n2 + p];
  if (active) {
    const size_t off = (size_t)cell * NC * n3;
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) {
        const size_t i = off + c * n3 + z * n2 + p;
        if (A.mode == MODE_APPLY) {
          A.dst[i] = y[c][z];
        } else if (A.mode == MODE_RESID) {
          A.dst[i] = __ldg(A.b + i) - y[c][z];
        } else {
          const double r = __ldg(A.b + i) - y[c][z];
          double dn = A.c_r * __ldg(A.dinv + i) * r;
          if (A.c_rho != 0.0) dn += A.c_rho * A.dvec[i];
          A.dvec[i] = dn;
          A.xout[i] = ucol[c][z] + dn;
        }
      }
  }
}

}  // namespace dgvv
