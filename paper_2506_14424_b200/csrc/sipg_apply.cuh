// sipg_apply.cuh — the hot kernel: matrix-free, sum-factorised SIPG operator apply
// (vector viscous operator, PAPER.md:1055-1111 eqn:viscous_term_weak; scalar Poisson,
// PAPER.md:713-758 eqn:pressure_step_weak) with fused epilogues (plain apply, residual
// b - A x, Chebyshev-Jacobi update of SURVEY §8(c) c1.6).
//
// Design: cell-centric.  A CTA holds CPB cells; each cell is a team of
// n^2 threads.  Thread (a,b) owns the z-column (x=a, y=b) in the volume phase and the face
// point (a,b) in the face phases.  With the Gauss-collocation basis (G1/G2) values at
// quadrature points are the coefficients, so the volume needs only derivative contractions:
// d/dxi_z in registers along the column, d/dxi_x, d/dxi_y from the cell's shared-memory
// copy.  Each of the 6 faces is evaluated from this cell's side only (own test functions),
// reading the neighbour's normal lines from L2/global: no atomics, every dst entry is
// written once by its owner (deterministic, and a multi-GPU run is bitwise equal to one
// GPU).  Dirichlet faces use the mirror state (G7), Neumann faces are skipped.
#pragma once
#include "common.cuh"

namespace dgvv {

template <int n>
struct Lines {
  static constexpr int n2 = n * n, n3 = n * n * n;
};

// Accumulate the flux coefficients at one face point from the own side ("-").
// gm/gp: physical gradients G[c][j] = d u_c / d x_j; um/up values; returns
// fv[c] (coefficient of v_c) and gk[c][k] (coefficient of d v_c / d xi_k), both times dA.
template <int NC, int FORM>
__device__ __forceinline__ void face_flux_impl(const double (&um)[NC], const double (&up)[NC],
                                          const double (&Gm)[NC][3], const double (&Gp)[NC][3],
                                          const double* nrm, double num, double nup, double tau,
                                          double dA, const double (&Jim)[9], double (&fv)[NC],
                                          double (&gk)[NC][3]) {
  static_assert(FORM == 1 || NC == 3, "divergence form needs 3 components");
  double jmp[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) jmp[c] = um[c] - up[c];
  double sbn[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double sm, sp;
      if constexpr (FORM == 0) {   // divergence: S = sym(G)
        sm = 0.5 * (Gm[c][j] + Gm[j][c]);
        sp = 0.5 * (Gp[c][j] + Gp[j][c]);
      } else {                     // laplace: S = G/2
        sm = 0.5 * Gm[c][j];
        sp = 0.5 * Gp[c][j];
      }
      acc += (num * sm + nup * sp) * nrm[j];
    }
    sbn[c] = acc;
  }
  double jn = 0.0;
  if (FORM == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) jn += jmp[c] * nrm[c];
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double pv = (FORM == 0) ? (jmp[c] + nrm[c] * jn) : jmp[c];
    fv[c] = dA * (-sbn[c] + tau * pv);
  }
  // gradient coefficient Gc[c][j] then to reference directions with own J^-1
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double Gc[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if constexpr (FORM == 0)
        Gc[j] = -num * 0.5 * (jmp[c] * nrm[j] + jmp[j] * nrm[c]);
      else
        Gc[j] = -num * 0.5 * jmp[c] * nrm[j];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
      gk[c][k] = dA * (Gc[0] * Jim[3 * k + 0] + Gc[1] * Jim[3 * k + 1] + Gc[2] * Jim[3 * k + 2]);
  }
}

// GEO: 0 = Cartesian (per-cell diagonal J^-1), 1 = general (streamed metric terms)
template <int n, int NC, int FORM, int GEO, int CPB>
__global__ void __launch_bounds__(CPB * n * n)
sipg_apply_kernel(const ApplyArgs A) {
  static_assert(FORM == 1 || NC == 3, "divergence form needs 3 components");
  constexpr int n2 = n * n, n3 = n * n * n;
  constexpr int CS = 4 * NC * n3;                 // doubles of smem per cell
  extern __shared__ double smem[];
  const Tab1D& T = c_tab[n];

  const int lc = threadIdx.x / n2;
  const int p = threadIdx.x - lc * n2;
  const int a = p % n, b = p / n;
  const int slot_raw = blockIdx.x * CPB + lc;
  const bool active = slot_raw < A.n_proc;
  const int slot = active ? slot_raw : (A.n_proc - 1);
  const int cell = A.cell_list ? A.cell_list[slot] : slot;

  double* su = smem + lc * CS;          // own cell values   [NC][n3]
  double* sy = su + NC * n3;            // output accumulator [NC][n3]
  double* sF = sy + NC * n3;            // volume fluxes x,y  [2][NC][n3] ; face buffers

  // per-thread rows/columns of the derivative matrix (thread-dependent -> registers)
  double Da[n], Db[n], DTa[n], DTb[n];
#pragma unroll
  for (int k = 0; k < n; ++k) {
    Da[k] = T.D[a * DGVV_NMAX + k];
    Db[k] = T.D[b * DGVV_NMAX + k];
    DTa[k] = T.D[k * DGVV_NMAX + a];
    DTb[k] = T.D[k * DGVV_NMAX + b];
  }

  // ---- stage own cell (coalesced: n^2 threads stride over NC n^3 contiguous doubles)
  const double* gsrc = A.src + (size_t)cell * NC * n3;
#pragma unroll
  for (int i = p; i < NC * n3; i += n2) su[i] = __ldg(gsrc + i);
  __syncthreads();

  // ---- geometry scalars of this cell
  double ih[3] = {0, 0, 0}, vol = 0.0, Hm = 0.0;
  if (GEO == 0) {
    const double* cg = A.cart + (size_t)cell * CART_STRIDE;
    ih[0] = cg[0]; ih[1] = cg[1]; ih[2] = cg[2]; Hm = cg[3]; vol = cg[4];
  } else {
    Hm = A.Hcell[cell];
  }

  // =============================================================== volume term
  {
    double ucol[NC][n];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) ucol[c][z] = su[c * n3 + z * n2 + p];
    double yz[NC][n];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) yz[c][z] = 0.0;
    const double wab = T.w[a] * T.w[b];

#pragma unroll
    for (int z = 0; z < n; ++z) {
      const int q = z * n2 + p;
      double gxi[NC][3];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double sx = 0.0, sy_ = 0.0, sz = 0.0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          sx += Da[k] * su[c * n3 + z * n2 + b * n + k];
          sy_ += Db[k] * su[c * n3 + z * n2 + k * n + a];
          sz += T.D[z * DGVV_NMAX + k] * ucol[c][k];
        }
        gxi[c][0] = sx; gxi[c][1] = sy_; gxi[c][2] = sz;
      }
      double Ji[9];
      double w;
      if (GEO == 0) {
        w = A.nu_cell[(size_t)cell * n3 + q] * wab * T.w[z] * vol;
      } else {
        const double* vm = A.vmet + (size_t)cell * VMET_NV * n3 + q;
#pragma unroll
        for (int r = 0; r < 9; ++r) Ji[r] = vm[r * n3];
        w = A.nu_cell[(size_t)cell * n3 + q] * vm[9 * n3];
      }
      // physical gradient
      double G[NC][3];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          G[c][j] = (GEO == 0) ? gxi[c][j] * ih[j]
                               : gxi[c][0] * Ji[j] + gxi[c][1] * Ji[3 + j] + gxi[c][2] * Ji[6 + j];
      // stress-like coefficient T[c][j] of d v_c / d x_j
      double Tc[NC][3];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < 3; ++j)
        {
          if constexpr (FORM == 0) Tc[c][j] = w * (G[c][j] + G[j][c]);
          else Tc[c][j] = w * G[c][j];
        }
      // to reference directions
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double F[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
          F[k] = (GEO == 0) ? Tc[c][k] * ih[k]
                            : Tc[c][0] * Ji[3 * k] + Tc[c][1] * Ji[3 * k + 1] + Tc[c][2] * Ji[3 * k + 2];
        sF[c * n3 + q] = F[0];
        sF[(NC + c) * n3 + q] = F[1];
#pragma unroll
        for (int z2 = 0; z2 < n; ++z2) yz[c][z2] += T.D[z * DGVV_NMAX + z2] * F[2];
      }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) {
        double acc = yz[c][z];
#pragma unroll
        for (int k = 0; k < n; ++k) {
          acc += DTa[k] * sF[c * n3 + z * n2 + b * n + k];
          acc += DTb[k] * sF[(NC + c) * n3 + z * n2 + k * n + a];
        }
        sy[c * n3 + z * n2 + p] = acc;
      }
    __syncthreads();
  }

  // =============================================================== face terms
  double* st = sF;                 // traces [2][NC][n2]
  double* sg = sF + 2 * NC * n2;   // tangential coefficients [2][NC][n2]
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
      const int nbv = A.nbr[cell * 6 + f];
      const bool interior = nbv >= 0;
      const bool act = interior || (nbv == NB_DIRICHLET);
      const double* lS = s ? T.l1 : T.l0;
      const double* dS = s ? T.d1 : T.d0;
      const double* lO = s ? T.l0 : T.l1;
      const double* dO = s ? T.d0 : T.d1;
      double um[NC], up[NC], dm[NC], dp[NC];
      if (act) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          double v = 0.0, g = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) {
            const double x = su[c * n3 + base + i * sd];
            v += lS[i] * x;
            g += dS[i] * x;
          }
          um[c] = v; dm[c] = g;
        }
        if (interior) {
          const double* pn = (nbv < A.n_owned) ? A.src + (size_t)nbv * NC * n3
                                               : A.ghost + (size_t)(nbv - A.n_owned) * NC * n3;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            double v = 0.0, g = 0.0;
#pragma unroll
            for (int i = 0; i < n; ++i) {
              const double x = __ldg(pn + c * n3 + base + i * sd);
              v += lO[i] * x;
              g += dO[i] * x;
            }
            up[c] = v; dp[c] = g;
          }
        } else {
#pragma unroll
          for (int c = 0; c < NC; ++c) { up[c] = -um[c]; dp[c] = dm[c]; }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          st[c * n2 + p] = um[c];
          st[(NC + c) * n2 + p] = up[c];
        }
      }
      __syncthreads();
      double fv[NC], gk[NC][3];
      if (act) {
        double gxm[NC][3], gxp[NC][3];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          double m1 = 0.0, m2 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
          for (int k = 0; k < n; ++k) {
            m1 += Da[k] * st[c * n2 + b * n + k];
            m2 += Db[k] * st[c * n2 + k * n + a];
          }
          if (interior) {
#pragma unroll
            for (int k = 0; k < n; ++k) {
              p1 += Da[k] * st[(NC + c) * n2 + b * n + k];
              p2 += Db[k] * st[(NC + c) * n2 + k * n + a];
            }
          }
          gxm[c][d] = dm[c]; gxm[c][t1] = m1; gxm[c][t2] = m2;
          gxp[c][d] = dp[c]; gxp[c][t1] = p1; gxp[c][t2] = p2;
        }
        double Jim[9], Jip[9], nrm[3], dA, num, nup, Hp;
        const double* nuf = A.nu_face + ((size_t)cell * 6 + f) * n2;
        num = nuf[p];
        if (GEO == 0) {
#pragma unroll
          for (int r = 0; r < 9; ++r) { Jim[r] = 0.0; Jip[r] = 0.0; }
          Jim[0] = ih[0]; Jim[4] = ih[1]; Jim[8] = ih[2];
          nrm[0] = nrm[1] = nrm[2] = 0.0;
          nrm[d] = s ? 1.0 : -1.0;
          dA = T.w[a] * T.w[b] * vol * ih[d];
        } else {
          const double* fm = A.fmet + ((size_t)cell * 6 + f) * FMET_NV * n2 + p;
#pragma unroll
          for (int r = 0; r < 9; ++r) Jim[r] = fm[r * n2];
          nrm[0] = fm[9 * n2]; nrm[1] = fm[10 * n2]; nrm[2] = fm[11 * n2];
          dA = fm[12 * n2];
        }
        if (interior) {
          nup = A.nu_face[((size_t)nbv * 6 + (f ^ 1)) * n2 + p];
          if (GEO == 0) {
            const double* cg = A.cart + (size_t)nbv * CART_STRIDE;
            Jip[0] = cg[0]; Jip[4] = cg[1]; Jip[8] = cg[2];
            Hp = cg[3];
          } else {
            const double* fm = A.fmet + ((size_t)nbv * 6 + (f ^ 1)) * FMET_NV * n2 + p;
#pragma unroll
            for (int r = 0; r < 9; ++r) Jip[r] = fm[r * n2];
            Hp = A.Hcell[nbv];
          }
        } else {
          nup = num; Hp = Hm;
#pragma unroll
          for (int r = 0; r < 9; ++r) Jip[r] = Jim[r];
#pragma unroll
          for (int c = 0; c < NC; ++c) { gxp[c][0] = gxm[c][0]; gxp[c][1] = gxm[c][1]; gxp[c][2] = gxm[c][2]; }
        }
        double Gm[NC][3], Gp[NC][3];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            Gm[c][j] = gxm[c][0] * Jim[j] + gxm[c][1] * Jim[3 + j] + gxm[c][2] * Jim[6 + j];
            Gp[c][j] = gxp[c][0] * Jip[j] + gxp[c][1] * Jip[3 + j] + gxp[c][2] * Jip[6 + j];
          }
        const double tau = A.pen * fmax(Hm, Hp) * 0.5 * (num + nup);
        face_flux_impl<NC, FORM>(um, up, Gm, Gp, nrm, num, nup, tau, dA, Jim, fv, gk);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          sg[c * n2 + p] = gk[c][t1];
          sg[(NC + c) * n2 + p] = gk[c][t2];
        }
      }
      __syncthreads();
      if (act) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          double val = fv[c];
#pragma unroll
          for (int k = 0; k < n; ++k) {
            val += DTa[k] * sg[c * n2 + b * n + k];
            val += DTb[k] * sg[(NC + c) * n2 + k * n + a];
          }
          const double gn = gk[c][d];
#pragma unroll
          for (int i = 0; i < n; ++i) sy[c * n3 + base + i * sd] += lS[i] * val + dS[i] * gn;
        }
      }
      __syncthreads();
    }
  }

  // =============================================================== epilogue
  if (active) {
    const size_t off = (size_t)cell * NC * n3;
    if (A.mode == MODE_APPLY) {
#pragma unroll
      for (int i = p; i < NC * n3; i += n2) A.dst[off + i] = sy[i];
    } else if (A.mode == MODE_RESID) {
#pragma unroll
      for (int i = p; i < NC * n3; i += n2) A.dst[off + i] = __ldg(A.b + off + i) - sy[i];
    } else {
#pragma unroll
      for (int i = p; i < NC * n3; i += n2) {
        const double r = __ldg(A.b + off + i) - sy[i];
        double dn = A.c_r * __ldg(A.dinv + off + i) * r;
        if (A.c_rho != 0.0) dn += A.c_rho * A.dvec[off + i];
        A.dvec[off + i] = dn;
        A.xout[off + i] = su[i] + dn;
      }
    }
  }
}

}  // namespace dgvv
