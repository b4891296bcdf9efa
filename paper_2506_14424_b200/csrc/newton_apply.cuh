// newton_apply.cuh — K2: Newton-linearised SIPG viscous apply (reading G10)
//   dst = J(u0) w = a(., w; nu0) + a(., u0; delta_nu[w]),
//   nu0 = eta(gd(eps(u0))),  delta_nu = 2 g(gd0) eps(u0):eps(w),  g = eta'(gd)/gd  (Carreau, G9)
// evaluated pointwise at every cell point and, per side, at every face point from that side's
// own traces (G8); the penalty uses (nu0- + nu0+)/2 and (dnu- + dnu+)/2.  nu0 and g are
// recomputed from eps(u0) in the kernel (the ε(u0) needed for delta_nu is formed anyway), so
// the stream is src + u_lin + dst.  Cell-centric like sipg_apply2.cuh: a team of
// n^2 threads per cell, z-columns in registers, faces one at a time (two fields double the
// live state), both fields' full face gradients (delta_nu needs all of eps).
#pragma once
#include "common.cuh"
#include "laws.cuh"


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


template <int n, int GEO>
struct NewtonCfg {
  static constexpr int n2 = n * n, n3 = n * n * n;
  static constexpr int WV = 6 * n3;                 // volume F_x, F_y of 3 components
  static constexpr int WF = 3 * n3 + 18 * n2;       // face accumulator + trace/coefficient buffers
  static constexpr int CS = 6 * n3 + (WV > WF ? WV : WF);   // w, u0 + work
};

template <int n, int GEO, int CPB, int MINB>
__global__ void __launch_bounds__(CPB * n * n, MINB) newton_apply_kernel(const ApplyArgs A) {
  using Cf = NewtonCfg<n, GEO>;
  constexpr int n2 = Cf::n2, n3 = Cf::n3;
  extern __shared__ double smem[];
  const Tab1D& T = c_tab[n];
  const int lc = threadIdx.x / n2;
  const int p = threadIdx.x - lc * n2;
  const int a = p % n, b = p / n;
  const int slot_raw = blockIdx.x * CPB + lc;
  const bool active = slot_raw < A.n_proc;
  const int slot = active ? slot_raw : (A.n_proc - 1);
  const int cell = A.cell_list ? A.cell_list[slot] : A.cell_base + slot;

  double* sw = smem + lc * Cf::CS;      // w  [3][n3]
  double* s0 = sw + 3 * n3;             // u0 [3][n3]
  double* W = s0 + 3 * n3;              // work
  double* Y = W;                        // face phase accumulator [3][n3]
  double* st = W + 3 * n3;              // traces [2 sides][2 fields][3][n2]
  double* sg = st + 12 * n2;            // tangential coefficients [2][3][n2]

  double Da[n], Db[n], DTa[n], DTb[n];
#pragma unroll
  for (int k = 0; k < n; ++k) {
    Da[k] = T.D[a * DGVV_NMAX + k];
    Db[k] = T.D[b * DGVV_NMAX + k];
    DTa[k] = T.D[k * DGVV_NMAX + a];
    DTb[k] = T.D[k * DGVV_NMAX + b];
  }
  for (int i = p; i < 3 * n3; i += n2) {
    sw[i] = __ldg(A.src + (size_t)cell * 3 * n3 + i);
    s0[i] = __ldg(A.ulin + (size_t)cell * 3 * n3 + i);
  }
  double ih[3] = {0, 0, 0}, vol = 0.0, Hm;
  if constexpr (GEO == 0) {
    const double* cg = A.cart + (size_t)cell * CART_STRIDE;
    ih[0] = cg[0]; ih[1] = cg[1]; ih[2] = cg[2]; Hm = cg[3]; vol = cg[4];
  } else {
    Hm = A.Hcell[cell];
  }
  __syncthreads();

  double y[3][n];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int z = 0; z < n; ++z) {        // Helmholtz mass term
      double jw = 0.0;
      if (A.mass != 0.0) jw = (GEO == 0) ? T.w[a] * T.w[b] * T.w[z] * vol : A.jxw[(size_t)cell * n3 + z * n2 + p];
      y[c][z] = A.mass * jw * sw[c * n3 + z * n2 + p];
    }

  auto to_phys = [&](const double (&gx)[3][3], const double (&Ji)[9], double (&G)[3][3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 3; ++j) G[c][j] = gx[c][0] * Ji[j] + gx[c][1] * Ji[3 + j] + gx[c][2] * Ji[6 + j];
  };
  auto epsdot = [&](const double (&G1)[3][3], const double (&G2)[3][3]) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 3; ++j) s += 0.5 * (G1[c][j] + G1[j][c]) * 0.5 * (G2[c][j] + G2[j][c]);
    return s;
  };
  auto cart_ji = [&](const double* h, double (&Ji)[9]) {
#pragma unroll
    for (int r = 0; r < 9; ++r) Ji[r] = 0.0;
    Ji[0] = h[0]; Ji[4] = h[1]; Ji[8] = h[2];
  };

  // =============================================================== volume
  {
    const double wab = T.w[a] * T.w[b];
#pragma unroll 1
    for (int z = 0; z < n; ++z) {
      const int q = z * n2 + p;
      double gw[3][3], g0[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double x1 = 0, y1 = 0, z1 = 0, x0 = 0, y0 = 0, z0 = 0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          x1 += Da[k] * sw[c * n3 + z * n2 + b * n + k];
          y1 += Db[k] * sw[c * n3 + z * n2 + k * n + a];
          z1 += T.D[z * DGVV_NMAX + k] * sw[c * n3 + k * n2 + p];
          x0 += Da[k] * s0[c * n3 + z * n2 + b * n + k];
          y0 += Db[k] * s0[c * n3 + z * n2 + k * n + a];
          z0 += T.D[z * DGVV_NMAX + k] * s0[c * n3 + k * n2 + p];
        }
        gw[c][0] = x1; gw[c][1] = y1; gw[c][2] = z1;
        g0[c][0] = x0; g0[c][1] = y0; g0[c][2] = z0;
      }
      double Ji[9], jxw;
      if constexpr (GEO == 0) {
        cart_ji(ih, Ji);
        jxw = wab * T.w[z] * vol;
      } else {
        const double* vm = A.vJi + (size_t)cell * 9 * n3 + q;
#pragma unroll
        for (int r = 0; r < 9; ++r) Ji[r] = __ldg(vm + r * n3);
        jxw = A.jxw[(size_t)cell * n3 + q];
      }
      double Gw[3][3], G0[3][3];
      to_phys(gw, Ji, Gw);
      to_phys(g0, Ji, G0);
      const double gd = sqrt(2.0 * epsdot(G0, G0));
      const double nu0 = carreau_eta(A.law, gd);
      const double dnu = 2.0 * carreau_g(A.law, gd) * epsdot(G0, Gw);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double Tc[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) Tc[j] = jxw * (nu0 * (Gw[c][j] + Gw[j][c]) + dnu * (G0[c][j] + G0[j][c]));
        double F[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) F[k] = Tc[0] * Ji[3 * k] + Tc[1] * Ji[3 * k + 1] + Tc[2] * Ji[3 * k + 2];
        W[c * n3 + q] = F[0];
        W[(3 + c) * n3 + q] = F[1];
#pragma unroll
        for (int z2 = 0; z2 < n; ++z2) y[c][z2] += T.D[z * DGVV_NMAX + z2] * F[2];
      }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          acc += DTa[k] * W[c * n3 + z * n2 + b * n + k];
          acc += DTb[k] * W[(3 + c) * n3 + z * n2 + k * n + a];
        }
        y[c][z] += acc;
      }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) Y[c * n3 + z * n2 + p] = 0.0;
  }

  // =============================================================== faces (one at a time)
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int d = f / 2, s = f % 2;
    const int sd = (d == 0) ? 1 : (d == 1 ? n : n2);
    const int st1 = (d == 0) ? n : 1;
    const int st2 = (d == 2) ? n : n2;
    const int t1 = face_t1(d), t2 = face_t2(d);
    const int base = a * st1 + b * st2;
    const int nbv = A.nbr[cell * 6 + f];
    const bool inter = nbv >= 0;
    const bool act = inter || nbv == NB_DIRICHLET;
    const double* lS = s ? T.l1 : T.l0;
    const double* dS = s ? T.d1 : T.d0;
    const double* lO = s ? T.l0 : T.l1;
    const double* dO = s ? T.d0 : T.d1;
    // values and normal derivatives: [field 0 = w, 1 = u0]
    double um[2][3], up[2][3], dm[2][3], dp[2][3];
#pragma unroll
    for (int fl = 0; fl < 2; ++fl) {
      const double* sf = fl ? s0 : sw;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v = 0, g = 0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const double x = sf[c * n3 + base + i * sd];
          v += lS[i] * x;
          g += dS[i] * x;
        }
        um[fl][c] = v; dm[fl][c] = g;
      }
    }
    if (inter) {
#pragma unroll
      for (int fl = 0; fl < 2; ++fl) {
        const double* gsrc = fl ? ((nbv < A.n_owned) ? A.ulin + (size_t)nbv * 3 * n3 : A.ulin_ghost + (size_t)(nbv - A.n_owned) * 3 * n3)
                                : ((nbv < A.n_owned) ? A.src + (size_t)nbv * 3 * n3 : A.ghost + (size_t)(nbv - A.n_owned) * 3 * n3);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double v = 0, g = 0;
#pragma unroll
          for (int i = 0; i < n; ++i) {
            const double x = __ldg(gsrc + c * n3 + base + i * sd);
            v += lO[i] * x;
            g += dO[i] * x;
          }
          up[fl][c] = v; dp[fl][c] = g;
        }
      }
    } else {
#pragma unroll
      for (int fl = 0; fl < 2; ++fl)
#pragma unroll
        for (int c = 0; c < 3; ++c) { up[fl][c] = -um[fl][c]; dp[fl][c] = dm[fl][c]; }
    }
#pragma unroll
    for (int fl = 0; fl < 2; ++fl)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        st[((0 * 2 + fl) * 3 + c) * n2 + p] = um[fl][c];
        st[((1 * 2 + fl) * 3 + c) * n2 + p] = up[fl][c];
      }
    __syncthreads();
    double fvt[3] = {0, 0, 0}, gkt[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    if (act) {
      double gxm[2][3][3], gxp[2][3][3];
#pragma unroll
      for (int fl = 0; fl < 2; ++fl)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double m1 = 0, m2 = 0, p1 = 0, p2 = 0;
          const double* sm_ = st + ((0 * 2 + fl) * 3 + c) * n2;
          const double* sp_ = st + ((1 * 2 + fl) * 3 + c) * n2;
#pragma unroll
          for (int k = 0; k < n; ++k) {
            m1 += Da[k] * sm_[b * n + k];
            m2 += Db[k] * sm_[k * n + a];
            p1 += Da[k] * sp_[b * n + k];
            p2 += Db[k] * sp_[k * n + a];
          }
          gxm[fl][c][d] = dm[fl][c]; gxm[fl][c][t1] = m1; gxm[fl][c][t2] = m2;
          if (inter) { gxp[fl][c][d] = dp[fl][c]; gxp[fl][c][t1] = p1; gxp[fl][c][t2] = p2; }
          else { gxp[fl][c][d] = dm[fl][c]; gxp[fl][c][t1] = m1; gxp[fl][c][t2] = m2; }
        }
      double Jim[9], Jip[9], nrm[3], dA, Hp = Hm;
      const double sgn = s ? 1.0 : -1.0;
      if constexpr (GEO == 0) {
        cart_ji(ih, Jim);
        nrm[0] = nrm[1] = nrm[2] = 0.0;
        nrm[d] = sgn;
        dA = T.w[a] * T.w[b] * vol * ih[d];
        if (inter) {
          const double* cg = A.cart + (size_t)nbv * CART_STRIDE;
          cart_ji(cg, Jip);
          Hp = cg[3];
        } else {
#pragma unroll
          for (int r = 0; r < 9; ++r) Jip[r] = Jim[r];
        }
      } else {
        const double* fm = A.fJi + ((size_t)cell * 6 + f) * 9 * n2 + p;
#pragma unroll
        for (int r = 0; r < 9; ++r) Jim[r] = __ldg(fm + r * n2);
        dA = A.fdA[((size_t)cell * 6 + f) * n2 + p];
        const double v0 = Jim[3 * d], v1 = Jim[3 * d + 1], v2 = Jim[3 * d + 2];
        const double il = sgn / sqrt(v0 * v0 + v1 * v1 + v2 * v2);
        nrm[0] = v0 * il; nrm[1] = v1 * il; nrm[2] = v2 * il;
        if (inter) {
          const double* fp = A.fJi + ((size_t)nbv * 6 + (f ^ 1)) * 9 * n2 + p;
#pragma unroll
          for (int r = 0; r < 9; ++r) Jip[r] = __ldg(fp + r * n2);
          Hp = A.Hcell[nbv];
        } else {
#pragma unroll
          for (int r = 0; r < 9; ++r) Jip[r] = Jim[r];
        }
      }
      double Gmw[3][3], Gm0[3][3], Gpw[3][3], Gp0[3][3];
      to_phys(gxm[0], Jim, Gmw);
      to_phys(gxm[1], Jim, Gm0);
      to_phys(gxp[0], Jip, Gpw);
      to_phys(gxp[1], Jip, Gp0);
      const double gdm = sqrt(2.0 * epsdot(Gm0, Gm0)), gdp = sqrt(2.0 * epsdot(Gp0, Gp0));
      const double num = carreau_eta(A.law, gdm), nup = carreau_eta(A.law, gdp);
      const double dnm = 2.0 * carreau_g(A.law, gdm) * epsdot(Gm0, Gmw);
      const double dnp = 2.0 * carreau_g(A.law, gdp) * epsdot(Gp0, Gpw);
      const double hmax = fmax(Hm, Hp);
      double fv[3], gk[3][3];
      // a(., w; nu0)
      face_flux_gen<3, 0>(um[0], up[0], Gmw, Gpw, nrm, num * dA, nup * dA, A.pen * hmax * 0.5 * (num + nup) * dA,
                          Jim, fv, gk);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        fvt[c] += fv[c];
#pragma unroll
        for (int k = 0; k < 3; ++k) gkt[c][k] += gk[c][k];
      }
      // a(., u0; delta nu)
      face_flux_gen<3, 0>(um[1], up[1], Gm0, Gp0, nrm, dnm * dA, dnp * dA, A.pen * hmax * 0.5 * (dnm + dnp) * dA,
                          Jim, fv, gk);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        fvt[c] += fv[c];
#pragma unroll
        for (int k = 0; k < 3; ++k) gkt[c][k] += gk[c][k];
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      sg[(0 * 3 + c) * n2 + p] = gkt[c][t1];
      sg[(1 * 3 + c) * n2 + p] = gkt[c][t2];
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double val = fvt[c];
#pragma unroll
        for (int k = 0; k < n; ++k)
          val += DTa[k] * sg[(0 * 3 + c) * n2 + b * n + k] + DTb[k] * sg[(1 * 3 + c) * n2 + k * n + a];
        const double gn = gkt[c][d];
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const double add = lS[i] * val + dS[i] * gn;
          if (d == 2) y[c][i] += add;
          else Y[c * n3 + base + i * sd] += add;
        }
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int z = 0; z < n; ++z) y[c][z] += Y[c * n3 + z * n2 + p];
  if (active) {
    const size_t off = (size_t)cell * 3 * n3;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) A.dst[off + c * n3 + z * n2 + p] = y[c][z];
  }
}

}  // namespace dgvv
