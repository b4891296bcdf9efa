// newton_apply2.cuh — K2 v2: Newton-linearised SIPG viscous apply on axis-aligned (Cartesian)
// cells (C3, C5).  Reading G10:
//   J(u0) w = a(., w; nu0) + a(., u0; dnu[w]),   dnu = 2 g(gd0) eps(u0):eps(w),  g = eta'(gd)/gd.
// a(.,.;nu) is linear in nu, so at every cell and face point the two terms are merged into one
// effective stress  nu0 eps(w) + dnu eps(u0)  (consistency), one effective jump
// nu0 [w] + dnu [u0]  (symmetry term) and two penalties tau(nu0) [w], tau(dnu) [u0].
// nu0 is the viscosity stored by dgvv_update_viscosity at the cell points and at each side's own
// face points (G8; same u_lin), and g follows from it without a second power:
//   Carreau (G9):  eta - eta_inf = (eta0 - eta_inf) P,  P = (1 + (lambda gd)^2)^((n-1)/2)
//   g = (eta0 - eta_inf)(n - 1) lambda^2 P / (1 + (lambda gd)^2)
//     = (n - 1) lambda^2 (nu0 - eta_inf) / (1 + (lambda gd0)^2),
// with gd0 = sqrt(2 eps(u0):eps(u0)) formed in the kernel (eps(u0) is needed for dnu anyway).
// Structure as sipg_apply2.cuh (team of n^2 threads per cell, padded smem, faces one at a time,
// no atomics); the general-geometry Newton apply stays in newton_apply.cuh.
#pragma once
#include "common.cuh"
#include "sipg_apply2.cuh"

namespace dgvv {

template <int n>
struct Newton2Cfg {
  using L = Lay<n>;
  static constexpr int VOL = 3 * L::CST;
  static constexpr int FB = 14 * L::FA;          // traces [m|p][w|u0][3] + G1, G2T (comp d)
  static constexpr int RW = (2 * VOL > VOL + FB) ? 2 * VOL : VOL + FB;
  static constexpr int CS = 2 * VOL + RW;
};

template <int n, int CPB, int MINB>
__global__ void __launch_bounds__(CPB * n * n, MINB) newton_apply2_kernel(const ApplyArgs A) {
  using L = Lay<n>;
  using Cf = Newton2Cfg<n>;
  constexpr int n2 = L::n2, n3 = L::n3, RS = L::RS, PS = L::PS, CST = L::CST, FA = L::FA;
  constexpr int VOL = Cf::VOL;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(16) double sD[n * RS];
  __shared__ __align__(16) double sDT[n * RS];
  __shared__ int sid[CPB];
  const Tab1D& T = c_tab[n];

  const int lc = threadIdx.x / n2;
  const int p = threadIdx.x - lc * n2;
  const int a = p % n, b = p / n;
  const int slot_raw = blockIdx.x * CPB + lc;
  const bool active = slot_raw < A.n_proc;
  const int slot = active ? slot_raw : (A.n_proc - 1);
  const int cell = A.cell_list ? A.cell_list[slot] : A.cell_base + slot;
  for (int i = threadIdx.x; i < n * RS; i += blockDim.x) {
    const int r = i / RS, k = i - r * RS;
    sD[i] = k < n ? T.D[r * DGVV_NMAX + k] : 0.0;
    sDT[i] = k < n ? T.D[k * DGVV_NMAX + r] : 0.0;
  }
  if (p == 0) sid[lc] = active ? cell : -1;

  double* sf[2];
  sf[0] = smem + lc * Cf::CS;            // w  [3][z][y][x]
  sf[1] = sf[0] + VOL;                   // u0 [3][z][y][x]
  double* R = sf[1] + VOL;               // W1 | W2T (volume);  Y | face buffers (faces)
  {
    const double* gw = A.src + (size_t)cell * 3 * n3;
    const double* g0 = A.ulin + (size_t)cell * 3 * n3;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) {
        sf[0][c * CST + z * PS + b * RS + a] = __ldg(gw + c * n3 + z * n2 + p);
        sf[1][c * CST + z * PS + b * RS + a] = __ldg(g0 + c * n3 + z * n2 + p);
      }
  }
  const double* cg = A.cart + (size_t)cell * CART_STRIDE;
  const double ih[3] = {cg[0], cg[1], cg[2]};
  const double Hm = cg[3], vol = cg[4];
  const double eta_inf = A.law[1], lam2 = A.law[2] * A.law[2], gfac = (A.law[3] - 1.0) * lam2;
  int nbf[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) nbf[f] = __ldg(A.nbr + cell * 6 + f);
  __syncthreads();

  double y[3][n];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int z = 0; z < n; ++z)          // Helmholtz mass term (the mass part of J is M itself)
      y[c][z] = A.mass == 0.0 ? 0.0 : A.mass * T.w[a] * T.w[b] * T.w[z] * vol * sf[0][c * CST + z * PS + b * RS + a];

  // =============================================================== volume
  {
    double Da[n], Db[n];
    ld_row<n>(sD + a * RS, Da);
    ld_row<n>(sD + b * RS, Db);
    const double wab = T.w[a] * T.w[b] * vol;
#pragma unroll 1
    for (int z = 0; z < n; ++z) {
      const int q = z * n2 + p;
      double G[2][3][3];                 // physical gradients of w (0) and u0 (1)
#pragma unroll
      for (int fl = 0; fl < 2; ++fl)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double* s = sf[fl] + c * CST;
          G[fl][c][0] = rowdot<n>(s + z * PS + b * RS, Da) * ih[0];
          double sy = 0.0, sz = 0.0;
#pragma unroll
          for (int k = 0; k < n; ++k) {
            sy = fma(Db[k], s[z * PS + k * RS + a], sy);
            sz = fma(T.D[z * DGVV_NMAX + k], s[k * PS + b * RS + a], sz);
          }
          G[fl][c][1] = sy * ih[1];
          G[fl][c][2] = sz * ih[2];
        }
      double e00 = 0.0, e0w = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double ew = 0.5 * (G[0][c][j] + G[0][j][c]), e0 = 0.5 * (G[1][c][j] + G[1][j][c]);
          e00 = fma(e0, e0, e00);
          e0w = fma(e0, ew, e0w);
        }
      const double nu0 = A.nu_cell[(size_t)cell * n3 + q];
      const double g = gfac * (nu0 - eta_inf) / (1.0 + lam2 * 2.0 * e00);
      const double dnu = 2.0 * g * e0w;
      const double jxw = wab * T.w[z];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double F[3];
#pragma unroll
        for (int j = 0; j < 3; ++j)
          F[j] = jxw * (nu0 * (G[0][c][j] + G[0][j][c]) + dnu * (G[1][c][j] + G[1][j][c])) * ih[j];
        R[c * CST + z * PS + b * RS + a] = F[0];
        R[VOL + c * CST + z * PS + a * RS + b] = F[1];
#pragma unroll
        for (int z2 = 0; z2 < n; ++z2) y[c][z2] = fma(T.D[z * DGVV_NMAX + z2], F[2], y[c][z2]);
      }
    }
    __syncthreads();
    double DTa[n], DTb[n];
    ld_row<n>(sDT + a * RS, DTa);
    ld_row<n>(sDT + b * RS, DTb);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z)
        y[c][z] += rowdot<n>(R + c * CST + z * PS + b * RS, DTa) + rowdot<n>(R + VOL + c * CST + z * PS + a * RS, DTb);
    __syncthreads();
  }

  // =============================================================== faces (one at a time)
  // buffers: trace arrays [side m|p][field w|u0][c] at R + VOL + ((side*2+fl)*3+c)*FA,
  //          G1 at R + VOL + 12 FA, G2T at R + VOL + 13 FA
  double* FBm = R + VOL;
#pragma unroll
  for (int dd = 0; dd < 3; ++dd) {
    const int d = (dd == 0) ? 2 : dd - 1;
    const int t1 = face_t1(d), t2 = face_t2(d);
    double val[2][3], gnn[2][3];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int f = 2 * d + s;
      const int nbv = nbf[f];
      const bool inter = nbv >= 0;
      const bool act = inter || (nbv == NB_DIRICHLET);
      const double* lS = s ? T.l1 : T.l0;
      const double* dS = s ? T.d1 : T.d0;
      // coefficient loads first
      const double num = A.nu_face[((size_t)cell * 6 + f) * n2 + p];
      double nup = num, Hp = Hm, ihp[3] = {ih[0], ih[1], ih[2]};
      if (inter) {
        const double* cgp = A.cart + (size_t)nbv * CART_STRIDE;
        ihp[0] = cgp[0]; ihp[1] = cgp[1]; ihp[2] = cgp[2]; Hp = cgp[3];
        nup = A.nu_face[((size_t)nbv * 6 + (f ^ 1)) * n2 + p];
      }
      // own and neighbour traces of both fields
      double um[2][3], dm[2][3], up[2][3], dp[2][3];
#pragma unroll
      for (int fl = 0; fl < 2; ++fl)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double x[n];
          const double* s_ = sf[fl] + c * CST;
          if (d == 0) ld_row<n>(s_ + b * PS + a * RS, x);
          else if (d == 1) {
#pragma unroll
            for (int i = 0; i < n; ++i) x[i] = s_[b * PS + i * RS + a];
          } else {
#pragma unroll
            for (int i = 0; i < n; ++i) x[i] = s_[i * PS + b * RS + a];
          }
          double v = 0.0, gg = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) { v = fma(lS[i], x[i], v); gg = fma(dS[i], x[i], gg); }
          um[fl][c] = v; dm[fl][c] = gg;
        }
      if (inter) {
        const double* lO = s ? T.l0 : T.l1;
        const double* dO = s ? T.d0 : T.d1;
        const int sl = lc + (nbv - cell);
        const bool in_cta = sl >= 0 && sl < CPB && sid[sl] == nbv;
#pragma unroll
        for (int fl = 0; fl < 2; ++fl) {
          const double* pn = fl == 0 ? (nbv < A.n_owned ? A.src + (size_t)nbv * 3 * n3
                                                        : A.ghost + (size_t)(nbv - A.n_owned) * 3 * n3)
                                     : (nbv < A.n_owned ? A.ulin + (size_t)nbv * 3 * n3
                                                        : A.ulin_ghost + (size_t)(nbv - A.n_owned) * 3 * n3);
          const double* ns = smem + (in_cta ? sl : 0) * Cf::CS + fl * VOL;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double x[n];
            if (in_cta) {
              if (d == 0) ld_row<n>(ns + c * CST + b * PS + a * RS, x);
              else if (d == 1) {
#pragma unroll
                for (int i = 0; i < n; ++i) x[i] = ns[c * CST + b * PS + i * RS + a];
              } else {
#pragma unroll
                for (int i = 0; i < n; ++i) x[i] = ns[c * CST + i * PS + b * RS + a];
              }
            } else {
              if (d == 0) {
                if constexpr ((n & 1) == 0) ldg_row<n>(pn + c * n3 + b * n2 + a * n, x);
                else {
#pragma unroll
                  for (int i = 0; i < n; ++i) x[i] = __ldg(pn + c * n3 + b * n2 + a * n + i);
                }
              } else if (d == 1) {
#pragma unroll
                for (int i = 0; i < n; ++i) x[i] = __ldg(pn + c * n3 + b * n2 + i * n + a);
              } else {
#pragma unroll
                for (int i = 0; i < n; ++i) x[i] = __ldg(pn + c * n3 + i * n2 + p);
              }
            }
            double v = 0.0, gg = 0.0;
#pragma unroll
            for (int i = 0; i < n; ++i) { v = fma(lO[i], x[i], v); gg = fma(dO[i], x[i], gg); }
            up[fl][c] = v; dp[fl][c] = gg;
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
          FBm[((0 * 2 + fl) * 3 + c) * FA + b * RS + a] = um[fl][c];
          FBm[((1 * 2 + fl) * 3 + c) * FA + b * RS + a] = up[fl][c];
        }
      __syncthreads();

      // per side: full physical gradients of w and u0, nu0, dnu, and column d of the
      // effective stress  nu0 eps(w) + dnu eps(u0)
      double Sn[2][3], dnuS[2];
      {
        double Da[n], Db[n];
        ld_row<n>(sD + a * RS, Da);
        ld_row<n>(sD + b * RS, Db);
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          if (side == 1 && !inter) {
#pragma unroll
            for (int c = 0; c < 3; ++c) Sn[1][c] = Sn[0][c];
            dnuS[1] = dnuS[0];
            continue;
          }
          const double* ihs = side ? ihp : ih;
          double G[2][3][3];
#pragma unroll
          for (int fl = 0; fl < 2; ++fl)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double* tr = FBm + ((side * 2 + fl) * 3 + c) * FA;
              double g2 = 0.0;
#pragma unroll
              for (int k = 0; k < n; ++k) g2 = fma(Db[k], tr[k * RS + a], g2);
              G[fl][c][d] = (side ? dp[fl][c] : dm[fl][c]) * ihs[d];
              G[fl][c][t1] = rowdot<n>(tr + b * RS, Da) * ihs[t1];
              G[fl][c][t2] = g2 * ihs[t2];
            }
          double e00 = 0.0, e0w = 0.0;
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              const double ew = 0.5 * (G[0][c][j] + G[0][j][c]), e0 = 0.5 * (G[1][c][j] + G[1][j][c]);
              e00 = fma(e0, e0, e00);
              e0w = fma(e0, ew, e0w);
            }
          const double nu0 = side ? nup : num;
          const double g = gfac * (nu0 - eta_inf) / (1.0 + lam2 * 2.0 * e00);
          const double dnu = 2.0 * g * e0w;
          dnuS[side] = dnu;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            Sn[side][c] = 0.5 * (nu0 * (G[0][c][d] + G[0][d][c]) + dnu * (G[1][c][d] + G[1][d][c]));
        }
      }
      const double sgn = s ? 1.0 : -1.0;
      const double dA = T.w[a] * T.w[b] * vol * ih[d];
      const double hm = A.pen * fmax(Hm, Hp);
      const double tw = hm * 0.5 * (num + nup), t0 = hm * 0.5 * (dnuS[0] + dnuS[1]);
      double gt1 = 0.0, gt2 = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double jw = um[0][c] - up[0][c], j0 = um[1][c] - up[1][c];
        const double pvw = (c == d) ? 2.0 * jw : jw, pv0 = (c == d) ? 2.0 * j0 : j0;
        val[s][c] = dA * (-sgn * (Sn[0][c] + Sn[1][c]) + tw * pvw + t0 * pv0);
        const double je = num * jw + dnuS[0] * j0;                      // effective jump
        gnn[s][c] = dA * ((c == d) ? -je * sgn : -0.5 * je * sgn) * ih[d];
        if (c == t1) gt1 = dA * (-0.5 * je * sgn) * ih[t1];
        if (c == t2) gt2 = dA * (-0.5 * je * sgn) * ih[t2];
      }
      if (!act) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { val[s][c] = 0.0; gnn[s][c] = 0.0; }
        gt1 = 0.0; gt2 = 0.0;
      }
      FBm[12 * FA + b * RS + a] = gt1;
      FBm[13 * FA + a * RS + b] = gt2;
      __syncthreads();
      {
        double DTa[n], DTb[n];
        ld_row<n>(sDT + a * RS, DTa);
        ld_row<n>(sDT + b * RS, DTb);
        val[s][d] += rowdot<n>(FBm + 12 * FA + b * RS, DTa) + rowdot<n>(FBm + 13 * FA + a * RS, DTb);
      }
    }
    // extrapolate both faces' coefficients along the normal line into the cell
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double add[n];
#pragma unroll
      for (int i = 0; i < n; ++i)
        add[i] = T.l0[i] * val[0][c] + T.d0[i] * gnn[0][c] + T.l1[i] * val[1][c] + T.d1[i] * gnn[1][c];
      if (d == 2) {
#pragma unroll
        for (int i = 0; i < n; ++i) y[c][i] += add[i];
      } else {
        st_row<n>(R + c * CST + b * PS + a * RS, add);
      }
    }
    if (d != 2) {
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int z = 0; z < n; ++z)
          y[c][z] += (d == 0) ? R[c * CST + z * PS + b * RS + a] : R[c * CST + z * PS + a * RS + b];
    }
  }

  if (active) {
    const size_t off = (size_t)cell * 3 * n3;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) A.dst[off + c * n3 + z * n2 + p] = y[c][z];
  }
}

}  // namespace dgvv
