// newton_apply3.cuh — K2 v3: Newton-linearised SIPG viscous apply on Cartesian cells from stored
// quadrature-point data of the linearisation point (reading G10):
//   J(u0) w = a(., w; nu0) + a(., u0; dnu[w]),   dnu = 2 g(gd0) eps(u0):eps(w).
// Everything that depends on u0 alone is fixed between two dgvv_update_viscosity calls, so it is
// derived once per linearisation (the paper's strategy for the viscosity) by
// newton_pointdata_kernel:
//   cell points:      S0 = grad u0 + grad u0^T (6 values), g = eta'(gd0)/gd0;
//   own face points:  S0 and g from this side's trace gradient (G8), and the trace u0 itself.
// The apply then needs only w: dnu = (g/2) S0:Sw with Sw = grad w + grad w^T, the effective stress
// nu0 Sw/2 + dnu S0/2, the effective jump nu0 [w] + dnu [u0] and the penalties tau(nu0)[w],
// tau(dnu)[u0] — no u0 staging, no u0 gradients, no u0 neighbour traces (v2 recomputed all of them
// every apply).  Team of n^2 threads per cell, padded smem, faces one at a time, no atomics.
#pragma once
#include "common.cuh"
#include "sipg_apply2.cuh"

namespace dgvv {

// layout of the stored point data
template <int n>
struct NewtonPD {
  static constexpr int n2 = n * n, n3 = n * n * n;
  static constexpr int CELL = 7 * n3;        // [cell][7][n^3]: S0xx S0yy S0zz S0xy S0xz S0yz g
  static constexpr int FACE = 6 * 10 * n2;   // [cell][6][10][n^2]: S0 (6), g, u0 trace (3)
};

// one thread per owned cell point or (owned or ghost) own-face point
template <int n>
__global__ void newton_pointdata_kernel(const ApplyArgs A, int n_total, double* pc, double* pf) {
  constexpr int n2 = n * n, n3 = n2 * n;
  using P = NewtonPD<n>;
  const Tab1D& T = c_tab[n];
  const double eta_inf = A.law[1], lam2 = A.law[2] * A.law[2], gfac = (A.law[3] - 1.0) * lam2;
  const long nvol = (long)A.n_owned * n3, nfac = (long)n_total * 6 * n2;
  for (long it = (long)blockIdx.x * blockDim.x + threadIdx.x; it < nvol + nfac; it += (long)gridDim.x * blockDim.x) {
    double G[3][3];
    double nu0, tr[3] = {0.0, 0.0, 0.0};
    size_t obase;
    int ostride;
    if (it < nvol) {
      const int cell = (int)(it / n3), q = (int)(it % n3);
      const int x = q % n, yy = (q / n) % n, z = q / n2;
      const double* u = A.ulin + (size_t)cell * 3 * n3;
      const double* cg = A.cart + (size_t)cell * CART_STRIDE;
      for (int c = 0; c < 3; ++c) {
        double g0 = 0.0, g1 = 0.0, g2 = 0.0;
        for (int k = 0; k < n; ++k) {
          g0 = fma(T.D[x * DGVV_NMAX + k], u[c * n3 + z * n2 + yy * n + k], g0);
          g1 = fma(T.D[yy * DGVV_NMAX + k], u[c * n3 + z * n2 + k * n + x], g1);
          g2 = fma(T.D[z * DGVV_NMAX + k], u[c * n3 + k * n2 + yy * n + x], g2);
        }
        G[c][0] = g0 * cg[0]; G[c][1] = g1 * cg[1]; G[c][2] = g2 * cg[2];
      }
      nu0 = A.nu_cell[(size_t)cell * n3 + q];
      obase = (size_t)cell * P::CELL + q;
      ostride = n3;
    } else {
      const long j = it - nvol;
      const int cell = (int)(j / (6 * n2)), f = (int)((j / n2) % 6), p = (int)(j % n2);
      const int a = p % n, b = p / n, d = f >> 1, s = f & 1;
      const int t1 = face_t1(d), t2 = face_t2(d);
      const double* u = cell < A.n_owned ? A.ulin + (size_t)cell * 3 * n3
                                         : A.ulin_ghost + (size_t)(cell - A.n_owned) * 3 * n3;
      const double* cg = A.cart + (size_t)cell * CART_STRIDE;
      const double* lS = s ? T.l1 : T.l0;
      const double* dS = s ? T.d1 : T.d0;
      auto line = [&](int c, int aa, int bb, int i) {     // point i of the normal line through (aa, bb)
        const int idx = (d == 2) ? i * n2 + bb * n + aa : (d == 0 ? bb * n2 + aa * n + i : bb * n2 + i * n + aa);
        return u[c * n3 + idx];
      };
      auto trace = [&](int c, int aa, int bb) {
        double v = 0.0;
        for (int i = 0; i < n; ++i) v = fma(lS[i], line(c, aa, bb, i), v);
        return v;
      };
      for (int c = 0; c < 3; ++c) {
        double gn = 0.0, gt1 = 0.0, gt2 = 0.0;
        for (int i = 0; i < n; ++i) gn = fma(dS[i], line(c, a, b, i), gn);
        for (int k = 0; k < n; ++k) {
          gt1 = fma(T.D[a * DGVV_NMAX + k], trace(c, k, b), gt1);
          gt2 = fma(T.D[b * DGVV_NMAX + k], trace(c, a, k), gt2);
        }
        G[c][d] = gn * cg[d];
        G[c][t1] = gt1 * cg[t1];
        G[c][t2] = gt2 * cg[t2];
        tr[c] = trace(c, a, b);
      }
      nu0 = A.nu_face[((size_t)cell * 6 + f) * n2 + p];
      obase = ((size_t)cell * 6 + f) * 10 * n2 + p;
      ostride = n2;
    }
    double S[3][3], e00 = 0.0;
    for (int c = 0; c < 3; ++c)
      for (int k = 0; k < 3; ++k) {
        S[c][k] = G[c][k] + G[k][c];
        e00 = fma(0.25 * S[c][k], S[c][k], e00);
      }
    const double g = gfac * (nu0 - eta_inf) / (1.0 + lam2 * 2.0 * e00);
    double* o = it < nvol ? pc : pf;
    o[obase + 0 * ostride] = S[0][0];
    o[obase + 1 * ostride] = S[1][1];
    o[obase + 2 * ostride] = S[2][2];
    o[obase + 3 * ostride] = S[0][1];
    o[obase + 4 * ostride] = S[0][2];
    o[obase + 5 * ostride] = S[1][2];
    o[obase + 6 * ostride] = g;
    if (it >= nvol)
      for (int c = 0; c < 3; ++c) o[obase + (7 + c) * ostride] = tr[c];
  }
}

template <int n>
struct Newton3Cfg {
  using L = Lay<n>;
  static constexpr int VOL = 3 * L::CST;
  static constexpr int FB = 8 * L::FA;           // w traces [m|p][3] + G1, G2T (comp d)
  static constexpr int RW = (2 * VOL > VOL + FB) ? 2 * VOL : VOL + FB;
  static constexpr int CS = VOL + RW;
};

// symmetric 3x3 from the stored 6 values at stride st
__device__ __forceinline__ void load_sym(const double* p, int st, double (&S)[3][3]) {
  S[0][0] = __ldg(p); S[1][1] = __ldg(p + st); S[2][2] = __ldg(p + 2 * st);
  S[0][1] = S[1][0] = __ldg(p + 3 * st);
  S[0][2] = S[2][0] = __ldg(p + 4 * st);
  S[1][2] = S[2][1] = __ldg(p + 5 * st);
}

template <int n, int CPB, int MINB>
__global__ void __launch_bounds__(CPB * n * n, MINB) newton_apply3_kernel(const ApplyArgs A) {
  using L = Lay<n>;
  using Cf = Newton3Cfg<n>;
  using P = NewtonPD<n>;
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

  double* sw = smem + lc * Cf::CS;       // w [3][z][y][x]
  double* R = sw + VOL;                  // W1 | W2T (volume);  Y | face buffers (faces)
  {
    const double* gw = A.src + (size_t)cell * 3 * n3;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) sw[c * CST + z * PS + b * RS + a] = __ldg(gw + c * n3 + z * n2 + p);
  }
  const double* cg = A.cart + (size_t)cell * CART_STRIDE;
  const double ih[3] = {cg[0], cg[1], cg[2]};
  const double Hm = cg[3], vol = cg[4];
  int nbf[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) nbf[f] = __ldg(A.nbr + cell * 6 + f);
  __syncthreads();

  double y[3][n];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int z = 0; z < n; ++z)          // Helmholtz mass term (the mass part of J is M itself)
      y[c][z] = A.mass == 0.0 ? 0.0 : A.mass * T.w[a] * T.w[b] * T.w[z] * vol * sw[c * CST + z * PS + b * RS + a];

  // =============================================================== volume
  {
    double Da[n], Db[n];
    ld_row<n>(sD + a * RS, Da);
    ld_row<n>(sD + b * RS, Db);
    const double wab = T.w[a] * T.w[b] * vol;
#pragma unroll 1
    for (int z = 0; z < n; ++z) {
      const int q = z * n2 + p;
      double G[3][3];                    // physical gradient of w
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double* s = sw + c * CST;
        G[c][0] = rowdot<n>(s + z * PS + b * RS, Da) * ih[0];
        double sy = 0.0, sz = 0.0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          sy = fma(Db[k], s[z * PS + k * RS + a], sy);
          sz = fma(T.D[z * DGVV_NMAX + k], s[k * PS + b * RS + a], sz);
        }
        G[c][1] = sy * ih[1];
        G[c][2] = sz * ih[2];
      }
      double S0[3][3];
      const double* pcq = A.npc + (size_t)cell * P::CELL + q;
      load_sym(pcq, n3, S0);
      const double g = __ldg(pcq + 6 * n3);
      double ss = 0.0;                   // S0 : Sw
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int j = 0; j < 3; ++j) ss = fma(S0[c][j], G[c][j] + G[j][c], ss);
      const double nu0 = A.nu_cell[(size_t)cell * n3 + q];
      const double dnu = 0.5 * g * ss;   // 2 g eps(u0):eps(w)
      const double jxw = wab * T.w[z];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double F[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) F[j] = jxw * (nu0 * (G[c][j] + G[j][c]) + dnu * S0[c][j]) * ih[j];
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
  // buffers: w trace arrays [side m|p][c] at R + VOL + (side*3+c)*FA; G1 at +6 FA, G2T at +7 FA
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
      // stored data of both sides first (one round trip)
      const double num = A.nu_face[((size_t)cell * 6 + f) * n2 + p];
      const double* pfm = A.npf + ((size_t)cell * 6 + f) * 10 * n2 + p;
      double S0[2][3][3], g0[2], u0m[3], u0p[3];
      load_sym(pfm, n2, S0[0]);
      g0[0] = __ldg(pfm + 6 * n2);
#pragma unroll
      for (int c = 0; c < 3; ++c) u0m[c] = __ldg(pfm + (7 + c) * n2);
      double nup = num, Hp = Hm, ihp[3] = {ih[0], ih[1], ih[2]};
      if (inter) {
        const double* cgp = A.cart + (size_t)nbv * CART_STRIDE;
        ihp[0] = cgp[0]; ihp[1] = cgp[1]; ihp[2] = cgp[2]; Hp = cgp[3];
        nup = A.nu_face[((size_t)nbv * 6 + (f ^ 1)) * n2 + p];
        const double* pfp = A.npf + ((size_t)nbv * 6 + (f ^ 1)) * 10 * n2 + p;
        load_sym(pfp, n2, S0[1]);
        g0[1] = __ldg(pfp + 6 * n2);
#pragma unroll
        for (int c = 0; c < 3; ++c) u0p[c] = __ldg(pfp + (7 + c) * n2);
      } else {                            // Dirichlet mirror (G7): u0+ = -u0-, grad u0+ = grad u0-
#pragma unroll
        for (int c = 0; c < 3; ++c) u0p[c] = -u0m[c];
      }
      // own and neighbour traces of w
      double um[3], dm[3], up[3], dp[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double x[n];
        const double* s_ = sw + c * CST;
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
        um[c] = v; dm[c] = gg;
      }
      if (inter) {
        const double* lO = s ? T.l0 : T.l1;
        const double* dO = s ? T.d0 : T.d1;
        const int sl = lc + (nbv - cell);
        const bool in_cta = sl >= 0 && sl < CPB && sid[sl] == nbv;
        const double* pn = nbv < A.n_owned ? A.src + (size_t)nbv * 3 * n3 : A.ghost + (size_t)(nbv - A.n_owned) * 3 * n3;
        const double* ns = smem + (in_cta ? sl : 0) * Cf::CS;
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
          up[c] = v; dp[c] = gg;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) { up[c] = -um[c]; dp[c] = dm[c]; }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        FBm[c * FA + b * RS + a] = um[c];
        FBm[(3 + c) * FA + b * RS + a] = up[c];
      }
      __syncthreads();

      // per side: gradient of w, dnu = (g/2) S0:Sw, column d of nu0 Sw/2 + dnu S0/2
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
          double G[3][3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double* tr = FBm + (side * 3 + c) * FA;
            double g2 = 0.0;
#pragma unroll
            for (int k = 0; k < n; ++k) g2 = fma(Db[k], tr[k * RS + a], g2);
            G[c][d] = (side ? dp[c] : dm[c]) * ihs[d];
            G[c][t1] = rowdot<n>(tr + b * RS, Da) * ihs[t1];
            G[c][t2] = g2 * ihs[t2];
          }
          double ss = 0.0;
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int j = 0; j < 3; ++j) ss = fma(S0[side][c][j], G[c][j] + G[j][c], ss);
          const double nu0 = side ? nup : num;
          const double dnu = 0.5 * g0[side] * ss;
          dnuS[side] = dnu;
#pragma unroll
          for (int c = 0; c < 3; ++c) Sn[side][c] = 0.5 * (nu0 * (G[c][d] + G[d][c]) + dnu * S0[side][c][d]);
        }
      }
      const double sgn = s ? 1.0 : -1.0;
      const double dA = T.w[a] * T.w[b] * vol * ih[d];
      const double hm = A.pen * fmax(Hm, Hp);
      const double tw = hm * 0.5 * (num + nup), t0 = hm * 0.5 * (dnuS[0] + dnuS[1]);
      double gt1 = 0.0, gt2 = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double jw = um[c] - up[c], j0 = u0m[c] - u0p[c];
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
      FBm[6 * FA + b * RS + a] = gt1;
      FBm[7 * FA + a * RS + b] = gt2;
      __syncthreads();
      {
        double DTa[n], DTb[n];
        ld_row<n>(sDT + a * RS, DTa);
        ld_row<n>(sDT + b * RS, DTb);
        val[s][d] += rowdot<n>(FBm + 6 * FA + b * RS, DTa) + rowdot<n>(FBm + 7 * FA + a * RS, DTb);
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
