// penalty_apply.cuh — §8(f) f2: the divergence/continuity penalty-step operator
// (eqn:penalty_step), homogeneous part, per cell e:
//   (v, u)_e + (div v, tau_div^e div u)_e + (v.n, tau_F [[u]].n)_{boundary of e}
// [[u]] = u(e) - u(neighbour) on interior/periodic faces, u on Dirichlet faces, no Neumann term;
// tau_F = (tau_cont^- + tau_cont^+)/2 on interior faces, the cell's own tau_cont on Dirichlet
// faces (readings P1/P2).  Same cell-centric structure and shared-memory layout as
// sipg_apply2.cuh (team of n^2 threads per cell, z-columns in registers, no atomics); the face
// terms need values only (no derivatives), on Cartesian cells only the normal component.
#pragma once
#include "common.cuh"
#include "sipg_apply2.cuh"

namespace dgvv {

// PenaltyArgs: see common.cuh

template <int n, int GEO>
struct PenaltyCfg {
  using L = Lay<n>;
  static constexpr int VOL = 3 * L::CST;
  static constexpr int CS = 3 * VOL;       // su | W1 W2T (volume) ; Y (faces)
};

template <int n, int GEO, int CPB>
#ifndef DGVV_PEN_MINB
#define DGVV_PEN_MINB 5   // min resident CTAs per SM (register cap), chosen by measurement:
                          // C2 0.206 -> 0.194 ms, C3 mesh 1.70 -> 1.54 ms (6: 0.242 / 1.65)
#endif
__global__ void __launch_bounds__(CPB * n * n, DGVV_PEN_MINB) penalty_apply_kernel(const PenaltyArgs A) {
  using L = Lay<n>;
  using Cf = PenaltyCfg<n, GEO>;
  constexpr int n2 = L::n2, n3 = L::n3, RS = L::RS, PS = L::PS, CST = L::CST, VOL = Cf::VOL;
  extern __shared__ __align__(16) double psmem[];
  __shared__ __align__(16) double sD[n * RS];
  __shared__ __align__(16) double sDT[n * RS];
  __shared__ int sid[CPB];
  const Tab1D& T = c_tab[n];
  const int lc = threadIdx.x / n2;
  const int p = threadIdx.x - lc * n2;
  const int a = p % n, b = p / n;
  const int slot_raw = blockIdx.x * CPB + lc;
  const bool active = slot_raw < A.n_proc;
  const int cell = A.cell_base + (active ? slot_raw : A.n_proc - 1);
  for (int i = threadIdx.x; i < n * RS; i += blockDim.x) {
    const int r = i / RS, k = i - r * RS;
    sD[i] = k < n ? T.D[r * DGVV_NMAX + k] : 0.0;
    sDT[i] = k < n ? T.D[k * DGVV_NMAX + r] : 0.0;
  }
  if (p == 0) sid[lc] = active ? cell : -1;
  double* su = psmem + lc * Cf::CS;
  double* WK = su + VOL;
  double ucol[3][n], y[3][n];
  const double* gsrc = A.src + (size_t)cell * 3 * n3;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int z = 0; z < n; ++z) {
      const double v = __ldg(gsrc + c * n3 + z * n2 + p);
      ucol[c][z] = v;
      su[c * CST + z * PS + b * RS + a] = v;
    }
  double ih[3] = {0, 0, 0}, vol = 0.0;
  if constexpr (GEO == 0) {
    const double* cg = A.cart + (size_t)cell * CART_STRIDE;
    ih[0] = cg[0]; ih[1] = cg[1]; ih[2] = cg[2]; vol = cg[4];
  }
  const double tdiv = A.tau_div[cell], tcm = A.tau_cont[cell];
  int nbf[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) nbf[f] = __ldg(A.nbr + cell * 6 + f);
  __syncthreads();

  // ------------------------------------------------------------ volume: mass + div-div
  {
    double Da[n], Db[n];
    ld_row<n>(sD + a * RS, Da);
    ld_row<n>(sD + b * RS, Db);
#pragma unroll
    for (int z = 0; z < n; ++z) {
      const int q = z * n2 + p;
      double jxw, Ji[9];
      if constexpr (GEO == 0) {
        jxw = T.w[a] * T.w[b] * T.w[z] * vol;
      } else {
        jxw = A.jxw[(size_t)cell * n3 + q];
#pragma unroll
        for (int r = 0; r < 9; ++r) Ji[r] = __ldg(A.vJi + (size_t)cell * 9 * n3 + r * n3 + q);
      }
      double dv = 0.0;                       // div u at q
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double gx = rowdot<n>(su + c * CST + z * PS + b * RS, Da);
        double gy = 0.0, gz = 0.0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          gy = fma(Db[k], su[c * CST + z * PS + k * RS + a], gy);
          gz = fma(T.D[z * DGVV_NMAX + k], ucol[c][k], gz);
        }
        if constexpr (GEO == 0) dv += (c == 0 ? gx : c == 1 ? gy : gz) * ih[c];
        else dv += gx * Ji[c] + gy * Ji[3 + c] + gz * Ji[6 + c];
      }
      const double Dq = tdiv * jxw * dv;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        // coefficient of d v_c / d xi_k = Dq * Ji[k][c]
        double F[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) F[k] = (GEO == 0) ? ((k == c) ? Dq * ih[c] : 0.0) : Dq * Ji[3 * k + c];
        WK[c * CST + z * PS + b * RS + a] = F[0];
        WK[VOL + c * CST + z * PS + a * RS + b] = F[1];
#pragma unroll
        for (int z2 = 0; z2 < n; ++z2) y[c][z2] = (z == 0 ? 0.0 : y[c][z2]) + T.D[z * DGVV_NMAX + z2] * F[2];
        y[c][z] += jxw * ucol[c][z];        // mass (v, u): diagonal with collocation (G2)
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
        y[c][z] += rowdot<n>(WK + c * CST + z * PS + b * RS, DTa) + rowdot<n>(WK + VOL + c * CST + z * PS + a * RS, DTb);
    __syncthreads();
  }

  // ------------------------------------------------------------ faces: continuity penalty
#pragma unroll
  for (int dd = 0; dd < 3; ++dd) {
    const int d = (dd == 0) ? 2 : dd - 1;
    double val[2][3];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int f = 2 * d + s;
      const int nbv = nbf[f];
      const double* lS = s ? T.l1 : T.l0;
      const double* lO = s ? T.l0 : T.l1;
#pragma unroll
      for (int c = 0; c < 3; ++c) val[s][c] = 0.0;
      if (nbv >= 0 || nbv == NB_DIRICHLET) {
        double nrm[3] = {0.0, 0.0, 0.0}, dA;
        const double sgn = s ? 1.0 : -1.0;
        if constexpr (GEO == 0) {
          nrm[d] = sgn;
          dA = T.w[a] * T.w[b] * vol * ih[d];
        } else {
          const double* fm = A.fJi + ((size_t)cell * 6 + f) * 9 * n2 + p;
          const double v0 = __ldg(fm + (3 * d) * n2), v1 = __ldg(fm + (3 * d + 1) * n2), v2 = __ldg(fm + (3 * d + 2) * n2);
          const double il = sgn * rsqrt(v0 * v0 + v1 * v1 + v2 * v2);
          nrm[0] = v0 * il; nrm[1] = v1 * il; nrm[2] = v2 * il;
          dA = A.fdA[((size_t)cell * 6 + f) * n2 + p];
        }
        double jn = 0.0, tauF = tcm;
        const int sl = nbv >= 0 ? lc + (nbv - cell) : -1;
        const bool in_cta = nbv >= 0 && sl >= 0 && sl < CPB && sid[sl] == nbv;
        const double* pn = nbv < 0 ? nullptr
                           : (nbv < A.n_owned ? A.src + (size_t)nbv * 3 * n3 : A.ghost + (size_t)(nbv - A.n_owned) * 3 * n3);
        const double* ns = psmem + (in_cta ? sl : 0) * Cf::CS;
        if (nbv >= 0) tauF = 0.5 * (tcm + A.tau_cont[nbv]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (GEO == 0 && c != d) continue;
          double um = 0.0, up = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) {
            const double xo = (d == 2) ? ucol[c][i] : (d == 0 ? su[c * CST + b * PS + a * RS + i] : su[c * CST + b * PS + i * RS + a]);
            um = fma(lS[i], xo, um);
            if (nbv >= 0) {
              double xn;
              if (in_cta) xn = (d == 2) ? ns[c * CST + i * PS + b * RS + a] : (d == 0 ? ns[c * CST + b * PS + a * RS + i] : ns[c * CST + b * PS + i * RS + a]);
              else xn = (d == 2) ? __ldg(pn + c * n3 + i * n2 + p) : (d == 0 ? __ldg(pn + c * n3 + b * n2 + a * n + i) : __ldg(pn + c * n3 + b * n2 + i * n + a));
              up = fma(lO[i], xn, up);
            }
          }
          jn += (um - up) * nrm[c];
        }
        const double coef = dA * tauF * jn;
#pragma unroll
        for (int c = 0; c < 3; ++c) val[s][c] = coef * nrm[c];
      }
    }
    // extrapolate both faces' value coefficients along the normal line into the cell
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double add[n];
#pragma unroll
      for (int i = 0; i < n; ++i) add[i] = T.l0[i] * val[0][c] + T.l1[i] * val[1][c];
      if (d == 2) {
#pragma unroll
        for (int i = 0; i < n; ++i) y[c][i] += add[i];
      } else {
        st_row<n>(WK + c * CST + b * PS + a * RS, add);
      }
    }
    if (d != 2) {
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int z = 0; z < n; ++z)
          y[c][z] += (d == 0) ? WK[c * CST + z * PS + b * RS + a] : WK[c * CST + z * PS + a * RS + b];
      __syncthreads();
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

namespace dgvv {

// Inverse diagonal of the penalty operator (Jacobi): with the collocation basis (G2)
//   D_ii = JxW_i + tau_div sum_{q on the 3 grid lines through i} JxW_q (d phi_i / d x_c (q))^2
//        + sum_{faces of the cell with phi_i != 0 on them} dA tau_F phi_i^2 n_c^2      (c = comp)
template <int n, int GEO>
__global__ void penalty_diag_kernel(const PenaltyArgs A) {
  constexpr int n2 = n * n, n3 = n2 * n;
  const Tab1D& T = c_tab[n];
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)A.n_owned * 3 * n3) return;
  const int cell = idx / (3 * n3);
  const int rem = idx % (3 * n3);
  const int comp = rem / n3, i = rem % n3;
  const int iv[3] = {i % n, (i / n) % n, i / n2};
  double ih[3] = {0, 0, 0}, vol = 0;
  if (GEO == 0) {
    const double* cg = A.cart + (size_t)cell * CART_STRIDE;
    ih[0] = cg[0]; ih[1] = cg[1]; ih[2] = cg[2]; vol = cg[4];
  }
  auto jxw_at = [&](int q) {
    return GEO == 0 ? T.w[q % n] * T.w[(q / n) % n] * T.w[q / n2] * vol : A.jxw[(size_t)cell * n3 + q];
  };
  double Dv = jxw_at(i);                                  // mass
  const double tdiv = A.tau_div[cell];
  auto add_point = [&](const int (&qv)[3], const double (&gxi)[3]) {
    const int q = qv[0] + n * qv[1] + n2 * qv[2];
    double g;                                             // d phi_i / d x_comp at q
    if (GEO == 0) g = gxi[comp] * ih[comp];
    else {
      const double* vm = A.vJi + (size_t)cell * 9 * n3 + q;
      g = gxi[0] * vm[comp * n3] + gxi[1] * vm[(3 + comp) * n3] + gxi[2] * vm[(6 + comp) * n3];
    }
    Dv += tdiv * jxw_at(q) * g * g;
  };
  {
    const double gxi[3] = {T.D[iv[0] * DGVV_NMAX + iv[0]], T.D[iv[1] * DGVV_NMAX + iv[1]], T.D[iv[2] * DGVV_NMAX + iv[2]]};
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
  for (int f = 0; f < 6; ++f) {
    const int d = f / 2, s = f % 2;
    const int nb = A.nbr[cell * 6 + f];
    if (nb == NB_NEUMANN) continue;
    const int pidx = iv[face_t1(d)] + n * iv[face_t2(d)];
    const double phi = s ? T.l1[iv[d]] : T.l0[iv[d]];
    double nc2, dA;
    if (GEO == 0) {
      nc2 = (comp == d) ? 1.0 : 0.0;
      dA = T.w[iv[face_t1(d)]] * T.w[iv[face_t2(d)]] * vol * ih[d];
    } else {
      const double* fm = A.fJi + ((size_t)cell * 6 + f) * 9 * n2 + pidx;
      const double v0 = fm[(3 * d) * n2], v1 = fm[(3 * d + 1) * n2], v2 = fm[(3 * d + 2) * n2];
      const double vc = comp == 0 ? v0 : comp == 1 ? v1 : v2;
      nc2 = vc * vc / (v0 * v0 + v1 * v1 + v2 * v2);
      dA = A.fdA[((size_t)cell * 6 + f) * n2 + pidx];
    }
    const double tauF = nb >= 0 ? 0.5 * (A.tau_cont[cell] + A.tau_cont[nb]) : A.tau_cont[cell];
    Dv += dA * tauF * phi * phi * nc2;
  }
  A.dst[idx] = 1.0 / Dv;
}

}  // namespace dgvv
