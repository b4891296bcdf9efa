// convective_apply.cuh — §8(f) f4: the upwind DG convective term (PAPER.md:686-711,
// eqn:convective_term_weak):  dst (+)= alpha * C(w) u  with
//   c_h^e(v, u; w) = (v, (w.grad) u)_e + (v, min({{w}}.n, 0) (u(nb) - u(e)))_{de}
// (readings F4a-F4c: (w.grad)u form; Dirichlet faces carry {{w}} = 0 under the
// mirror state, Neumann faces have no jump, so only interior/periodic faces contribute).
// With the collocation basis (G2) the volume test functions are point values: no transposed
// contraction, y_c(q) += alpha JxW_q (w.grad u_c)(q).  The transport field enters only through
// quadrature-point data derived once per field (conv_pointdata_kernel), used by the standalone
// apply below and by the fused viscous + convective apply (sipg_apply2.cuh, CONV).
#pragma once
#include "common.cuh"
#include "sipg_apply2.cuh"

namespace dgvv {

// Quadrature-point data of the convective term for the fused viscous + convective apply
// (sipg_apply2.cuh, CONV), derived once per transport field (the analogue of the stored viscosity):
//   wref[cell][k][q]  = JxW_q sum_j Ji[k][j](q) w_j(q)     (reference transport direction times JxW)
//   wface[cell][f][p] = min({{w}}.n, 0) dA                  (own side; 0 on boundary faces, F4b)
// One thread per cell point / face point, plain global loads (setup-time kernel).
template <int n, int GEO>
__global__ void conv_pointdata_kernel(const ConvArgs A, double* wref, double* wface) {
  constexpr int n2 = n * n, n3 = n2 * n;
  const Tab1D& T = c_tab[n];
  const long nvol = (long)A.n_owned * n3, nfac = (long)A.n_owned * 6 * n2;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nvol + nfac; i += (long)gridDim.x * blockDim.x) {
    if (i < nvol) {
      const int cell = (int)(i / n3), q = (int)(i % n3);
      const int a = q % n, b = (q / n) % n, z = q / n2;
      const double* w = A.w + (size_t)cell * 3 * n3 + q;
      const double w0 = w[0], w1 = w[n3], w2 = w[2 * n3];
      double r[3];
      if constexpr (GEO == 0) {
        const double* cg = A.cart + (size_t)cell * CART_STRIDE;
        const double jxw = T.w[a] * T.w[b] * T.w[z] * cg[4];
        r[0] = jxw * cg[0] * w0; r[1] = jxw * cg[1] * w1; r[2] = jxw * cg[2] * w2;
      } else {
        const double* Ji = A.vJi + (size_t)cell * 9 * n3 + q;
        const double jxw = A.jxw[(size_t)cell * n3 + q];
#pragma unroll
        for (int k = 0; k < 3; ++k) r[k] = jxw * (Ji[(3 * k) * n3] * w0 + Ji[(3 * k + 1) * n3] * w1 + Ji[(3 * k + 2) * n3] * w2);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) wref[(size_t)cell * 3 * n3 + k * n3 + q] = r[k];
    } else {
      const long j = i - nvol;
      const int cell = (int)(j / (6 * n2)), f = (int)((j / n2) % 6), p = (int)(j % n2);
      const int a = p % n, b = p / n, d = f >> 1, s = f & 1;
      const int nbv = A.nbr[cell * 6 + f];
      double out = 0.0;
      if (nbv >= 0) {
        const double* wo = A.w + (size_t)cell * 3 * n3;
        const double* wn = nbv < A.n_owned ? A.w + (size_t)nbv * 3 * n3 : A.wghost + (size_t)(nbv - A.n_owned) * 3 * n3;
        const double* lS = s ? T.l1 : T.l0;
        const double* lO = s ? T.l0 : T.l1;
        const double sgn = s ? 1.0 : -1.0;
        auto trace = [&](const double* base, int c, const double* l) {
          double v = 0.0;
          for (int ii = 0; ii < n; ++ii) {
            const int idx = (d == 2) ? ii * n2 + p : (d == 0 ? b * n2 + a * n + ii : b * n2 + ii * n + a);
            v = fma(l[ii], base[c * n3 + idx], v);
          }
          return v;
        };
        double wnv, dA;
        if constexpr (GEO == 0) {
          const double* cg = A.cart + (size_t)cell * CART_STRIDE;
          wnv = 0.5 * (trace(wo, d, lS) + trace(wn, d, lO)) * sgn;
          dA = T.w[a] * T.w[b] * cg[4] * cg[d];
        } else {
          const double* fm = A.fJi + ((size_t)cell * 6 + f) * 9 * n2 + p;
          const double v0 = fm[(3 * d) * n2], v1 = fm[(3 * d + 1) * n2], v2 = fm[(3 * d + 2) * n2];
          const double il = sgn * rsqrt(v0 * v0 + v1 * v1 + v2 * v2);
          const double nr[3] = {v0 * il, v1 * il, v2 * il};
          wnv = 0.0;
          for (int c = 0; c < 3; ++c) wnv += 0.5 * (trace(wo, c, lS) + trace(wn, c, lO)) * nr[c];
          dA = A.fdA[((size_t)cell * 6 + f) * n2 + p];
        }
        out = wnv < 0.0 ? wnv * dA : 0.0;
      }
      wface[j] = out;
    }
  }
}

// dst (+)= alpha C(w) src from the stored point data (wref, wface of conv_pointdata_kernel): no
// geometry and no transport-field traces in the apply; the neighbour trace is read only where
// this side is an inflow side (wface != 0).  Team of n^2 threads per cell, column ownership and
// the padded smem layout of sipg_apply2.cuh.
template <int n, int CPB>
// (no register cap: 6 / 8 resident CTAs measured slower, C3 mesh 1.26 -> 1.56 / 2.07 ms)
__global__ void __launch_bounds__(CPB * n * n) convective_pd_kernel(const ConvArgs A, const double* wref,
                                                                     const double* wface) {
  using L = Lay<n>;
  constexpr int n2 = L::n2, n3 = L::n3, RS = L::RS, PS = L::PS, CST = L::CST, VOL = 3 * L::CST;
  constexpr int CS = 2 * VOL;              // u | Y
  extern __shared__ __align__(16) double csmem[];
  __shared__ __align__(16) double sD[n * RS];
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
  }
  if (p == 0) sid[lc] = active ? cell : -1;
  double* su = csmem + lc * CS;
  double* Y = su + VOL;
  double ucol[3][n], y[3][n];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int z = 0; z < n; ++z) {
      const double v = __ldg(A.src + (size_t)cell * 3 * n3 + c * n3 + z * n2 + p);
      ucol[c][z] = v;
      su[c * CST + z * PS + b * RS + a] = v;
    }
  int nbf[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) nbf[f] = __ldg(A.nbr + cell * 6 + f);
  __syncthreads();
  {
    double Da[n], Db[n];
    ld_row<n>(sD + a * RS, Da);
    ld_row<n>(sD + b * RS, Db);
#pragma unroll
    for (int z = 0; z < n; ++z) {
      const double* gw = wref + (size_t)cell * 3 * n3 + z * n2 + p;
      const double wr0 = A.alpha * __ldg(gw), wr1 = A.alpha * __ldg(gw + n3), wr2 = A.alpha * __ldg(gw + 2 * n3);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double gx = rowdot<n>(su + c * CST + z * PS + b * RS, Da);
        double gy = 0.0, gz = 0.0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          gy = fma(Db[k], su[c * CST + z * PS + k * RS + a], gy);
          gz = fma(T.D[z * DGVV_NMAX + k], ucol[c][k], gz);
        }
        y[c][z] = gx * wr0 + gy * wr1 + gz * wr2;
      }
    }
  }
#pragma unroll
  for (int dd = 0; dd < 3; ++dd) {
    const int d = (dd == 0) ? 2 : dd - 1;
    double val[2][3];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int f = 2 * d + s;
      const int nbv = nbf[f];
#pragma unroll
      for (int c = 0; c < 3; ++c) val[s][c] = 0.0;
      const double cf = nbv >= 0 ? A.alpha * __ldg(wface + ((size_t)cell * 6 + f) * n2 + p) : 0.0;
      if (cf != 0.0) {                         // inflow side of this cell: upwind from the neighbour
        const double* lS = s ? T.l1 : T.l0;
        const double* lO = s ? T.l0 : T.l1;
        const int sl = lc + (nbv - cell);
        const bool in_cta = sl >= 0 && sl < CPB && sid[sl] == nbv;
        const double* pu = nbv < A.n_owned ? A.src + (size_t)nbv * 3 * n3 : A.ghost + (size_t)(nbv - A.n_owned) * 3 * n3;
        const double* nsu = csmem + (in_cta ? sl : 0) * CS;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double um = 0.0, up = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) {
            const double xm = (d == 2) ? ucol[c][i] : (d == 0 ? su[c * CST + b * PS + a * RS + i] : su[c * CST + b * PS + i * RS + a]);
            double xp;
            if (in_cta)
              xp = (d == 2) ? nsu[c * CST + i * PS + b * RS + a]
                            : (d == 0 ? nsu[c * CST + b * PS + a * RS + i] : nsu[c * CST + b * PS + i * RS + a]);
            else
              xp = (d == 2) ? __ldg(pu + c * n3 + i * n2 + p)
                            : (d == 0 ? __ldg(pu + c * n3 + b * n2 + a * n + i) : __ldg(pu + c * n3 + b * n2 + i * n + a));
            um = fma(lS[i], xm, um);
            up = fma(lO[i], xp, up);
          }
          val[s][c] = cf * (up - um);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double add[n];
#pragma unroll
      for (int i = 0; i < n; ++i) add[i] = T.l0[i] * val[0][c] + T.l1[i] * val[1][c];
      if (d == 2) {
#pragma unroll
        for (int i = 0; i < n; ++i) y[c][i] += add[i];
      } else {
        st_row<n>(Y + c * CST + b * PS + a * RS, add);
      }
    }
    if (d != 2) {
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int z = 0; z < n; ++z) y[c][z] += (d == 0) ? Y[c * CST + z * PS + b * RS + a] : Y[c * CST + z * PS + a * RS + b];
      __syncthreads();
    }
  }
  if (active) {
    const size_t off = (size_t)cell * 3 * n3;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) {
        double* o = A.dst + off + c * n3 + z * n2 + p;
        *o = A.accumulate ? *o + y[c][z] : y[c][z];
      }
  }
}

}  // namespace dgvv
