// tables.cpp — see tables.h.
#include "tables.h"

#include <cmath>
#include <cstring>

namespace dgvv {

// Legendre P_n(t) and P_n'(t) by the three-term recurrence.
static void legendre(int n, long double t, long double* P, long double* dP) {
  long double p0 = 1.0L, p1 = t;
  if (n == 0) { *P = 1.0L; *dP = 0.0L; return; }
  for (int k = 2; k <= n; ++k) {
    long double pk = ((2.0L * k - 1.0L) * t * p1 - (k - 1.0L) * p0) / k;
    p0 = p1;
    p1 = pk;
  }
  *P = p1;
  *dP = n * (t * p1 - p0) / (t * t - 1.0L);
}

void gauss01(int n, double* x, double* w) {
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < n; ++i) {
    long double t = -cosl(pi * (i + 0.75L) / (n + 0.5L));  // ascending initial guess
    for (int it = 0; it < 100; ++it) {
      long double P, dP;
      legendre(n, t, &P, &dP);
      long double dt = P / dP;
      t -= dt;
      if (fabsl(dt) < 1e-19L) break;
    }
    long double P, dP;
    legendre(n, t, &P, &dP);
    x[i] = (double)(0.5L * (1.0L + t));
    w[i] = (double)(1.0L / ((1.0L - t * t) * dP * dP));      // 2/((1-t^2)P'^2) / 2
  }
}

void gll01(int m, double* x) {
  const long double pi = 3.141592653589793238462643383279502884L;
  x[0] = 0.0;
  x[m] = 1.0;
  for (int i = 1; i < m; ++i) {
    long double t = -cosl(pi * i / m);
    for (int it = 0; it < 100; ++it) {
      long double P, dP;
      legendre(m, t, &P, &dP);
      // P'' from the Legendre ODE: (1-t^2) P'' = 2 t P' - m(m+1) P
      long double d2P = (2.0L * t * dP - m * (m + 1.0L) * P) / (1.0L - t * t);
      long double dt = dP / d2P;
      t -= dt;
      if (fabsl(dt) < 1e-19L) break;
    }
    x[i] = (double)(0.5L * (1.0L + t));
  }
}

void lagrange_at(const double* nodes, int np, double x, double* val, double* der) {
  // barycentric weights
  long double bw[DGVV_NMAX];
  for (int i = 0; i < np; ++i) {
    long double p = 1.0L;
    for (int j = 0; j < np; ++j)
      if (j != i) p *= ((long double)nodes[i] - nodes[j]);
    bw[i] = 1.0L / p;
  }
  int hit = -1;
  for (int i = 0; i < np; ++i)
    if ((long double)x == (long double)nodes[i]) hit = i;
  if (hit < 0) {
    // l_i(x) = l(x) bw_i / (x - x_i), l(x) = prod (x - x_j);  l_i'(x) = l_i(x) sum_{j != i} 1/(x - x_j)
    long double l = 1.0L;
    for (int j = 0; j < np; ++j) l *= ((long double)x - nodes[j]);
    for (int i = 0; i < np; ++i) {
      long double li = l * bw[i] / ((long double)x - nodes[i]);
      long double s = 0.0L;
      for (int j = 0; j < np; ++j)
        if (j != i) s += 1.0L / ((long double)x - nodes[j]);
      val[i] = (double)li;
      der[i] = (double)(li * s);
    }
  } else {
    // at a node: l_i = delta; derivative by the differentiation-matrix formula
    long double dsum = 0.0L;
    for (int i = 0; i < np; ++i) {
      val[i] = (i == hit) ? 1.0 : 0.0;
      if (i != hit) {
        long double d = (bw[i] / bw[hit]) / ((long double)nodes[hit] - nodes[i]);
        der[i] = (double)d;
        dsum += d;
      }
    }
    der[hit] = (double)(-dsum);
  }
}

void make_tab(int n, Tab1D* t) {
  std::memset(t, 0, sizeof(Tab1D));
  gauss01(n, t->x, t->w);
  for (int q = 0; q < n; ++q) {
    double v[DGVV_NMAX], d[DGVV_NMAX];
    lagrange_at(t->x, n, t->x[q], v, d);
    for (int i = 0; i < n; ++i) t->D[q * DGVV_NMAX + i] = d[i];
  }
  lagrange_at(t->x, n, 0.0, t->l0, t->d0);
  lagrange_at(t->x, n, 1.0, t->l1, t->d1);
}

void transfer_matrix(int nf, int nc, double* P1) {
  double xf[DGVV_NMAX], wf[DGVV_NMAX], xc[DGVV_NMAX], wc[DGVV_NMAX];
  gauss01(nf, xf, wf);
  gauss01(nc, xc, wc);
  for (int i = 0; i < nf; ++i) {
    double v[DGVV_NMAX], d[DGVV_NMAX];
    lagrange_at(xc, nc, xf[i], v, d);
    for (int j = 0; j < nc; ++j) P1[i * nc + j] = v[j];
  }
}

void make_geotab(int m, int n, GeoTab* g) {
  std::memset(g, 0, sizeof(GeoTab));
  g->m = m;
  g->n = n;
  double gn[DGVV_NMAX];
  gll01(m, gn);
  gauss01(n, g->x, g->w);
  for (int q = 0; q < n; ++q) lagrange_at(gn, m + 1, g->x[q], g->L[q], g->dL[q]);
  lagrange_at(gn, m + 1, 0.0, g->E[0], g->dE[0]);
  lagrange_at(gn, m + 1, 1.0, g->E[1], g->dE[1]);
}

}  // namespace dgvv
