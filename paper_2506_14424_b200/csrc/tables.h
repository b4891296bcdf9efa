// tables.h — host-side 1D tables (Gauss-Legendre rule, Lagrange basis on the Gauss
// points, Gauss-Lobatto geometry basis, p-transfer matrices).  Own implementation:
// Newton iteration on the Legendre three-term recurrence in long double, barycentric
// Lagrange formulas.  Shares nothing with the oracle (oracle/basis.py).
#pragma once
#include "common.cuh"

namespace dgvv {

// Gauss-Legendre points/weights of [0,1] (n points); readings G1/G2.
void gauss01(int n, double* x, double* w);
// Gauss-Lobatto points of [0,1] of degree m (m+1 points, endpoints included).
void gll01(int m, double* x);
// Fill the Tab1D of the degree n-1 collocation basis.
void make_tab(int n, Tab1D* t);
// Values / derivatives of the Lagrange basis on `nodes` (np points) at x.
void lagrange_at(const double* nodes, int np, double x, double* val, double* der);
// P1[i_f * nc + j_c] = l^(c)_j(xi^(f)_i)  (reading G18)
void transfer_matrix(int nf, int nc, double* P1);

struct GeoTab {                 // geometry basis (degree m GLL Lagrange) at the Gauss points
  int m, n;
  double L[DGVV_NMAX][DGVV_NMAX];    // L[q][a]  = L_a(x_q)
  double dL[DGVV_NMAX][DGVV_NMAX];   // dL[q][a] = L_a'(x_q)
  double E[2][DGVV_NMAX];            // L_a(0), L_a(1)
  double dE[2][DGVV_NMAX];           // L_a'(0), L_a'(1)
  double w[DGVV_NMAX];               // Gauss weights
  double x[DGVV_NMAX];               // Gauss points
};
void make_geotab(int m, int n, GeoTab* g);

}  // namespace dgvv
