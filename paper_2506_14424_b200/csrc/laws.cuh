// laws.cuh — coefficient laws at a point (device).  PAPER.md:172-195 (shear rate, eqn:viscosity_general),
// readings G9 (Carreau: kappa = 1, a = 2, b = n) and G10 (g = eta'/gd).
#pragma once
#include "common.cuh"

namespace dgvv {

// ----------------------------------------------------------------- laws (device)
__device__ __forceinline__ double eval_law(int kind, const double* p, double x, double y, double z) {
  const double twopi = 6.283185307179586476925286766559;
  if (kind == 0) return p[0];
  if (kind == 1) return p[0] + p[1] * sin(twopi * x) * sin(twopi * y) * sin(twopi * z);
  if (kind == 2) return exp(p[0] * (x + y + z));
  return nan("");
}

// Carreau eta(gd) = eta_inf + (eta0 - eta_inf) (1 + (lambda gd)^2)^((n-1)/2)   (G9)
// (1 + (lambda gd)^2)^e with e = (n-1)/2 as exp(e log(.)): the base is >= 1 and |e log| stays
// O(10), so the result keeps ~1e-16 relative accuracy at a fraction of pow()'s cost.
__device__ __forceinline__ double carreau_eta(const double* L, double gd) {
  const double lg = L[2] * gd;
  return L[1] + (L[0] - L[1]) * exp(0.5 * (L[3] - 1.0) * log1p(lg * lg));
}
// g = eta'(gd)/gd = (eta0-eta_inf)(n-1) lambda^2 (1+(lambda gd)^2)^((n-3)/2)    (G10)
__device__ __forceinline__ double carreau_g(const double* L, double gd) {
  const double lg = L[2] * gd;
  return (L[0] - L[1]) * (L[3] - 1.0) * L[2] * L[2] * pow(1.0 + lg * lg, 0.5 * (L[3] - 3.0));
}

}  // namespace dgvv
