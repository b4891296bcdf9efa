"""Viscosity laws and shear rate (oracle).  Test infrastructure only — see oracle/__init__.py.

PAPER.md:172-176 (§2): shear rate  gamma_dot = sqrt(2 grad^S u : grad^S u).
PAPER.md:180-195 (§2, eqn:viscosity_general): generalized Newtonian law
    eta(gd) = eta_inf + (eta_0 - eta_inf) [kappa + (lambda gd)^a]^((b-1)/a);
Carreau is kappa = 1, a = 2, b = n (reading G9).
Analytic fields of the BASELINE configurations:
    C1 nu = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z)
    C2 nu = exp(ln(100) (x+y+z)/3)
    C4 c  = exp(-ln(1e4) (x+y+z)/3)         (reading G16)
"""
from __future__ import annotations

import numpy as np


def shear_rate(eps: np.ndarray) -> np.ndarray:
    """gamma_dot = sqrt(2 eps:eps) for eps [..., 3, 3]."""
    return np.sqrt(2.0 * np.einsum("...ij,...ij->...", eps, eps))


def generalized_newtonian(gd, eta0, eta_inf, lam, a, b, kappa):
    """eqn:viscosity_general, written out literally."""
    return eta_inf + (eta0 - eta_inf) * (kappa + (lam * gd) ** a) ** ((b - 1.0) / a)


def carreau(gd, eta0, eta_inf, lam, n):
    """Carreau: kappa = 1, a = 2, b = n (G9)."""
    return generalized_newtonian(gd, eta0, eta_inf, lam, 2.0, n, 1.0)


def carreau_g(gd, eta0, eta_inf, lam, n):
    """g = eta'(gd)/gd for Carreau (G10), finite at gd = 0:
    eta' = (eta0-eta_inf) (n-1) lam^2 gd (1 + (lam gd)^2)^((n-3)/2)."""
    return (eta0 - eta_inf) * (n - 1.0) * lam ** 2 * (1.0 + (lam * gd) ** 2) ** ((n - 3.0) / 2.0)


def analytic(law: dict, x: np.ndarray) -> np.ndarray:
    """Evaluate an analytic coefficient law at physical points x [..., 3]."""
    kind = law["kind"]
    if kind == "const":
        return np.full(x.shape[:-1], float(law["value"]))
    if kind == "sin3":   # C1
        return law.get("mean", 1.0) + law.get("amp", 0.5) * (
            np.sin(2 * np.pi * x[..., 0]) * np.sin(2 * np.pi * x[..., 1]) * np.sin(2 * np.pi * x[..., 2]))
    if kind == "exp":    # C2 (rate = ln(100)/3), C4 (rate = -ln(1e4)/3)
        return np.exp(law["rate"] * (x[..., 0] + x[..., 1] + x[..., 2]))
    if kind == "affine":  # P6 manufactured-solution pin: nu = c0 + g . x
        return law["c0"] + x @ np.asarray(law["grad"], dtype=np.float64)
    raise ValueError(kind)


C1_LAW = {"kind": "sin3", "mean": 1.0, "amp": 0.5}
C2_LAW = {"kind": "exp", "rate": np.log(100.0) / 3.0}
C4_LAW = {"kind": "exp", "rate": -np.log(1.0e4) / 3.0}
C3_CARREAU = {"kind": "carreau", "eta0": 1.0, "eta_inf": 1.0e-3, "lam": 1.0, "n": 0.5}
C5_CARREAU = {"kind": "carreau", "eta0": 1.0, "eta_inf": 1.0e-4, "lam": 10.0, "n": 0.5}
