"""1D bases and quadrature (oracle).  Test infrastructure only — see oracle/__init__.py.

PAPER.md:592-596 (§4): Q_k on the reference hexahedron "constructed by tensor-product shape
functions"; PAPER.md:1523-1527 (§5.3): operator action "realized via numerical quadrature".
Readings: G1 Gauss-Legendre with n_q = k+1 points per direction;
G2 Lagrange basis on the k+1 Gauss points.  The reference interval is [0,1].
"""
from __future__ import annotations

import numpy as np


def gauss01(n: int):
    """n-point Gauss-Legendre rule on [0,1] (G1).  numpy.leggauss is the library primitive."""
    t, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (1.0 + t), 0.5 * w


def gll01(m: int) -> np.ndarray:
    """Gauss-Lobatto points of degree m on [0,1]: endpoints and roots of P_m' (geometry nodes)."""
    if m == 1:
        return np.array([0.0, 1.0])
    c = np.zeros(m + 1)
    c[m] = 1.0
    r = np.polynomial.legendre.Legendre(c).deriv().roots().real
    return 0.5 * (1.0 + np.concatenate([[-1.0], np.sort(r), [1.0]]))


def lagrange(nodes: np.ndarray, x) -> np.ndarray:
    """L[p, i] = l_i(x_p) = prod_{j != i} (x_p - x_j) / (x_i - x_j)  (product formula)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = len(nodes)
    L = np.ones((len(x), n))
    for i in range(n):
        for j in range(n):
            if j != i:
                L[:, i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
    return L


def lagrange_deriv(nodes: np.ndarray, x) -> np.ndarray:
    """dL[p, i] = l_i'(x_p) = sum_{m != i} 1/(x_i - x_m) prod_{j != i, m} (x_p - x_j)/(x_i - x_j)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = len(nodes)
    dL = np.zeros((len(x), n))
    for i in range(n):
        for m in range(n):
            if m == i:
                continue
            term = np.full(len(x), 1.0 / (nodes[i] - nodes[m]))
            for j in range(n):
                if j != i and j != m:
                    term *= (x - nodes[j]) / (nodes[i] - nodes[j])
            dL[:, i] += term
    return dL


def tensor_points(xi: np.ndarray) -> np.ndarray:
    """All 3D points of a tensor rule, lexicographic with x fastest: [n^3, 3]."""
    gz, gy, gx = np.meshgrid(xi, xi, xi, indexing="ij")
    return np.stack([gx.reshape(-1), gy.reshape(-1), gz.reshape(-1)], axis=-1)


def tensor_weights(w: np.ndarray) -> np.ndarray:
    wz, wy, wx = np.meshgrid(w, w, w, indexing="ij")
    return (wx * wy * wz).reshape(-1)


def tabulate(nodes: np.ndarray, pts: np.ndarray):
    """Full-tensor tabulation of the 3D tensor Lagrange basis on `nodes` at 3D points pts [P,3].

    Returns Phi[P, N] with N = n^3 basis functions (index i = ix + n iy + n^2 iz) and
    dPhi[3, P, N] = d phi_i / d xi_d.  Dense — no sum factorisation.
    """
    n = len(nodes)
    Lx, Ly, Lz = (lagrange(nodes, pts[:, d]) for d in range(3))
    dLx, dLy, dLz = (lagrange_deriv(nodes, pts[:, d]) for d in range(3))
    idx = np.arange(n ** 3)
    ix, iy, iz = idx % n, (idx // n) % n, idx // (n * n)
    Phi = Lx[:, ix] * Ly[:, iy] * Lz[:, iz]
    dPhi = np.stack([dLx[:, ix] * Ly[:, iy] * Lz[:, iz],
                     Lx[:, ix] * dLy[:, iy] * Lz[:, iz],
                     Lx[:, ix] * Ly[:, iy] * dLz[:, iz]])
    return Phi, dPhi


FACE_AXES = {0: (1, 2), 1: (0, 2), 2: (0, 1)}   # tangential axes of a face with normal axis d


def face_points(xi: np.ndarray, f: int) -> np.ndarray:
    """Reference points of local face f (0..5 = -x,+x,-y,+y,-z,+z) for a 1D rule xi:
    lexicographic over the two tangential axes in increasing axis order, first fastest."""
    d, s = f // 2, f % 2
    t1, t2 = FACE_AXES[d]
    gb, ga = np.meshgrid(xi, xi, indexing="ij")
    P = np.zeros((len(xi) ** 2, 3))
    P[:, d] = float(s)
    P[:, t1] = ga.reshape(-1)
    P[:, t2] = gb.reshape(-1)
    return P


def face_weights(w: np.ndarray) -> np.ndarray:
    wb, wa = np.meshgrid(w, w, indexing="ij")
    return (wa * wb).reshape(-1)
