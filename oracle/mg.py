"""p-multigrid pieces (oracle): transfer, Chebyshev-Jacobi smoother, V-cycle, Lanczos,
diagonal.  Test infrastructure only — see oracle/__init__.py.

PAPER.md:1531-1541 (§5.3): hp-multigrid, polynomial degree lowered level by level
(p-coarsening); readings G17 (5 -> 3 -> 2 -> 1), G18 (P = exact DG embedding, R = P^T).
PAPER.md:1553-1557: V-cycles with a Chebyshev-accelerated Jacobi smoother (Adams 2003),
inverse diagonal precomputed per level, residual via the level operator.
Readings G12-G15: degree 5, range [lambda_hi/20, lambda_hi], lambda_hi = 1.2 lambda_hat,
1 pre- + 1 post-smoothing, coarsest level = Chebyshev(5) from 0.
PAPER.md:1536-1545: after p-coarsening, h-coarsening on the grids "created by
refining an initial coarse grid" and, on the coarsest level, "a direct solver if the system size
falls below 2000 DoFs": h-transfer (readings H1-H3) and the direct coarse solve.
"""
from __future__ import annotations

import numpy as np

from . import basis as B


def transfer_1d(kf: int, kc: int) -> np.ndarray:
    """P1[i_f, j_c] = l^(kc)_j(xi^(kf)_i): coarse Lagrange basis (on the kc+1 Gauss points)
    evaluated at the fine Gauss points (G18)."""
    xf, _ = B.gauss01(kf + 1)
    xc, _ = B.gauss01(kc + 1)
    return B.lagrange(xc, xf)


def transfer_3d(kf: int, kc: int) -> np.ndarray:
    """Per-cell prolongation (n_f^3 x n_c^3), lexicographic x fastest: kron(P1, P1, P1)."""
    P1 = transfer_1d(kf, kc)
    return np.kron(P1, np.kron(P1, P1))


def prolongate(coarse, kf, kc, n_cells, ncomp=1):
    P = transfer_3d(kf, kc)
    C = coarse.reshape(n_cells * ncomp, -1)
    return (C @ P.T).reshape(-1)


def restrict(fine, kf, kc, n_cells, ncomp=1):
    P = transfer_3d(kf, kc)
    F = fine.reshape(n_cells * ncomp, -1)
    return (F @ P).reshape(-1)


def h_transfer_1d(k: int) -> np.ndarray:
    """Ph[o, i_f, j_c] = l^(k)_j((xi_i + o) / 2), o in {0, 1}: the parent's degree-k Lagrange basis
    (on its Gauss points, G2) evaluated at the Gauss points of the child occupying the half
    [o/2, (o+1)/2] of the parent's reference interval (reading H1: nested refinement in
    reference coordinates; P = exact DG embedding of the coarse space, as G18 for p)."""
    xi, _ = B.gauss01(k + 1)
    return np.stack([B.lagrange(xi, 0.5 * (xi + o)) for o in (0, 1)])


def h_transfer_3d(k: int, octant: int) -> np.ndarray:
    """Per-child prolongation (n^3 x n^3), lexicographic x fastest; octant = ox + 2 oy + 4 oz."""
    Ph = h_transfer_1d(k)
    ox, oy, oz = octant & 1, (octant >> 1) & 1, (octant >> 2) & 1
    return np.kron(Ph[oz], np.kron(Ph[oy], Ph[ox]))


def h_prolongate(coarse, k, parent, octant, ncomp=1):
    """fine[f, c] = P_{octant[f]} coarse[parent[f], c] (reading H1)."""
    n3 = (k + 1) ** 3
    C = np.asarray(coarse).reshape(-1, ncomp, n3)
    out = np.empty((len(parent), ncomp, n3))
    for f in range(len(parent)):
        out[f] = C[parent[f]] @ h_transfer_3d(k, int(octant[f])).T
    return out.reshape(-1)


def h_restrict(fine, k, parent, octant, n_coarse, ncomp=1):
    """R = P^T: coarse[p, c] = sum over the children f of p of P_{octant[f]}^T fine[f, c] (H2)."""
    n3 = (k + 1) ** 3
    F = np.asarray(fine).reshape(-1, ncomp, n3)
    out = np.zeros((n_coarse, ncomp, n3))
    for f in range(len(parent)):
        out[parent[f]] += F[f] @ h_transfer_3d(k, int(octant[f]))
    return out.reshape(-1)


def chebyshev(apply, Dinv, b, x0, lam_lo, lam_hi, m=5):
    """Chebyshev semi-iteration on D^-1 A (Adams 2003 via PAPER.md:1555):
      theta = (hi+lo)/2, delta = (hi-lo)/2, sigma = theta/delta, rho_0 = 1/sigma
      r_0 = b - A x_0; d_0 = D^-1 r_0 / theta; x_1 = x_0 + d_0
      j = 1..m-1: r_j = b - A x_j; rho_j = 1/(2 sigma - rho_{j-1});
                  d_j = rho_j rho_{j-1} d_{j-1} + (2 rho_j/delta) D^-1 r_j; x_{j+1} = x_j + d_j
    Returns x_m."""
    theta = 0.5 * (lam_hi + lam_lo)
    delta = 0.5 * (lam_hi - lam_lo)
    sigma = theta / delta
    rho = 1.0 / sigma
    x = np.array(x0, dtype=np.float64, copy=True)
    r = b - apply(x)
    dvec = Dinv * r / theta
    x = x + dvec
    for _ in range(1, m):
        r = b - apply(x)
        rho_new = 1.0 / (2.0 * sigma - rho)
        dvec = rho_new * rho * dvec + (2.0 * rho_new / delta) * Dinv * r
        rho = rho_new
        x = x + dvec
    return x


def vcycle(levels, b, lvl=None, m=5):
    """V(l, b) per SURVEY.md §8(c) c1.7.  `levels` is finest-first; each entry a dict with
    apply, Dinv, lam_hi, and (except the coarsest) restrict(r) / prolongate(xc) to the next
    coarser level.  lam_lo = lam_hi / 20 (G12).  If the coarsest entry carries "solve", that
    direct solve replaces its Chebyshev smoothing (reading H3)."""
    if lvl is None:
        lvl = 0
    L = levels[lvl]
    if lvl == len(levels) - 1 and "solve" in L:
        return L["solve"](b)
    lo, hi = L["lam_hi"] / 20.0, L["lam_hi"]
    zero = np.zeros_like(b)
    if lvl == len(levels) - 1:
        return chebyshev(L["apply"], L["Dinv"], b, zero, lo, hi, m)
    x = chebyshev(L["apply"], L["Dinv"], b, zero, lo, hi, m)
    r = b - L["apply"](x)
    xc = vcycle(levels, L["restrict"](r), lvl + 1, m)
    x = x + L["prolongate"](xc)
    return chebyshev(L["apply"], L["Dinv"], b, x, lo, hi, m)


def lanczos_lambda_max(apply, Dinv, v0, steps=20):
    """Largest eigenvalue estimate of D^-1 A by `steps` Lanczos steps (reading G12) on the
    symmetric form D^-1/2 A D^-1/2, start vector D^1/2-weighted v0; Ritz value = largest
    eigenvalue of the tridiagonal matrix."""
    s = np.sqrt(Dinv)
    q = v0 / s
    q = q / np.linalg.norm(q)
    q_prev = np.zeros_like(q)
    alpha, beta = [], []
    b_prev = 0.0
    for _ in range(steps):
        w = s * apply(s * q)
        a = q @ w
        w = w - a * q - b_prev * q_prev
        alpha.append(a)
        bn = np.linalg.norm(w)
        if bn == 0.0:
            break
        beta.append(bn)
        q_prev, q = q, w / bn
        b_prev = bn
    k = len(alpha)
    T = np.diag(alpha) + np.diag(beta[:k - 1], 1) + np.diag(beta[:k - 1], -1)
    return float(np.linalg.eigvalsh(T).max())


def diagonal_entries(apply_cells, n_dofs_cell, idx, ncomp=1):
    """D_ii = a(phi_i, phi_i) = (A e_i)_i for sampled global DoF indices idx, evaluated with
    the matrix-free oracle restricted to the DoF's own cell: apply_cells(e, cells) -> y rows."""
    out = np.empty(len(idx))
    per_cell = ncomp * n_dofs_cell
    for t, i in enumerate(idx):
        c = int(i) // per_cell
        e = np.zeros(per_cell)
        e[int(i) % per_cell] = 1.0
        out[t] = apply_cells(c, e)[int(i) % per_cell]
    return out


def pcg(apply, b, x0, precond, rtol, maxit):
    """Preconditioned conjugate gradients (Hestenes-Stiefel), the Krylov solver the paper uses
    for the symmetric viscous and pressure steps:
      r = b - A x; z = P r; p = z; rz = (r, z)
      repeat: q = A p; alpha = rz / (p, q); x += alpha p; r -= alpha q;
              stop when ||r|| <= rtol ||b|| (or maxit); z = P r; beta = (r, z)_new / rz; p = z + beta p
    `precond(r)` returns P r (identity for plain CG).  Returns (x, iterations, ||r||/||b||)."""
    x = np.array(x0, dtype=np.float64, copy=True)
    bn = np.sqrt(b @ b)
    r = b - apply(x)
    rn = np.sqrt(r @ r)
    if bn == 0.0 or rn <= rtol * bn:
        return x, 0, (rn / bn if bn else 0.0)
    z = precond(r)
    p = z.copy()
    rz = r @ z
    it = 0
    while it < maxit:
        it += 1
        q = apply(p)
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        rn = np.sqrt(r @ r)
        if rn <= rtol * bn:
            break
        z = precond(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it, rn / bn


def gmres(apply, b, x0, precond, rtol, restart, maxit):
    """Restarted GMRES(m) with right preconditioning and modified Gram-Schmidt Arnoldi (Saad,
    Iterative Methods, Alg. 9.5) — the Krylov solver for the non-symmetric viscous step with the
    convective term:
      r = b - A x; beta = ||r||; V_1 = r/beta
      for j = 1..m: z_j = P V_j; w = A z_j; h_ij = (w, V_i), w -= h_ij V_i (i <= j); h_{j+1,j} = ||w||
        Givens-rotate column j; |g_{j+1}| = ||b - A x_j||; stop at rtol ||b||
      x += P (V y),  y from the triangular solve;  restart.
    Returns (x, total iterations, ||r|| / ||b||)."""
    x = np.array(x0, dtype=np.float64, copy=True)
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return x, 0, 0.0
    total = 0
    r = b - apply(x)
    rn = np.linalg.norm(r)
    while rn > rtol * bn and total < maxit:
        m = min(restart, maxit - total)
        V = np.zeros((m + 1, len(b)))
        Z = np.zeros((m, len(b)))
        H = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = rn
        V[0] = r / rn
        j_done = 0
        for j in range(m):
            Z[j] = precond(V[j])
            wv = apply(Z[j])
            for i in range(j + 1):
                H[i, j] = wv @ V[i]
                wv = wv - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(wv)
            if H[j + 1, j] > 0:
                V[j + 1] = wv / H[j + 1, j]
            for i in range(j):                       # apply the previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            j_done = j + 1
            if abs(g[j + 1]) <= rtol * bn:
                break
        yk = np.zeros(j_done)
        for i in range(j_done - 1, -1, -1):
            yk[i] = (g[i] - H[i, i + 1:j_done] @ yk[i + 1:]) / H[i, i]
        x = x + yk @ Z[:j_done]
        r = b - apply(x)
        rn = np.linalg.norm(r)
    return x, total, rn / bn
