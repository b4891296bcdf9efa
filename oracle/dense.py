"""Dense assembly of the SIPG operators on tiny meshes (oracle).
Test infrastructure only — see oracle/__init__.py.

An independent encoding of the same forms (PAPER.md:1055-1111 viscous; PAPER.md:713-758
Poisson), written as quadratic forms: at each quadrature point the element/face state
s = B U (values and physical gradients) and the integrand s_v^T Q s_u, with Q spelled
out from Appendix A:
  face Q = -E^T M - M^T E + tau E^T N E,   E s = [u] (jump),  M s = sigma_bar(u) n,
  N = I + n n^T (divergence, reading G5) or I (laplace / Poisson).
Dirichlet faces: the trial state is mirrored (u+ = -u-, grad u+ = grad u-, nu+ = nu-),
the test state has v+ = 0 (reading G7).  The matrix-free oracle must satisfy
y = A_dense x to rounding.
"""
from __future__ import annotations

import numpy as np

from .dg import Disc


def _grad_B(dPhi, Jinv):
    """G[p, j, n] = d phi_n / d x_j at points (dPhi [3,P,N], Jinv [P,3,3])."""
    return np.einsum("dpn,pdj->pjn", dPhi, Jinv)


def _vec_state(Phi, gphi):
    """Vector field state at points: s = [u(3), grad u(9) with index 3i+j] -> [P, 12, 3N]."""
    P, N = Phi.shape
    S = np.zeros((P, 12, 3 * N))
    for i in range(3):
        S[:, i, i * N:(i + 1) * N] = Phi
        for j in range(3):
            S[:, 3 + 3 * i + j, i * N:(i + 1) * N] = gphi[:, j, :]
    return S


def _sym_n(n, div):
    """M_side [3, 9]: (S(G) n)_i as a linear map of G (index 3a+b)."""
    M = np.zeros((3, 9))
    for i in range(3):
        for a in range(3):
            for b in range(3):
                if div:
                    M[i, 3 * a + b] += 0.5 * ((i == a) * n[b] + (i == b) * n[a])
                else:
                    M[i, 3 * a + b] += 0.5 * (i == a) * n[b]
    return M


def assemble_viscous(disc: Disc, nu, formulation="divergence"):
    d = disc
    nc, N = d.mesh.n_cells, d.N
    nd = 3 * N
    A = np.zeros((nc * nd, nc * nd))
    div = formulation == "divergence"
    pen = d.ip * (d.k + 1) ** 2
    cells = np.arange(nc)
    H = d.H(cells)
    Psym = np.zeros((9, 9))
    for i in range(3):
        for j in range(3):
            Psym[3 * i + j, 3 * i + j] += 0.5
            Psym[3 * i + j, 3 * j + i] += 0.5
    _, JxW, Jinv = d.vol_geom(cells)
    nuv = nu.vol(cells)
    for c in range(nc):
        Kc = np.zeros((nd, nd))
        for q in range(d.N):
            S = _vec_state(d.Phi[q:q + 1], _grad_B(d.dPhi[:, q:q + 1], Jinv[c, q:q + 1]))[0, 3:]
            C = (2.0 * Psym if div else np.eye(9)) * nuv[c, q] * JxW[c, q]
            Kc += S.T @ C @ S
        A[c * nd:(c + 1) * nd, c * nd:(c + 1) * nd] += Kc

    E = np.zeros((3, 24))
    E[:, 0:3] = np.eye(3)
    E[:, 12:15] = -np.eye(3)
    inter, bnd = d.unique_faces(cells)
    for (a, fa), b in inter.items():
        fb, perm, _ = d.match_faces(np.array([a]), fa, np.array([b]))
        fb, perm = int(fb[0]), perm[0]
        _, Ja, n, dA = d.face_geom(np.array([a]), fa)
        _, Jb, _, _ = d.face_geom(np.array([b]), fb)
        nua, nub = nu.face(np.array([a]), fa)[0], nu.face(np.array([b]), fb)[0]
        Sa = _vec_state(d.PhiF[fa], _grad_B(d.dPhiF[fa], Ja[0]))
        Sb = _vec_state(d.PhiF[fb][perm], _grad_B(d.dPhiF[fb][:, perm], Jb[0][perm]))
        blk = np.zeros((2 * nd, 2 * nd))
        for p in range(d.P):
            S = np.zeros((24, 2 * nd))
            S[:12, :nd] = Sa[p]
            S[12:, nd:] = Sb[p]
            nn = n[0, p]
            M = np.zeros((3, 24))
            M[:, 3:12] = nua[p] * _sym_n(nn, div)
            M[:, 15:24] = nub[perm[p]] * _sym_n(nn, div)
            tau = pen * max(H[a], H[b]) * 0.5 * (nua[p] + nub[perm[p]])
            Nm = np.eye(3) + (np.outer(nn, nn) if div else 0.0)
            Q = -E.T @ M - M.T @ E + tau * E.T @ Nm @ E
            blk += dA[0, p] * S.T @ Q @ S
        idx = np.concatenate([np.arange(a * nd, (a + 1) * nd), np.arange(b * nd, (b + 1) * nd)])
        A[np.ix_(idx, idx)] += blk
    # Dirichlet faces
    Tu = np.zeros((24, 12))
    Tu[:12, :] = np.eye(12)
    Tu[12:15, 0:3] = -np.eye(3)
    Tu[15:24, 3:12] = np.eye(9)
    Tv = np.zeros((24, 12))
    Tv[:12, :] = np.eye(12)
    for (a, f, t) in bnd:
        if t != 1:
            continue
        _, Ja, n, dA = d.face_geom(np.array([a]), f)
        nua = nu.face(np.array([a]), f)[0]
        Sa = _vec_state(d.PhiF[f], _grad_B(d.dPhiF[f], Ja[0]))
        blk = np.zeros((nd, nd))
        for p in range(d.P):
            nn = n[0, p]
            M = np.zeros((3, 24))
            M[:, 3:12] = nua[p] * _sym_n(nn, div)
            M[:, 15:24] = nua[p] * _sym_n(nn, div)
            tau = pen * H[a] * nua[p]
            Nm = np.eye(3) + (np.outer(nn, nn) if div else 0.0)
            Q = -E.T @ M - M.T @ E + tau * E.T @ Nm @ E
            blk += dA[0, p] * Sa[p].T @ (Tv.T @ Q @ Tu) @ Sa[p]
        A[a * nd:(a + 1) * nd, a * nd:(a + 1) * nd] += blk
    return A


def assemble_poisson(disc: Disc, coef):
    d = disc
    nc, N = d.mesh.n_cells, d.N
    A = np.zeros((nc * N, nc * N))
    pen = d.ip * (d.k + 1) ** 2
    cells = np.arange(nc)
    H = d.H(cells)
    _, JxW, Jinv = d.vol_geom(cells)
    cv = coef.vol(cells)
    for c in range(nc):
        Kc = np.zeros((N, N))
        for q in range(d.N):
            g = _grad_B(d.dPhi[:, q:q + 1], Jinv[c, q:q + 1])[0]     # [3, N]
            Kc += cv[c, q] * JxW[c, q] * g.T @ g
        A[c * N:(c + 1) * N, c * N:(c + 1) * N] += Kc

    def state(Phi, gphi):                                          # [P, 4, N]
        return np.concatenate([Phi[:, None, :], gphi], axis=1)

    E = np.array([[1.0, 0, 0, 0, -1.0, 0, 0, 0]])
    inter, bnd = d.unique_faces(cells)
    for (a, fa), b in inter.items():
        fb, perm, _ = d.match_faces(np.array([a]), fa, np.array([b]))
        fb, perm = int(fb[0]), perm[0]
        _, Ja, n, dA = d.face_geom(np.array([a]), fa)
        _, Jb, _, _ = d.face_geom(np.array([b]), fb)
        ca, cb = coef.face(np.array([a]), fa)[0], coef.face(np.array([b]), fb)[0]
        Sa = state(d.PhiF[fa], _grad_B(d.dPhiF[fa], Ja[0]))
        Sb = state(d.PhiF[fb][perm], _grad_B(d.dPhiF[fb][:, perm], Jb[0][perm]))
        blk = np.zeros((2 * N, 2 * N))
        for p in range(d.P):
            S = np.zeros((8, 2 * N))
            S[:4, :N] = Sa[p]
            S[4:, N:] = Sb[p]
            M = np.zeros((1, 8))
            M[0, 1:4] = 0.5 * ca[p] * n[0, p]
            M[0, 5:8] = 0.5 * cb[perm[p]] * n[0, p]
            tau = pen * max(H[a], H[b]) * 0.5 * (ca[p] + cb[perm[p]])
            Q = -E.T @ M - M.T @ E + tau * E.T @ E
            blk += dA[0, p] * S.T @ Q @ S
        idx = np.concatenate([np.arange(a * N, (a + 1) * N), np.arange(b * N, (b + 1) * N)])
        A[np.ix_(idx, idx)] += blk
    Tu = np.zeros((8, 4))
    Tu[:4] = np.eye(4)
    Tu[4, 0] = -1.0
    Tu[5:8, 1:4] = np.eye(3)
    Tv = np.zeros((8, 4))
    Tv[:4] = np.eye(4)
    for (a, f, t) in bnd:
        if t != 1:
            continue
        _, Ja, n, dA = d.face_geom(np.array([a]), f)
        ca = coef.face(np.array([a]), f)[0]
        Sa = state(d.PhiF[f], _grad_B(d.dPhiF[f], Ja[0]))
        blk = np.zeros((N, N))
        for p in range(d.P):
            M = np.zeros((1, 8))
            M[0, 1:4] = 0.5 * ca[p] * n[0, p]
            M[0, 5:8] = 0.5 * ca[p] * n[0, p]
            tau = pen * H[a] * ca[p]
            Q = -E.T @ M - M.T @ E + tau * E.T @ E
            blk += dA[0, p] * Sa[p].T @ (Tv.T @ Q @ Tu) @ Sa[p]
        A[a * N:(a + 1) * N, a * N:(a + 1) * N] += blk
    return A
