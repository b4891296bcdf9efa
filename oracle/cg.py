"""c-level of the cph hierarchy (oracle): continuous Q1 space below the DG levels.
Test infrastructure only — see oracle/__init__.py.

PAPER.md:1533-1536 (§5.3): "first the conversion from a discontinuous to a continuous polynomial
space is performed, whereafter the polynomial degree is lowered … after which h-coarsening is
performed" (cph-multigrid, Fehn2020).  Readings C1-C3:
  C1  the continuous level is Q1 (one value per mesh vertex and component) on the mesh of the
      degree-1 DG level; its embedding P_c into DG_1 is the nodal interpolation of the
      trilinear function at the DG Gauss points, per cell E = E1 (x) E1 (x) E1 with
      E1[i][o] = (1 - xi_i, xi_i)[o] (o = corner bit, xi_i the 2 Gauss points of [0,1]);
  C2  the continuous-level operator is the Galerkin product A_c = P_c^T A_DG P_c (for continuous
      functions every interior-face term of the SIPG form vanishes, so this is the conforming
      Q1 operator with the SIPG (Nitsche) Dirichlet terms); its smoother diagonal is diag(A_c);
  C3  h-levels of the continuous space: nested Q1 interpolation — a fine vertex takes the
      trilinear interpolant of its parent cell's 8 vertex values at its position (reference
      coordinates (corner bit + octant bit) / 2 per axis); restriction = transpose.
Vertices are identified here by their physical coordinates (periodic images folded with the
mesh periods), independently of the library's topological numbering.
"""
from __future__ import annotations

import numpy as np

from . import basis as B


def corner_positions(mesh) -> np.ndarray:
    """[n_cells, 8, 3] physical corner positions, corner = vx + 2 vy + 4 vz."""
    m = mesh.map_degree
    idx = [(vx * m) + (m + 1) * (vy * m) + (m + 1) ** 2 * (vz * m)
           for vz in (0, 1) for vy in (0, 1) for vx in (0, 1)]
    return mesh.nodes[:, idx, :]


def vertex_numbering(mesh, tol: float = 1e-9):
    """vid[cell, corner] and the vertex count, vertices matched by coordinates (periodic wrap).
    Numbering = order of first appearance in (cell, corner) order."""
    X = corner_positions(mesh).reshape(-1, 3).copy()
    per = np.asarray(mesh.periods, dtype=np.float64)
    ext = np.ptp(mesh.nodes.reshape(-1, 3), axis=0).max()
    for d in range(3):
        if per[d] > 0:
            lo = mesh.nodes[:, :, d].min()
            t = np.mod(X[:, d] - lo, per[d])
            t[np.abs(t - per[d]) < tol * ext] = 0.0
            X[:, d] = t
    key = np.round(X / (tol * ext * 10)).astype(np.int64)
    ids = {}
    vid = np.empty(len(key), dtype=np.int64)
    for i, kk in enumerate(map(tuple, key)):
        vid[i] = ids.setdefault(kk, len(ids))
    return vid.reshape(mesh.n_cells, 8), len(ids)


def embedding_1d() -> np.ndarray:
    """E1[i, o] = value of the linear corner function o at the i-th Gauss point of [0,1] (C1)."""
    xi, _ = B.gauss01(2)
    return np.stack([1.0 - xi, xi], axis=1)


def embedding(mesh, vid, nv) -> np.ndarray:
    """Dense P_c: (n_cells * 8) x nv, DG_1 scalar layout [cell][q] (q lexicographic x fastest)."""
    E1 = embedding_1d()
    E = np.kron(E1, np.kron(E1, E1))        # [q, corner], corner = vx + 2 vy + 4 vz
    P = np.zeros((mesh.n_cells * 8, nv))
    for c in range(mesh.n_cells):
        for o in range(8):
            P[c * 8:(c + 1) * 8, vid[c, o]] += E[:, o]
    return P


def h_transfer(vid_f, nvf, vid_c, nvc, parent, octant) -> np.ndarray:
    """Dense nested-Q1 prolongation (C3): nvf x nvc.  Every incidence of a fine vertex must give
    the same row (continuity of the coarse interpolant)."""
    P = np.full((nvf, nvc), np.nan)
    for f in range(len(parent)):
        p, oc = int(parent[f]), int(octant[f])
        for o in range(8):
            t = [((o >> a) & 1) * 0.5 + ((oc >> a) & 1) * 0.5 for a in range(3)]
            row = np.zeros(nvc)
            for co in range(8):
                w = 1.0
                for a in range(3):
                    w *= t[a] if (co >> a) & 1 else 1.0 - t[a]
                row[vid_c[p, co]] += w
            v = vid_f[f, o]
            if np.isnan(P[v, 0]):
                P[v] = row
            else:
                assert np.allclose(P[v], row, atol=1e-14), "non-nested vertex"
    assert not np.isnan(P).any()
    return P


def expand(P, ncomp):
    """Component-blocked version of a scalar transfer for vector fields.
    DG side layout [cell][c][q] (8 per cell), CG side layout [c][v]."""
    if ncomp == 1:
        return P
    ndg, nv = P.shape
    ncell = ndg // 8
    out = np.zeros((ndg * ncomp, nv * ncomp))
    for c in range(ncomp):
        rows = (np.arange(ncell)[:, None] * ncomp * 8 + c * 8 + np.arange(8)[None, :]).reshape(-1)
        out[rows, c * nv:(c + 1) * nv] = P
    return out
