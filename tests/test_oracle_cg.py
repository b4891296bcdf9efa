"""Pins of the oracle's c-level (continuous Q1 space of the cph hierarchy; SURVEY §8(f) f3,
PAPER.md:1533-1536), CPU only: vertex counts of closed/periodic meshes, exact reproduction of
global trilinear functions by the DG embedding and by the nested Q1 h-transfer, the textbook
27-point Q1 stiffness stencil (diagonal 8h/3, face diagonals -h/6, body diagonals -h/12, edge
neighbours 0) recovered from P_c^T A_DG P_c, and a symmetric contracting V-cycle
DG p -> c -> CG h -> direct."""
import numpy as np
import pytest

from inputs import cube, cube_parent_map, uniform
from inputs.meshes import NEUMANN
from inputs.vectors import node_positions
from oracle import cg, dense, dg, laws, mg


def _trilinear(x):
    X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
    return 1.0 + X - 2.0 * Y + 0.5 * Z + 3.0 * X * Y - 0.7 * Y * Z + 1.3 * X * Z - 2.1 * X * Y * Z


def test_vertex_counts():
    assert cg.vertex_numbering(cube(3))[1] == 64
    assert cg.vertex_numbering(cube(3, periodic=(True, True, True)))[1] == 27
    assert cg.vertex_numbering(cube(3, periodic=(False, False, True)))[1] == 48


def _vertex_values(mesh, vid, nv, f):
    X = cg.corner_positions(mesh)
    v = np.full(nv, np.nan)
    for c in range(mesh.n_cells):
        for o in range(8):
            v[vid[c, o]] = f(X[c, o])
    return v


def test_embedding_reproduces_trilinear_functions():
    m = cube(3)
    vid, nv = cg.vertex_numbering(m)
    P = cg.embedding(m, vid, nv)
    vals = _vertex_values(m, vid, nv, _trilinear)
    ref = _trilinear(node_positions(m, 1)).reshape(-1)        # DG_1 nodal values at the Gauss points
    assert np.abs(P @ vals - ref).max() < 1e-13
    # each cell row block sums to 1 (partition of unity of the corner functions)
    assert np.allclose(P.sum(axis=1), 1.0, atol=1e-15)


def test_h_transfer_reproduces_trilinear_functions():
    mf, mc = cube(4), cube(2)
    parent, octant = cube_parent_map(4)
    vf, nvf = cg.vertex_numbering(mf)
    vc, nvc = cg.vertex_numbering(mc)
    Ph = cg.h_transfer(vf, nvf, vc, nvc, parent, octant)
    xc = _vertex_values(mc, vc, nvc, _trilinear)
    xf = _vertex_values(mf, vf, nvf, _trilinear)
    assert np.abs(Ph @ xc - xf).max() < 1e-13


def test_galerkin_q1_stiffness_is_the_textbook_stencil():
    N = 4
    h = 1.0 / N
    m = cube(N, bc=NEUMANN)
    d = dg.Disc(m, 1)
    Adg = dense.assemble_poisson(d, dg.AnalyticNu(d, {"kind": "const", "value": 1.0}))
    vid, nv = cg.vertex_numbering(m)
    P = cg.embedding(m, vid, nv)
    Ac = P.T @ Adg @ P
    X = _vertex_values(m, vid, nv, lambda x: 0.0)              # just to size
    pos = np.zeros((nv, 3))
    C = cg.corner_positions(m)
    for c in range(m.n_cells):
        for o in range(8):
            pos[vid[c, o]] = C[c, o]
    idx = np.round(pos / h).astype(int)
    interior = np.all((idx > 0) & (idx < N), axis=1)
    assert len(X) == nv and interior.sum() == (N - 1) ** 3
    for v in np.nonzero(interior)[0]:
        dist = np.abs(idx - idx[v]).sum(axis=1)
        cheb = np.abs(idx - idx[v]).max(axis=1)
        row = Ac[v]
        assert abs(row[v] - 8.0 * h / 3.0) < 1e-13
        assert np.allclose(row[(cheb == 1) & (dist == 1)], 0.0, atol=1e-13)
        assert np.allclose(row[(cheb == 1) & (dist == 2)], -h / 6.0, atol=1e-13)
        assert np.allclose(row[(cheb == 1) & (dist == 3)], -h / 12.0, atol=1e-13)
        assert np.allclose(row[cheb > 1], 0.0, atol=1e-13)
    assert np.abs(Ac.sum(axis=1)).max() < 1e-12                 # constants: all-Neumann kernel


def test_cph_vcycle_with_c_level_is_symmetric_contraction():
    """Poisson (C4 law) on cube(4): DG k = 2 -> 1, then the c-level (Q1 on cube(4)), the CG h-level
    Q1 on cube(2) with the direct solve.  V symmetric, spectral radius of I - V A below 1."""
    law = laws.C4_LAW
    mf, mc = cube(4), cube(2)
    parent, octant = cube_parent_map(4)
    levels = []
    for k in (2, 1):
        d = dg.Disc(mf, k)
        Ad = dense.assemble_poisson(d, dg.AnalyticNu(d, law))
        levels.append({"A": Ad})
    vf, nvf = cg.vertex_numbering(mf)
    vc, nvc = cg.vertex_numbering(mc)
    Pc = cg.embedding(mf, vf, nvf)
    Acf = Pc.T @ levels[1]["A"] @ Pc
    Ph = cg.h_transfer(vf, nvf, vc, nvc, parent, octant)
    dcc = dg.Disc(mc, 1)
    Pcc = cg.embedding(mc, vc, nvc)
    Acc = Pcc.T @ dense.assemble_poisson(dcc, dg.AnalyticNu(dcc, law)) @ Pcc
    levels.append({"A": Acf})
    for L in levels:
        L["apply"] = (lambda x, Ad=L["A"]: Ad @ x)
        L["Dinv"] = 1.0 / np.diag(L["A"])
        L["lam_hi"] = 1.2 * mg.lanczos_lambda_max(L["apply"], L["Dinv"], uniform(2, len(L["Dinv"])), 20)
    levels[0]["restrict"] = lambda r: mg.restrict(r, 2, 1, mf.n_cells)
    levels[0]["prolongate"] = lambda x: mg.prolongate(x, 2, 1, mf.n_cells)
    levels[1]["restrict"] = lambda r: Pc.T @ r
    levels[1]["prolongate"] = lambda x: Pc @ x
    levels[2]["restrict"] = lambda r: Ph.T @ r
    levels[2]["prolongate"] = lambda x: Ph @ x
    levels.append({"apply": (lambda x: Acc @ x), "solve": lambda b: np.linalg.solve(Acc, b)})
    A0 = levels[0]["A"]
    n = A0.shape[0]
    V = np.array([mg.vcycle(levels, e) for e in np.eye(n)]).T
    assert np.abs(V - V.T).max() < 1e-10 * np.abs(V).max()
    rho = np.abs(np.linalg.eigvals(np.eye(n) - V @ A0)).max()
    assert rho < 1.0
