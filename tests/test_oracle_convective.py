"""Pins of the oracle's upwind convective term and GMRES, CPU only:
the closed form int (w.grad) u_c for a continuous linear field, the exact upwind energy
identity u^T C(w) u = 1/2 sum_F int |w.n| |[u]|^2 on a periodic mesh with constant w (the face
values of the right-hand side are evaluated independently with the 1D Lagrange basis), and
GMRES against numpy's dense solver / textbook termination properties."""
import numpy as np
import pytest

from inputs import cube, uniform
from inputs.meshes import NEUMANN
from inputs.vectors import field_to_dofs, node_positions
from oracle import basis as B
from oracle import dg, mg


def test_linear_field_closed_form():
    """u = (x, 0, 0), w = (1, 0, 0): sum_i y[0,i] = int (w.grad) u_x = |Omega| = 1."""
    for bc in (1, NEUMANN):
        m = cube(3, bc=bc)
        k = 2
        d = dg.Disc(m, k)
        X = node_positions(m, k)
        uv = np.zeros_like(X)
        uv[..., 0] = X[..., 0]
        wv = np.zeros_like(X)
        wv[..., 0] = 1.0
        y = dg.convective_apply(d, field_to_dofs(uv), field_to_dofs(wv)).reshape(m.n_cells, 3, d.N)
        assert abs(y[:, 0].sum() - 1.0) < 1e-12 and abs(y[:, 1:].sum()) < 1e-12


@pytest.mark.parametrize("k", [1, 2, 3])
def test_upwind_energy_identity_periodic(k):
    N = 3
    m = cube(N, periodic=(True, True, True))
    d = dg.Disc(m, k)
    n = k + 1
    u = uniform(0, m.n_cells * 3 * d.N)
    wconst = np.array([0.7, -0.4, 0.25])
    w = np.zeros((m.n_cells, 3, d.N))
    w[:, :, :] = wconst[None, :, None]
    lhs = u @ dg.convective_apply(d, u, w.reshape(-1))
    # right-hand side: independent face evaluation, 1D Lagrange basis on the Gauss points
    xi, wq = B.gauss01(n)
    l0, l1 = B.lagrange(xi, np.array([0.0]))[0], B.lagrange(xi, np.array([1.0]))[0]
    h = 1.0 / N
    U = u.reshape(N, N, N, 3, n, n, n)          # [k][j][i][c][z][y][x]
    rhs = 0.0
    for ax in range(3):
        for kk in range(N):
            for jj in range(N):
                for ii in range(N):
                    idx = [kk, jj, ii]
                    nb = list(idx)
                    nb[2 - ax] = (nb[2 - ax] + 1) % N            # +axis neighbour (x is the last index)
                    um = np.tensordot(U[tuple(idx)], l1, axes=([3 - ax], [0]))   # trace at +face
                    up = np.tensordot(U[tuple(nb)], l0, axes=([3 - ax], [0]))   # neighbour at its -face
                    jump2 = ((um - up) ** 2).sum(axis=0)                        # [n][n] face points
                    rhs += 0.5 * abs(wconst[ax]) * (np.outer(wq, wq) * jump2).sum() * h * h
    assert abs(lhs - rhs) < 1e-12 * abs(rhs)


def test_gmres_against_dense_and_termination():
    rng = np.random.default_rng(1)
    n = 30
    A = np.eye(n) * 4 + rng.standard_normal((n, n))
    b = rng.standard_normal(n)
    x, it, rr = mg.gmres(lambda v: A @ v, b, np.zeros(n), lambda r: r, 1e-12, n, 200)
    assert it <= n and rr < 1e-12
    assert np.linalg.norm(x - np.linalg.solve(A, b)) < 1e-10 * np.linalg.norm(x)
    Ai = np.linalg.inv(A)
    x, it, rr = mg.gmres(lambda v: A @ v, b, np.zeros(n), lambda r: Ai @ r, 1e-12, 10, 50)
    assert it == 1
    # restarted GMRES(5) converges when the field of values stays away from 0 (A2 = 10 I + R)
    A2 = np.eye(n) * 10 + rng.standard_normal((n, n))
    x, it, rr = mg.gmres(lambda v: A2 @ v, b, np.zeros(n), lambda r: r, 1e-10, 5, 400)
    assert rr < 1e-10 and np.linalg.norm(x - np.linalg.solve(A2, b)) < 1e-8 * np.linalg.norm(x)
