"""Pins of the oracle's Helmholtz mass term and preconditioned CG, CPU only.

mass_apply is pinned by exact polynomial integrals and the domain volume (closed forms);
pcg by textbook properties (exact termination after as many iterations as distinct
eigenvalues, one iteration with the exact inverse as preconditioner) and by numpy's dense
solver on the assembled Helmholtz matrix."""
import numpy as np
import pytest

from inputs import bfs, cube, deformed_cube, uniform
from inputs.vectors import node_positions
from oracle import dense, dg, laws, mg


def test_mass_volume_closed_form():
    """sum_c e_c^T M e_c = 3 |Omega|: unit cube (1) and the BFS channel (10x1x4 + 40x2x4 = 360)."""
    for m, vol in ((cube(3), 1.0), (bfs(nx_in=3, ny_in=2, nx_out=5, nz=2), 360.0)):
        d = dg.Disc(m, 2)
        e = np.ones(m.n_cells * 3 * d.N)
        assert abs(e @ dg.mass_apply(d, e) - 3.0 * vol) < 1e-12 * vol


@pytest.mark.parametrize("k", [1, 2, 3])
def test_mass_exact_polynomial_integrals(k):
    """v^T M u = int_Omega v.u exactly for polynomial u, v of degree <= k per direction on an
    affine mesh (Gauss with k+1 points integrates degree 2k+1); exact value from
    int_0^1 x^p dx = 1/(p+1)."""
    m = cube(2)
    d = dg.Disc(m, k)
    X = node_positions(m, k)                       # [cells, N, 3] physical nodes (collocation)
    rng = np.random.default_rng(4)
    pu, pv = rng.integers(0, k + 1, 3), rng.integers(0, k + 1, 3)
    fu = X[..., 0] ** pu[0] * X[..., 1] ** pu[1] * X[..., 2] ** pu[2]
    fv = X[..., 0] ** pv[0] * X[..., 1] ** pv[1] * X[..., 2] ** pv[2]
    u = np.zeros((m.n_cells, 3, d.N))
    v = np.zeros((m.n_cells, 3, d.N))
    u[:, 1] = fu
    v[:, 1] = fv
    exact = np.prod([1.0 / (pu[i] + pv[i] + 1) for i in range(3)])
    got = v.reshape(-1) @ dg.mass_apply(d, u.reshape(-1))
    assert abs(got - exact) < 1e-13


def test_mass_is_diagonal_with_collocation_and_positive():
    m = deformed_cube(2, 2)
    d = dg.Disc(m, 2)
    n = m.n_cells * 3 * d.N
    for i in (0, 7, n // 2, n - 1):
        e = np.zeros(n)
        e[i] = 1.0
        y = dg.mass_apply(d, e)
        off = np.delete(y, i)
        assert y[i] > 0 and np.abs(off).max() < 1e-15 * y[i]


def test_pcg_terminates_after_distinct_eigenvalues():
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    lam = np.repeat([1.0, 3.0, 10.0], [10, 20, 10])
    A = (Q * lam) @ Q.T
    b = rng.standard_normal(40)
    x, it, rr = mg.pcg(lambda v: A @ v, b, np.zeros(40), lambda r: r, 1e-12, 50)
    assert it == 3 and rr < 1e-12
    assert np.linalg.norm(x - np.linalg.solve(A, b)) < 1e-10 * np.linalg.norm(x)
    # exact inverse as preconditioner: one iteration
    Ai = np.linalg.inv(A)
    x, it, rr = mg.pcg(lambda v: A @ v, b, np.zeros(40), lambda r: Ai @ r, 1e-12, 50)
    assert it == 1


def test_pcg_helmholtz_matches_dense_solve():
    """CG on (mass M + A(nu)) with a Jacobi preconditioner converges to numpy's dense solution."""
    m = deformed_cube(2, 2)
    k = 2
    d = dg.Disc(m, k)
    nu = dg.AnalyticNu(d, laws.C2_LAW)
    A = dense.assemble_viscous(d, nu)
    mass = 50.0
    Mdiag = dg.mass_apply(d, np.ones(A.shape[0]))
    H = A + mass * np.diag(Mdiag)
    b = uniform(0, A.shape[0])
    Dinv = 1.0 / np.diag(H)
    x, it, rr = mg.pcg(lambda v: dg.helmholtz_apply(d, v, nu, mass), b, np.zeros(len(b)),
                       lambda r: Dinv * r, 1e-11, 2000)
    assert rr <= 1e-11
    ref = np.linalg.solve(H, b)
    assert np.linalg.norm(x - ref) < 1e-8 * np.linalg.norm(ref)
    # the dense Helmholtz matrix is the matrix-free one
    v = uniform(1, len(b))
    assert np.linalg.norm(H @ v - dg.helmholtz_apply(d, v, nu, mass)) < 1e-12 * np.linalg.norm(H @ v)
