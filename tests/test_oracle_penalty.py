"""Pins of the oracle's divergence/continuity penalty-step operator (PAPER.md:1190-1224,
eqn:penalty_step), CPU only: closed-form energies of constant and linear
fields, the divergence-free kernel (A = M on continuous solenoidal fields), symmetry with
non-uniform per-cell parameters (reading P2) and positive definiteness."""
import numpy as np
import pytest

from inputs import bfs, cube, deformed_cube, uniform
from inputs.meshes import NEUMANN
from inputs.vectors import field_to_dofs, node_positions
from oracle import dg


def test_constant_field_energy_dirichlet_cube():
    """e_c^T A e_c = |Omega| + tau_c * sum over boundary faces of int n_c^2 = 1 + 2 tau_c."""
    m = cube(4)
    d = dg.Disc(m, 2)
    td, tc = np.full(m.n_cells, 0.7), np.full(m.n_cells, 3.0)
    for c in range(3):
        e = np.zeros((m.n_cells, 3, d.N))
        e[:, c] = 1.0
        e = e.reshape(-1)
        assert abs(e @ dg.penalty_apply(d, e, td, tc) - (1.0 + 2.0 * 3.0)) < 1e-12


def test_linear_field_energy_neumann_cube():
    """u = (x, 0, 0) on an all-Neumann affine mesh: u^T A u = int x^2 + tau_div int (div u)^2
    = 1/3 + tau_div (continuous field: no jumps; Neumann: no boundary term)."""
    m = cube(3, bc=NEUMANN)
    k = 2
    d = dg.Disc(m, k)
    X = node_positions(m, k)
    vals = np.zeros_like(X)
    vals[..., 0] = X[..., 0]
    u = field_to_dofs(vals)
    td = np.full(m.n_cells, 2.5)
    tc = np.full(m.n_cells, 11.0)
    assert abs(u @ dg.penalty_apply(d, u, td, tc) - (1.0 / 3.0 + 2.5)) < 1e-12


def test_solenoidal_continuous_field_sees_only_the_mass():
    """u = (-y, x, 0): div u = 0 and [[u]] = 0, so A u = M u (all-Neumann cube)."""
    m = cube(3, bc=NEUMANN)
    k = 2
    d = dg.Disc(m, k)
    X = node_positions(m, k)
    vals = np.stack([-X[..., 1], X[..., 0], np.zeros_like(X[..., 0])], axis=-1)
    u = field_to_dofs(vals)
    rng = np.random.default_rng(3)
    td, tc = rng.uniform(0.5, 5.0, m.n_cells), rng.uniform(0.5, 5.0, m.n_cells)
    y = dg.penalty_apply(d, u, td, tc)
    ref = dg.mass_apply(d, u)
    assert np.linalg.norm(y - ref) < 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("mk,k", [(lambda: deformed_cube(2, 2), 2), (lambda: bfs(nx_in=2, ny_in=1, nx_out=3, nz=2), 2)])
def test_symmetric_and_positive_definite(mk, k):
    m = mk()
    d = dg.Disc(m, k)
    rng = np.random.default_rng(7)
    td, tc = rng.uniform(0.1, 10.0, m.n_cells), rng.uniform(0.1, 10.0, m.n_cells)
    n = m.n_cells * 3 * d.N
    u, v = uniform(0, n), uniform(1, n)
    a, b = v @ dg.penalty_apply(d, u, td, tc), u @ dg.penalty_apply(d, v, td, tc)
    assert abs(a - b) < 1e-12 * abs(a)
    if n <= 1000:
        A = np.array([dg.penalty_apply(d, e, td, tc) for e in np.eye(n)]).T
        assert np.linalg.norm(A - A.T) < 1e-12 * np.linalg.norm(A)
        assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > 0
