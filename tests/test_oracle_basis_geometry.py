"""Oracle pins: basis/quadrature (P12), geometry (G3 worked H values, closed-surface
identities, exact volume), face pairing vs the input neighbour table."""
import json
import os

import numpy as np
import pytest

from inputs import bfs, cube, deformed_cube
from oracle import basis as B
from oracle import dg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7])
def test_gauss_exactness(n):
    """P12: n-point Gauss integrates x^m exactly on [0,1] for m <= 2n-1, not for m = 2n."""
    x, w = B.gauss01(n)
    for m in range(2 * n):
        assert abs(w @ x ** m - 1.0 / (m + 1)) < 1e-14
    assert abs(w @ x ** (2 * n) - 1.0 / (2 * n + 1)) > 1e-12
    assert np.all(w > 0) and abs(w.sum() - 1) < 1e-15


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_lagrange_partition_of_unity_and_derivative(n):
    """P12: sum l_i = 1, sum l_i' = 0, l_i(x_j) = delta_ij; l' against central differences."""
    x, _ = B.gauss01(n)
    t = np.random.default_rng(0).uniform(-0.2, 1.2, 50)
    L, dL = B.lagrange(x, t), B.lagrange_deriv(x, t)
    assert np.abs(L.sum(1) - 1).max() < 1e-12
    assert np.abs(dL.sum(1)).max() < 1e-10
    assert np.abs(B.lagrange(x, x) - np.eye(n)).max() < 1e-13
    h = 1e-6
    fd = (B.lagrange(x, t + h) - B.lagrange(x, t - h)) / (2 * h)
    assert np.abs(fd - dL).max() < 1e-6 * max(1, np.abs(dL).max())


def test_gll_points_closed_form():
    """GLL points of degree 2 and 3 on [0,1]: {0,1/2,1}, {0,(1-1/sqrt5)/2,(1+1/sqrt5)/2,1}."""
    assert np.allclose(B.gll01(2), [0, 0.5, 1], atol=1e-15)
    s = 1 / np.sqrt(5)
    assert np.allclose(B.gll01(3), [0, (1 - s) / 2, (1 + s) / 2, 1], atol=1e-15)


def test_penalty_length_scale_worked_example():
    """G3 worked example (tests/golden/penalty_H.json): 12 / 14 / 16 / 18 on the h=1/4 cube."""
    gold = json.load(open(os.path.join(GOLD, "penalty_H.json")))
    m = cube(4)
    d = dg.Disc(m, 2)
    H = d.H(np.arange(m.n_cells))
    nb = (m.neighbor < 0).sum(1)
    for c in range(m.n_cells):
        assert abs(H[c] - gold["H_by_boundary_faces"][str(nb[c])]) < 1e-12


def test_deformed_geometry_closed_surface_and_volume():
    """C2-type iso-parametric mesh: total volume of [0,1]^3 is 1, boundary area 6, and
    int_{dK} n dA = 0 on every cell (Nanson cofactor integrand is exactly integrated)."""
    m = deformed_cube(3, 3)
    d = dg.Disc(m, 3)
    cells = np.arange(m.n_cells)
    _, JxW, _ = d.vol_geom(cells)
    assert abs(JxW.sum() - 1.0) < 1e-13
    area_b = 0.0
    closure = np.zeros((m.n_cells, 3))
    for f in range(6):
        _, _, n, dA = d.face_geom(cells, f)
        closure += np.einsum("cp,cpi->ci", dA, n)
        area_b += dA[m.neighbor[:, f] < 0].sum()
    assert abs(area_b - 6.0) < 1e-13
    assert np.abs(closure).max() < 1e-14
    # the map really is deformed
    assert np.ptp(JxW / d.vol_w) > 0.1 * np.mean(JxW / d.vol_w) / 27


def test_face_pairing_matches_neighbour_table():
    """The oracle's geometric pairing (centroids, periodic shift) reproduces the input
    neighbour table of a BFS mesh with periodic z and a block interface."""
    m = bfs(nx_in=3, ny_in=2, nx_out=4, nz=3)
    d = dg.Disc(m, 1)
    cells = np.arange(m.n_cells)
    for f in range(6):
        sel = m.neighbor[:, f] >= 0
        fb, perm, shift = d.match_faces(cells[sel], f, m.neighbor[sel, f])
        assert np.all(fb == f ^ 1)
        # structured + aligned meshes: identity point permutation (convention of the ABI)
        assert np.all(perm == np.arange(d.P)[None, :])
        if f >= 4:
            assert np.all(np.isin(np.round(np.abs(shift[:, 2]), 12), [0.0, 4.0]))
