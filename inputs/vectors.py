"""Seeded random vectors and smooth random fields (SURVEY.md §8(c) G20, §8(d) input recipe)."""
from __future__ import annotations

import numpy as np


def uniform(seed: int, n: int) -> np.ndarray:
    """G20: numpy.random.default_rng(seed).uniform(-1, 1, n) in canonical DoF order."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def fourier_modes(seed: int = 1, n_modes: int = 8):
    """C3 recipe: drawn from rng(seed) in this order: k_m = integers(1,4,(8,3)),
    a_m = uniform(-1,1,(8,3)), phi_m = uniform(0, 2 pi, 8)."""
    rng = np.random.default_rng(seed)
    k = rng.integers(1, 4, (n_modes, 3))
    a = rng.uniform(-1.0, 1.0, (n_modes, 3))
    phi = rng.uniform(0.0, 2.0 * np.pi, n_modes)
    return k, a, phi


def fourier_field(x: np.ndarray, modes) -> np.ndarray:
    """u(x) = sum_m a_m sin(2 pi k_m . x + phi_m); x [..., 3] -> [..., 3]."""
    k, a, phi = modes
    arg = 2.0 * np.pi * np.tensordot(x, k.T.astype(np.float64), axes=([-1], [0])) + phi  # [..., M]
    return np.tensordot(np.sin(arg), a, axes=([-1], [0]))


def node_positions(mesh, degree: int) -> np.ndarray:
    """Sampling positions used to build smooth input vectors on axis-aligned box cells:
    x = x0 + h * xi with xi the Gauss-Legendre points of [0,1] (numpy.leggauss), tensor
    order x fastest.  Returns [n_cells, (degree+1)^3, 3].  Sampling the field here gives
    the nodal interpolant under the collocation basis of SURVEY.md G2; it is an input
    recipe only (the value of the vector, not how either side uses it)."""
    if mesh.map_degree != 1:
        raise ValueError("node_positions: box meshes only")
    t, _ = np.polynomial.legendre.leggauss(degree + 1)
    xi = 0.5 * (1.0 + t)
    gz, gy, gx = np.meshgrid(xi, xi, xi, indexing="ij")
    ref = np.stack([gx.reshape(-1), gy.reshape(-1), gz.reshape(-1)], axis=-1)
    x0 = mesh.nodes[:, 0, :]
    h = mesh.nodes[:, 7, :] - x0
    return x0[:, None, :] + h[:, None, :] * ref[None, :, :]


def field_to_dofs(values: np.ndarray) -> np.ndarray:
    """[cells, n^3, 3] point values -> canonical vector layout [cell][component][z][y][x]."""
    return np.ascontiguousarray(np.transpose(values, (0, 2, 1))).reshape(-1)


def c3_linearization(mesh, degree: int = 4, seed: int = 1) -> np.ndarray:
    """C3 u_lin: nodal interpolant of the 8-mode Fourier field drawn from rng(seed)."""
    x = node_positions(mesh, degree)
    return field_to_dofs(fourier_field(x, fourier_modes(seed)))


def c5_linearization(mesh, degree: int = 3, seed: int = 1) -> np.ndarray:
    """C5 u_lin: Poiseuille per block (inlet 6(y-1)(2-y), outlet 0.75 y(2-y), x-component)
    plus 0.1 x the 8-mode field in coordinates scaled to the unit box ((x+10)/50, y/2, z/4)."""
    x = node_positions(mesh, degree)
    u = np.zeros_like(x)
    inlet = x[..., 0] < 0.0
    y = x[..., 1]
    u[..., 0] = np.where(inlet, 6.0 * (y - 1.0) * (2.0 - y), 0.75 * y * (2.0 - y))
    xs = np.stack([(x[..., 0] + 10.0) / 50.0, x[..., 1] / 2.0, x[..., 2] / 4.0], axis=-1)
    u += 0.1 * fourier_field(xs, fourier_modes(seed))
    return field_to_dofs(u)
