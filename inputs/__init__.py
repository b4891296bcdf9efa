"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no basis, quadrature, geometry metric,
viscosity law or operator).  It only produces the inputs both sides consume:
  * structured hexahedral meshes (corner vertices or iso-parametric node positions,
    face-neighbour tables with boundary ids, periodicity vectors), and
  * seeded random vectors / smooth random fields (SURVEY.md §8(c) G20, §8(d) input recipe).
Positions of mapping nodes and of sampling points are produced with library
primitives (numpy Legendre roots); both the oracle and the CUDA library re-derive
every quantity they need from these positions with their own code.
"""
from .meshes import Mesh, cube, cube_parent_map, deformed_cube, bfs, box_block, config_mesh  # noqa: F401
from .vectors import uniform, fourier_modes, fourier_field, node_positions  # noqa: F401
