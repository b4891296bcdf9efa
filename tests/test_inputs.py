"""Input generators: mesh sizes/topology of the BASELINE configs."""
import numpy as np

from inputs import bfs, config_mesh, cube, uniform
from inputs.meshes import DIRICHLET, NEUMANN, bc_code


def test_config_sizes():
    assert config_mesh(1).n_cells == 64
    m5 = bfs()
    assert m5.n_cells == 999424
    assert m5.meta["n_inlet"] == 81920
    # boundary face counts of C5 (37,888 boundary faces)
    assert int((m5.neighbor < 0).sum()) == 37888
    assert int((m5.neighbor == bc_code(NEUMANN)).sum()) == 64 * 32
    c3 = cube(64)
    assert int((c3.neighbor < 0).sum()) == 24576


def test_uniform_recipe():
    assert np.array_equal(uniform(0, 5), np.random.default_rng(0).uniform(-1, 1, 5))


def test_bfs_grading():
    m = bfs()
    x = m.nodes[:, :, 0]
    dx = x[:, 7] - x[:, 0]
    out = m.meta["n_inlet"]
    assert abs(dx[out:].min() - 0.0239) < 1e-3 and abs(dx[out:].max() - 0.22) < 1e-2
    assert np.all(dx > 0)
