"""Structured hexahedral meshes for the five BASELINE configurations.

Conventions (shared input format, also the C-ABI's `dgvv_mesh`, include/dgvv.h):
  * local faces are ordered (-x, +x, -y, +y, -z, +z);
  * neighbor[c, f] >= 0 is the global id of the cell across face f (periodic faces are
    ordinary neighbours); a boundary face stores -1 - bc with bc = 1 (Dirichlet) or
    2 (Neumann);
  * geometry is given as mapping nodes: nodes[c, a, :] is the physical position of the
    a-th node of a degree-`map_degree` tensor-product Lagrange map on the
    Gauss-Lobatto points of [0,1], lexicographic with x fastest.  map_degree = 1 means
    the 8 corner vertices (a = vx + 2 vy + 4 vz);
  * `periods[d]` > 0 marks direction d as periodic with that period (used only by the
    oracle's independent geometric face pairing).
No quantity of the method (metric, normal, penalty, ...) is computed here.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DIRICHLET = 1
NEUMANN = 2


def bc_code(bc: int) -> int:
    return -1 - bc


@dataclass
class Mesh:
    n_cells: int
    neighbor: np.ndarray          # int64 [n_cells, 6]
    nodes: np.ndarray             # float64 [n_cells, (map_degree+1)^3, 3]
    map_degree: int
    periods: tuple = (0.0, 0.0, 0.0)
    name: str = ""
    meta: dict = field(default_factory=dict)

    def validate(self) -> None:
        assert self.neighbor.shape == (self.n_cells, 6)
        m1 = self.map_degree + 1
        assert self.nodes.shape == (self.n_cells, m1 ** 3, 3)
        nb = self.neighbor
        inner = nb >= 0
        assert np.all(nb[inner] < self.n_cells)
        # reciprocity: if c --f--> c2 then c2 --f^1--> c
        c_idx, f_idx = np.nonzero(inner)
        back = nb[nb[c_idx, f_idx], f_idx ^ 1]
        assert np.all(back == c_idx), "neighbour table is not reciprocal"
        assert np.all((nb >= 0) | (nb == bc_code(DIRICHLET)) | (nb == bc_code(NEUMANN)))


def gll_points01(m: int) -> np.ndarray:
    """Gauss-Lobatto points of degree m on [0,1] (endpoints + roots of P_m'); input sampling only."""
    if m == 1:
        return np.array([0.0, 1.0])
    c = np.zeros(m + 1)
    c[m] = 1.0
    inner = np.polynomial.legendre.Legendre(c).deriv().roots()
    t = np.concatenate([[-1.0], np.sort(inner.real), [1.0]])
    return 0.5 * (1.0 + t)


def box_block(xs, ys, zs, order="xyz"):
    """Cells of one structured block with grid lines xs, ys, zs.

    order="xyz": id = i + nx*j + nx*ny*k  (x fastest; z-slabs are contiguous ranges)
    order="yzx": id = j + ny*k + ny*nz*i  (x slowest; x-slabs are contiguous ranges)
    Returns (ids[nx,ny,nz], vertices[n,8,3]) with vertices ordered by id.
    """
    xs, ys, zs = (np.asarray(a, dtype=np.float64) for a in (xs, ys, zs))
    nx, ny, nz = len(xs) - 1, len(ys) - 1, len(zs) - 1
    I, J, K = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    if order == "xyz":
        ids = I + nx * J + nx * ny * K
    elif order == "yzx":
        ids = J + ny * K + ny * nz * I
    else:
        raise ValueError(order)
    n = nx * ny * nz
    verts = np.empty((n, 8, 3))
    flat = ids.reshape(-1)
    Ii, Jj, Kk = I.reshape(-1), J.reshape(-1), K.reshape(-1)
    for v in range(8):
        vx, vy, vz = v & 1, (v >> 1) & 1, (v >> 2) & 1
        verts[flat, v, 0] = xs[Ii + vx]
        verts[flat, v, 1] = ys[Jj + vy]
        verts[flat, v, 2] = zs[Kk + vz]
    return ids, verts


def _block_neighbors(ids, nb, lo_bc, hi_bc, periodic):
    """Fill nb for cells of one block.  lo_bc/hi_bc[d]: boundary code on the low/high side
    of direction d (ignored when periodic[d])."""
    shape = ids.shape
    for d in range(3):
        n_d = shape[d]
        for side, step in ((0, -1), (1, +1)):
            f = 2 * d + side
            idx = np.arange(n_d)
            tgt = idx + step
            sl_src = [slice(None)] * 3
            for i in range(n_d):
                sl_src[d] = i
                src_ids = ids[tuple(sl_src)].reshape(-1)
                t = tgt[i]
                if 0 <= t < n_d or periodic[d]:
                    t %= n_d
                    sl_t = list(sl_src)
                    sl_t[d] = t
                    nb[src_ids, f] = ids[tuple(sl_t)].reshape(-1)
                else:
                    nb[src_ids, f] = (lo_bc if side == 0 else hi_bc)[d]


def cube(N: int, lo=0.0, hi=1.0, bc=DIRICHLET, periodic=(False, False, False), grid=None) -> Mesh:
    """[lo,hi]^3 with N^3 axis-aligned cells, id = i + N j + N^2 k (configs C1, C3, C4)."""
    g = np.linspace(lo, hi, N + 1) if grid is None else np.asarray(grid)
    ids, verts = box_block(g, g, g, "xyz")
    nb = np.empty((N ** 3, 6), dtype=np.int64)
    code = bc_code(bc)
    _block_neighbors(ids, nb, [code] * 3, [code] * 3, periodic)
    L = hi - lo
    periods = tuple(L if p else 0.0 for p in periodic)
    m = Mesh(N ** 3, nb, verts, 1, periods, name=f"cube{N}")
    m.meta["grid"] = (g, g, g)
    m.validate()
    return m


def cube_parent_map(N: int):
    """Nested refinement of cube(N // 2) into cube(N) (cell id = i + N j + N^2 k): the coarse
    parent id of every fine cell and its octant ox + 2 oy + 4 oz (which half of the parent it
    occupies along x, y, z).  Index bookkeeping only (h-levels)."""
    assert N % 2 == 0
    k, j, i = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    i, j, k = i.reshape(-1), j.reshape(-1), k.reshape(-1)
    Nc = N // 2
    parent = (i // 2) + Nc * (j // 2) + Nc * Nc * (k // 2)
    octant = (i % 2) + 2 * (j % 2) + 4 * (k % 2)
    return parent.astype(np.int32), octant.astype(np.int8)


def deformed_cube(N: int, map_degree: int, amp: float = 0.05, bc=DIRICHLET, nz_mult: int = 1) -> Mesh:
    """C2: [0,1]^3, N^3 cells, X = x^ + amp sin(2 pi x^) sin(2 pi y^) sin(2 pi z^) (1,1,1),
    sampled at the degree-`map_degree` GLL nodes of every cell (iso-parametric map).
    nz_mult > 1 stacks nz_mult such unit cubes in z ([0,1]^2 x [0,nz_mult], N x N x N nz_mult
    cells; the weak-scaling workload: one C2 cube per GPU)."""
    if nz_mult == 1:
        base = cube(N, bc=bc)
    else:
        g = np.linspace(0.0, 1.0, N + 1)
        gz = np.linspace(0.0, float(nz_mult), N * nz_mult + 1)
        ids, verts = box_block(g, g, gz, "xyz")
        nb = np.empty((ids.size, 6), dtype=np.int64)
        code = bc_code(bc)
        _block_neighbors(ids, nb, [code] * 3, [code] * 3, (False, False, False))
        base = Mesh(ids.size, nb, verts, 1)
    m1 = map_degree + 1
    g = gll_points01(map_degree)
    gz, gy, gx = np.meshgrid(g, g, g, indexing="ij")        # lexicographic, x fastest
    ref = np.stack([gx.reshape(-1), gy.reshape(-1), gz.reshape(-1)], axis=-1)  # [m1^3, 3]
    x0 = base.nodes[:, 0, :]
    h = base.nodes[:, 7, :] - base.nodes[:, 0, :]
    xh = x0[:, None, :] + h[:, None, :] * ref[None, :, :]
    s = np.sin(2 * np.pi * xh[..., 0]) * np.sin(2 * np.pi * xh[..., 1]) * np.sin(2 * np.pi * xh[..., 2])
    X = xh + amp * s[..., None]
    assert X.shape == (base.n_cells, m1 ** 3, 3)
    m = Mesh(base.n_cells, base.neighbor, X, map_degree, (0.0, 0.0, 0.0), name=f"deformed{N}_m{map_degree}x{nz_mult}")
    m.meta["amp"] = amp
    m.validate()
    return m


def bfs(nx_in=80, ny_in=32, nx_out=448, nz=32, r_out=1.005 ** 448, r_in=1.02 ** 80) -> Mesh:
    """C5 backward-facing step, h = 1, expansion ratio 2.

    Inlet block  [-10,0] x [1,2] x [0,4]: nx_in x ny_in x nz cells.
    Outlet block [0,40]  x [0,2] x [0,4]: nx_out x 2 ny_in x nz cells.
    x-grading is geometric toward x = 0 (the step); r_out / r_in are the TOTAL
    growth factors r^n (defaults 1.005^448 and 1.02^80 of the full-size mesh).
    Cells are ordered with x slowest (x-slabs are contiguous id ranges), inlet first.
    BCs: inlet x=-10 Dirichlet; outlet x=40 Neumann; walls and step face Dirichlet;
    z periodic (period 4).
    """
    ny_out = 2 * ny_in
    ro = r_out ** (1.0 / nx_out)
    ri = r_in ** (1.0 / nx_in)
    io = np.arange(nx_out + 1)
    xs_out = 40.0 * (ro ** io - 1.0) / (ro ** nx_out - 1.0)
    ii = np.arange(nx_in + 1)
    xs_in = -10.0 * (ri ** (nx_in - ii) - 1.0) / (ri ** nx_in - 1.0)
    xs_in[-1] = 0.0
    xs_out[0] = 0.0
    zs = np.linspace(0.0, 4.0, nz + 1)
    ys_in = np.linspace(1.0, 2.0, ny_in + 1)
    ys_out = np.linspace(0.0, 2.0, ny_out + 1)
    ids_in, v_in = box_block(xs_in, ys_in, zs, "yzx")
    ids_out, v_out = box_block(xs_out, ys_out, zs, "yzx")
    n_in = ids_in.size
    ids_out = ids_out + n_in
    n = n_in + ids_out.size
    nb = np.empty((n, 6), dtype=np.int64)
    D, Nm = bc_code(DIRICHLET), bc_code(NEUMANN)
    _block_neighbors(ids_in, nb, [D, D, 0], [D, D, 0], (False, False, True))
    _block_neighbors(ids_out, nb, [D, D, 0], [Nm, D, 0], (False, False, True))
    # block interface at x = 0: inlet (nx_in-1, j, k) <-> outlet (0, j + ny_in, k)
    for j in range(ny_in):
        a = ids_in[nx_in - 1, j, :]
        b = ids_out[0, j + ny_in, :]
        nb[a, 1] = b
        nb[b, 0] = a
    verts = np.concatenate([v_in, v_out], axis=0)
    m = Mesh(n, nb, verts, 1, (0.0, 0.0, 4.0), name=f"bfs{n}")
    m.meta.update(n_inlet=n_in, layer_out=ny_out * nz, nx_out=nx_out, nx_in=nx_in, layer_in=ny_in * nz)
    m.validate()
    return m


def config_mesh(cfg: int, small: bool = False) -> Mesh:
    """Mesh of BASELINE config C1..C5 (small=True: a reduced mesh of the same shape for tests)."""
    if cfg == 1:
        return cube(4)
    if cfg == 2:
        return deformed_cube(4 if small else 32, 3)
    if cfg in (3, 4):
        return cube(4 if small else 64)
    if cfg == 5:
        if small:
            return bfs(nx_in=6, ny_in=2, nx_out=20, nz=3)
        return bfs()
    raise ValueError(cfg)
