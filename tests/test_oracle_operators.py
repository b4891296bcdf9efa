"""Oracle pins for the SIPG operators (c1.9).

Everything here is CPU-only (-m "not gpu").  Each test pins the oracle against something
other than itself: an invariant of SIPG, a closed form, an exact consistency property,
an independent symbolic (sympy) brute-force integration, or worked values computed
outside this repo (tests/golden/)."""
import json
import os

import numpy as np
import pytest
import sympy as sp

from inputs import bfs, cube, deformed_cube, uniform
from inputs.meshes import NEUMANN, Mesh
from oracle import dense, dg, laws

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sheared(N):
    """Affine (globally sheared) mesh: x -> A x + b applied to a Cartesian cube."""
    m = cube(N)
    A = np.array([[1.0, 0.2, 0.1], [0.0, 0.9, 0.15], [0.05, 0.0, 1.1]])
    nodes = m.nodes @ A.T + np.array([0.1, -0.2, 0.3])
    return Mesh(m.n_cells, m.neighbor, nodes, 1, (0.0, 0.0, 0.0), name=f"sheared{N}")


MESHES = {
    "cube2": lambda: cube(2),
    "deformed2": lambda: deformed_cube(2, 2),
    "bfs_small": lambda: bfs(nx_in=2, ny_in=1, nx_out=3, nz=3),
    "sheared2": lambda: sheared(2),
}


# ----------------------------------------------------------------- P1 symmetry + c1.9 dense
@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("k", [1, 2])
def test_symmetry_and_dense_equivalence(name, k):
    """P1: v^T A u = u^T A v for the matrix-free oracle (any nu field; north_star);
    c1.9: matrix-free == independently encoded dense assembly to rounding."""
    m = MESHES[name]()
    d = dg.Disc(m, k)
    nu = dg.AnalyticNu(d, laws.C2_LAW)
    n = m.n_cells * 3 * d.N
    u, v = uniform(0, n), uniform(1, n)
    for form in ("divergence", "laplace"):
        Au = dg.viscous_apply(d, u, nu, formulation=form)
        Av = dg.viscous_apply(d, v, nu, formulation=form)
        assert abs(v @ Au - u @ Av) < 1e-13 * np.linalg.norm(Au) * np.linalg.norm(v)
        A = dense.assemble_viscous(d, nu, form)
        assert np.linalg.norm(A @ u - Au) < 1e-14 * np.linalg.norm(Au) * 10
    p, q = uniform(0, m.n_cells * d.N), uniform(1, m.n_cells * d.N)
    Ap, Aq = dg.poisson_apply(d, p, nu), dg.poisson_apply(d, q, nu)
    assert abs(q @ Ap - p @ Aq) < 1e-13 * np.linalg.norm(Ap) * np.linalg.norm(q)
    AP = dense.assemble_poisson(d, nu)
    assert np.linalg.norm(AP @ p - Ap) < 1e-13 * np.linalg.norm(Ap)


# ----------------------------------------------------------------- P2 positive definiteness
def test_positive_definite_c1():
    """P2: Cholesky of the C1 operator (4^3, k=2, sin nu, all Dirichlet) succeeds."""
    m = cube(4)
    d = dg.Disc(m, 2)
    A = dense.assemble_viscous(d, dg.AnalyticNu(d, laws.C1_LAW))
    np.linalg.cholesky(A)
    assert np.abs(A - A.T).max() < 1e-13 * np.abs(A).max()


@pytest.mark.parametrize("k", [1, 3])
def test_positive_definite_high_contrast(k):
    """P2 at 1e4 coefficient contrast (C4 law, C5-like BFS with a Neumann outlet)."""
    bfs_law = {"kind": "exp", "rate": -np.log(1.0e4) / 55.0}     # x+y+z spans 55 on the BFS
    for m, law in ((cube(3), laws.C4_LAW), (bfs(nx_in=2, ny_in=1, nx_out=3, nz=3), bfs_law)):
        d = dg.Disc(m, k)
        c = dg.AnalyticNu(d, law)
        assert np.linalg.eigvalsh(dense.assemble_poisson(d, c)).min() > 0
        assert np.linalg.eigvalsh(dense.assemble_viscous(d, c)).min() > 0


# ----------------------------------------------------------------- P3 rigid-body modes
def rigid_modes(d):
    x, _, _ = d.vol_geom(np.arange(d.mesh.n_cells))          # collocation nodes = points
    modes = []
    for a in np.eye(3):
        modes.append(np.broadcast_to(a, x.shape))
    for w in np.eye(3):
        modes.append(np.cross(w, x))
    return [np.transpose(mo, (0, 2, 1)).reshape(-1) for mo in modes]


@pytest.mark.parametrize("mk", ["cube", "deformed"])
def test_rigid_body_kernel(mk):
    """P3: u = a + w x x is in the kernel with all-Neumann BCs; with Dirichlet BCs the rows
    of cells without a Dirichlet face vanish (the interior eps-form kills rigid motions)."""
    m = cube(3, bc=NEUMANN) if mk == "cube" else deformed_cube(3, 2, bc=NEUMANN)
    d = dg.Disc(m, 2)
    nu = dg.AnalyticNu(d, laws.C1_LAW)
    scale = np.linalg.norm(dg.viscous_apply(d, uniform(0, m.n_cells * 3 * d.N), nu))
    for u in rigid_modes(d):
        assert np.linalg.norm(dg.viscous_apply(d, u, nu)) < 1e-12 * scale * max(1, np.linalg.norm(u))
    md = cube(3)
    dd = dg.Disc(md, 2)
    nud = dg.AnalyticNu(dd, laws.C1_LAW)
    inner = np.nonzero((md.neighbor >= 0).all(1))[0]
    assert len(inner) == 1
    for u in rigid_modes(dd):
        y = dg.viscous_apply(dd, u, nud).reshape(md.n_cells, 3, -1)
        assert np.abs(y[inner]).max() < 1e-12 * scale


# ----------------------------------------------------------------- P4 homogeneity in nu
def test_homogeneity_in_nu():
    m = deformed_cube(2, 2)
    d = dg.Disc(m, 2)
    u = uniform(0, m.n_cells * 3 * d.N)
    y1 = dg.viscous_apply(d, u, dg.AnalyticNu(d, {"kind": "const", "value": 1.0}))
    y3 = dg.viscous_apply(d, u, dg.AnalyticNu(d, {"kind": "const", "value": 3.0}))
    assert np.linalg.norm(y3 - 3 * y1) < 1e-14 * np.linalg.norm(y3) * 4


# ----------------------------------------------------------------- P5 vector Laplacian
@pytest.mark.parametrize("name", ["cube2", "deformed2", "bfs_small"])
def test_laplace_part_is_vector_poisson(name):
    """P5: with formulation=laplace and nu == c, A_L u = c (I_3 (x) A_Poisson(1)) u
    (two separately written forms: Appendix A.3 vs A.2)."""
    m = MESHES[name]()
    d = dg.Disc(m, 2)
    c = 2.5
    u = uniform(0, m.n_cells * 3 * d.N)
    yL = dg.viscous_apply(d, u, dg.AnalyticNu(d, {"kind": "const", "value": c}), formulation="laplace")
    one = dg.AnalyticNu(d, {"kind": "const", "value": 1.0})
    U = u.reshape(m.n_cells, 3, d.N)
    yP = np.stack([dg.poisson_apply(d, U[:, i].reshape(-1), one).reshape(m.n_cells, d.N) for i in range(3)], 1)
    assert np.linalg.norm(yL - c * yP.reshape(-1)) < 1e-13 * np.linalg.norm(yL)


# ----------------------------------------------------------------- P6 manufactured solution
X, Y, Z = sp.symbols("x y z")


def _poly(rng, k):
    terms = [X ** a * Y ** b * Z ** c for a in range(k + 1) for b in range(k + 1) for c in range(k + 1) if a + b + c <= k]
    return sum(sp.Float(rng.uniform(-1, 1)) * t for t in terms)


@pytest.mark.parametrize("mk", ["cube", "sheared"])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_manufactured_polynomial_viscous(mk, k):
    """P6: for u in [P_k]^3 and affine nu on affine cells, A u_I = F(f, g) to rounding with
    f = -div(2 nu eps(u)) (sympy) and Dirichlet data g = u (Appendix A.5): SIPG consistency
    with exactly integrated (n_q = k+1) terms."""
    m = cube(2) if mk == "cube" else sheared(2)
    d = dg.Disc(m, k)
    rng = np.random.default_rng(7)
    u = [_poly(rng, k) for _ in range(3)]
    g = np.array([0.3, -0.2, 0.25])
    nu_s = 2.0 + g[0] * X + g[1] * Y + g[2] * Z
    law = {"kind": "affine", "c0": 2.0, "grad": g}
    xs = (X, Y, Z)
    eps = [[(sp.diff(u[i], xs[j]) + sp.diff(u[j], xs[i])) / 2 for j in range(3)] for i in range(3)]
    f = [-sum(sp.diff(2 * nu_s * eps[i][j], xs[j]) for j in range(3)) for i in range(3)]
    fu = sp.lambdify((X, Y, Z), u, "numpy")
    ff = sp.lambdify((X, Y, Z), f, "numpy")

    def ev(fun, x):
        return np.stack([np.broadcast_to(np.asarray(v, dtype=float), x.shape[:-1]) for v in fun(x[..., 0], x[..., 1], x[..., 2])], -1)

    cells = np.arange(m.n_cells)
    xq, JxW, _ = d.vol_geom(cells)
    uI = np.transpose(ev(fu, xq), (0, 2, 1)).reshape(-1)
    y = dg.viscous_apply(d, uI, dg.AnalyticNu(d, law)).reshape(m.n_cells, 3, d.N)

    F = np.einsum("cq,qn,cqi->cin", JxW, d.Phi, ev(ff, xq))
    H = d.H(cells)
    pen = (k + 1) ** 2
    for f_ in range(6):
        bc = np.nonzero(m.neighbor[:, f_] < 0)[0]
        if len(bc) == 0:
            continue
        xf, Jinv, n, dA = d.face_geom(bc, f_)
        gq = ev(fu, xf)
        nuq = laws.analytic(law, xf)
        tau = pen * H[bc][:, None] * nuq
        gphi = np.einsum("dpn,cpdj->cpnj", d.dPhiF[f_], Jinv)            # grad phi_n
        gn = np.einsum("cpi,cpi->cp", gq, n)
        for comp in range(3):
            # g . eps(phi e_comp) n = 1/2 (g_comp grad phi . n + n_comp g . grad phi)
            gen = 0.5 * (gq[..., comp, None] * np.einsum("cpnj,cpj->cpn", gphi, n)
                         + n[..., comp, None] * np.einsum("cpnj,cpj->cpn", gphi, gq))
            val = d.PhiF[f_][None] * (gq[..., comp] + n[..., comp] * gn)[..., None]
            F[bc, comp] += np.einsum("cp,cpn->cn", dA, -2 * nuq[..., None] * gen + 2 * tau[..., None] * val)
    assert np.linalg.norm(y - F) < 1e-12 * np.linalg.norm(F)


@pytest.mark.parametrize("mk", ["cube", "sheared"])
@pytest.mark.parametrize("k", [1, 2, 4])
def test_manufactured_polynomial_poisson(mk, k):
    """P6 (Poisson): p in P_k, c affine: A_P p_I = (q, f) + sum_D dA(-g c grad q.n + 2 tau q g),
    f = -div(c grad p)."""
    m = cube(2) if mk == "cube" else sheared(2)
    d = dg.Disc(m, k)
    rng = np.random.default_rng(3)
    p = _poly(rng, k)
    g = np.array([0.3, -0.2, 0.25])
    c_s = 2.0 + g[0] * X + g[1] * Y + g[2] * Z
    law = {"kind": "affine", "c0": 2.0, "grad": g}
    xs = (X, Y, Z)
    f = -sum(sp.diff(c_s * sp.diff(p, v), v) for v in xs)
    fp = sp.lambdify((X, Y, Z), p, "numpy")
    ff = sp.lambdify((X, Y, Z), f, "numpy")
    cells = np.arange(m.n_cells)
    xq, JxW, _ = d.vol_geom(cells)
    pI = np.broadcast_to(fp(xq[..., 0], xq[..., 1], xq[..., 2]), xq.shape[:-1]).reshape(-1)
    y = dg.poisson_apply(d, pI, dg.AnalyticNu(d, law)).reshape(m.n_cells, d.N)
    F = np.einsum("cq,qn,cq->cn", JxW, d.Phi, np.broadcast_to(ff(xq[..., 0], xq[..., 1], xq[..., 2]), xq.shape[:-1]))
    H = d.H(cells)
    for f_ in range(6):
        bc = np.nonzero(m.neighbor[:, f_] < 0)[0]
        xf, Jinv, n, dA = d.face_geom(bc, f_)
        gq = np.broadcast_to(fp(xf[..., 0], xf[..., 1], xf[..., 2]), xf.shape[:-1])
        cq = laws.analytic(law, xf)
        tau = (k + 1) ** 2 * H[bc][:, None] * cq
        gphin = np.einsum("dpn,cpdj,cpj->cpn", d.dPhiF[f_], Jinv, n)
        F[bc] += np.einsum("cp,cpn->cn", dA, -(gq * cq)[..., None] * gphin + (2 * tau * gq)[..., None] * d.PhiF[f_][None])
    assert np.linalg.norm(y - F) < 1e-12 * np.linalg.norm(F)


# ----------------------------------------------------------------- P7 exact brute force
# Exact integration independent of the oracle's tabulation/quadrature: every basis function
# is a product of three 1D monomial-coefficient polynomials (numpy.polynomial, built from
# the Gauss nodes as roots), nu is affine, so every integrand of Appendix A.1 is a sum of
# separable products and each integral is a product of exact 1D polynomial integrals.
from numpy.polynomial import Polynomial as Poly1


class Sep:
    """sum_t coef_t * px_t(x) py_t(y) pz_t(z)."""

    def __init__(self, terms):
        self.t = [t for t in terms if t[0] != 0.0]

    def __add__(self, o):
        return Sep(self.t + o.t)

    def __sub__(self, o):
        return Sep(self.t + [(-c, p) for c, p in o.t])

    def __mul__(self, o):
        if isinstance(o, (int, float)):
            return Sep([(c * o, p) for c, p in self.t])
        return Sep([(c1 * c2, tuple(a * b for a, b in zip(p1, p2))) for c1, p1 in self.t for c2, p2 in o.t])

    __rmul__ = __mul__

    def box(self, lo, hi):
        tot = 0.0
        for c, p in self.t:
            v = c
            for d_ in range(3):
                I = p[d_].integ()
                v *= I(hi[d_]) - I(lo[d_])
            tot += v
        return tot

    def face(self, lo, hi, dim, val):
        tot = 0.0
        for c, p in self.t:
            v = c * p[dim](val)
            for d_ in range(3):
                if d_ != dim:
                    I = p[d_].integ()
                    v *= I(hi[d_]) - I(lo[d_])
            tot += v
        return tot


ONE = Poly1([1.0])
ZERO_SEP = Sep([])


def _basis_1d(k, lo, h):
    t = np.polynomial.legendre.Legendre.basis(k + 1).roots()
    nodes = lo + h * (1 + np.sort(t)) / 2
    out = []
    for i in range(k + 1):
        others = np.delete(nodes, i)
        p = Poly1.fromroots(others)
        out.append(p / p(nodes[i]))
    return out


def _cell_basis(k, lo, h):
    """phi_i and d phi_i/dx_s (as Sep) for the 3D tensor basis on box [lo, lo+h]."""
    b1 = [_basis_1d(k, lo[d_], h[d_]) for d_ in range(3)]
    n = k + 1
    phi, dphi = [], []
    for i in range(n ** 3):
        ii = (i % n, (i // n) % n, i // (n * n))
        f = [b1[d_][ii[d_]] for d_ in range(3)]
        phi.append(Sep([(1.0, tuple(f))]))
        g = []
        for s_ in range(3):
            fs = list(f)
            fs[s_] = fs[s_].deriv()
            g.append(Sep([(1.0, tuple(fs))]))
        dphi.append(g)
    return phi, dphi


def _brute_force_viscous(cells_geo, k, nu_c0, nu_g, nbs, H, ip=1.0, rows=None):
    """Exact a(phi_a e_i, phi_b e_j) (Appendix A.1) on axis-aligned boxes."""
    N = (k + 1) ** 3
    nd = 3 * N
    nC = len(cells_geo)
    A = np.zeros((nC * nd, nC * nd))
    X1 = Poly1([0.0, 1.0])
    nu = Sep([(nu_c0, (ONE, ONE, ONE)), (nu_g[0], (X1, ONE, ONE)), (nu_g[1], (ONE, X1, ONE)), (nu_g[2], (ONE, ONE, X1))])
    bases = [_cell_basis(k, lo, h) for lo, h in cells_geo]
    pen = ip * (k + 1) ** 2

    def vec(c, a, i):
        """value (list of 3 Sep) and gradient G[r][s] = d v_r/d x_s of phi_a e_i in cell c."""
        val = [ZERO_SEP] * 3
        val[i] = bases[c][0][a]
        G = [[ZERO_SEP] * 3 for _ in range(3)]
        G[i] = list(bases[c][1][a])
        return val, G

    def eps(G):
        return [[(G[r][s] + G[s][r]) * 0.5 for s in range(3)] for r in range(3)]

    for c, (lo, h) in enumerate(cells_geo):
        hi = tuple(l_ + h_ for l_, h_ in zip(lo, h))
        for a in range(N):
            for i in range(3):
                if rows is not None and (c, a, i) not in rows:
                    continue
                ev = eps(vec(c, a, i)[1])
                for b in range(N):
                    for j in range(3):
                        eu = eps(vec(c, b, j)[1])
                        e = ZERO_SEP
                        for r in range(3):
                            for s_ in range(3):
                                e = e + ev[r][s_] * eu[r][s_]
                        A[c * nd + i * N + a, c * nd + j * N + b] += (2.0 * nu * e).box(lo, hi)

    for c, (lo, h) in enumerate(cells_geo):
        hi = tuple(l_ + h_ for l_, h_ in zip(lo, h))
        for f in range(6):
            dim, side = f // 2, f % 2
            n = np.zeros(3)
            n[dim] = 1.0 if side else -1.0
            val = hi[dim] if side else lo[dim]
            nb = nbs[c][f]
            if nb == "N" or (nb != "D" and nb < c):
                continue
            sides = [c] if nb == "D" else [c, nb]
            Hf = H[c] if nb == "D" else max(H[c], H[nb])
            for ca in sides:
                for a in range(N):
                    for i in range(3):
                        if rows is not None and (ca, a, i) not in rows:
                            continue
                        va, Ga = vec(ca, a, i)
                        sv = 1.0 if ca == c else -1.0
                        jv = [t * sv for t in va]                          # [v]
                        Ev = eps(Ga)
                        svn = [nu * sum((Ev[r][s_] * n[s_] for s_ in range(3)), ZERO_SEP) for r in range(3)]
                        for cb in sides:
                            for b in range(N):
                                for j in range(3):
                                    ub, Gb = vec(cb, b, j)
                                    Eu = eps(Gb)
                                    if nb == "D":                          # mirror trial state
                                        ju = [t * 2.0 for t in ub]
                                        mult = 2.0
                                        tau_s = nu * (pen * Hf)
                                    else:
                                        su = 1.0 if cb == c else -1.0
                                        ju = [t * su for t in ub]
                                        mult = 1.0
                                        tau_s = nu * (pen * Hf)
                                    sun = [nu * sum((Eu[r][s_] * n[s_] for s_ in range(3)), ZERO_SEP) * mult for r in range(3)]
                                    jun = sum((ju[r] * n[r] for r in range(3)), ZERO_SEP)
                                    jvn = sum((jv[r] * n[r] for r in range(3)), ZERO_SEP)
                                    e = ZERO_SEP
                                    for r in range(3):
                                        e = e - jv[r] * sun[r] - ju[r] * svn[r] + tau_s * (jv[r] * ju[r])
                                    e = e + tau_s * (jvn * jun)
                                    A[ca * nd + i * N + a, cb * nd + j * N + b] += e.face(lo, hi, dim, val)
    return A


@pytest.mark.parametrize("k", [1, 2])
def test_brute_force_exact_two_cells(k):
    """P7: two Cartesian cells [0,.5]^3 and [.5,1]x[0,.5]^2, affine nu, Dirichlet outer faces:
    every entry of the oracle's A equals the exact integral of Appendix A.1."""
    from inputs.meshes import box_block
    _, verts = box_block([0, 0.5, 1.0], [0, 0.5], [0, 0.5])
    nb = np.array([[-2, 1, -2, -2, -2, -2], [0, -2, -2, -2, -2, -2]], dtype=np.int64)
    m = Mesh(2, nb, verts, 1)
    d = dg.Disc(m, k)
    law = {"kind": "affine", "c0": 1.5, "grad": [0.4, -0.3, 0.2]}
    A_or = dense.assemble_viscous(d, dg.AnalyticNu(d, law))
    H = [(0.5 * 0.25 + 5 * 0.25) / 0.125] * 2                      # G3 by hand: 11
    geo = [((0.0, 0.0, 0.0), (0.5, 0.5, 0.5)), ((0.5, 0.0, 0.0), (0.5, 0.5, 0.5))]
    nbs = [["D", 1, "D", "D", "D", "D"], [0, "D", "D", "D", "D", "D"]]
    N = (k + 1) ** 3
    rows = None
    if k == 2:   # full k=2 takes minutes: check the rows of a few basis functions touching the faces
        rows = {(c, a, i) for c in (0, 1) for a in (0, 4, 14, 26) for i in range(3)}
    A_bf = _brute_force_viscous(geo, k, 1.5, (0.4, -0.3, 0.2), nbs, H, rows=rows)
    if rows is not None:
        idx = [c * 3 * N + i * N + a for (c, a, i) in sorted(rows)]
        A_bf, A_or = A_bf[idx], A_or[idx]
    assert np.abs(A_bf).max() > 0
    assert np.abs(A_bf - A_or).max() < 1e-12 * np.abs(A_bf).max()


# ----------------------------------------------------------------- P13 worked values
def _closed_form_p13(N, k):
    """sum over boundary faces of 2 tau |F| (weights) with tau = (k+1)^2 H_K, H_K from G3 on
    an N^3 Cartesian unit cube (count of boundary faces per cell), computed independently."""
    h = 1.0 / N
    tot_p = 0.0
    tot_v = np.zeros(3)
    for i in range(N):
        for j in range(N):
            for l in range(N):
                idx = (i, j, l)
                nbf = sum((t == 0) + (t == N - 1) for t in idx) if N > 1 else 6
                H = (0.5 * (6 - nbf) * h * h + nbf * h * h) / h ** 3
                for dim in range(3):
                    for end in (0, N - 1):
                        if idx[dim] == end:
                            cnt = 2 if N == 1 else 1
                            if N > 1 and end == 0 and end == N - 1:
                                cnt = 2
                            w = 2 * (k + 1) ** 2 * H * h * h * (cnt if N == 1 else 1)
                            if N == 1:
                                w /= 2          # loop visits end 0 and N-1 (same index) twice
                            tot_p += w
                            for c in range(3):
                                tot_v[c] += w * (1 + (c == dim))
    return tot_v, tot_p


@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "constant_energy_p13.json")))["cases"][:3])
def test_constant_field_energy_worked_values(case):
    """P13 worked values (golden) == oracle == independent closed form."""
    N, k = case["N"], case["k"]
    m = cube(N)
    d = dg.Disc(m, k)
    one = dg.AnalyticNu(d, {"kind": "const", "value": 1.0})
    cf_v, cf_p = _closed_form_p13(N, k)
    for c in range(3):
        e = np.zeros((m.n_cells, 3, d.N))
        e[:, c] = 1.0
        val = e.reshape(-1) @ dg.viscous_apply(d, e.reshape(-1), one)
        assert abs(val - case["viscous"]) < 1e-12 * case["viscous"]
        assert abs(cf_v[c] - case["viscous"]) < 1e-12 * case["viscous"]
    e = np.ones(m.n_cells * d.N)
    val = e @ dg.poisson_apply(d, e, one)
    assert abs(val - case["poisson"]) < 1e-12 * case["poisson"]
    assert abs(cf_p - case["poisson"]) < 1e-12 * case["poisson"]


def test_closed_form_matches_large_worked_values():
    """The independent closed form reproduces the survey's large-mesh values (C2/C3/C4 sizes);
    the GPU tests check dot(e_c, apply(e_c)) against these at full size."""
    for case in json.load(open(os.path.join(GOLD, "constant_energy_p13.json")))["cases"]:
        v, p = _closed_form_p13(case["N"], case["k"])
        assert abs(v[0] - case["viscous"]) < 1e-9 * case["viscous"]
        assert abs(p - case["poisson"]) < 1e-9 * case["poisson"]
