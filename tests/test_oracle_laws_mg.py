"""Oracle pins: viscosity laws (P9), Newton linearisation vs finite differences (P8),
Chebyshev closed form (P10), transfer / V-cycle / diagonal / Lanczos identities (P11)."""
import json
import os

import numpy as np
import pytest

from inputs import cube, deformed_cube, uniform
from inputs.vectors import c3_linearization
from oracle import dense, dg, laws, mg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------- P9 laws
def test_carreau_worked_values():
    gold = json.load(open(os.path.join(GOLD, "laws_worked_values.json")))
    for key in ("c3_law", "c5_law"):
        L = gold[key]
        for gd, val in L["eta"]:
            assert abs(laws.carreau(gd, L["eta0"], L["eta_inf"], L["lam"], L["n"]) - val) < 1e-15 * abs(val) * 4
        for gd, val in L["g"]:
            assert abs(laws.carreau_g(gd, L["eta0"], L["eta_inf"], L["lam"], L["n"]) - val) < 1e-14 * abs(val)
    ex = gold["spec_example_kappa2_a1"]
    p = ex["params"]
    v = laws.generalized_newtonian(ex["gd"], p["eta0"], p["eta_inf"], p["lam"], p["a"], p["b"], p["kappa"])
    assert abs(v - ex["eta"]) < 1e-4 * ex["eta"]
    c1 = gold["c1_nu_cell0_q0"]
    m = cube(4)
    d = dg.Disc(m, 2)
    x, _, _ = d.vol_geom(np.array([0]))
    assert np.allclose(x[0, 0], c1["x"], rtol=0, atol=1e-16)
    assert abs(laws.analytic(laws.C1_LAW, x[0, 0]) - c1["nu"]) < 1e-15


def test_carreau_special_cases_and_monotonicity():
    """eta(0) = eta0; n = 1 is Newtonian; n = 0 gives eta_inf + (eta0-eta_inf)/sqrt(1+(lam gd)^2);
    decreasing toward eta_inf for n < 1; g = eta'/gd against a central difference."""
    e0, ei, lam = 1.0, 1e-3, 2.0
    assert laws.carreau(0.0, e0, ei, lam, 0.5) == e0
    gd = np.logspace(-3, 4, 50)
    assert np.allclose(laws.carreau(gd, e0, ei, lam, 1.0), e0, rtol=1e-15)
    assert np.allclose(laws.carreau(gd, e0, ei, lam, 0.0), ei + (e0 - ei) / np.sqrt(1 + (lam * gd) ** 2), rtol=1e-14)
    eta = laws.carreau(gd, e0, ei, lam, 0.5)
    assert np.all(np.diff(eta) < 0) and np.all(eta > ei)
    assert abs(laws.carreau(1e12, e0, ei, lam, 0.5) - ei) < 1e-5
    h = 1e-4 * gd
    fd = (laws.carreau(gd + h, e0, ei, lam, 0.5) - laws.carreau(gd - h, e0, ei, lam, 0.5)) / (2 * h)
    assert np.allclose(laws.carreau_g(gd, e0, ei, lam, 0.5) * gd, fd, rtol=1e-5, atol=0)


def test_shear_rate_examples():
    """gamma_dot for simple shear u = (y,0,0) is 1, for a rigid rotation 0;
    adding a skew-symmetric gradient leaves eta unchanged."""
    G = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 0.0], [0.0, 0.0, 0.0]])
    assert abs(laws.shear_rate(dg.sym(G)) - 1.0) < 1e-15
    R = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 0.0]])
    assert laws.shear_rate(dg.sym(R)) == 0.0
    rng = np.random.default_rng(0)
    A = rng.normal(size=(3, 3))
    W = rng.normal(size=(3, 3))
    W = W - W.T
    assert abs(laws.shear_rate(dg.sym(A + W)) - laws.shear_rate(dg.sym(A))) < 1e-15


# ----------------------------------------------------------------- P8 Newton vs FD
@pytest.mark.parametrize("mk", ["cube", "deformed"])
def test_newton_matches_finite_differences(mk):
    """P8: (R(u0+hw) - R(u0-hw))/2h -> J(u0) w at O(h^2): error drops ~4x per halving."""
    m = cube(2) if mk == "cube" else deformed_cube(2, 2)
    k = 2
    d = dg.Disc(m, k)
    law = laws.C3_CARREAU
    if mk == "cube":
        u0 = c3_linearization(m, k)
    else:
        u0 = 3.0 * uniform(4, m.n_cells * 3 * d.N)
    w = uniform(0, len(u0))
    Jw = dg.newton_apply(d, u0, w, law)
    errs = []
    for h in (1e-3, 5e-4, 2.5e-4):
        hh = h * np.linalg.norm(u0) / np.linalg.norm(w)
        fd = (dg.carreau_residual(d, u0 + hh * w, law) - dg.carreau_residual(d, u0 - hh * w, law)) / (2 * hh)
        errs.append(np.linalg.norm(fd - Jw) / np.linalg.norm(Jw))
    assert errs[-1] < 1e-6
    assert 3.0 < errs[0] / errs[1] < 5.0 and 3.0 < errs[1] / errs[2] < 5.0


def test_newton_volume_part_monotone():
    """P8 extra: for Carreau n > 0 the linearised volume term is positive ((J w, w) > 0 for the
    volume-only operator) because the stress eta(gd) gd is monotone in gd."""
    from inputs.meshes import NEUMANN
    # volume-only: a single all-Neumann cell has no face terms
    m1 = cube(1, bc=NEUMANN)
    d1 = dg.Disc(m1, 2)
    u0 = 5.0 * uniform(2, 3 * d1.N)
    for s in range(5):
        w = uniform(10 + s, 3 * d1.N)
        assert w @ dg.newton_apply(d1, u0, w, laws.C3_CARREAU) > 0


# ----------------------------------------------------------------- P10 Chebyshev
def test_chebyshev_closed_form():
    """P10: e_m = T_m((theta - D^-1 A)/delta) e_0 / T_m(theta/delta), via the eigendecomposition
    of D^-1/2 A D^-1/2 (b = 0 so x_m = e_m)."""
    m = cube(2)
    d = dg.Disc(m, 2)
    A = dense.assemble_poisson(d, dg.AnalyticNu(d, laws.C4_LAW))
    D = np.diag(A)
    Dinv = 1.0 / D
    S = A / np.sqrt(np.outer(D, D))
    lam, V = np.linalg.eigh(S)
    hi = 1.2 * lam.max()
    lo = hi / 20
    theta, delta = (hi + lo) / 2, (hi - lo) / 2
    x0 = uniform(3, len(D))
    xm = mg.chebyshev(lambda x: A @ x, Dinv, np.zeros_like(x0), x0, lo, hi, 5)
    Tm = np.polynomial.chebyshev.Chebyshev.basis(5)
    pm = Tm((theta - lam) / delta) / Tm(theta / delta)
    ref = (V @ (pm * (V.T @ (np.sqrt(D) * x0)))) / np.sqrt(D)
    assert np.linalg.norm(xm - ref) < 1e-12 * np.linalg.norm(x0)
    # A = D: e_m = p_m(1) e_0
    xd = mg.chebyshev(lambda x: D * x, Dinv, np.zeros_like(x0), x0, lo, hi, 5)
    assert np.linalg.norm(xd - Tm((theta - 1) / delta) / Tm(theta / delta) * x0) < 1e-13 * np.linalg.norm(x0)


# ----------------------------------------------------------------- P11 transfer / V-cycle
@pytest.mark.parametrize("kf,kc", [(5, 3), (3, 2), (2, 1), (4, 4)])
def test_transfer_reproduces_coarse_polynomials(kf, kc):
    """P11: P maps the coarse interpolant of any polynomial of degree <= kc (per direction) to
    its fine interpolant; <R r, x_c> = <r, P x_c>."""
    xf, _ = np.polynomial.legendre.leggauss(kf + 1)
    xc, _ = np.polynomial.legendre.leggauss(kc + 1)
    xf, xc = (1 + xf) / 2, (1 + xc) / 2
    rng = np.random.default_rng(1)
    cx, cy, cz = rng.normal(size=(3, kc + 1))
    f = lambda x, y, z: np.polyval(cx, x) * np.polyval(cy, y) * np.polyval(cz, z)

    def grid(p):
        Z_, Y_, X_ = np.meshgrid(p, p, p, indexing="ij")
        return f(X_, Y_, Z_).reshape(-1)
    fine = mg.prolongate(grid(xc), kf, kc, 1)
    assert np.abs(fine - grid(xf)).max() < 1e-13 * np.abs(grid(xf)).max()
    r = rng.normal(size=(3, (kf + 1) ** 3)).reshape(-1)
    xcv = rng.normal(size=(3, (kc + 1) ** 3)).reshape(-1)
    assert abs(mg.restrict(r, kf, kc, 3) @ xcv - r @ mg.prolongate(xcv, kf, kc, 3)) < 1e-12 * np.linalg.norm(r) * np.linalg.norm(xcv)


def _levels(m, degrees, law):
    levels = []
    for li, k in enumerate(degrees):
        d = dg.Disc(m, k)
        A = dense.assemble_poisson(d, dg.AnalyticNu(d, law))
        Dinv = 1.0 / np.diag(A)
        lam = mg.lanczos_lambda_max(lambda x, A=A: A @ x, Dinv, uniform(2, len(Dinv)), 20)
        L = {"apply": (lambda x, A=A: A @ x), "Dinv": Dinv, "lam_hi": 1.2 * lam, "A": A, "k": k}
        if li + 1 < len(degrees):
            kc = degrees[li + 1]
            L["restrict"] = lambda r, k=k, kc=kc: mg.restrict(r, k, kc, m.n_cells)
            L["prolongate"] = lambda x, k=k, kc=kc: mg.prolongate(x, k, kc, m.n_cells)
        levels.append(L)
    return levels


def test_vcycle_linear_symmetric_and_contracting():
    """P11: V is linear and symmetric (pre/post Chebyshev adjoint); it reduces the error."""
    m = cube(2)
    levels = _levels(m, [5, 3, 2, 1], laws.C4_LAW)
    n = len(levels[0]["Dinv"])
    r1, r2 = uniform(0, n), uniform(1, n)
    V1, V2 = mg.vcycle(levels, r1), mg.vcycle(levels, r2)
    assert abs(r2 @ V1 - r1 @ V2) < 1e-12 * np.linalg.norm(V1) * np.linalg.norm(r2)
    V12 = mg.vcycle(levels, r1 + 2 * r2)
    assert np.linalg.norm(V12 - V1 - 2 * V2) < 1e-12 * np.linalg.norm(V12)
    A = levels[0]["A"]
    # error propagation I - V A is a contraction in the A-norm
    e = uniform(5, n)
    e1 = e - mg.vcycle(levels, A @ e)
    assert np.sqrt(e1 @ A @ e1) < 0.5 * np.sqrt(e @ A @ e)


def test_diagonal_and_lanczos():
    """D_ii from the matrix-free apply on e_i == diag(A_dense); Lanczos(20) on a <= 20-dim
    problem is exact; otherwise its Ritz value lies inside the spectrum of D^-1 A."""
    m = cube(2)
    d = dg.Disc(m, 1)
    nu = dg.AnalyticNu(d, laws.C1_LAW)
    A = dense.assemble_viscous(d, nu)
    n = A.shape[0]
    per = 3 * d.N

    def ap(c, e):
        full = np.zeros(n)
        full[c * per:(c + 1) * per] = e
        return dg.viscous_apply(d, full, nu, cells=[c]).reshape(-1)
    idx = np.arange(0, n, 7)
    assert np.allclose(mg.diagonal_entries(ap, d.N, idx, ncomp=3), np.diag(A)[idx], rtol=1e-13, atol=0)
    Dinv = 1.0 / np.diag(A)
    S = A * np.sqrt(np.outer(Dinv, Dinv))
    ev = np.linalg.eigvalsh(S)
    lam = mg.lanczos_lambda_max(lambda x: A @ x, Dinv, uniform(2, n), 20)
    assert ev.min() <= lam <= ev.max() * (1 + 1e-12) and lam > 0.9 * ev.max()
    small = A[:16, :16]
    Ds = 1.0 / np.diag(small)
    ev_s = np.linalg.eigvalsh(small * np.sqrt(np.outer(Ds, Ds)))
    lam_s = mg.lanczos_lambda_max(lambda x: small @ x, Ds, uniform(2, 16), 20)
    assert abs(lam_s - ev_s.max()) < 1e-10 * ev_s.max()


# ----------------------------------------------------------------- G19 coarse-level viscosity
def _nodal(disc, fn):
    """Nodal (collocation) coefficients of a physical vector field fn(x [...,3]) -> [...,3]."""
    x, _, _ = disc.vol_geom(np.arange(disc.mesh.n_cells))
    return np.ascontiguousarray(np.transpose(fn(x), (0, 2, 1))).reshape(-1)


@pytest.mark.parametrize("mk,kf,kc", [(lambda: cube(3), 4, 2), (lambda: deformed_cube(2, 2), 4, 2),
                                      (lambda: cube(2), 3, 1)])
def test_coarse_level_nu_g19_linear_field_is_exact(mk, kf, kc):
    """G19 pin (closed form): for u = A x the strain is sym(A) everywhere.  x(xi) is Q_{map
    degree} per cell, so u_lin's fine nodal interpolant and its coarse interpolation are both
    exact when the map degree <= k_c: the coarse nu must equal eta(gamma_dot(sym A)) at every
    coarse cell point and every face point of every side."""
    m = mk()
    df, dc = dg.Disc(m, kf), dg.Disc(m, kc)
    Amat = np.array([[0.3, -1.2, 0.5], [0.7, 0.1, -0.4], [-0.2, 0.9, -0.4]])
    ulin = _nodal(df, lambda x: x @ Amat.T)
    nu = dg.coarse_level_nu(df, dc, ulin, laws.C3_CARREAU)
    p = laws.C3_CARREAU
    eps = 0.5 * (Amat + Amat.T)
    expect = laws.carreau(np.sqrt(2.0 * np.sum(eps * eps)), p["eta0"], p["eta_inf"], p["lam"], p["n"])
    cells = np.arange(m.n_cells)
    assert np.allclose(nu.vol(cells), expect, rtol=1e-12, atol=0)
    for f in range(6):
        assert np.allclose(nu.face(cells, f), expect, rtol=1e-12, atol=0)
    # and the interpolated coefficients are the field's values at the coarse Gauss points
    assert np.allclose(dg.coarse_level_ulin(df, dc, ulin), _nodal(dc, lambda x: x @ Amat.T), rtol=0, atol=1e-13)


def test_coarse_level_nu_g19_quadratic_field():
    """G19 pin: a quadratic field is reproduced exactly by the k=2 level on box cells, so the
    coarse-level nu equals eta of the analytic strain at the coarse physical points (cell and
    face points); a transposed or wrongly ordered interpolation fails it."""
    m = cube(3)
    df, dc = dg.Disc(m, 4), dg.Disc(m, 2)

    def u(x):
        X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
        return np.stack([X * Y + 0.3 * Z * Z, -0.5 * X * X + Y * Z, 0.2 * X * Z - Y * Y], axis=-1)

    def grad(x):
        X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
        G = np.zeros(x.shape[:-1] + (3, 3))
        G[..., 0, 0], G[..., 0, 1], G[..., 0, 2] = Y, X, 0.6 * Z
        G[..., 1, 0], G[..., 1, 1], G[..., 1, 2] = -X, Z, Y
        G[..., 2, 0], G[..., 2, 1], G[..., 2, 2] = 0.2 * Z, -2.0 * Y, 0.2 * X
        return G

    p = laws.C3_CARREAU
    nu = dg.coarse_level_nu(df, dc, _nodal(df, u), p)

    def eta(x):
        e = 0.5 * (grad(x) + np.swapaxes(grad(x), -1, -2))
        return laws.carreau(np.sqrt(2.0 * np.einsum("...ij,...ij->...", e, e)), p["eta0"], p["eta_inf"], p["lam"], p["n"])

    cells = np.arange(m.n_cells)
    xq, _, _ = dc.vol_geom(cells)
    assert np.allclose(nu.vol(cells), eta(xq), rtol=1e-12, atol=0)
    for f in range(6):
        xf = dc.face_geom(cells, f)[0]
        assert np.allclose(nu.face(cells, f), eta(xf), rtol=1e-12, atol=0)
