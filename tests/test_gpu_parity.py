"""GPU parity: libdgvv.so (through the C ABI) against the CPU oracle on the same seeded
inputs.  Tolerance: relative L2 <= 1e-12 in FP64 (BASELINE north_star; reading G25)."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import bfs, cube, deformed_cube, uniform                       # noqa: E402
from inputs.vectors import c3_linearization                               # noqa: E402
from oracle import dense, dg, laws, mg                                    # noqa: E402

TOL = 1e-12
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def Ctx(*a, **k):
    from paper_2506_14424_b200.dgvv import Context
    return Context(*a, **k)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def gpu_apply(ctx, u, level=0, op="visc"):
    s = dev(u)
    y = torch.empty_like(s)
    (ctx.apply_viscous if op == "visc" else ctx.apply_poisson)(s, y, level)
    return host(y)


# ------------------------------------------------------------------ viscous apply
CASES = [
    ("C1 cube4 k2 sin", lambda: cube(4), 2, laws.C1_LAW),
    ("C2-shape deformed4 k3 exp", lambda: deformed_cube(4, 3), 3, laws.C2_LAW),
    ("deformed3 k2 (map deg 2)", lambda: deformed_cube(3, 2), 2, laws.C1_LAW),
    ("BFS small k3", lambda: bfs(nx_in=3, ny_in=2, nx_out=5, nz=3), 3, laws.C1_LAW),
    ("cube3 k1", lambda: cube(3), 1, laws.C2_LAW),
    ("cube3 k4", lambda: cube(3), 4, laws.C2_LAW),
    ("cube2 k5", lambda: cube(2), 5, laws.C1_LAW),
]


@pytest.mark.parametrize("name,mk,k,law", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("form", ["divergence", "laplace"])
def test_viscous_apply_parity(name, mk, k, law, form):
    m = mk()
    d = dg.Disc(m, k)
    u = uniform(0, m.n_cells * 3 * d.N)
    ref = dg.viscous_apply(d, u, dg.AnalyticNu(d, law), formulation=form)
    ctx = Ctx(m, k, visc_law=law, formulation=form)
    assert rel(gpu_apply(ctx, u), ref) < TOL


def test_viscous_apply_deterministic_and_alias_rejected():
    m = deformed_cube(4, 3)
    ctx = Ctx(m, 3, visc_law=laws.C2_LAW)
    s = dev(uniform(0, m.n_cells * 3 * 64))
    y1, y2 = torch.empty_like(s), torch.empty_like(s)
    ctx.apply_viscous(s, y1)
    for _ in range(5):
        ctx.apply_viscous(s, y2)
    assert torch.equal(y1, y2)
    from paper_2506_14424_b200 import DgvvError
    with pytest.raises(DgvvError):
        ctx.apply_viscous(s, s)


# ------------------------------------------------------------------ Poisson
@pytest.mark.parametrize("mk", [lambda: cube(3), lambda: deformed_cube(3, 2), lambda: bfs(nx_in=2, ny_in=1, nx_out=4, nz=3)])
def test_poisson_apply_parity_all_levels(mk):
    m = mk()
    degs = [5, 3, 2, 1]
    law = laws.C4_LAW if m.periods == (0.0, 0.0, 0.0) else {"kind": "exp", "rate": -np.log(1e4) / 55}
    ctx = Ctx(m, 5, poisson_law=law, degrees=degs)
    for l, k in enumerate(degs):
        d = dg.Disc(m, k)
        p = uniform(l, m.n_cells * d.N)
        ref = dg.poisson_apply(d, p, dg.AnalyticNu(d, law))
        assert rel(gpu_apply(ctx, p, l, op="pois"), ref) < TOL, (l, k)


def test_laplace_equals_vector_poisson_on_gpu():
    """P5 on the GPU: apply_viscous(laplace, nu=c) == c * per-component apply_poisson(c=1)."""
    m = deformed_cube(3, 2)
    c = 2.5
    cv = Ctx(m, 2, visc_law={"kind": "const", "value": c}, formulation="laplace")
    cp = Ctx(m, 2, poisson_law={"kind": "const", "value": 1.0})
    u = uniform(0, m.n_cells * 3 * 27)
    yv = gpu_apply(cv, u).reshape(m.n_cells, 3, 27)
    U = u.reshape(m.n_cells, 3, 27)
    for i in range(3):
        yp = gpu_apply(cp, np.ascontiguousarray(U[:, i]).reshape(-1), op="pois").reshape(m.n_cells, 27)
        assert rel(yv[:, i], c * yp) < TOL


# ------------------------------------------------------------------ diagonal
@pytest.mark.parametrize("op", ["visc", "pois"])
@pytest.mark.parametrize("mk", [lambda: cube(2), lambda: deformed_cube(2, 2), lambda: bfs(nx_in=2, ny_in=1, nx_out=3, nz=3)])
def test_inverse_diagonal(op, mk):
    m = mk()
    k = 2
    d = dg.Disc(m, k)
    law = laws.C1_LAW
    if op == "visc":
        A = dense.assemble_viscous(d, dg.AnalyticNu(d, law))
        ctx = Ctx(m, k, visc_law=law)
        out = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
        ctx.inverse_diagonal(0, out)
    else:
        A = dense.assemble_poisson(d, dg.AnalyticNu(d, law))
        ctx = Ctx(m, k, poisson_law=law)
        out = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
        ctx.inverse_diagonal(1, out)
    assert rel(host(out), 1.0 / np.diag(A)) < TOL


# ------------------------------------------------------------------ transfer
@pytest.mark.parametrize("pair", [(5, 3), (3, 2), (2, 1), (4, 2), (3, 1), (5, 1)])
def test_transfer_parity(pair):
    kf, kc = pair
    m = cube(3)
    ctx = Ctx(m, kf, poisson_law=laws.C4_LAW, degrees=[kf, kc])
    nf, nc = (kf + 1) ** 3, (kc + 1) ** 3
    xc = uniform(1, m.n_cells * nc)
    xf0 = uniform(2, m.n_cells * nf)
    f = dev(xf0.copy())
    ctx.prolongate(1, 0, dev(xc), f, beta=1.0)
    assert rel(host(f), mg.prolongate(xc, kf, kc, m.n_cells) + xf0) < TOL
    r = uniform(3, m.n_cells * nf)
    c = dev(np.zeros(m.n_cells * nc))
    ctx.restrict(1, 0, dev(r), c, beta=0.0)
    assert rel(host(c), mg.restrict(r, kf, kc, m.n_cells)) < TOL


@pytest.mark.parametrize("pair", [(4, 2), (3, 2), (2, 1)])
def test_transfer_parity_vector(pair):
    """Three-component transfer (the viscous operator's levels): each component block is transferred
    on its own, cell-major [cell][c][point]; ragged last CTA (5^3 cells); beta != 0 on both sides."""
    kf, kc = pair
    m = cube(5)
    ctx = Ctx(m, kf, visc_law=laws.C1_LAW, degrees=[kf, kc])
    nf, nc = (kf + 1) ** 3, (kc + 1) ** 3
    xc = uniform(1, 3 * m.n_cells * nc)
    xf0 = uniform(2, 3 * m.n_cells * nf)
    f = dev(xf0.copy())
    ctx.prolongate(0, 0, dev(xc), f, beta=0.5)
    assert rel(host(f), mg.prolongate(xc, kf, kc, 3 * m.n_cells) + 0.5 * xf0) < TOL
    r = uniform(3, 3 * m.n_cells * nf)
    c0 = uniform(4, 3 * m.n_cells * nc)
    c = dev(c0.copy())
    ctx.restrict(0, 0, dev(r), c, beta=-2.0)
    assert rel(host(c), mg.restrict(r, kf, kc, 3 * m.n_cells) - 2.0 * c0) < TOL


# ------------------------------------------------------------------ smoother / V-cycle
def _oracle_levels(m, degs, law):
    levels = []
    for li, k in enumerate(degs):
        d = dg.Disc(m, k)
        nu = dg.AnalyticNu(d, law)
        A = dense.assemble_poisson(d, nu)
        L = {"apply": (lambda x, A=A: A @ x), "Dinv": 1.0 / np.diag(A), "A": A}
        if li + 1 < len(degs):
            kc = degs[li + 1]
            L["restrict"] = lambda r, k=k, kc=kc: mg.restrict(r, k, kc, m.n_cells)
            L["prolongate"] = lambda x, k=k, kc=kc: mg.prolongate(x, k, kc, m.n_cells)
        levels.append(L)
    return levels


def test_chebyshev_and_vcycle_parity():
    m = cube(2)
    degs = [5, 3, 2, 1]
    law = laws.C4_LAW
    ctx = Ctx(m, 5, poisson_law=law, degrees=degs)
    levels = _oracle_levels(m, degs, law)
    n0 = len(levels[0]["Dinv"])
    # Lanczos estimate parity (same start vector)
    lams = []
    for l, L in enumerate(levels):
        v0 = uniform(2, len(L["Dinv"]))
        lo = mg.lanczos_lambda_max(L["apply"], L["Dinv"], v0, 20)
        lg = ctx.estimate_lambda_max(1, dev(v0), level=l, steps=20)
        assert abs(lg - lo) < 1e-10 * lo, (l, lg, lo)
        lams.append(1.2 * lo)
        L["lam_hi"] = 1.2 * lo
    b = uniform(0, n0)
    hi = lams[0]
    # Chebyshev from zero and from x0
    x = dev(np.zeros(n0))
    ctx.chebyshev_smooth(1, x, dev(b), hi / 20, hi, 5, x_is_zero=True)
    ref = mg.chebyshev(levels[0]["apply"], levels[0]["Dinv"], b, np.zeros(n0), hi / 20, hi, 5)
    assert rel(host(x), ref) < TOL
    x0 = uniform(3, n0)
    x = dev(x0)
    ctx.chebyshev_smooth(1, x, dev(b), hi / 20, hi, 5, x_is_zero=False)
    ref = mg.chebyshev(levels[0]["apply"], levels[0]["Dinv"], b, x0, hi / 20, hi, 5)
    assert rel(host(x), ref) < TOL
    # V-cycle
    xv = dev(np.zeros(n0))
    ctx.vcycle(1, dev(b), xv, lams)
    assert rel(host(xv), mg.vcycle(levels, b)) < TOL


# ------------------------------------------------------------------ Carreau
@pytest.mark.parametrize("mk,k", [(lambda: cube(3), 4), (lambda: bfs(nx_in=2, ny_in=1, nx_out=4, nz=3), 3)])
def test_carreau_viscosity_and_apply(mk, k):
    m = mk()
    d = dg.Disc(m, k)
    law = laws.C3_CARREAU
    if m.periods == (0.0, 0.0, 0.0):
        ulin = c3_linearization(m, k)
    else:
        from inputs.vectors import c5_linearization
        ulin = c5_linearization(m, k)
    nu = dg.CarreauNu(d, ulin, law)
    u = uniform(0, len(ulin))
    ref = dg.viscous_apply(d, u, nu)
    ctx = Ctx(m, k, visc_law=law)
    from paper_2506_14424_b200 import DgvvError
    with pytest.raises(DgvvError):           # ESTATE before the first update
        ctx.apply_viscous(dev(u), dev(u * 0))
    ul = dev(ulin)
    ctx.update_viscosity(ul)
    assert rel(gpu_apply(ctx, u), ref) < TOL
    lo, hi = ctx.coefficient_range(0)
    cells = np.arange(m.n_cells)
    allv = np.concatenate([nu.vol(cells).ravel()] + [nu.face(cells, f).ravel() for f in range(6)])
    assert abs(lo - allv.min()) < 1e-13 and abs(hi - allv.max()) < 1e-13


# ------------------------------------------------------------------ P13 at full size
@pytest.mark.parametrize("N,k", [(32, 3), (64, 4)])
def test_constant_field_energy_full_size(N, k):
    """P13 worked values (golden) on the full C2/C3-size Cartesian meshes, nu = 1."""
    gold = {(c["N"], c["k"]): c for c in json.load(open(os.path.join(GOLD, "constant_energy_p13.json")))["cases"]}
    m = cube(N)
    ctx = Ctx(m, k, visc_law={"kind": "const", "value": 1.0})
    n3 = (k + 1) ** 3
    e = torch.zeros(m.n_cells, 3, n3, dtype=torch.float64, device="cuda")
    e[:, 0] = 1.0
    e = e.reshape(-1)
    y = torch.empty_like(e)
    ctx.apply_viscous(e, y)
    val = ctx.dot(e, y, ncomp=3)
    assert abs(val - gold[(N, k)]["viscous"]) < 1e-11 * gold[(N, k)]["viscous"]


def test_poisson_constant_energy_c4_size():
    gold = {(c["N"], c["k"]): c for c in json.load(open(os.path.join(GOLD, "constant_energy_p13.json")))["cases"]}
    m = cube(64)
    ctx = Ctx(m, 5, poisson_law={"kind": "const", "value": 1.0})
    e = torch.ones(m.n_cells * 216, dtype=torch.float64, device="cuda")
    y = torch.empty_like(e)
    ctx.apply_poisson(e, y)
    assert abs(ctx.dot(e, y) - gold[(64, 5)]["poisson"]) < 1e-11 * gold[(64, 5)]["poisson"]


# ------------------------------------------------------------------ full-size sampled parity
def _sample_cells(m, count, seed=5):
    rng = np.random.default_rng(seed)
    bnd = np.nonzero((m.neighbor < 0).any(1))[0]
    inner = np.nonzero((m.neighbor >= 0).all(1))[0]
    pick = [rng.choice(bnd, min(len(bnd), count // 2), replace=False),
            rng.choice(inner, min(len(inner), count - count // 2), replace=False)]
    return np.sort(np.concatenate(pick))


def test_c2_full_size_sampled():
    """C2 at full size (32^3 deformed, k=3, 6.3M DoFs): GPU apply vs oracle on 64 sampled cells."""
    m = deformed_cube(32, 3)
    d = dg.Disc(m, 3)
    u = uniform(0, m.n_cells * 3 * 64)
    ctx = Ctx(m, 3, visc_law=laws.C2_LAW)
    y = gpu_apply(ctx, u).reshape(m.n_cells, 3, 64)
    cells = _sample_cells(m, 64)
    ref = dg.viscous_apply(d, u, dg.AnalyticNu(d, laws.C2_LAW), cells=cells)
    assert rel(y[cells], ref) < TOL


def test_c3_full_size_sampled_carreau():
    """C3 at full size (64^3, k=4, Carreau from the 8-mode field): sampled cells."""
    m = cube(64)
    k = 4
    d = dg.Disc(m, k)
    ulin = c3_linearization(m, k)
    u = uniform(0, len(ulin))
    ctx = Ctx(m, k, visc_law=laws.C3_CARREAU)
    ctx.update_viscosity(dev(ulin))
    y = gpu_apply(ctx, u).reshape(m.n_cells, 3, 125)
    cells = _sample_cells(m, 48)
    ref = dg.viscous_apply(d, u, dg.CarreauNu(d, ulin, laws.C3_CARREAU), cells=cells)
    assert rel(y[cells], ref) < TOL


# ------------------------------------------------------------------ Newton (K2)
@pytest.mark.parametrize("mk,k", [(lambda: cube(3), 4), (lambda: deformed_cube(3, 2), 2),
                                  (lambda: bfs(nx_in=2, ny_in=1, nx_out=4, nz=3), 3), (lambda: cube(2), 1)])
def test_newton_apply_parity(mk, k):
    """J(u0) w on the GPU == oracle newton_apply (reading G10; FD-pinned in the oracle tests)."""
    m = mk()
    d = dg.Disc(m, k)
    law = laws.C3_CARREAU
    if m.map_degree == 1 and m.periods == (0.0, 0.0, 0.0):
        u0 = c3_linearization(m, k)
    else:
        u0 = 2.0 * uniform(7, m.n_cells * 3 * d.N)
    w = uniform(0, len(u0))
    ref = dg.newton_apply(d, u0, w, law)
    ctx = Ctx(m, k, visc_law=law)
    from paper_2506_14424_b200 import DgvvError
    with pytest.raises(DgvvError):
        ctx.apply_linearized_viscous(dev(w), dev(w * 0))
    ul = dev(u0)
    ctx.update_viscosity(ul)
    y = torch.empty_like(ul)
    ctx.apply_linearized_viscous(dev(w), y)
    assert rel(host(y), ref) < TOL


def test_newton_full_size_sampled_c3():
    m = cube(64)
    k = 4
    d = dg.Disc(m, k)
    u0 = c3_linearization(m, k)
    w = uniform(0, len(u0))
    ctx = Ctx(m, k, visc_law=laws.C3_CARREAU)
    ul = dev(u0)
    ctx.update_viscosity(ul)
    y = torch.empty_like(ul)
    ctx.apply_linearized_viscous(dev(w), y)
    y = host(y).reshape(m.n_cells, 3, 125)
    cells = _sample_cells(m, 32)
    ref = dg.newton_apply(d, u0, w, laws.C3_CARREAU, cells=cells)
    assert rel(y[cells], ref) < TOL


def test_c4_full_size_sampled_poisson_and_chebyshev_step():
    """C4 at full size (64^3, k=5, c = exp(-ln(1e4)(x+y+z)/3), 56.6M DoFs): the Poisson apply vs
    the oracle on sampled cells; then the fused Chebyshev step (K6 epilogue, x0 != 0, m = 1) must
    equal its unfused definition x1 = x0 + D^-1 (b - A x0)/theta built from
    the library's own apply and diagonal — a fusion property at full size (the oracle pins A x0
    here, D^-1 and Chebyshev on the dense oracle in the small-mesh tests above)."""
    m = cube(64)
    k = 5
    d = dg.Disc(m, k)
    n3 = (k + 1) ** 3
    ctx = Ctx(m, k, poisson_law=laws.C4_LAW)
    x0 = uniform(3, m.n_cells * n3)
    b = uniform(0, m.n_cells * n3)
    cells = _sample_cells(m, 32)
    y = gpu_apply(ctx, x0, op="pois")
    Ax = dg.poisson_apply(d, x0, dg.AnalyticNu(d, laws.C4_LAW), cells=cells)
    assert rel(y.reshape(m.n_cells, n3)[cells], Ax) < TOL
    dinv = torch.empty(m.n_cells * n3, dtype=torch.float64, device="cuda")
    ctx.inverse_diagonal(1, dinv)
    lo, hi = 0.05, 1.0
    x = dev(x0)
    ctx.chebyshev_smooth(1, x, dev(b), lo, hi, 1, x_is_zero=False)
    theta = 0.5 * (hi + lo)
    ref = x0 + host(dinv) * (b - y) / theta
    assert rel(host(x), ref) < 1e-14


def test_c4_full_size_vcycle_is_symmetric():
    """V-cycle 5->3->2->1 at full C4 size is linear and symmetric (P11: pre- and post-Chebyshev
    are adjoint): <V r1, r2> = <r1, V r2> and V(r1 + 2 r2) = V r1 + 2 V r2 to rounding."""
    m = cube(64)
    degs = [5, 3, 2, 1]
    ctx = Ctx(m, 5, poisson_law=laws.C4_LAW, degrees=degs)
    lams = [1.2 * ctx.estimate_lambda_max(1, dev(uniform(2, ctx.n_dofs(l))), level=l, steps=20)
            for l in range(len(degs))]
    n0 = ctx.n_dofs(0)
    r1, r2 = dev(uniform(0, n0)), dev(uniform(1, n0))
    v1, v2, v3 = (torch.zeros(n0, dtype=torch.float64, device="cuda") for _ in range(3))
    ctx.vcycle(1, r1, v1, lams)
    ctx.vcycle(1, r2, v2, lams)
    ctx.vcycle(1, r1 + 2.0 * r2, v3, lams)
    a, bb = ctx.dot(v1, r2), ctx.dot(r1, v2)
    assert abs(a - bb) < 1e-10 * abs(a)
    assert rel(host(v3), host(v1) + 2.0 * host(v2)) < 1e-12


def test_c5_full_size_sampled_carreau():
    """C5 at full size (BFS, 999,424 graded cells, k=3, Carreau contrast 1e4, periodic z,
    Neumann outlet): GPU apply vs oracle on sampled cells (boundary and interior)."""
    from inputs.vectors import c5_linearization
    m = bfs()
    k = 3
    d = dg.Disc(m, k)
    ulin = c5_linearization(m, k)
    u = uniform(0, len(ulin))
    ctx = Ctx(m, k, visc_law=laws.C5_CARREAU)
    ctx.update_viscosity(dev(ulin))
    y = gpu_apply(ctx, u).reshape(m.n_cells, 3, 64)
    cells = _sample_cells(m, 48)
    ref = dg.viscous_apply(d, u, dg.CarreauNu(d, ulin, laws.C5_CARREAU), cells=cells)
    assert rel(y[cells], ref) < TOL


def test_newton_point_data_follow_the_linearisation():
    """The Newton apply reads point data derived from u_lin (K2 v3): a second update_viscosity
    with another u_lin must be honoured (no stale data)."""
    m = cube(3)
    k = 4
    d = dg.Disc(m, k)
    law = laws.C3_CARREAU
    u0 = c3_linearization(m, k)
    u1 = 0.5 * c3_linearization(m, k, seed=3)
    w = uniform(0, len(u0))
    ctx = Ctx(m, k, visc_law=law)
    y = torch.empty(len(w), dtype=torch.float64, device="cuda")
    for ul in (u0, u1):
        ctx.update_viscosity(dev(ul))
        ctx.apply_linearized_viscous(dev(w), y)
        assert rel(host(y), dg.newton_apply(d, ul, w, law)) < TOL
