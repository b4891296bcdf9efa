"""GPU parity, round-2 gaps (VERDICT r1 "What's weak" 1): the coarse-level Carreau viscosity of
reading G19, the Helmholtz V-cycle after update_viscosity in FP64 and with
FP32 levels, and multi-sweep Chebyshev / V-cycle parity on meshes WITH interior cells, all
against the CPU oracle (matrix-free oracle applies; the dense oracle only supplies diagonals).
Tolerances: 1e-12 relative L2 in FP64 (G25); FP32 levels 2e-5 (reading F1)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import cube, deformed_cube, uniform                            # noqa: E402
from inputs.vectors import c3_linearization                               # noqa: E402
from oracle import dense, dg, laws, mg                                    # noqa: E402

TOL = 1e-12
TOL32 = 2e-5
OP_VISC, OP_POIS = 0, 1


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


# ------------------------------------------------------------------ G19 coarse-level nu
G19_CASES = [
    ("cube3 k4->2->1 C3 u_lin", lambda: cube(3), [4, 2, 1], "c3"),
    ("deformed3 (map deg 3) k3->2->1 random u_lin", lambda: deformed_cube(3, 3), [3, 2, 1], "rand"),
]


def _g19_setup(mk, degs, ulin_kind):
    m = mk()
    kf = degs[0]
    n_f = m.n_cells * 3 * (kf + 1) ** 3
    ulin = c3_linearization(m, kf) if ulin_kind == "c3" else uniform(7, n_f)
    law = laws.C3_CARREAU
    discs = [dg.Disc(m, k) for k in degs]
    nus = [dg.CarreauNu(discs[0], ulin, law)] + [dg.coarse_level_nu(discs[0], d, ulin, law) for d in discs[1:]]
    ctx = Ctx(m, kf, visc_law=law, degrees=degs)
    ctx.update_viscosity(dev(ulin))
    return m, discs, nus, ctx


@pytest.mark.parametrize("name,mk,degs,ulin_kind", G19_CASES, ids=[c[0] for c in G19_CASES])
def test_coarse_level_carreau_apply_g19(name, mk, degs, ulin_kind):
    """apply_viscous on every level after update_viscosity == oracle viscous_apply with the G19
    coarse-level viscosity (u_lin interpolated to the level's Gauss points, then Carreau)."""
    m, discs, nus, ctx = _g19_setup(mk, degs, ulin_kind)
    for lvl, (d, nu) in enumerate(zip(discs, nus)):
        u = uniform(10 + lvl, m.n_cells * 3 * d.N)
        y = torch.empty(len(u), dtype=torch.float64, device="cuda")
        ctx.apply_viscous(dev(u), y, lvl)
        err = rel(host(y), dg.viscous_apply(d, u, nu))
        assert err < TOL, (lvl, err)
        lo, hi = ctx.coefficient_range(OP_VISC, lvl)
        cells = np.arange(m.n_cells)
        allv = np.concatenate([nu.vol(cells).ravel()] + [nu.face(cells, f).ravel() for f in range(6)])
        assert abs(lo - allv.min()) <= 1e-13 * allv.max() and abs(hi - allv.max()) <= 1e-13 * allv.max(), lvl


def _visc_levels(m, discs, nus, mass):
    levels = []
    for li, (d, nu) in enumerate(zip(discs, nus)):
        Md = dg.mass_apply(d, np.ones(m.n_cells * 3 * d.N), 3)              # diagonal mass (G2)
        Ad = dense.assemble_viscous(d, nu)
        L = {"apply": (lambda x, d=d, nu=nu, Md=Md: dg.viscous_apply(d, x, nu) + mass * Md * x),
             "Dinv": 1.0 / (np.diag(Ad) + mass * Md)}
        del Ad
        if li + 1 < len(discs):
            kf, kc = d.k, discs[li + 1].k
            L["restrict"] = lambda r, kf=kf, kc=kc: mg.restrict(r, kf, kc, m.n_cells, 3)
            L["prolongate"] = lambda x, kf=kf, kc=kc: mg.prolongate(x, kf, kc, m.n_cells, 3)
        levels.append(L)
    lams = []
    for li, L in enumerate(levels):
        lam = 1.2 * mg.lanczos_lambda_max(L["apply"], L["Dinv"], uniform(2, len(L["Dinv"])), 20)
        L["lam_hi"] = lam
        lams.append(lam)
    return levels, lams


@pytest.mark.parametrize("name,mk,degs,ulin_kind", G19_CASES, ids=[c[0] for c in G19_CASES])
def test_helmholtz_vcycle_after_update_viscosity(name, mk, degs, ulin_kind):
    """The viscous-step V-cycle (mass 1e2 + A(nu), G19 nu on every level, FP64 levels and the
    paper's FP32 levels) against the oracle V-cycle built from matrix-free oracle applies.  Also
    the library's own inverse diagonal on every level against the dense oracle's diagonal."""
    m, discs, nus, ctx = _g19_setup(mk, degs, ulin_kind)
    mass = 1e2
    ctx.set_mass(OP_VISC, mass)
    levels, lams = _visc_levels(m, discs, nus, mass)
    for lvl, L in enumerate(levels):
        dv = torch.empty(len(L["Dinv"]), dtype=torch.float64, device="cuda")
        ctx.inverse_diagonal(OP_VISC, dv, lvl)
        assert rel(host(dv), L["Dinv"]) < TOL, lvl
    b = uniform(0, len(levels[0]["Dinv"]))
    ref = mg.vcycle(levels, b)
    x = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    ctx.vcycle(OP_VISC, dev(b), x, lams)
    assert rel(host(x), ref) < TOL
    x32 = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    ctx.vcycle_fp32(OP_VISC, dev(b), x32, lams)
    err = rel(host(x32), ref)
    assert err < TOL32, err
    assert err > 1e-12                       # the FP32 levels really ran in single precision


# ------------------------------------------------------------------ Chebyshev / V-cycle with interior cells
def test_poisson_chebyshev_vcycle_parity_interior_cells():
    """C4's p-sequence 5->3->2->1 on cube(3) (one interior cell, every face type): Lanczos,
    Chebyshev(5) from 0 and from x0, and the V-cycle, FP64 and FP32, vs matrix-free oracle applies."""
    m = cube(3)
    degs = [5, 3, 2, 1]
    law = laws.C4_LAW
    ctx = Ctx(m, 5, poisson_law=law, degrees=degs)
    levels = []
    for li, k in enumerate(degs):
        d = dg.Disc(m, k)
        nu = dg.AnalyticNu(d, law)
        Ad = dense.assemble_poisson(d, nu)
        L = {"apply": (lambda x, d=d, nu=nu: dg.poisson_apply(d, x, nu)), "Dinv": 1.0 / np.diag(Ad)}
        del Ad
        if li + 1 < len(degs):
            kc = degs[li + 1]
            L["restrict"] = lambda r, k=k, kc=kc: mg.restrict(r, k, kc, m.n_cells)
            L["prolongate"] = lambda x, k=k, kc=kc: mg.prolongate(x, k, kc, m.n_cells)
        levels.append(L)
    lams = []
    for lvl, L in enumerate(levels):
        v0 = uniform(2, len(L["Dinv"]))
        lo = mg.lanczos_lambda_max(L["apply"], L["Dinv"], v0, 20)
        lg = ctx.estimate_lambda_max(OP_POIS, dev(v0), level=lvl, steps=20)
        assert abs(lg - lo) < 1e-10 * lo, (lvl, lg, lo)
        L["lam_hi"] = 1.2 * lo
        lams.append(1.2 * lo)
    n0 = len(levels[0]["Dinv"])
    b = uniform(0, n0)
    hi = lams[0]
    x = dev(np.zeros(n0))
    ctx.chebyshev_smooth(OP_POIS, x, dev(b), hi / 20, hi, 5, x_is_zero=True)
    assert rel(host(x), mg.chebyshev(levels[0]["apply"], levels[0]["Dinv"], b, np.zeros(n0), hi / 20, hi, 5)) < TOL
    x0 = uniform(3, n0)
    x = dev(x0)
    ctx.chebyshev_smooth(OP_POIS, x, dev(b), hi / 20, hi, 5, x_is_zero=False)
    assert rel(host(x), mg.chebyshev(levels[0]["apply"], levels[0]["Dinv"], b, x0, hi / 20, hi, 5)) < TOL
    ref = mg.vcycle(levels, b)
    xv = dev(np.zeros(n0))
    ctx.vcycle(OP_POIS, dev(b), xv, lams)
    assert rel(host(xv), ref) < TOL
    x32 = dev(np.zeros(n0))
    ctx.vcycle_fp32(OP_POIS, dev(b), x32, lams)
    assert rel(host(x32), ref) < TOL32
