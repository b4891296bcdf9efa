"""§8(f) f4 on the GPU: the upwind DG convective term (dgvv_apply_convective), the viscous-step
operator with linearly implicit convection mass M + A(nu) + alpha_c C(w) (dgvv_apply_oseen) and
the right-preconditioned restarted GMRES (dgvv_gmres_solve) against the CPU oracle
(oracle.dg.convective_apply / helmholtz_apply and oracle.mg.gmres, pinned in
test_oracle_convective.py) on the same seeded inputs; the full-size C2 mesh on sampled cells;
and the multi-rank path (bitwise vs one context)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import bfs, cube, deformed_cube, uniform                       # noqa: E402
from inputs.meshes import NEUMANN                                         # noqa: E402
from oracle import dense, dg, laws, mg                                    # noqa: E402
from paper_2506_14424_b200 import _abi as A                               # noqa: E402

TOL = 1e-12


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


CASES = [("cube3 k3 Dirichlet", lambda: cube(3), 3), ("deformed3 k3", lambda: deformed_cube(3, 3), 3),
         ("bfs periodic/Neumann k2", lambda: bfs(nx_in=2, ny_in=1, nx_out=4, nz=3), 2),
         ("cube3 Neumann k4", lambda: cube(3, bc=NEUMANN), 4), ("cube2 k1", lambda: cube(2), 1),
         ("cube2 periodic k5", lambda: cube(2, periodic=(True, True, True)), 5)]


@pytest.mark.parametrize("name,mk,k", CASES, ids=[c[0] for c in CASES])
def test_convective_apply_parity(name, mk, k):
    m = mk()
    d = dg.Disc(m, k)
    n = m.n_cells * 3 * d.N
    u = uniform(0, n)
    w = uniform(1, n)                 # transport field: every face sees inflow on one side
    ctx = Ctx(m, k, visc_law=laws.C1_LAW)
    from paper_2506_14424_b200 import DgvvError
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    with pytest.raises(DgvvError):    # ESTATE before the transport field is set
        ctx.apply_convective(dev(u), y)
    ctx.set_transport(dev(w))
    y.fill_(7.0)                      # overwritten, not accumulated
    ctx.apply_convective(dev(u), y)
    assert rel(host(y), dg.convective_apply(d, u, w)) < TOL
    bad = w.copy()
    bad[3] = np.nan
    with pytest.raises(DgvvError):
        ctx.set_transport(dev(bad))


def test_convective_constant_transport_is_skew_on_periodic_mesh():
    """Property at any size: with constant w on a periodic mesh, u^T C u = 1/2 sum |w.n| |[u]|^2 >= 0
    and C + C^T is the upwind jump term only, so (u, C u) equals the oracle's on the same u."""
    m = cube(4, periodic=(True, True, True))
    k = 3
    d = dg.Disc(m, k)
    n = m.n_cells * 3 * d.N
    w = np.zeros((m.n_cells, 3, d.N))
    w[:] = np.array([0.7, -0.4, 0.25])[None, :, None]
    w = w.reshape(-1)
    u = uniform(0, n)
    ctx = Ctx(m, k, visc_law=laws.C1_LAW)
    ctx.set_transport(dev(w))
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    ctx.apply_convective(dev(u), y)
    e = float(u @ host(y))
    assert e > 0.0 and abs(e - float(u @ dg.convective_apply(d, u, w))) < 1e-12 * abs(e)


@pytest.mark.parametrize("mk,k,law", [(lambda: cube(3), 3, laws.C1_LAW), (lambda: deformed_cube(3, 3), 3, laws.C2_LAW)])
def test_oseen_apply_parity(mk, k, law):
    m = mk()
    d = dg.Disc(m, k)
    nu = dg.AnalyticNu(d, law)
    n = m.n_cells * 3 * d.N
    u, w = uniform(0, n), uniform(1, n)
    mass = 25.0
    ctx = Ctx(m, k, visc_law=law)
    ctx.set_mass(0, mass)
    ctx.set_transport(dev(w))
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for ac in (1.0, 0.0, -0.5):
        ctx.apply_oseen(dev(u), y, alpha_c=ac)
        ref = dg.helmholtz_apply(d, u, nu, mass) + ac * dg.convective_apply(d, u, w)
        assert rel(host(y), ref) < TOL


def _levels(m, degs, law, mass):
    levels = []
    for li, k in enumerate(degs):
        d = dg.Disc(m, k)
        nu = dg.AnalyticNu(d, law)
        Ad = dense.assemble_viscous(d, nu)
        Ad = Ad + mass * np.diag(dg.mass_apply(d, np.ones(Ad.shape[0])))
        L = {"apply": (lambda x, Ad=Ad: Ad @ x), "Dinv": 1.0 / np.diag(Ad)}
        if li + 1 < len(degs):
            kc = degs[li + 1]
            L["restrict"] = lambda r, k=k, kc=kc: mg.restrict(r, k, kc, m.n_cells, ncomp=3)
            L["prolongate"] = lambda x, k=k, kc=kc: mg.prolongate(x, k, kc, m.n_cells, ncomp=3)
        levels.append(L)
    return levels


@pytest.mark.parametrize("precond", ["none", "jacobi", "vcycle"])
def test_gmres_parity_fixed_iterations(precond):
    """rtol = 0, GMRES(4), 10 iterations (two restarts): GPU and oracle run the same iterations
    on mass M + A(nu) + C(w); the preconditioner is the symmetric part's Jacobi or V-cycle."""
    m = deformed_cube(2, 3)
    degs = [3, 2, 1]
    mass, law = 20.0, laws.C2_LAW
    d = dg.Disc(m, 3)
    nu = dg.AnalyticNu(d, law)
    ctx = Ctx(m, 3, visc_law=law, degrees=degs)
    ctx.set_mass(0, mass)
    levels = _levels(m, degs, law, mass)
    lams = []
    for L in levels:
        v0 = uniform(2, len(L["Dinv"]))
        lam = 1.2 * mg.lanczos_lambda_max(L["apply"], L["Dinv"], v0, 20)
        L["lam_hi"] = lam
        lams.append(lam)
    n0 = len(levels[0]["Dinv"])
    w = 30.0 * uniform(1, n0)                       # strong convection: non-symmetric
    ctx.set_transport(dev(w))
    op = lambda v: levels[0]["apply"](v) + dg.convective_apply(d, v, w)
    b = uniform(0, n0)
    x0 = 0.1 * uniform(5, n0)
    P = {"none": lambda r: r, "jacobi": lambda r: levels[0]["Dinv"] * r,
         "vcycle": lambda r: mg.vcycle(levels, r)}[precond]
    xr, itr, rrr = mg.gmres(op, b, x0, P, 0.0, 4, 10)
    x = dev(x0)
    it, rr = ctx.gmres_solve(dev(b), x, alpha_c=1.0, rtol=0.0, restart=4, maxit=10, precond=precond,
                             lam_hi_per_level=lams)
    assert it == itr == 10
    assert rel(host(x), xr) < 1e-10
    assert abs(rr - rrr) < 1e-8 * rrr


def test_gmres_converges_and_residual_is_independent():
    """GMRES(30) with the V-cycle of the symmetric part to rtol 1e-10 on cube(4) k=3; the returned
    x is checked with the oracle operator (not the GPU's)."""
    m = cube(4)
    degs = [3, 2, 1]
    k = 3
    d = dg.Disc(m, k)
    nu = dg.AnalyticNu(d, laws.C1_LAW)
    mass = 50.0
    ctx = Ctx(m, k, visc_law=laws.C1_LAW, degrees=degs)
    ctx.set_mass(0, mass)
    n = m.n_cells * 3 * d.N
    w = 5.0 * uniform(1, n)
    ctx.set_transport(dev(w))
    lams = [1.2 * ctx.estimate_lambda_max(0, dev(uniform(2, 3 * m.n_cells * (kk + 1) ** 3)), level=l, steps=20)
            for l, kk in enumerate(degs)]
    b = uniform(0, n)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    it, rr = ctx.gmres_solve(dev(b), x, rtol=1e-10, restart=30, maxit=200, precond="vcycle", lam_hi_per_level=lams)
    assert rr <= 1e-10 and 0 < it < 200
    xs = host(x)
    res = b - dg.helmholtz_apply(d, xs, nu, mass) - dg.convective_apply(d, xs, w)
    assert np.linalg.norm(res) <= 1.01e-10 * np.linalg.norm(b) + 1e-13 * np.linalg.norm(b)
    x2 = torch.zeros_like(x)
    it2, rr2 = ctx.gmres_solve(dev(b), x2, rtol=1e-10, restart=30, maxit=200, precond="vcycle_fp32",
                               lam_hi_per_level=lams)
    assert rr2 <= 1e-10 and it2 <= it + 3


def test_convective_full_size_c2_sampled_and_gmres():
    """C2 mesh (32^3 deformed, k=3): convective apply vs oracle on sampled cells; GMRES with the
    V-cycle of mass M + A(nu) (mass = gamma_0/dt for a CFL-limited dt) to rtol 1e-8."""
    m = deformed_cube(32, 3)
    k = 3
    degs = [3, 2, 1]
    d = dg.Disc(m, k)
    n = m.n_cells * 3 * d.N
    ctx = Ctx(m, k, visc_law=laws.C2_LAW, degrees=degs)
    u = uniform(0, n)
    w = uniform(1, n)
    ctx.set_transport(dev(w))
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    ctx.apply_convective(dev(u), y)
    rng = np.random.default_rng(5)
    cells = np.sort(rng.choice(m.n_cells, 48, replace=False))
    ref = dg.convective_apply(d, u, w, cells=cells)
    assert rel(host(y).reshape(m.n_cells, 3, d.N)[cells], ref) < TOL
    ctx.set_mass(0, 1.0e3)
    lams = [1.2 * ctx.estimate_lambda_max(0, dev(uniform(2, 3 * m.n_cells * (kk + 1) ** 3)), level=l, steps=15)
            for l, kk in enumerate(degs)]
    b = dev(u)
    x = torch.zeros_like(b)
    it, rr = ctx.gmres_solve(b, x, rtol=1e-8, restart=30, maxit=300, precond="vcycle", lam_hi_per_level=lams)
    assert rr <= 1e-8 and it < 300
    ctx.apply_oseen(x, y, alpha_c=1.0)
    assert float(torch.linalg.norm(b - y) / torch.linalg.norm(b)) <= 1.01e-8


def test_convective_multirank_bitwise():
    from test_gpu_multirank import fill_ghosts, make_ranks   # tests/ is on sys.path (rootdir-less import)
    m = deformed_cube(4, 3)
    k, R = 3, 3
    per = 3 * (k + 1) ** 3
    u = uniform(0, m.n_cells * per)
    w = uniform(1, m.n_cells * per)
    ref_ctx = Ctx(m, k, visc_law=laws.C2_LAW)
    ref_ctx.set_transport(dev(w))
    src = dev(u)
    ref = torch.empty_like(src)
    ref_ctx.apply_convective(src, ref)
    parts, ctxs = make_ranks(m, R, k, visc_law=laws.C2_LAW)
    wd = dev(w)
    wl = [wd[p.first * per:(p.first + p.n_owned) * per].contiguous() for p in parts]
    for c, x in zip(ctxs, wl):
        c.set_transport(x)
    fill_ghosts(parts, ctxs, wl, A.GHOST_TRANSPORT, per)
    locs = [src[p.first * per:(p.first + p.n_owned) * per].contiguous() for p in parts]
    fill_ghosts(parts, ctxs, locs, A.GHOST_VISCOUS, per)
    outs = []
    for c, x in zip(ctxs, locs):
        y = torch.empty_like(x)
        c.apply_convective(x, y)
        outs.append(y)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs), ref)
    from test_gpu_multirank import oracle_close
    d = dg.Disc(m, k)
    oracle_close(torch.cat(outs), dg.convective_apply(d, u, w))
    # the fused operator mass M + A + C (one kernel) is partition-independent too
    for c in [ref_ctx] + ctxs:
        c.set_mass(0, 7.0)
    ref_ctx.apply_oseen(src, ref, alpha_c=1.0)
    outs = []
    for c, x in zip(ctxs, locs):
        y = torch.empty_like(x)
        c.apply_oseen(x, y, alpha_c=1.0)
        outs.append(y)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs), ref)
    oracle_close(torch.cat(outs), dg.helmholtz_apply(d, u, dg.AnalyticNu(d, laws.C2_LAW), 7.0)
                 + dg.convective_apply(d, u, w))


def test_transport_point_data_follow_set_transport():
    """The convective applies read point data derived from w: a new set_transport must be honoured
    by both the standalone and the fused apply."""
    m = cube(3)
    k = 3
    d = dg.Disc(m, k)
    nu = dg.AnalyticNu(d, laws.C1_LAW)
    n = m.n_cells * 3 * d.N
    u = uniform(0, n)
    ctx = Ctx(m, k, visc_law=laws.C1_LAW)
    ctx.set_mass(0, 5.0)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for seed in (1, 4):
        w = uniform(seed, n)
        ctx.set_transport(dev(w))
        ctx.apply_oseen(dev(u), y, alpha_c=1.0)
        assert rel(host(y), dg.helmholtz_apply(d, u, nu, 5.0) + dg.convective_apply(d, u, w)) < TOL
        ctx.apply_convective(dev(u), y)
        assert rel(host(y), dg.convective_apply(d, u, w)) < TOL
