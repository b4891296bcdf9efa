"""§8(f) f2 on the GPU: the divergence/continuity penalty-step operator (dgvv_apply_penalty),
its inverse diagonal and the Jacobi-PCG solve of the penalty step against the CPU oracle
(oracle.dg.penalty_apply, pinned in test_oracle_penalty.py) on the same seeded inputs, the
full-size C2 mesh on sampled cells, and the multi-rank path (bitwise vs one context)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import bfs, cube, deformed_cube, uniform                       # noqa: E402
from inputs.meshes import NEUMANN                                         # noqa: E402
from oracle import dg, laws, mg                                           # noqa: E402
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


def taus(n, seed=7):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.1, 10.0, n), rng.uniform(0.1, 10.0, n)


CASES = [("cube3 k3 Dirichlet", lambda: cube(3), 3), ("deformed3 k3", lambda: deformed_cube(3, 3), 3),
         ("bfs periodic/Neumann k2", lambda: bfs(nx_in=2, ny_in=1, nx_out=4, nz=3), 2),
         ("cube3 Neumann k4", lambda: cube(3, bc=NEUMANN), 4), ("cube2 k1", lambda: cube(2), 1)]


@pytest.mark.parametrize("name,mk,k", CASES, ids=[c[0] for c in CASES])
def test_penalty_apply_parity(name, mk, k):
    m = mk()
    d = dg.Disc(m, k)
    td, tc = taus(m.n_cells)
    ctx = Ctx(m, k, visc_law=laws.C1_LAW)
    from paper_2506_14424_b200 import DgvvError
    u = uniform(0, m.n_cells * 3 * d.N)
    with pytest.raises(DgvvError):                    # ESTATE before the parameters are set
        ctx.apply_penalty(dev(u), dev(u * 0))
    ctx.set_penalty_parameters(td, tc)
    y = torch.empty(len(u), dtype=torch.float64, device="cuda")
    ctx.apply_penalty(dev(u), y)
    assert rel(host(y), dg.penalty_apply(d, u, td, tc)) < TOL
    with pytest.raises(DgvvError):
        ctx.set_penalty_parameters(-td, tc)


@pytest.mark.parametrize("mk,k", [(lambda: cube(2), 2), (lambda: deformed_cube(2, 2), 2)])
def test_penalty_diagonal_and_jacobi_pcg(mk, k):
    m = mk()
    d = dg.Disc(m, k)
    td, tc = taus(m.n_cells, 3)
    ctx = Ctx(m, k, visc_law=laws.C1_LAW)
    ctx.set_penalty_parameters(td, tc)
    n = m.n_cells * 3 * d.N
    Adense = np.array([dg.penalty_apply(d, e, td, tc) for e in np.eye(n)]).T
    dinv = torch.empty(n, dtype=torch.float64, device="cuda")
    ctx.inverse_diagonal(A.OP_PENALTY, dinv)
    Dinv = 1.0 / np.diag(Adense)
    assert rel(host(dinv), Dinv) < TOL
    b = uniform(0, n)
    xr, itr, rrr = mg.pcg(lambda v: Adense @ v, b, np.zeros(n), lambda r: Dinv * r, 0.0, 8)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    it, rr = ctx.cg_solve(A.OP_PENALTY, dev(b), x, rtol=0.0, maxit=8, precond="jacobi")
    assert it == itr == 8 and rel(host(x), xr) < 1e-10


def test_penalty_full_size_c2_sampled_and_solve():
    """C2 mesh (32^3 deformed, k=3): apply vs oracle on sampled cells; Jacobi-PCG of the penalty
    step to rtol 1e-10 checked with an independent apply."""
    m = deformed_cube(32, 3)
    k = 3
    d = dg.Disc(m, k)
    # parameters of the size Fehn2018b's choice gives (tau_div ~ |u| h dt, tau_cont ~ |u| dt with
    # |u| in [0.1, 2], h = 1/32 and a CFL-limited dt = 1e-3 for k = 3): the penalty step is then
    # mass-dominated and Jacobi-PCG converges in tens of iterations (with tau = O(1) the
    # div-div term makes it ill-conditioned: kappa ~ tau (n^2/h)^2)
    rng = np.random.default_rng(11)
    speed = rng.uniform(0.1, 2.0, m.n_cells)
    td, tc = speed * (1.0 / 32) * 1e-3, speed * 1e-3
    ctx = Ctx(m, k, visc_law=laws.C2_LAW)
    ctx.set_penalty_parameters(td, tc)
    u = uniform(0, m.n_cells * 3 * d.N)
    y = torch.empty(len(u), dtype=torch.float64, device="cuda")
    ctx.apply_penalty(dev(u), y)
    rng = np.random.default_rng(5)
    cells = np.sort(rng.choice(m.n_cells, 48, replace=False))
    ref = dg.penalty_apply(d, u, td, tc, cells=cells)
    assert rel(host(y).reshape(m.n_cells, 3, d.N)[cells], ref) < TOL
    b = dev(u)
    x = torch.zeros_like(b)
    it, rr = ctx.cg_solve(A.OP_PENALTY, b, x, rtol=1e-10, maxit=500, precond="jacobi")
    assert rr <= 1e-10 and it < 500
    ctx.apply_penalty(x, y)
    assert float(torch.linalg.norm(b - y) / torch.linalg.norm(b)) <= 1.01e-10


def test_penalty_multirank_bitwise():
    from test_gpu_multirank import fill_ghosts, make_ranks   # tests/ is on sys.path (rootdir-less import)
    m = deformed_cube(4, 3)
    k, R = 3, 3
    per = 3 * (k + 1) ** 3
    td, tc = taus(m.n_cells, 2)
    u = uniform(0, m.n_cells * per)
    ref_ctx = Ctx(m, k, visc_law=laws.C2_LAW)
    ref_ctx.set_penalty_parameters(td, tc)
    src = dev(u)
    ref = torch.empty_like(src)
    ref_ctx.apply_penalty(src, ref)
    parts, ctxs = make_ranks(m, R, k, visc_law=laws.C2_LAW)
    locs = [src[p.first * per:(p.first + p.n_owned) * per].contiguous() for p in parts]
    for p, c in zip(parts, ctxs):
        rows = np.concatenate([np.arange(p.first, p.first + p.n_owned), np.asarray(p.ghost_global_id)])
        c.set_penalty_parameters(td[rows], tc[rows])
    fill_ghosts(parts, ctxs, locs, A.GHOST_VISCOUS, per)
    outs = []
    for c, x in zip(ctxs, locs):
        y = torch.empty_like(x)
        c.apply_penalty(x, y)
        outs.append(y)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs), ref)
    from test_gpu_multirank import oracle_close
    oracle_close(torch.cat(outs), dg.penalty_apply(dg.Disc(m, k), u, td, tc))


# ------------------------------------------------------------------ f2 multigrid
def _checkerboard_diag(apply, m, per_cell):
    """diag(A) of an operator that couples only face neighbours, from len(per_cell)*2 applies:
    the unit vectors of one local index in every cell of one checkerboard colour at once (cells
    of a colour share no face on a non-periodic cube, so no off-diagonal entry is picked up)."""
    ijk = np.array(np.unravel_index(np.arange(m.n_cells), (round(m.n_cells ** (1 / 3)),) * 3))
    colour = ijk.sum(axis=0) % 2
    D = np.zeros(m.n_cells * per_cell)
    for col in (0, 1):
        cells = np.nonzero(colour == col)[0]
        for j in range(per_cell):
            e = np.zeros_like(D)
            e[cells * per_cell + j] = 1.0
            y = apply(e)
            D[cells * per_cell + j] = y[cells * per_cell + j]
    return D


def test_penalty_multigrid_levels_vcycle_and_pcg():
    """The penalty-step operator on every p-level (3 -> 2 -> 1) of cube(3) (interior cell), its
    inverse diagonal, Lanczos lambda_max, Chebyshev(5) from x0, the V-cycle and V-cycle-PCG
    (6 fixed iterations) against the oracle built from oracle.dg.penalty_apply."""
    m = cube(3)
    degs = [3, 2, 1]
    td, tc = taus(m.n_cells, 4)
    ctx = Ctx(m, 3, visc_law=laws.C1_LAW, degrees=degs)
    ctx.set_penalty_parameters(td, tc)
    levels = []
    for lvl, k in enumerate(degs):
        d = dg.Disc(m, k)
        app = (lambda x, d=d: dg.penalty_apply(d, x, td, tc))
        n = m.n_cells * 3 * d.N
        u = uniform(20 + lvl, n)
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        ctx.apply_penalty(dev(u), y, level=lvl)
        assert rel(host(y), app(u)) < TOL, lvl
        Dinv = 1.0 / _checkerboard_diag(app, m, 3 * d.N)
        dv = torch.empty(n, dtype=torch.float64, device="cuda")
        ctx.inverse_diagonal(A.OP_PENALTY, dv, level=lvl)
        assert rel(host(dv), Dinv) < TOL, lvl
        v0 = uniform(2, n)
        lo = mg.lanczos_lambda_max(app, Dinv, v0, 20)
        lg = ctx.estimate_lambda_max(A.OP_PENALTY, dev(v0), level=lvl, steps=20)
        assert abs(lg - lo) < 1e-10 * lo, (lvl, lg, lo)
        L = {"apply": app, "Dinv": Dinv, "lam_hi": 1.2 * lo}
        if lvl + 1 < len(degs):
            L["restrict"] = lambda r, k=k, kc=degs[lvl + 1]: mg.restrict(r, k, kc, m.n_cells, 3)
            L["prolongate"] = lambda x, k=k, kc=degs[lvl + 1]: mg.prolongate(x, k, kc, m.n_cells, 3)
        levels.append(L)
    lams = [L["lam_hi"] for L in levels]
    n0 = len(levels[0]["Dinv"])
    b = uniform(0, n0)
    x0 = uniform(3, n0)
    hi = lams[0]
    x = dev(x0)
    ctx.chebyshev_smooth(A.OP_PENALTY, x, dev(b), hi / 20, hi, 5, x_is_zero=False)
    assert rel(host(x), mg.chebyshev(levels[0]["apply"], levels[0]["Dinv"], b, x0, hi / 20, hi, 5)) < TOL
    ref = mg.vcycle(levels, b)
    xv = dev(np.zeros(n0))
    ctx.vcycle(A.OP_PENALTY, dev(b), xv, lams)
    assert rel(host(xv), ref) < TOL
    xr, itr, _ = mg.pcg(levels[0]["apply"], b, np.zeros(n0), lambda r: mg.vcycle(levels, r), 0.0, 6)
    xg = dev(np.zeros(n0))
    it, _ = ctx.cg_solve(A.OP_PENALTY, dev(b), xg, rtol=0.0, maxit=6, precond="vcycle", lam_hi_per_level=lams)
    assert it == itr == 6 and rel(host(xg), xr) < 1e-10


def test_penalty_vcycle_pcg_beats_jacobi_c2_mesh():
    """Full-size C2 mesh (32^3 deformed, k = 3 -> 2 -> 1), Fehn2018b-sized tau: V-cycle-PCG reaches
    rtol 1e-10 in far fewer iterations than Jacobi-PCG; the solution is checked with an
    independent apply."""
    m = deformed_cube(32, 3)
    rng = np.random.default_rng(11)
    speed = rng.uniform(0.1, 2.0, m.n_cells)
    td, tc = speed * (1.0 / 32) * 1e-3, speed * 1e-3
    ctx = Ctx(m, 3, visc_law=laws.C2_LAW, degrees=[3, 2, 1])
    ctx.set_penalty_parameters(td, tc)
    lams = [1.2 * ctx.estimate_lambda_max(A.OP_PENALTY, dev(uniform(2, 3 * ctx.n_dofs(l))), level=l, steps=20)
            for l in range(3)]
    b = dev(uniform(0, 3 * ctx.n_dofs(0)))
    xj = torch.zeros_like(b)
    itj, rrj = ctx.cg_solve(A.OP_PENALTY, b, xj, rtol=1e-10, maxit=500, precond="jacobi")
    xv = torch.zeros_like(b)
    itv, rrv = ctx.cg_solve(A.OP_PENALTY, b, xv, rtol=1e-10, maxit=500, precond="vcycle", lam_hi_per_level=lams)
    assert rrv <= 1e-10 and itv < itj / 3, (itv, itj)
    y = torch.empty_like(b)
    ctx.apply_penalty(xv, y)
    assert float(torch.linalg.norm(b - y) / torch.linalg.norm(b)) <= 1.01e-10
