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
