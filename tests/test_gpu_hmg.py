"""§8(f) f3 on the GPU: h-transfer between nested refinements (dgvv_prolongate_h / dgvv_restrict_h),
the direct coarse solver (dgvv_setup_coarse_solver) and the V-cycle over p- and h-levels
(dgvv_set_coarse_context) against the CPU oracle (oracle.mg.h_prolongate / h_restrict / vcycle,
dense oracle operators solved with numpy; pinned in test_oracle_hmg.py) on the same seeded
inputs; full-size C4 PCG with the cph V-cycle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import cube, cube_parent_map, uniform                         # noqa: E402
from oracle import dense, dg, laws, mg                                    # noqa: E402
from paper_2506_14424_b200 import _abi as A                               # noqa: E402


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


@pytest.mark.parametrize("k", [1, 2, 3, 5])
@pytest.mark.parametrize("op", [A.OP_VISCOUS, A.OP_POISSON])
def test_h_transfer_parity(k, op):
    mf, mc = cube(4), cube(2)
    parent, octant = cube_parent_map(4)
    nc = 3 if op == A.OP_VISCOUS else 1
    kw = {"visc_law": laws.C1_LAW} if op == A.OP_VISCOUS else {"poisson_law": laws.C4_LAW}
    fine, coarse = Ctx(mf, k, **kw), Ctx(mc, k, **kw)
    fine.set_coarse_context(coarse, parent, octant)
    n3 = (k + 1) ** 3
    xc = uniform(0, mc.n_cells * nc * n3)
    xf = uniform(1, mf.n_cells * nc * n3)
    yf = dev(xf)
    fine.prolongate_h(op, dev(xc), yf, beta=0.5)
    ref = mg.h_prolongate(xc, k, parent, octant, nc) + 0.5 * xf
    assert rel(host(yf), ref) < 1e-14
    yc = dev(xc)
    fine.restrict_h(op, dev(xf), yc, beta=-2.0)
    ref = mg.h_restrict(xf, k, parent, octant, mc.n_cells, nc) - 2.0 * xc
    assert rel(host(yc), ref) < 1e-14


def test_set_coarse_context_validation():
    from paper_2506_14424_b200 import DgvvError
    mf, mc = cube(4), cube(2)
    parent, octant = cube_parent_map(4)
    fine, coarse = Ctx(mf, 2, visc_law=laws.C1_LAW, degrees=[2, 1]), Ctx(mc, 1, visc_law=laws.C1_LAW)
    bad = octant.copy()
    bad[1] = bad[0]                                  # two children in one octant
    with pytest.raises(DgvvError):
        fine.set_coarse_context(coarse, parent, bad)
    with pytest.raises(DgvvError):                   # degree mismatch (coarse k=2 vs fine coarsest k=1)
        fine.set_coarse_context(Ctx(mc, 2, visc_law=laws.C1_LAW), parent, octant)
    with pytest.raises(DgvvError):                   # ESTATE: no coarse context yet
        fine.prolongate_h(A.OP_VISCOUS, torch.zeros(mc.n_cells * 24, dtype=torch.float64, device="cuda"),
                          torch.zeros(mf.n_cells * 24, dtype=torch.float64, device="cuda"))
    fine.set_coarse_context(coarse, parent, octant)


@pytest.mark.parametrize("op", [A.OP_VISCOUS, A.OP_POISSON])
def test_direct_coarse_solver(op):
    """x = V(b) on a single-level context with the direct solver == numpy's solve of the dense
    oracle matrix (viscous: cube(2) k=1 + mass, 192 DoFs; Poisson: cube(4) k=1, 512 DoFs)."""
    if op == A.OP_VISCOUS:
        m, k, law, mass = cube(2), 1, laws.C1_LAW, 3.0
        ctx = Ctx(m, k, visc_law=law)
        d = dg.Disc(m, k)
        Ad = dense.assemble_viscous(d, dg.AnalyticNu(d, law)) + mass * np.diag(dg.mass_apply(d, np.ones(m.n_cells * 3 * d.N)))
    else:
        m, k, law, mass = cube(4), 1, laws.C4_LAW, 0.0
        ctx = Ctx(m, k, poisson_law=law)
        d = dg.Disc(m, k)
        Ad = dense.assemble_poisson(d, dg.AnalyticNu(d, law))
    ctx.set_mass(op, mass)
    n = ctx.setup_coarse_solver(op)
    assert n == Ad.shape[0]
    b = uniform(0, n)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    ctx.vcycle(op, dev(b), x, [1.0])
    ref = np.linalg.solve(Ad, b)
    assert rel(host(x), ref) < 1e-10 * max(1.0, np.linalg.cond(Ad) / 1e4)
    from paper_2506_14424_b200 import DgvvError
    ctx.set_mass(op, mass + 1.0)                    # the inverse is now stale
    with pytest.raises(DgvvError):
        ctx.vcycle(op, dev(b), x, [1.0])


def _oracle_chain(op, law, mf, mc, degs, parent, octant, mass):
    levels = []
    for li, k in enumerate(degs):
        d = dg.Disc(mf, k)
        if op == A.OP_VISCOUS:
            Ad = dense.assemble_viscous(d, dg.AnalyticNu(d, law)) + mass * np.diag(dg.mass_apply(d, np.ones(mf.n_cells * 3 * d.N)))
        else:
            Ad = dense.assemble_poisson(d, dg.AnalyticNu(d, law)) + mass * np.diag(dg.mass_apply(d, np.ones(mf.n_cells * d.N), ncomp=1))
        levels.append({"apply": (lambda x, Ad=Ad: Ad @ x), "Dinv": 1.0 / np.diag(Ad)})
    nc = 3 if op == A.OP_VISCOUS else 1
    for li in range(len(degs) - 1):
        kf, kc = degs[li], degs[li + 1]
        levels[li]["restrict"] = lambda r, kf=kf, kc=kc: mg.restrict(r, kf, kc, mf.n_cells, ncomp=nc)
        levels[li]["prolongate"] = lambda x, kf=kf, kc=kc: mg.prolongate(x, kf, kc, mf.n_cells, ncomp=nc)
    kl = degs[-1]
    levels[-1]["restrict"] = lambda r: mg.h_restrict(r, kl, parent, octant, mc.n_cells, nc)
    levels[-1]["prolongate"] = lambda x: mg.h_prolongate(x, kl, parent, octant, nc)
    dcc = dg.Disc(mc, kl)
    if op == A.OP_VISCOUS:
        Ac = dense.assemble_viscous(dcc, dg.AnalyticNu(dcc, law)) + mass * np.diag(dg.mass_apply(dcc, np.ones(mc.n_cells * 3 * dcc.N)))
    else:
        Ac = dense.assemble_poisson(dcc, dg.AnalyticNu(dcc, law)) + mass * np.diag(dg.mass_apply(dcc, np.ones(mc.n_cells * dcc.N), ncomp=1))
    levels.append({"apply": (lambda x: Ac @ x), "Dinv": 1.0 / np.diag(Ac), "solve": lambda b: np.linalg.solve(Ac, b)})
    for L in levels[:-1]:
        L["lam_hi"] = 1.2 * mg.lanczos_lambda_max(L["apply"], L["Dinv"], uniform(2, len(L["Dinv"])), 20)
    return levels


@pytest.mark.parametrize("op", [A.OP_VISCOUS, A.OP_POISSON])
def test_cph_vcycle_parity(op):
    """cube(4) p-levels 2 -> 1, h-level cube(2) k = 1 with the direct solve: GPU V-cycle == oracle."""
    mf, mc = cube(4), cube(2)
    parent, octant = cube_parent_map(4)
    degs = [2, 1]
    law = laws.C1_LAW if op == A.OP_VISCOUS else laws.C4_LAW
    mass = 10.0 if op == A.OP_VISCOUS else 0.0
    kw = {"visc_law": law} if op == A.OP_VISCOUS else {"poisson_law": law}
    fine, coarse = Ctx(mf, 2, degrees=degs, **kw), Ctx(mc, 1, **kw)
    fine.set_mass(op, mass)
    coarse.set_mass(op, mass)
    coarse.setup_coarse_solver(op)
    fine.set_coarse_context(coarse, parent, octant)
    levels = _oracle_chain(op, law, mf, mc, degs, parent, octant, mass)
    lams = [L["lam_hi"] for L in levels[:-1]] + [1.0]
    assert fine.chain_levels() == 3
    b = uniform(0, len(levels[0]["Dinv"]))
    x = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    fine.vcycle(op, dev(b), x, lams)
    ref = mg.vcycle(levels, b)
    assert rel(host(x), ref) < 1e-10
    # the FP32 V-cycle follows the same chain (direct solve in FP64): within the FP32 reading F1
    xf = torch.zeros_like(x)
    fine.vcycle_fp32(op, dev(b), xf, lams)
    assert rel(host(xf), ref) < 2e-5


def test_cph_pcg_full_size_c4():
    """C4 at full size: Poisson 64^3, k = 5 -> 3 -> 2 -> 1, then h-levels 32^3 ... 4^3 at k = 1 and
    the direct solve on 4^3 (512 DoFs).  PCG with this cph V-cycle converges to 1e-8 in fewer
    iterations than with the p-only V-cycle (Chebyshev on the 64^3 k = 1 level)."""
    law = laws.C4_LAW
    ctxs, m_prev = [], None
    fine = Ctx(cube(64), 5, poisson_law=law, degrees=[5, 3, 2, 1])
    lams = []
    for l, k in enumerate([5, 3, 2, 1]):
        lams.append(1.2 * fine.estimate_lambda_max(A.OP_POISSON, dev(uniform(2, 64 ** 3 * (k + 1) ** 3)), level=l, steps=20))
    b = dev(uniform(0, fine.n_dofs(0)))
    x = torch.zeros_like(b)
    it_p, rr_p = fine.cg_solve(A.OP_POISSON, b, x, rtol=1e-8, maxit=300, precond="vcycle", lam_hi_per_level=lams)
    prev, N = fine, 64
    while N > 4:
        N //= 2
        c = Ctx(cube(N), 1, poisson_law=law)
        parent, octant = cube_parent_map(2 * N)
        prev.set_coarse_context(c, parent, octant)
        ctxs.append(c)
        if N > 4:
            lams.append(1.2 * c.estimate_lambda_max(A.OP_POISSON, dev(uniform(2, N ** 3 * 8)), level=0, steps=20))
        prev = c
    assert ctxs[-1].setup_coarse_solver(A.OP_POISSON) == 512
    lams.append(1.0)
    assert fine.chain_levels() == len(lams) == 8
    x.zero_()
    it_h, rr_h = fine.cg_solve(A.OP_POISSON, b, x, rtol=1e-8, maxit=300, precond="vcycle", lam_hi_per_level=lams)
    assert rr_h <= 1e-8 and it_h < it_p
    y = torch.empty_like(b)
    fine.apply_poisson(x, y)
    assert float(torch.linalg.norm(b - y) / torch.linalg.norm(b)) <= 1.01e-8
    x.zero_()                                     # the paper's configuration: FP32 cph V-cycle in FP64 CG
    it_f, rr_f = fine.cg_solve(A.OP_POISSON, b, x, rtol=1e-8, maxit=300, precond="vcycle_fp32", lam_hi_per_level=lams)
    assert rr_f <= 1e-8 and it_f <= it_h + 2
