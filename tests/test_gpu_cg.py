"""§8(f) f3 c-level on the GPU: the continuous Q1 level below the DG levels (dgvv_set_continuous_level,
dgvv_embed_continuous, dgvv_apply_continuous, Lanczos on the continuous level, V-cycle
DG-p -> c -> CG-h -> direct) against the CPU oracle (oracle.cg: coordinate-matched vertices,
dense P_c and nested Q1 transfer, Galerkin operator; pinned in test_oracle_cg.py) on the same
seeded inputs; full-size C4 PCG with the c-level."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import cube, cube_parent_map, uniform                         # noqa: E402
from oracle import cg, dense, dg, laws, mg                                # noqa: E402
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


def _kw(op, law):
    return {"visc_law": law} if op == A.OP_VISCOUS else {"poisson_law": law}


def _dense_dg(op, d, law, mass, n_cells):
    if op == A.OP_VISCOUS:
        return dense.assemble_viscous(d, dg.AnalyticNu(d, law)) + mass * np.diag(dg.mass_apply(d, np.ones(n_cells * 3 * d.N)))
    return dense.assemble_poisson(d, dg.AnalyticNu(d, law)) + mass * np.diag(dg.mass_apply(d, np.ones(n_cells * d.N), ncomp=1))


@pytest.mark.parametrize("op", [A.OP_VISCOUS, A.OP_POISSON])
@pytest.mark.parametrize("mk", [lambda: cube(3), lambda: cube(3, periodic=(True, False, True))], ids=["cube3", "cube3-periodic-xz"])
def test_continuous_embedding_and_operator_parity(op, mk):
    m = mk()
    law = laws.C1_LAW if op == A.OP_VISCOUS else laws.C4_LAW
    nc = 3 if op == A.OP_VISCOUS else 1
    ctx = Ctx(m, 1, **_kw(op, law))
    nv, ncol = ctx.set_continuous_level()
    vid, nvo = cg.vertex_numbering(m)
    assert nv == nvo and ncol >= 8
    P = cg.expand(cg.embedding(m, vid, nvo), nc)
    x = uniform(0, nc * nv)
    ydg = torch.empty(m.n_cells * nc * 8, dtype=torch.float64, device="cuda")
    ctx.embed_continuous(op, dev(x), ydg)
    assert rel(host(ydg), P @ x) < 1e-14
    r = uniform(1, m.n_cells * nc * 8)
    ycg = dev(x)
    ctx.embed_continuous(op, dev(r), ycg, transpose=True, beta=0.5)
    assert rel(host(ycg), P.T @ r + 0.5 * x) < 1e-14
    Ad = _dense_dg(op, dg.Disc(m, 1), law, 0.0, m.n_cells)
    y = torch.empty(nc * nv, dtype=torch.float64, device="cuda")
    ctx.apply_continuous(op, dev(x), y)
    assert rel(host(y), P.T @ (Ad @ (P @ x))) < 1e-12


def _oracle_c_chain(op, law, mf, mc, degs, parent, octant, mass):
    nc = 3 if op == A.OP_VISCOUS else 1
    levels = []
    for k in degs:
        d = dg.Disc(mf, k)
        levels.append({"A": _dense_dg(op, d, law, mass, mf.n_cells)})
    vf, nvf = cg.vertex_numbering(mf)
    vc, nvc = cg.vertex_numbering(mc)
    Pc = cg.expand(cg.embedding(mf, vf, nvf), nc)
    Ph = np.kron(np.eye(nc), cg.h_transfer(vf, nvf, vc, nvc, parent, octant))
    Pcc = cg.expand(cg.embedding(mc, vc, nvc), nc)
    Acc = Pcc.T @ _dense_dg(op, dg.Disc(mc, 1), law, mass, mc.n_cells) @ Pcc
    levels.append({"A": Pc.T @ levels[-1]["A"] @ Pc})
    for L in levels:
        L["apply"] = (lambda x, Ad=L["A"]: Ad @ x)
        L["Dinv"] = 1.0 / np.diag(L["A"])
        L["lam_hi"] = 1.2 * mg.lanczos_lambda_max(L["apply"], L["Dinv"], uniform(2, len(L["Dinv"])), 20)
    for li in range(len(degs) - 1):
        kf, kc = degs[li], degs[li + 1]
        levels[li]["restrict"] = lambda r, kf=kf, kc=kc: mg.restrict(r, kf, kc, mf.n_cells, ncomp=nc)
        levels[li]["prolongate"] = lambda x, kf=kf, kc=kc: mg.prolongate(x, kf, kc, mf.n_cells, ncomp=nc)
    levels[len(degs) - 1]["restrict"] = lambda r: Pc.T @ r
    levels[len(degs) - 1]["prolongate"] = lambda x: Pc @ x
    levels[-1]["restrict"] = lambda r: Ph.T @ r
    levels[-1]["prolongate"] = lambda x: Ph @ x
    levels.append({"apply": (lambda x: Acc @ x), "solve": lambda b: np.linalg.solve(Acc, b)})
    return levels


@pytest.mark.parametrize("op", [A.OP_VISCOUS, A.OP_POISSON])
def test_c_level_vcycle_parity(op):
    """cube(4): DG k = 2 -> 1, c-level Q1 on cube(4), CG h-level Q1 on cube(2) with the direct solve:
    GPU V-cycle == oracle; GPU Lanczos on the continuous level == oracle's."""
    mf, mc = cube(4), cube(2)
    parent, octant = cube_parent_map(4)
    degs = [2, 1]
    law = laws.C1_LAW if op == A.OP_VISCOUS else laws.C4_LAW
    mass = 10.0 if op == A.OP_VISCOUS else 0.0
    fine, coarse = Ctx(mf, 2, degrees=degs, **_kw(op, law)), Ctx(mc, 1, **_kw(op, law))
    fine.set_mass(op, mass)
    coarse.set_mass(op, mass)
    fine.set_coarse_context(coarse, parent, octant)
    fine.set_continuous_level()
    coarse.set_continuous_level()
    coarse.setup_coarse_solver(op)
    levels = _oracle_c_chain(op, law, mf, mc, degs, parent, octant, mass)
    assert fine.chain_levels() == 4
    v0 = uniform(2, len(levels[2]["Dinv"]))
    lam_gpu = fine.estimate_lambda_max_continuous(op, dev(v0), steps=20)
    assert abs(lam_gpu - levels[2]["lam_hi"] / 1.2) < 1e-10 * lam_gpu
    lams = [L["lam_hi"] for L in levels[:3]] + [1.0]
    b = uniform(0, len(levels[0]["Dinv"]))
    x = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    fine.vcycle(op, dev(b), x, lams)
    assert rel(host(x), mg.vcycle(levels, b)) < 1e-10


def test_c_level_pcg_full_size_c4():
    """C4 at full size: DG k = 5 -> 3 -> 2 -> 1 on 64^3, the c-level (Q1 on 64^3, 274,625 vertices),
    Q1 h-levels 32^3 ... 4^3 and the direct solve on 4^3 (125 vertices): PCG to 1e-8."""
    law = laws.C4_LAW
    op = A.OP_POISSON
    fine = Ctx(cube(64), 5, poisson_law=law, degrees=[5, 3, 2, 1])
    lams = [1.2 * fine.estimate_lambda_max(op, dev(uniform(2, 64 ** 3 * (k + 1) ** 3)), level=l, steps=20)
            for l, k in enumerate([5, 3, 2, 1])]
    ctxs, prev, N = [fine], fine, 64
    while N > 4:
        N //= 2
        c = Ctx(cube(N), 1, poisson_law=law)
        parent, octant = cube_parent_map(2 * N)
        prev.set_coarse_context(c, parent, octant)
        ctxs.append(c)
        prev = c
    for c in ctxs:
        nv, _ = c.set_continuous_level()
    for c in ctxs[:-1]:
        lams.append(1.2 * c.estimate_lambda_max_continuous(op, dev(uniform(2, c.n_vertices)), steps=20))
    assert ctxs[-1].setup_coarse_solver(op) == 125
    lams.append(1.0)
    assert fine.chain_levels() == len(lams) == 4 + 5
    b = dev(uniform(0, fine.n_dofs(0)))
    x = torch.zeros_like(b)
    it, rr = fine.cg_solve(op, b, x, rtol=1e-8, maxit=300, precond="vcycle", lam_hi_per_level=lams)
    assert rr <= 1e-8 and it < 60
    y = torch.empty_like(b)
    fine.apply_poisson(x, y)
    assert float(torch.linalg.norm(b - y) / torch.linalg.norm(b)) <= 1.01e-8
