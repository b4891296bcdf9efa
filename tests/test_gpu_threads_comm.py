"""The multi-rank library path executed end to end on ONE GPU: R ranks, each a host
thread with its own context and CUDA stream, joined by the library's in-process communicator
(dgvv_thread_group_*).  Unlike the external-exchange tests this runs the library's own collective
path — setup handshake, grouped ghost exchange on the comm stream overlapped with the interior
cells, allreduced dots, and therefore the multi-rank Lanczos, Chebyshev, V-cycle and CG.
Results: applies bitwise equal to one context (each cell's sum is partition-independent) and
within 1e-12 of the CPU oracle; solvers match the one-context run (dots are summed rank-wise, so
only to rounding)."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import bfs, cube, uniform                                      # noqa: E402
from inputs.vectors import c3_linearization                               # noqa: E402
from oracle import dg, laws                                               # noqa: E402
from paper_2506_14424_b200 import _abi as A                               # noqa: E402
from paper_2506_14424_b200.partition import slab_partition                # noqa: E402

TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_ranks(m, R, k, body, **kw):
    """body(rank, ctx, part) in R threads (each on its own stream); returns the per-rank results."""
    from paper_2506_14424_b200.dgvv import Context, ThreadGroup
    g = ThreadGroup(R)
    parts = [slab_partition(m, R, r) for r in range(R)]
    out, err = [None] * R, [None] * R

    def worker(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                p = parts[r]
                ctx = Context(p, k, n_owned=p.n_owned, n_ghost=p.n_ghost, ghost_global_id=p.ghost_global_id,
                              ghost_owner=p.ghost_owner, first_global_cell=p.first, nccl_comm=g.comm(r), **kw)
                out[r] = body(r, ctx, p)
                torch.cuda.current_stream().synchronize()
                ctx.close()
        except BaseException as e:          # noqa: BLE001 - re-raised in the main thread
            err[r] = e

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    g.close()
    for e in err:
        if e is not None:
            raise e
    return parts, out


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name,mk,k,R", [("cube4 k4 R2", lambda: cube(4), 4, 2), ("cube5 k3 R3", lambda: cube(5), 3, 3),
                                         ("bfs small k3 R3", lambda: bfs(nx_in=4, ny_in=2, nx_out=8, nz=3), 3, 3)])
def test_thread_group_viscous_and_poisson_apply(name, mk, k, R):
    from paper_2506_14424_b200.dgvv import Context
    m = mk()
    per = 3 * (k + 1) ** 3
    u = uniform(0, m.n_cells * per)
    ref_ctx = Context(m, k, visc_law=laws.C2_LAW, poisson_law=laws.C4_LAW)
    ref = torch.empty(len(u), dtype=torch.float64, device="cuda")
    ref_ctx.apply_viscous(torch.from_numpy(u).cuda(), ref)
    ps = uniform(1, m.n_cells * (k + 1) ** 3)
    refp = torch.empty(len(ps), dtype=torch.float64, device="cuda")
    ref_ctx.apply_poisson(torch.from_numpy(ps).cuda(), refp)

    def body(r, ctx, p):
        x = torch.from_numpy(u[p.first * per:(p.first + p.n_owned) * per].copy()).cuda()
        y = torch.empty_like(x)
        for _ in range(3):                     # repeated exchanges reuse the buffers
            ctx.apply_viscous(x, y)
        n1 = (k + 1) ** 3
        xp = torch.from_numpy(ps[p.first * n1:(p.first + p.n_owned) * n1].copy()).cuda()
        yp = torch.empty_like(xp)
        ctx.apply_poisson(xp, yp)
        d = ctx.dot(x, x, 3)                   # allreduced
        # a5: the exchange moves face traces, 2 NC n^2 doubles per cut face (not NC n^3 per cell)
        sent, recv = ctx.exchange_bytes(0)
        cut = sum(1 for cc in range(p.n_owned) for f in range(6)
                  if p.neighbor[cc, f] >= 0 and not (p.first <= p.neighbor[cc, f] < p.first + p.n_owned))
        assert sent == cut * 2 * 3 * (k + 1) ** 2 * 8 and recv > 0
        return y.cpu(), yp.cpu(), d

    parts, out = run_ranks(m, R, k, body, visc_law=laws.C2_LAW, poisson_law=laws.C4_LAW)
    y = torch.cat([o[0] for o in out])
    assert torch.equal(y, ref.cpu())
    assert torch.equal(torch.cat([o[1] for o in out]), refp.cpu())
    assert all(abs(o[2] - float(u @ u)) <= 1e-13 * float(u @ u) for o in out)
    assert len({o[2] for o in out}) == 1      # every rank holds the same allreduced bits
    d = dg.Disc(m, k)
    assert rel(y.numpy(), dg.viscous_apply(d, u, dg.AnalyticNu(d, laws.C2_LAW))) < TOL


def test_thread_group_carreau_newton():
    """Carreau update (ghost u_lin exchange, coarse-level nu), Picard and Newton applies on 2 ranks."""
    from paper_2506_14424_b200.dgvv import Context
    m = cube(4)
    k, R = 4, 2
    per = 3 * 125
    ul = c3_linearization(m, k)
    w = uniform(0, m.n_cells * per)
    rc = Context(m, k, visc_law=laws.C3_CARREAU, degrees=[4, 2])
    rc.update_viscosity(torch.from_numpy(ul).cuda())
    refp, refn = torch.empty(len(w), dtype=torch.float64, device="cuda"), torch.empty(len(w), dtype=torch.float64, device="cuda")
    rc.apply_viscous(torch.from_numpy(w).cuda(), refp)
    rc.apply_linearized_viscous(torch.from_numpy(w).cuda(), refn)

    def body(r, ctx, p):
        sl = slice(p.first * per, (p.first + p.n_owned) * per)
        ctx.update_viscosity(torch.from_numpy(ul[sl].copy()).cuda())
        x = torch.from_numpy(w[sl].copy()).cuda()
        y1, y2 = torch.empty_like(x), torch.empty_like(x)
        ctx.apply_viscous(x, y1)
        ctx.apply_linearized_viscous(x, y2)
        return y1.cpu(), y2.cpu()

    _, out = run_ranks(m, R, k, body, visc_law=laws.C3_CARREAU, degrees=[4, 2])
    assert torch.equal(torch.cat([o[0] for o in out]), refp.cpu())
    assert torch.equal(torch.cat([o[1] for o in out]), refn.cpu())
    d = dg.Disc(m, k)
    assert rel(torch.cat([o[1] for o in out]).numpy(), dg.newton_apply(d, ul, w, laws.C3_CARREAU)) < TOL


@pytest.mark.parametrize("op,precond", [(0, "vcycle"), (1, "vcycle"), (0, "jacobi"), (2, "vcycle"),
                                        (0, "vcycle_fp32"), (1, "vcycle_fp32")])
def test_thread_group_pcg_matches_one_context(op, precond):
    """Multi-rank Lanczos, V-cycle and PCG on 3 ranks vs one context: lambda_max to rounding (the
    Lanczos dots are allreduced rank-wise); with the same bounds one V-cycle (FP64 or FP32 levels, no
    dot inside) is bitwise the one-context V-cycle; PCG to rtol 1e-9 then differs only through the
    rounding of its dots: iteration counts within one, solutions within 1e-6."""
    from paper_2506_14424_b200.dgvv import Context
    m = cube(6)
    R = 3
    degs = [3, 2, 1]
    kw = dict(visc_law=laws.C2_LAW, poisson_law=laws.C4_LAW, degrees=degs)
    nc = 1 if op == 1 else 3
    per = nc * 64
    rng = np.random.default_rng(3)
    td, tc = rng.uniform(1e-3, 1e-2, m.n_cells), rng.uniform(1e-3, 1e-2, m.n_cells)   # Fehn2018b-sized (DESIGN P1)
    b = uniform(0, m.n_cells * per)
    one = Context(m, 3, **kw)
    if op == 0:
        one.set_mass(0, 10.0)
    if op == 2:
        one.set_penalty_parameters(td, tc)
    v0s = [uniform(2, m.n_cells * nc * (kk + 1) ** 3) for kk in degs]
    lams = [1.2 * one.estimate_lambda_max(op, torch.from_numpy(v0s[l]).cuda(), level=l, steps=15)
            for l in range(len(degs))]
    bd = torch.from_numpy(b).cuda()
    v1 = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    if precond != "jacobi":
        (one.vcycle_fp32 if precond == "vcycle_fp32" else one.vcycle)(op, bd, v1, lams)
    x1 = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    it1, rr1 = one.cg_solve(op, bd, x1, rtol=1e-9, maxit=2000, precond=precond, lam_hi_per_level=lams)

    def body(r, ctx, p):
        if op == 0:
            ctx.set_mass(0, 10.0)
        if op == 2:
            rows = np.concatenate([np.arange(p.first, p.first + p.n_owned), np.asarray(p.ghost_global_id, dtype=np.int64)])
            ctx.set_penalty_parameters(td[rows], tc[rows])
        lam = []
        for l, kk in enumerate(degs):
            q = nc * (kk + 1) ** 3
            lam.append(1.2 * ctx.estimate_lambda_max(op, torch.from_numpy(v0s[l][p.first * q:(p.first + p.n_owned) * q].copy()).cuda(),
                                                     level=l, steps=15))
        bb = torch.from_numpy(b[p.first * per:(p.first + p.n_owned) * per].copy()).cuda()
        v = torch.zeros(p.n_owned * per, dtype=torch.float64, device="cuda")
        if precond != "jacobi":
            (ctx.vcycle_fp32 if precond == "vcycle_fp32" else ctx.vcycle)(op, bb, v, lams)
        x = torch.zeros(p.n_owned * per, dtype=torch.float64, device="cuda")
        it, rr = ctx.cg_solve(op, bb, x, rtol=1e-9, maxit=2000, precond=precond, lam_hi_per_level=lams)
        return x.cpu(), it, rr, lam, v.cpu()

    _, out = run_ranks(m, R, 3, body, **kw)
    for o in out:
        assert np.allclose(o[3], lams, rtol=1e-10, atol=0), (o[3], lams)
        assert abs(o[1] - it1) <= 1, (o[1], it1)
    assert torch.equal(torch.cat([o[4] for o in out]), v1.cpu())
    x = torch.cat([o[0] for o in out]).numpy()
    assert rel(x, x1.cpu().numpy()) < 1e-6
    assert rr1 <= 1e-9 and max(o[2] for o in out) <= 1e-9


def test_thread_group_cph_vcycle_h_levels():
    """h-levels across ranks (nested z-slabs): the cph V-cycle 8^3 k=2 -> k=1 -> 4^3 k=1 -> 2^3 k=1
    (coarsest: Chebyshev) on 2 ranks is bitwise the one-context V-cycle; PCG with it matches."""
    from inputs import cube_parent_map
    from paper_2506_14424_b200.dgvv import Context, ThreadGroup
    R = 2
    law = laws.C2_LAW
    meshes = [cube(8), cube(4), cube(2)]
    degs0 = [2, 1]
    b = uniform(0, meshes[0].n_cells * 3 * 27)

    def chain(ctxs, parts):
        for lvl in range(len(ctxs) - 1):
            par, octa = cube_parent_map(meshes[lvl].n_cells and round(meshes[lvl].n_cells ** (1 / 3)))
            pf, pc = parts[lvl], parts[lvl + 1]
            sl = slice(pf.first, pf.first + pf.n_owned)
            ctxs[lvl].set_coarse_context(ctxs[lvl + 1], par[sl] - pc.first, octa[sl])

    # one context
    one = [Context(meshes[0], 2, visc_law=law, degrees=degs0), Context(meshes[1], 1, visc_law=law),
           Context(meshes[2], 1, visc_law=law)]
    for c in one:
        c.set_mass(0, 10.0)

    class _P:
        first, n_owned = 0, None
    full = []
    for m in meshes:
        p = _P()
        p.n_owned = m.n_cells
        full.append(p)
    chain(one, full)
    nlev = 4
    v0 = [uniform(2, 3 * meshes[0].n_cells * 27), uniform(2, 3 * meshes[0].n_cells * 8),
          uniform(3, 3 * meshes[1].n_cells * 8), uniform(4, 3 * meshes[2].n_cells * 8)]
    lams = [1.2 * one[0].estimate_lambda_max(0, torch.from_numpy(v0[0]).cuda(), level=0, steps=15),
            1.2 * one[0].estimate_lambda_max(0, torch.from_numpy(v0[1]).cuda(), level=1, steps=15),
            1.2 * one[1].estimate_lambda_max(0, torch.from_numpy(v0[2]).cuda(), level=0, steps=15),
            1.2 * one[2].estimate_lambda_max(0, torch.from_numpy(v0[3]).cuda(), level=0, steps=15)]
    assert one[0].chain_levels() == nlev
    v1 = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    one[0].vcycle(0, torch.from_numpy(b).cuda(), v1, lams)
    x1 = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    it1, _ = one[0].cg_solve(0, torch.from_numpy(b).cuda(), x1, rtol=1e-9, maxit=200, precond="vcycle", lam_hi_per_level=lams)

    g = ThreadGroup(R)
    parts = [[slab_partition(m, R, r) for m in meshes] for r in range(R)]
    out, err = [None] * R, [None] * R

    def worker(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                ps = parts[r]
                kws = [dict(degrees=degs0), {}, {}]
                ks = [2, 1, 1]
                ctxs = [Context(p, k, visc_law=law, n_owned=p.n_owned, n_ghost=p.n_ghost, ghost_global_id=p.ghost_global_id,
                                ghost_owner=p.ghost_owner, first_global_cell=p.first, nccl_comm=g.comm(r), **kw)
                        for p, k, kw in zip(ps, ks, kws)]
                for c in ctxs:
                    c.set_mass(0, 10.0)
                chain(ctxs, ps)
                per = 3 * 27
                bb = torch.from_numpy(b[ps[0].first * per:(ps[0].first + ps[0].n_owned) * per].copy()).cuda()
                v = torch.zeros_like(bb)
                ctxs[0].vcycle(0, bb, v, lams)
                x = torch.zeros_like(bb)
                it, rr = ctxs[0].cg_solve(0, bb, x, rtol=1e-9, maxit=200, precond="vcycle", lam_hi_per_level=lams)
                torch.cuda.current_stream().synchronize()
                out[r] = (v.cpu(), x.cpu(), it, rr)
                for c in ctxs:
                    c.close()
        except BaseException as e:          # noqa: BLE001
            err[r] = e

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    g.close()
    for e in err:
        if e is not None:
            raise e
    assert torch.equal(torch.cat([o[0] for o in out]), v1.cpu())
    assert all(abs(o[2] - it1) <= 1 for o in out)
    assert rel(torch.cat([o[1] for o in out]).numpy(), x1.cpu().numpy()) < 1e-6


@pytest.mark.parametrize("op,R", [(A.OP_VISCOUS, 2), (A.OP_POISSON, 3)])
def test_thread_group_direct_coarse_solver(op, R):
    """The direct coarse solve across ranks (dgvv_setup_coarse_solver on communicator contexts):
    x = V(b) on a single-level context == numpy's solve of the dense ORACLE matrix (viscous: cube(2)
    k=1 + mass, 192 DoFs on 2 ranks; Poisson: cube(3) k=1, 216 DoFs on 3 ranks), FP64 and FP32."""
    from oracle import dense
    if op == A.OP_VISCOUS:
        m, k, law, mass, kw = cube(2), 1, laws.C1_LAW, 3.0, {"visc_law": laws.C1_LAW}
        d = dg.Disc(m, k)
        Ad = dense.assemble_viscous(d, dg.AnalyticNu(d, law)) + mass * np.diag(dg.mass_apply(d, np.ones(m.n_cells * 3 * d.N)))
        per = 3 * 8
    else:
        m, k, law, mass, kw = cube(3), 1, laws.C4_LAW, 0.0, {"poisson_law": laws.C4_LAW}
        d = dg.Disc(m, k)
        Ad = dense.assemble_poisson(d, dg.AnalyticNu(d, law))
        per = 8
    b = uniform(0, Ad.shape[0])
    ref = np.linalg.solve(Ad, b)

    def body(r, ctx, p):
        ctx.set_mass(op, mass)
        n = ctx.setup_coarse_solver(op)
        bb = torch.from_numpy(b[p.first * per:(p.first + p.n_owned) * per].copy()).cuda()
        x = torch.zeros_like(bb)
        ctx.vcycle(op, bb, x, [1.0])
        xf = torch.zeros_like(bb)
        ctx.vcycle_fp32(op, bb, xf, [1.0])
        return n, x.cpu(), xf.cpu()

    parts, out = run_ranks(m, R, k, body, **kw)
    assert all(o[0] == Ad.shape[0] for o in out)
    x = torch.cat([o[1] for o in out]).numpy()
    xf = torch.cat([o[2] for o in out]).numpy()
    cond = np.linalg.cond(Ad)
    assert rel(x, ref) < 1e-10 * max(1.0, cond / 1e4)
    assert rel(xf, ref) < 1e-5 * max(1.0, cond / 1e4)      # b and x in FP32, the solve in FP64 (reading F1)


def test_thread_group_cph_direct_solve():
    """cph V-cycle whose coarsest h-level ends in the direct solve, on 2 ranks (nested slabs):
    equal to the one-context V-cycle to rounding (the gathered solve sums the same terms)."""
    from inputs import cube_parent_map
    from paper_2506_14424_b200.dgvv import Context, ThreadGroup
    R = 2
    law = laws.C4_LAW
    meshes = [cube(4), cube(2)]
    b = uniform(0, meshes[0].n_cells * 27)

    def chain(ctxs, parts):
        par, octa = cube_parent_map(4)
        pf, pc = parts[0], parts[1]
        sl = slice(pf.first, pf.first + pf.n_owned)
        ctxs[0].set_coarse_context(ctxs[1], par[sl] - pc.first, octa[sl])

    class _P:
        first, n_owned = 0, None
    full = []
    for mm in meshes:
        p = _P()
        p.n_owned = mm.n_cells
        full.append(p)
    one = [Context(meshes[0], 2, poisson_law=law, degrees=[2, 1]), Context(meshes[1], 1, poisson_law=law)]
    assert one[1].setup_coarse_solver(A.OP_POISSON) == 64
    chain(one, full)
    v0 = [uniform(2, meshes[0].n_cells * 27), uniform(2, meshes[0].n_cells * 8)]
    lams = [1.2 * one[0].estimate_lambda_max(1, torch.from_numpy(v0[0]).cuda(), level=0, steps=15),
            1.2 * one[0].estimate_lambda_max(1, torch.from_numpy(v0[1]).cuda(), level=1, steps=15), 1.0]
    v1 = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    one[0].vcycle(A.OP_POISSON, torch.from_numpy(b).cuda(), v1, lams)

    g = ThreadGroup(R)
    parts = [[slab_partition(mm, R, r) for mm in meshes] for r in range(R)]
    out, err = [None] * R, [None] * R

    def worker(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                ps = parts[r]
                ctxs = [Context(p, k, poisson_law=law, n_owned=p.n_owned, n_ghost=p.n_ghost, ghost_global_id=p.ghost_global_id,
                                ghost_owner=p.ghost_owner, first_global_cell=p.first, nccl_comm=g.comm(r), **kw)
                        for p, k, kw in zip(ps, [2, 1], [dict(degrees=[2, 1]), {}])]
                ctxs[1].setup_coarse_solver(A.OP_POISSON)
                chain(ctxs, ps)
                bb = torch.from_numpy(b[ps[0].first * 27:(ps[0].first + ps[0].n_owned) * 27].copy()).cuda()
                v = torch.zeros_like(bb)
                ctxs[0].vcycle(A.OP_POISSON, bb, v, lams)
                torch.cuda.current_stream().synchronize()
                out[r] = v.cpu()
                for c in ctxs:
                    c.close()
        except BaseException as e:          # noqa: BLE001
            err[r] = e

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    g.close()
    for e in err:
        if e is not None:
            raise e
    assert rel(torch.cat(out).numpy(), v1.cpu().numpy()) < 1e-12
