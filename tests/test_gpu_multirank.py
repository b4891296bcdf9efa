"""Multi-rank path on ONE GPU (external-exchange mode): R contexts, one per slab partition,
whose ghost buffers are filled from the peers' packed send buffers (the library's own pack
kernel and ghost ordering; NCCL only moves those same buffers).  The gathered result must be
BITWISE equal to the single-context apply: each cell's output is a fixed-order sum of its
own volume and face terms, independent of the partition.  Every
gathered result is also compared with the CPU oracle (relative L2 <= 1e-12, reading G25), so
the multi-rank path is held to the same bar as the one-context path, not only to itself."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import bfs, cube, deformed_cube, uniform                       # noqa: E402
from inputs.vectors import c3_linearization                               # noqa: E402
from oracle import dg, laws                                                # noqa: E402
from paper_2506_14424_b200 import _abi as A                               # noqa: E402
from paper_2506_14424_b200.partition import slab_partition                # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


TOL = 1e-12


def oracle_close(y, ref):
    """Gathered multi-rank result vs the oracle: relative L2 <= 1e-12 (G25)."""
    y = y.cpu().numpy()
    err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert err < TOL, err


def make_ranks(m, R, k, **kw):
    from paper_2506_14424_b200.dgvv import Context
    parts = [slab_partition(m, R, r) for r in range(R)]
    ctxs = [Context(p, k, n_owned=p.n_owned, n_ghost=p.n_ghost, ghost_global_id=p.ghost_global_id,
                    ghost_owner=p.ghost_owner, first_global_cell=p.first, **kw) for p in parts]
    return parts, ctxs


def fill_ghosts(parts, ctxs, locals_, kind, per):
    """Transport stand-in: copy every rank's packed send block into its peers' ghost buffers."""
    R = len(parts)
    packed, offs = [], []
    for r in range(R):
        lay = ctxs[r].ghost_layout()
        tot = sum(s for _, s, _ in lay) * per
        buf = torch.empty(max(tot, 1), dtype=torch.float64, device="cuda")
        if tot:
            ctxs[r].pack_ghosts(kind, locals_[r], buf)
        d, o = {}, 0
        for peer, s, _ in lay:
            d[peer] = (o, s)
            o += s * per
        packed.append(buf)
        offs.append(d)
    for r in range(R):
        if parts[r].n_ghost == 0:
            continue
        gb = ctxs[r].ghost_buffer(kind, parts[r].n_ghost)
        pos = 0
        for peer, _, rc in ctxs[r].ghost_layout():
            o, cnt = offs[peer][r]
            assert cnt == rc
            gb[pos * per:(pos + rc) * per] = packed[peer][o:o + cnt * per]
            pos += rc
    torch.cuda.synchronize()


@pytest.mark.parametrize("name,mk,k,R", [
    ("deformed4 k3 R2", lambda: deformed_cube(4, 3), 3, 2),
    ("deformed4 k3 R4", lambda: deformed_cube(4, 3), 3, 4),
    ("cube4 k4 R3", lambda: cube(4), 4, 3),
    ("bfs small k3 R4", lambda: bfs(nx_in=4, ny_in=2, nx_out=8, nz=3), 3, 4),
])
def test_viscous_multirank_bitwise(name, mk, k, R):
    from paper_2506_14424_b200.dgvv import Context
    m = mk()
    n3 = (k + 1) ** 3
    per = 3 * n3
    u = uniform(0, m.n_cells * per)
    ref_ctx = Context(m, k, visc_law=laws.C2_LAW)
    src = torch.from_numpy(u).cuda()
    ref = torch.empty_like(src)
    ref_ctx.apply_viscous(src, ref)
    parts, ctxs = make_ranks(m, R, k, visc_law=laws.C2_LAW)
    locs = [src[p.first * per:(p.first + p.n_owned) * per].contiguous() for p in parts]
    fill_ghosts(parts, ctxs, locs, A.GHOST_VISCOUS, per)
    outs = []
    for p, c, x in zip(parts, ctxs, locs):
        y = torch.empty_like(x)
        c.apply_viscous(x, y)
        outs.append(y)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs), ref)
    d = dg.Disc(m, k)
    oracle_close(torch.cat(outs), dg.viscous_apply(d, u, dg.AnalyticNu(d, laws.C2_LAW)))


def test_poisson_and_carreau_multirank_bitwise():
    from paper_2506_14424_b200.dgvv import Context
    m = cube(4)
    # Poisson k=5
    n3 = 216
    p_ = uniform(1, m.n_cells * n3)
    src = torch.from_numpy(p_).cuda()
    ref = torch.empty_like(src)
    Context(m, 5, poisson_law=laws.C4_LAW).apply_poisson(src, ref)
    parts, ctxs = make_ranks(m, 2, 5, poisson_law=laws.C4_LAW)
    locs = [src[p.first * n3:(p.first + p.n_owned) * n3].contiguous() for p in parts]
    fill_ghosts(parts, ctxs, locs, A.GHOST_POISSON, n3)
    outs = []
    for c, x in zip(ctxs, locs):
        y = torch.empty_like(x)
        c.apply_poisson(x, y)
        outs.append(y)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs), ref)
    dp = dg.Disc(m, 5)
    oracle_close(torch.cat(outs), dg.poisson_apply(dp, p_, dg.AnalyticNu(dp, laws.C4_LAW)))
    # Carreau (ghost u_lin) + Picard and Newton applies, k=4
    k, per = 4, 3 * 125
    ul = torch.from_numpy(c3_linearization(m, k)).cuda()
    w = torch.from_numpy(uniform(0, m.n_cells * per)).cuda()
    rc = Context(m, k, visc_law=laws.C3_CARREAU)
    rc.update_viscosity(ul)
    refp, refn = torch.empty_like(w), torch.empty_like(w)
    rc.apply_viscous(w, refp)
    rc.apply_linearized_viscous(w, refn)
    parts, ctxs = make_ranks(m, 2, k, visc_law=laws.C3_CARREAU)
    uls = [ul[p.first * per:(p.first + p.n_owned) * per].contiguous() for p in parts]
    ws = [w[p.first * per:(p.first + p.n_owned) * per].contiguous() for p in parts]
    fill_ghosts(parts, ctxs, uls, A.GHOST_ULIN, per)
    for c, x in zip(ctxs, uls):
        c.update_viscosity(x)
    fill_ghosts(parts, ctxs, ws, A.GHOST_VISCOUS, per)
    op, on = [], []
    for c, x in zip(ctxs, ws):
        y1, y2 = torch.empty_like(x), torch.empty_like(x)
        c.apply_viscous(x, y1)
        c.apply_linearized_viscous(x, y2)
        op.append(y1)
        on.append(y2)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(op), refp)
    assert torch.equal(torch.cat(on), refn)
    d = dg.Disc(m, k)
    ul_h, w_h = ul.cpu().numpy(), w.cpu().numpy()
    oracle_close(torch.cat(op), dg.viscous_apply(d, w_h, dg.CarreauNu(d, ul_h, laws.C3_CARREAU)))
    oracle_close(torch.cat(on), dg.newton_apply(d, ul_h, w_h, laws.C3_CARREAU))
