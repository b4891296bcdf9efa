"""Error behaviour of the C ABI entry points added for §8(f) (include/dgvv.h): status codes, never
exceptions across the ABI, no state change on failure."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import cube, cube_parent_map, deformed_cube, uniform           # noqa: E402
from oracle import laws                                                   # noqa: E402
from paper_2506_14424_b200 import _abi as A                               # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def Ctx(*a, **k):
    from paper_2506_14424_b200.dgvv import Context
    return Context(*a, **k)


def status_of(fn):
    from paper_2506_14424_b200 import DgvvError
    with pytest.raises(DgvvError) as e:
        fn()
    return e.value.status


def test_gmres_and_oseen_errors():
    m = cube(2)
    ctx = Ctx(m, 2, visc_law=laws.C1_LAW)
    n = m.n_cells * 3 * 27
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    assert status_of(lambda: ctx.gmres_solve(b, x, alpha_c=1.0)) == A.ESTATE            # no transport field
    assert status_of(lambda: ctx.apply_oseen(b, x, alpha_c=1.0)) == A.ESTATE
    ctx.set_transport(torch.from_numpy(uniform(1, n)).cuda())
    assert status_of(lambda: ctx.gmres_solve(b, x, restart=0)) == A.EINVAL
    assert status_of(lambda: ctx.gmres_solve(b, x, restart=500)) == A.EINVAL
    assert status_of(lambda: ctx.gmres_solve(b, x, rtol=-1.0)) == A.EINVAL
    assert status_of(lambda: ctx.gmres_solve(b, x, precond="vcycle", lam_hi_per_level=None)) == A.EINVAL
    assert status_of(lambda: ctx.apply_oseen(b, b, alpha_c=1.0)) == A.EINVAL           # aliasing
    ctx.set_mass(0, 200.0)                                                               # still usable
    it, rr = ctx.gmres_solve(b, x, rtol=1e-6, restart=30, maxit=400, precond="jacobi")
    assert rr <= 1e-6 and it < 400


def test_coarse_solver_and_hierarchy_errors():
    mf, mc = cube(4), cube(2)
    parent, octant = cube_parent_map(4)
    big = Ctx(cube(8), 1, poisson_law=laws.C4_LAW)                  # 4096 scalar DoFs: allowed
    assert big.setup_coarse_solver(A.OP_POISSON) == 4096
    too_big = Ctx(cube(6), 2, poisson_law=laws.C4_LAW)              # 5832 > 4096
    assert status_of(lambda: too_big.setup_coarse_solver(A.OP_POISSON)) == A.EINVAL
    fine = Ctx(mf, 1, visc_law=laws.C1_LAW)
    coarse = Ctx(mc, 1, visc_law=laws.C1_LAW)
    assert status_of(lambda: fine.set_coarse_context(fine, parent, octant)) == A.EINVAL   # self
    with pytest.raises(ValueError):                                      # binding checks the array lengths
        fine.set_coarse_context(coarse, parent[:8], octant[:8])
    bad = parent.copy()
    bad[0] = 99                                                          # parent out of range
    assert status_of(lambda: fine.set_coarse_context(coarse, bad, octant)) == A.EINVAL
    fine.set_coarse_context(coarse, parent, octant)
    z8 = np.zeros(mc.n_cells, dtype=np.int32)
    assert status_of(lambda: coarse.set_coarse_context(fine, z8, z8.astype(np.int8))) == A.EINVAL  # would form a cycle
    assert status_of(lambda: Ctx(mf, 2, visc_law=laws.C1_LAW).set_continuous_level()) == A.EINVAL  # degree 2


def test_continuous_level_requires_chain():
    mf, mc = cube(4), cube(2)
    parent, octant = cube_parent_map(4)
    fine = Ctx(mf, 1, visc_law=laws.C1_LAW)
    coarse = Ctx(mc, 1, visc_law=laws.C1_LAW)
    fine.set_coarse_context(coarse, parent, octant)
    fine.set_continuous_level()                          # coarse context not enabled -> ESTATE
    b = torch.ones(mf.n_cells * 3 * 8, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    assert status_of(lambda: fine.vcycle(A.OP_VISCOUS, b, x, [1.0, 1.0, 1.0])) == A.ESTATE
    coarse.set_continuous_level()
    coarse.setup_coarse_solver(A.OP_VISCOUS)
    lam = fine.estimate_lambda_max(A.OP_VISCOUS, torch.from_numpy(uniform(2, len(b))).cuda())
    lamc = fine.estimate_lambda_max_continuous(A.OP_VISCOUS, torch.from_numpy(uniform(2, 3 * fine.n_vertices)).cuda())
    fine.vcycle(A.OP_VISCOUS, b, x, [1.2 * lam, 1.2 * lamc, 1.0])
    assert torch.isfinite(x).all()
    assert status_of(lambda: fine.vcycle_fp32(A.OP_VISCOUS, b, x, [1.2 * lam, 1.2 * lamc, 1.0])) == A.EUNSUPPORTED


def test_carreau_domain_check_in_kernel():
    """update_viscosity checks nu > 0 and finite at every point inside the K3 kernel (one host read):
    a non-finite u_lin gives DGVV_EDOMAIN and leaves the operator unusable until a valid update."""
    from inputs.vectors import c3_linearization
    m = cube(2)
    ctx = Ctx(m, 4, visc_law=laws.C3_CARREAU)
    u0 = c3_linearization(m, 4)
    bad = u0.copy()
    bad[5] = np.nan
    w = torch.from_numpy(uniform(0, len(u0))).cuda()
    y = torch.empty_like(w)
    assert status_of(lambda: ctx.update_viscosity(torch.from_numpy(bad).cuda())) == A.EDOMAIN
    assert status_of(lambda: ctx.apply_viscous(w, y)) == A.ESTATE
    ctx.update_viscosity(torch.from_numpy(u0).cuda())
    ctx.apply_viscous(w, y)
    assert torch.isfinite(y).all()
