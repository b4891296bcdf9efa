"""dgvv_apply_viscous_host (host buffers, slab-pipelined copies) == dgvv_apply_viscous on device
buffers, bitwise (same kernel, same cells, only the launch is split into slabs), and == the CPU
oracle within the parity tolerance.  Meshes cover slab-crossing neighbours in every direction,
periodic faces that connect the first and the last slab (BFS, z periodic), general geometry."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import bfs, cube, deformed_cube, uniform                       # noqa: E402
from oracle import dg, laws                                                # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = [
    ("cube16 k3", lambda: cube(16), 3, laws.C2_LAW),
    ("deformed12 k3", lambda: deformed_cube(12, 3), 3, laws.C2_LAW),
    ("bfs periodic k2", lambda: bfs(nx_in=4, ny_in=4, nx_out=24, nz=8), 2, laws.C1_LAW),
    ("cube9 k4", lambda: cube(9), 4, laws.C1_LAW),
]


@pytest.mark.parametrize("name,mk,k,law", CASES, ids=[c[0] for c in CASES])
def test_host_apply_equals_device_apply(name, mk, k, law):
    from paper_2506_14424_b200.dgvv import Context
    m = mk()
    ctx = Context(m, k, visc_law=law)
    u = uniform(0, m.n_cells * 3 * (k + 1) ** 3)
    ref_dev = torch.empty(len(u), dtype=torch.float64, device="cuda")
    ctx.apply_viscous(torch.from_numpy(u).cuda(), ref_dev)
    hs = torch.from_numpy(u).pin_memory()
    hd = torch.full((len(u),), np.nan, dtype=torch.float64).pin_memory()
    for _ in range(2):                       # second call reuses the staging buffers
        ctx.apply_viscous_host(hs, hd)
        torch.cuda.synchronize()
        assert torch.equal(hd, ref_dev.cpu())
    # pageable host memory is accepted too
    hp = torch.from_numpy(u.copy())
    dp = torch.empty(len(u), dtype=torch.float64)
    ctx.apply_viscous_host(hp, dp)
    torch.cuda.synchronize()
    assert torch.equal(dp, ref_dev.cpu())
    if m.n_cells <= 2000:
        d = dg.Disc(m, k)
        ref = dg.viscous_apply(d, u, dg.AnalyticNu(d, law))
        assert np.linalg.norm(dp.numpy() - ref) / np.linalg.norm(ref) < 1e-12


def test_host_apply_rejects_bad_buffers():
    from paper_2506_14424_b200.dgvv import Context
    m = cube(2)
    ctx = Context(m, 1, visc_law=laws.C2_LAW)
    n = m.n_cells * 3 * 8
    with pytest.raises(ValueError):
        ctx.apply_viscous_host(torch.zeros(n, dtype=torch.float64, device="cuda"), torch.zeros(n, dtype=torch.float64))
    with pytest.raises(ValueError):
        ctx.apply_viscous_host(torch.zeros(n - 1, dtype=torch.float64), torch.zeros(n, dtype=torch.float64))
