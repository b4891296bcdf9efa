"""Launch a few Helmholtz applies (or Chebyshev sweeps) on one p-level of the C5 hierarchy, for
ncu:  ncu --set full -k regex:sipg_apply2 -s 2 -c 1 python scripts/prof_level.py <level> [cheb]"""
import sys
import torch
sys.path.insert(0, ".")
from inputs import bfs, uniform
from inputs.vectors import c5_linearization
from scripts.bench_ops import C5_LAW, dev
from paper_2506_14424_b200 import _abi as A
from paper_2506_14424_b200.dgvv import Context

lvl = int(sys.argv[1])
m = bfs()
ctx = Context(m, 3, visc_law=C5_LAW, degrees=[3, 2, 1])
ctx.set_mass(A.OP_VISCOUS, 1.0e3)
ctx.update_viscosity(dev(c5_linearization(m, 3)))
N = 3 * ctx.n_dofs(lvl)
s, d = dev(uniform(3, N)), torch.empty(N, dtype=torch.float64, device="cuda")
if len(sys.argv) > 2:
    wk = torch.empty(2 * N, dtype=torch.float64, device="cuda")
    ctx.inverse_diagonal(A.OP_VISCOUS, wk[:N], level=lvl)
    for _ in range(2):
        ctx.chebyshev_smooth(A.OP_VISCOUS, d, s, 1.0, 20.0, degree=5, x_is_zero=True, work=wk, level=lvl)
else:
    for _ in range(6):
        ctx.apply_viscous(s, d, level=lvl)
torch.cuda.synchronize()
print("done")
