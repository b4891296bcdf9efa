"""Split the 'diagonals + lambda' phase of the Picard step (bench_ops.py run_step) into the inverse
diagonals of the three p-levels and the Lanczos estimates (C3 mesh, Carreau, mass 1e3)."""
import sys
import torch
sys.path.insert(0, ".")
from inputs import cube, uniform
from inputs.vectors import c3_linearization
from scripts.bench_ops import C3_LAW, dev
from paper_2506_14424_b200 import _abi as A
from paper_2506_14424_b200.dgvv import Context

m = cube(64)
ctx = Context(m, 4, visc_law=C3_LAW, degrees=[4, 2, 1])
ctx.set_mass(A.OP_VISCOUS, 1.0e3)
ul = dev(c3_linearization(m, 4))
v0 = [dev(uniform(2, 3 * ctx.n_dofs(l))) for l in range(3)]
dinv = [torch.empty(3 * ctx.n_dofs(l), dtype=torch.float64, device="cuda") for l in range(3)]
for rep in range(2):
    ctx.update_viscosity(ul)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record()
    for l in range(3):
        ctx.inverse_diagonal(A.OP_VISCOUS, dinv[l], level=l)
        ev[1 + l].record()
    for l in range(3):
        ctx.estimate_lambda_max(A.OP_VISCOUS, v0[l], level=l, steps=15)
        ev[4 + l].record()
    ev[6].synchronize()
    print("diag per level (ms):", [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(0, 3)],
          "lanczos per level (ms):", [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(3, 6)])
