import sys, torch
sys.path.insert(0, ".")
from inputs import cube, uniform
from inputs.vectors import c3_linearization
from scripts.bench_ops import C3_LAW, dev
from paper_2506_14424_b200.dgvv import Context
m = cube(64)
ctx = Context(m, 4, visc_law=C3_LAW)
ul = dev(c3_linearization(m, 4))
w = dev(uniform(0, 3 * ctx.n_dofs(0)))
y = torch.empty_like(w)
for rep in range(3):
    ctx.update_viscosity(ul)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); ctx.apply_linearized_viscous(w, y); e[1].record(); ctx.apply_linearized_viscous(w, y); e[2].record()
    e[2].synchronize()
    print(f"first Newton apply after update {e[0].elapsed_time(e[1]):.2f} ms, next {e[1].elapsed_time(e[2]):.2f} ms")
