# f4 timings (bench_ops) and one ncu --set full capture of the convective kernel on the C2 mesh.
set -e
mkdir -p gpurun_out
python scripts/bench_ops.py --configs f4 --reps 5 > gpurun_out/ops_f4.json 2> gpurun_out/ops_f4.err
cat > /tmp/conv_once.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from inputs import deformed_cube, uniform
from scripts.bench_ops import C2_LAW, dev
from paper_2506_14424_b200.dgvv import Context
m = deformed_cube(32, 3)
ctx = Context(m, 3, visc_law=C2_LAW)
N = 3 * ctx.n_dofs(0)
src = dev(uniform(0, N)); ctx.set_transport(dev(uniform(1, N))); dst = torch.empty_like(src)
for _ in range(6):
    ctx.apply_convective(src, dst)
torch.cuda.synchronize()
PY
python /tmp/conv_once.py
ncu --set full --clock-control none --import-source on -k regex:convective -s 3 -c 1 \
    -o gpurun_out/prof_conv_c2 python /tmp/conv_once.py > gpurun_out/ncu_conv_c2.log 2>&1
