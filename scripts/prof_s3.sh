# Session-3 captures after the Cartesian face staging and the fused Oseen kernel (one GPU):
# plain runs first (must exit 0), then one ncu --set full capture per changed kernel.
set -e
mkdir -p gpurun_out
python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/s3_plain_c5.json
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 5 -c 1 -o gpurun_out/s3_c5_apply \
    python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/s3_ncu_c5.log 2>&1
cat > /tmp/oseen_once.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from inputs import deformed_cube, uniform
from scripts.bench_ops import C2_LAW, dev
from paper_2506_14424_b200.dgvv import Context
m = deformed_cube(32, 3)
ctx = Context(m, 3, visc_law=C2_LAW)
N = 3 * ctx.n_dofs(0)
src = dev(uniform(0, N)); ctx.set_transport(dev(uniform(1, N))); ctx.set_mass(0, 1.0e3); dst = torch.empty_like(src)
for _ in range(6):
    ctx.apply_oseen(src, dst, 1.0)
torch.cuda.synchronize()
PY
python /tmp/oseen_once.py
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 3 -c 1 -o gpurun_out/s3_c2_oseen \
    python /tmp/oseen_once.py > gpurun_out/s3_ncu_oseen.log 2>&1

# reduce to CSV pages on the box (the reports exceed gpurun's 64 MiB pull limit)
for r in s3_c5_apply s3_c2_oseen; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_sass.csv
  rm -f gpurun_out/$r.ncu-rep
done
echo done
