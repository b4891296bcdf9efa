# source-level ncu captures of the apply kernels (C5 viscous k=3, C4 Poisson k=5), exported here
set -e
mkdir -p gpurun_out
python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline --no-ops > gpurun_out/ps_plain_c5.json
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 5 -c 1 -o gpurun_out/ps_c5 \
    python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline --no-ops > gpurun_out/ps_ncu_c5.log 2>&1
ncu -i gpurun_out/ps_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/ps_c5_sass.csv 2>/dev/null || true
ncu -i gpurun_out/ps_c5.ncu-rep --page source --csv > gpurun_out/ps_c5_src.csv 2>/dev/null || true
bash scripts/prof_c4.sh
ncu -i gpurun_out/p4_pois.ncu-rep --page source --csv > gpurun_out/p4_src.csv 2>/dev/null || true
echo done
ncu -i gpurun_out/ps_c5.ncu-rep --page raw --csv > gpurun_out/ps_c5_raw.csv
ncu -i gpurun_out/p4_pois.ncu-rep --page raw --csv > gpurun_out/p4_raw.csv
ncu -i gpurun_out/p4_pois.ncu-rep --page source --csv --print-source sass > gpurun_out/p4_sass.csv 2>/dev/null || true
rm -f gpurun_out/*.ncu-rep
gzip -f gpurun_out/*_src.csv gpurun_out/*_sass.csv
ls -la gpurun_out
