# source-level ncu capture of the C4 Poisson apply (k = 5), exported as compressed CSV
set -e
mkdir -p gpurun_out
python scripts/bench_ops.py --configs 4 --reps 1 > gpurun_out/p4_plain.json
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 8 -c 1 -o gpurun_out/p4_pois \
    python scripts/bench_ops.py --configs 4 --reps 1 > gpurun_out/p4_ncu.log 2>&1
ncu -i gpurun_out/p4_pois.ncu-rep --page source --csv --print-source sass > gpurun_out/p4b_src.csv 2>/dev/null || true
ncu -i gpurun_out/p4_pois.ncu-rep --page raw --csv > gpurun_out/p4b_raw.csv
rm -f gpurun_out/*.ncu-rep
gzip -f gpurun_out/p4b_src.csv
