# Round-2 artifacts (one GPU): GPU tests, the default bench line (C5 + ops + cpu baseline), the
# reference arm, the ncu launch list of the bench command, one --set full capture of the benched
# C5 kernel (raw page CSV for scripts/ncu_summary.py), and the per-op table of every §8 row.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_gputests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo ref=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_c5.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-ops > gpurun_out/f_ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 5 -c 1 -o gpurun_out/f_c5 \
    python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-ops > gpurun_out/f_ncu_c5.log 2>&1; echo ncu=$?
ncu -i gpurun_out/f_c5.ncu-rep --page raw --csv > gpurun_out/f_c5_raw.csv
ncu -i gpurun_out/f_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/f_c5_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
gzip -f gpurun_out/f_c5_src.csv
timeout 1500 python scripts/bench_ops.py --configs 2,3,4,5,f1,f2,f3,f4,step --reps 5 > gpurun_out/f_ops.json 2> gpurun_out/f_ops.err; echo ops=$?
echo done
