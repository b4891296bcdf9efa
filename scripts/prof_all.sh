# Round profile capture (one GPU): plain runs first, then ncu launch list of the bench command and
# one `--set full` capture per hot kernel.  Output: gpurun_out/r_*.{csv,ncu-rep,log}
set -e
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r_plain_c2.json
python bench.py --config 3 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r_plain_c3.json
python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r_plain_c5.json
python scripts/bench_ops.py --configs 3 --reps 1 > gpurun_out/r_plain_ops3.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r_launches_c2.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 5 -c 1 -o gpurun_out/r_c2_apply \
    python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r_ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 5 -c 1 -o gpurun_out/r_c3_apply \
    python bench.py --config 3 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r_ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 5 -c 1 -o gpurun_out/r_c5_apply \
    python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r_ncu_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:newton_apply2 -s 3 -c 1 -o gpurun_out/r_c3_newton \
    python scripts/bench_ops.py --configs 3 --reps 1 > gpurun_out/r_ncu_newton.log 2>&1
echo done
