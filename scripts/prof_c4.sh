set -e
python scripts/bench_ops.py --configs 4 --reps 1 > gpurun_out/p4_plain.json
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 8 -c 1 -o gpurun_out/p4_pois \
    python scripts/bench_ops.py --configs 4 --reps 1 > gpurun_out/p4_ncu.log 2>&1
echo done
