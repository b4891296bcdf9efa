# End-of-session artifacts (one GPU): bench lines C2 (default), C3, C5, the oracle reference arm,
# and the per-op table of every §8 row (bench_ops: C2-C5, f1-f4, the end-to-end step).
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/fin_bench_c2.json 2> gpurun_out/fin_bench_c2.err
python bench.py --config 3 --steps 50 --no-cpu-baseline > gpurun_out/fin_bench_c3.json 2> gpurun_out/fin_bench_c3.err
python bench.py --config 5 --steps 50 --no-cpu-baseline > gpurun_out/fin_bench_c5.json 2> gpurun_out/fin_bench_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
python scripts/bench_ops.py --configs 2,3,4,5,f1,f2,f3,f4,step --reps 5 > gpurun_out/fin_ops.json 2> gpurun_out/fin_ops.err
echo done
