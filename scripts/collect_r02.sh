# Copy the outputs of scripts/final_r02.sh (gpurun_out/f_*) into profiles/ as the round-2 artifacts.
set -e
cp gpurun_out/f_bench_c5.json profiles/r02_bench_c5.json
cp gpurun_out/f_bench_ref.json profiles/r02_bench_ref.json
cp gpurun_out/f_c5_src.csv.gz profiles/r02_c5_sass_source.csv.gz
cp gpurun_out/f_gputests.log profiles/r02_gpu_tests.log
cp gpurun_out/f_launches_c5.csv profiles/r02_launches_c5.csv
cp gpurun_out/f_ops.json profiles/r02_ops_final.json
NCU_TRAFFIC=profiles/r02_ncu_traffic.json python scripts/ncu_summary.py C5=gpurun_out/f_c5_raw.csv > profiles/r02_ncu_c5_final.json
