# usage: bash scripts/gpu_variants.sh "<configs>" "<parity-test variant>" <variant>...
#   bench lines per variant/config (scripts/bench_variants.sh), C4 ops per variant, then the
#   apply parity tests against the chosen variant's library
cfgs=$1; tv=$2; shift 2
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "$@"; do bash scripts/bench_variants.sh "$cfgs" $v; done
done
for v in "$@"; do bash scripts/bench_pois_variants.sh $v; done
if [ -n "$tv" ]; then
  DGVV_LIB_PATH=$PWD/build/var_$tv/libdgvv.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_threads_comm.py -q -x > gpurun_out/var_tests_$tv.log 2>&1
  echo "tests($tv)=$?"; tail -2 gpurun_out/var_tests_$tv.log
fi
