# usage: bash scripts/bench_variants.sh <configs> <variant>...   (bench lines per variant/config)
cfgs=$1; shift
for v in "$@"; do for c in $cfgs; do
  DGVV_LIB_PATH=$PWD/build/var_$v/libdgvv.so timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/var_${v}_c$c.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/var_${v}_c$c.json').read().strip().splitlines()[-1]); print('$v C$c', round(d['ms_per_step']*1e3,1), 'us', round(d['value']/1e9,2), 'GDoF/s')" || tail -3 gpurun_out/var_${v}_c$c.json
done; done
