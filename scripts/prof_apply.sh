# usage: bash scripts/prof_apply.sh <config> <tag> [kernel-regex]
# plain run first (must exit 0), then one ncu --set full capture of the apply kernel.
set -e
cfg=$1; tag=$2; kre=${3:-sipg_apply}
mkdir -p gpurun_out
python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$tag.json 2> gpurun_out/plain_$tag.err
ncu --set full --clock-control none --import-source on -k regex:$kre -s 5 -c 1 \
    -o gpurun_out/prof_$tag python bench.py --config $cfg --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
