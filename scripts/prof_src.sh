# source-level ncu capture of the C5 apply kernel (SASS + stall samples), exported as compressed CSV
# usage: bash scripts/prof_src.sh <tag> [config]
set -e
tag=${1:-c5}; cfg=${2:-5}
mkdir -p gpurun_out
python bench.py --config $cfg --steps 6 --warmup 3 --no-cpu-baseline --no-ops > gpurun_out/ps_plain_$tag.json
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 5 -c 1 -o gpurun_out/ps_$tag \
    python bench.py --config $cfg --steps 6 --warmup 3 --no-cpu-baseline --no-ops > gpurun_out/ps_ncu_$tag.log 2>&1
ncu -i gpurun_out/ps_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ps_${tag}_src.csv 2>/dev/null || true
ncu -i gpurun_out/ps_$tag.ncu-rep --page raw --csv > gpurun_out/ps_${tag}_raw.csv
rm -f gpurun_out/*.ncu-rep
gzip -f gpurun_out/ps_${tag}_src.csv
