# ncu --set full of one launch of the apply kernel on a p-level of the C5 hierarchy (raw + SASS source pages as CSV)
# usage: bash scripts/prof_level.sh <level> [cheb]
set -e
lvl=$1; mode=$2; tag=l${lvl}${mode}
mkdir -p gpurun_out
python scripts/prof_level.py $lvl $mode > gpurun_out/pl_plain_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sipg_apply2 -s 2 -c 1 -o gpurun_out/pl_$tag \
    python scripts/prof_level.py $lvl $mode > gpurun_out/pl_ncu_$tag.log 2>&1
ncu -i gpurun_out/pl_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/pl_${tag}_src.csv 2>/dev/null || true
ncu -i gpurun_out/pl_$tag.ncu-rep --page raw --csv > gpurun_out/pl_${tag}_raw.csv
rm -f gpurun_out/pl_$tag.ncu-rep
gzip -f gpurun_out/pl_${tag}_src.csv
