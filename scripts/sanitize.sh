#!/bin/bash
# compute-sanitizer runs (memcheck, racecheck, synccheck) over the small-mesh GPU tests:
# every kernel family (sipg_apply2 TMA/TMAC paths, newton, penalty, convective, FP32 levels,
# h-transfer, c-level, direct solve) at sizes the sanitizer finishes in minutes.
# usage: scripts/sanitize.sh <tool> [pytest -k expr]   (writes gpurun_out/sanitize_<tool>.log)
set -u
tool=$1
sel=${2:-"not full and not c2_full and not c3_full and not c4_full and not c5_full and not fp32_full"}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
extra=""
if [ "$tool" = "racecheck" ]; then extra="--racecheck-report all"; fi
timeout 1500 $CS --tool "$tool" $extra --print-limit 50 --error-exitcode 99 --target-processes all \
  --log-file gpurun_out/sanitize_${tool}.raw \
  python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$sel" > gpurun_out/sanitize_${tool}.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_${tool}.log
tail -5 gpurun_out/sanitize_${tool}.raw >> gpurun_out/sanitize_${tool}.log 2>/dev/null
