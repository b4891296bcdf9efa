# C5 hierarchy per-level rows (bench_ops.py --configs 5) per library variant
mkdir -p gpurun_out build/var_base
cp paper_2506_14424_b200/lib/libdgvv.so build/var_base/libdgvv.so
for v in base "$@"; do
  DGVV_LIB_PATH=$PWD/build/var_$v/libdgvv.so timeout 300 python scripts/bench_ops.py --configs 5 --reps 3 > gpurun_out/lv_$v.json 2>&1
  echo "== $v"; grep -h "level1\|vcycle" gpurun_out/lv_$v.json | cut -c17-100
done
