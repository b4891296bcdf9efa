# ncu --set full captures (raw page CSV) of the other hot kernels of §8(a) on one GPU: C2 and C3
# Picard applies, the C3 Newton apply (v3), update_viscosity (K3), the C4 Poisson k = 5 apply and
# its FP32 multigrid-level twin.  Summarised by scripts/ncu_summary.py into profiles/.
mkdir -p gpurun_out
cap() {  # cap <tag> <kernel regex> <skip> <command...>
  tag=$1; rx=$2; sk=$3; shift 3
  ncu --set full --clock-control none -k "regex:$rx" -s $sk -c 1 -o gpurun_out/p_$tag "$@" > gpurun_out/p_$tag.log 2>&1
  ncu -i gpurun_out/p_$tag.ncu-rep --page raw --csv > gpurun_out/p_${tag}_raw.csv 2>/dev/null
  rm -f gpurun_out/p_$tag.ncu-rep
  echo "$tag: $(wc -l < gpurun_out/p_${tag}_raw.csv) lines"
}
cap c2 sipg_apply2 5 python bench.py --config 2 --steps 6 --warmup 3 --no-cpu-baseline --no-ops
cap c3 sipg_apply2 5 python bench.py --config 3 --steps 6 --warmup 3 --no-cpu-baseline --no-ops
cap c3newton newton_apply3 3 python scripts/bench_ops.py --configs 3 --reps 1
cap c3nu carreau_nu 3 python scripts/bench_ops.py --configs 3 --reps 1
cap c4pois 'sipg_apply2_kernel<double, 6' 5 python scripts/bench_ops.py --configs 4 --reps 1
cap c4pois32 'sipg_apply2_kernel<float, 6' 5 python scripts/bench_ops.py --configs 4 --reps 1
echo done
