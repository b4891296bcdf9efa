# C4 Poisson k = 5 launch shapes after the Chebyshev epilogue fix (tree = 4 cells x 4 CTAs/SM)
set -x
mkdir -p gpurun_out build/var_base
cp paper_2506_14424_b200/lib/libdgvv.so build/var_base/libdgvv.so
for rep in 1 2; do bash scripts/bench_pois_variants.sh base "$@"; done
for v in base "$@"; do grep -h "vcycle_5_3_2_1_fp32" gpurun_out/pv_$v.json | cut -c1-90; done
echo done
