# usage: bash scripts/bench_variants_ops.sh <variant>...  C5/C3/C2 bench lines + C4 ops per variant
for v in "$@"; do
  bash scripts/bench_variants.sh "5 3 2" $v
  bash scripts/bench_pois_variants.sh $v
done
