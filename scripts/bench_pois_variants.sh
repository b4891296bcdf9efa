# usage: bash scripts/bench_pois_variants.sh <variant>...   (C4 Poisson apply per variant)
for v in "$@"; do
  DGVV_LIB_PATH=$PWD/build/var_$v/libdgvv.so timeout 300 python scripts/bench_ops.py --configs 4 --reps 3 > gpurun_out/pv_$v.json 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
for line in open(f"gpurun_out/pv_{v}.json"):
    if line.startswith("{"):
        d = json.loads(line)
        if d.get("op") in ("apply_poisson_k5", "chebyshev5_from_zero_k5", "vcycle_5_3_2_1"):
            print(v, d["op"], d["ms"])
PY
done
