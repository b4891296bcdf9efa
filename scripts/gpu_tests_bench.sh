# GPU parity suite + C5 bench line (+ C3/C2 quick lines)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -5 gpurun_out/gputests.log
for c in 5 3 2; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline --no-ops > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c=$?
  python -c "import json; d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1]); print('C$c', d['ms_per_step'], d['value']/1e9, d['roofline']['frac'])"
done
