# quick GPU check: parity tests, then C2/C3/C5 bench lines (no cpu baseline)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -5 gpurun_out/gputests.log
for c in 2 3 5; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c=$?
  python -c "import json; d=json.load(open('gpurun_out/bench_c$c.json')); print('C$c', d['ms_per_step'], d['value']/1e9, d['roofline']['frac'], d['roofline']['bound'])"
done
