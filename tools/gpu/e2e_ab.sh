# analyze_many per-call copy stream (B2L_MANY_FRESH_STREAM=1, the old behaviour) vs one per device:
# per-step times and the bench's e2e lines; then the single-pass front sweep
for mode in fresh persistent; do
  if [ $mode = fresh ]; then export B2L_MANY_FRESH_STREAM=1; else unset B2L_MANY_FRESH_STREAM; fi
  echo "== $mode"
  timeout -k 5 300 python tools/e2e_steps.py 2>&1 | tail -3
  timeout -k 10 900 python bench.py --no-cpu > gpurun_out/bench_$mode.json 2> /dev/null
  python - $mode <<'PY'
import json, sys
d = json.loads(open(f'gpurun_out/bench_{sys.argv[1]}.json').read().strip().splitlines()[-1])
a = d['analysis']['e2e']; print('C2 e2e', a['value'], a['step_ms_min_median_max'], a['slowest_step'])
for c in d['configs']:
    e = c.get('e2e') or {}
    if 'step_ms_min_median_max' in e: print(c['name'], e['value'], e['step_ms_min_median_max'], e['slowest_step'])
PY
done
bash tools/gpu/sweep_front.sh 2>&1 | tail -5
