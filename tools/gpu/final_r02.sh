# closing numbers after the single-pass front: GPU tests, smoke, bench (ours), analysis traffic at
# 1M / 10M, and the host/GPU phase timelines at 1M / 10M
timeout -k 10 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
bash tools/gpu/traffic.sh > gpurun_out/traffic_medians.txt 2>&1
cp gpurun_out/analysis_traffic_c2_*.json profiles/ 2>/dev/null
timeout -k 10 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
B2L_TRACE=ev timeout -k 5 300 python tools/evlog.py --n 10000000 --iters 4 2>&1 | sed -n '/=== last call/,$p' > gpurun_out/timeline_10m.txt
B2L_SYNC_STATS=2 B2L_TRACE=ev timeout -k 5 300 python tools/evlog.py --n 1000000 2>&1 | sed -n '/=== last call/,$p' > gpurun_out/timeline_1m.txt
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/traffic_medians.txt
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print('bench', d.get('value'), d.get('unit'), 'e2e', (d.get('e2e') or {}).get('value'))
a = d.get('analysis') or {}
print('  analysis', a.get('value'), a.get('ms_per_step'), a.get('verified'), (a.get('e2e') or {}).get('value'))
for c in d.get('configs') or []:
    print('  ', c.get('name'), c.get('value'), c.get('unit'), c.get('ms_per_step'), 'ver', c.get('verified'), 'e2e', (c.get('e2e') or {}).get('value'))
PY
