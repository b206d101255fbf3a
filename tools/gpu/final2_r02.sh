# closing run after the K2 retune: ncu of K2 (16-buffer and single launches), GPU tests, smoke,
# bench (ours), K2 timings
sed -n '/^cat > \/tmp\/k2many.py/,/^PY$/p' tools/gpu/evidence_r02b.sh > /tmp/mk2.sh; bash /tmp/mk2.sh
timeout -k 10 900 ncu --set full --import-source on --clock-control none -k regex:k_hash_planes -s 2 -c 1 -o gpurun_out/k2_many_full -f python /tmp/k2many.py > gpurun_out/k2many_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/k2_many_full.ncu-rep gpurun_out/k2_many_ncu_summary.json --algo-bytes 4294967296 > /dev/null 2>&1
bash tools/gpu/k2ncu.sh > /dev/null 2>&1
cp gpurun_out/k2_many_ncu_summary.json gpurun_out/k2_ncu_summary.json profiles/ 2>/dev/null
timeout -k 10 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout -k 10 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -k 10 200 python tools/k2_time.py > gpurun_out/k2_time.txt 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/k2_time.txt
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print('bench', d.get('value'), d.get('unit'), 'e2e', (d.get('e2e') or {}).get('value'))
a = d.get('analysis') or {}
print('  analysis', a.get('value'), a.get('ms_per_step'), a.get('verified'), (a.get('e2e') or {}).get('value'))
for c in d.get('configs') or []:
    print('  ', c.get('name'), c.get('value'), c.get('unit'), c.get('ms_per_step'), 'ver', c.get('verified'), 'e2e', (c.get('e2e') or {}).get('value'), 'traffic', (c.get('roofline') or {}).get('traffic'))
PY
