# round-2 evidence: GPU tests, smoke, both bench arms, analysis traffic (1M, 10M), the hash
# launch list, ncu --set full of the C1 batch (split pairs) and of the C2 hash kernel, and the
# §8(d) config lines -- everything into gpurun_out/ (summaries are copied to profiles/ after)
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
for n in 1000000 10000000; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/traffic_c2_$n.csv python tools/time_analysis.py --device --config c2 --n $n --iters 2 > /dev/null 2>&1
  python tools/analysis_traffic.py gpurun_out/traffic_c2_$n.csv 2 $n gpurun_out/analysis_traffic_c2_$n.json > /dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/hash_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-large --no-configs > gpurun_out/bench_ncu.log 2>&1
sed -n '/^cat > \/tmp\/c1t.py/,/^PY$/p' tools/gpu/c1split.sh > /tmp/mk.sh; bash /tmp/mk.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hash_warp -s 3 -c 1 -o gpurun_out/c1_split -f python /tmp/c1t.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_hash_coop -s 2 -c 1 -o gpurun_out/hash_c2 -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-large --no-configs > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/c1_split.ncu-rep gpurun_out/c1_split_ncu_summary.json > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/hash_c2.ncu-rep gpurun_out/hash_c2_ncu_summary.json > /dev/null 2>&1
timeout 900 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
python - <<'PY'
import json
for f in ('gpurun_out/bench.json', 'gpurun_out/bench_ref.json'):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'unparsable', e); continue
    print(f, d.get('value'), d.get('unit'), 'e2e', (d.get('e2e') or {}).get('value'))
    a = d.get('analysis') or {}
    print('  analysis', a.get('value'), a.get('verified'), (a.get('e2e') or {}).get('value'))
    for c in d.get('configs') or []:
        print('  ', c.get('name'), c.get('value'), c.get('unit'), 'ver', c.get('verified'), 'e2e', (c.get('e2e') or {}).get('value'), 'cpu', (c.get('cpu_baseline') or {}).get('value'))
PY
