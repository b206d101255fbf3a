# the driver's two bench arms (N=1): ours then the reference, full default configs
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 1500 gpurun_out/bench.err; tail -c 600 gpurun_out/bench_ref.err
python -c "
import json
for f in ('gpurun_out/bench.json','gpurun_out/bench_ref.json'):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'unparsable', e); continue
    print(f, d.get('value'), d.get('unit'), 'e2e', (d.get('e2e') or {}).get('value'))
    a=d.get('analysis') or {}
    print('  analysis', a.get('value'), a.get('verified'), (a.get('e2e') or {}).get('value'), (a.get('cpu_baseline') or {}).get('value'))
    for c in d.get('configs') or []:
        print('  ', c.get('name'), c.get('value'), c.get('unit'), 'ver', c.get('verified'), c.get('verified_strict_rt'), 'e2e', (c.get('e2e') or {}).get('value'), 'cpu', (c.get('cpu_baseline') or {}).get('value'), c.get('error') or c.get('not_run','')[:40])
"
